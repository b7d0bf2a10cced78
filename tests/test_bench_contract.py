"""bench.py's job accounting (CPU): `value` is the whole-job aggregate over
all ranks, with the rank shards covering the job exactly."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_job_pixels_is_the_sum_of_the_rank_shards(bench, world):
    from paper_2110_14934_b200.shard import row_shard, stream_shard

    for name, (_, W, H, S, M, shard) in bench.WORKLOADS.items():
        total = bench.job_pixels(shard, W, H, S, world)
        if shard == "stream":
            parts = [W * H * (b - a) for a, b in (stream_shard(S, r, world) for r in range(world))]
        elif shard == "rows":
            parts = [W * (b - a) for a, b in (row_shard(H, r, world) for r in range(world))]
        else:
            parts = [W * H * S] * world
        assert sum(parts) == total, (name, world)
