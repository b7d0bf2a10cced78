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


def test_traffic_table_from_ncu_csv(tmp_path, monkeypatch):
    """profiles/traffic_from_ncu.py folds an ncu --csv launch list into
    per-pixel DRAM bytes (the roofline's `achieved` basis)."""
    import importlib.util
    import json
    import shutil

    prof = tmp_path / "profiles"
    prof.mkdir()
    shutil.copy(os.path.join(ROOT, "profiles", "traffic_from_ncu.py"), prof)
    spec = importlib.util.spec_from_file_location("tfn", prof / "traffic_from_ncu.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    npx = 256 * 640 * 480
    rows = ['"ID","Kernel Name","Metric Name","Metric Unit","Metric Value"']
    for i, (rd, wr, t) in enumerate([(5.3, 2.5, 1.5), (5.5, 2.7, 1.6)]):
        rows += [f'"{i}","k_fused_ldg","dram__bytes_read.sum","Gbyte","{rd}"',
                 f'"{i}","k_fused_ldg","dram__bytes_write.sum","Gbyte","{wr}"',
                 f'"{i}","k_fused_ldg","gpu__time_duration.sum","ms","{t}"']
    csv_path = tmp_path / "traffic_streams256_auto.csv"
    csv_path.write_text("==PROF== noise line\n" + "\n".join(rows) + "\n")
    mod.main([str(csv_path)])
    rec = json.load(open(prof / "traffic.json"))["per_px"]["streams256:auto"]
    assert rec["launches"] == 2
    assert abs(rec["read_bytes_per_px"] - 5.4e9 / npx) < 0.01
    assert abs(rec["bytes_per_px"] - (5.4e9 + 2.6e9) / npx) < 0.01
    assert abs(rec["ncu_ms"] - 1.55) < 1e-9
