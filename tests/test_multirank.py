"""Multi-GPU partitioning, tested on CPU with world_size 2 over gloo.

bench.py shards the path one process per GPU with no data-path collective:
config 4 by camera stream, config 5 by row tile (paper_2110_14934_b200/shard.py).
Here each rank runs the oracle on exactly the shard bench.py would give it,
the ranks all_gather their fused masks and bank words, and rank 0 checks the
gathered result is bit-identical to one process doing all the work -- the
analogue of the reference's worker-count invariance (test_segmenter.cpp:103-130,
acceptance.cpp:206-237)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2110_14934_b200.shard import contiguous_split, row_shard, stream_shard


def test_contiguous_split_matches_parallel_for_rows():
    """engine.cpp:20-29: base = h / workers, the first h % workers ranges
    get one extra row; ranges are contiguous and cover [0, h) once."""
    for total in (1, 7, 480, 1080, 8192, 256):
        for world in (1, 2, 3, 4, 8):
            spans = [contiguous_split(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            base, extra = divmod(total, world)
            assert sizes == [base + (1 if r < extra else 0) for r in range(world)]
    assert stream_shard(256, 3, 8) == (96, 128)
    assert row_shard(8192, 7, 8) == (7168, 8192)
    with pytest.raises(ValueError):
        contiguous_split(10, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _frames(port, streams, w, h, nframes):
    import oracle as O

    scenes = [O.PortScene(port, "A", w, h, seed=s + 1) for s in range(streams)]
    out = []
    for f in range(nframes):
        frs = [sc.render(95 + f) for sc in scenes]
        d = np.stack([fr.depth for fr in frs])
        if f % 3 == 1:
            d[:, 2:6, 3:11] = 0
        out.append((np.stack([fr.r for fr in frs]), np.stack([fr.g for fr in frs]),
                    np.stack([fr.b for fr in frs]), d))
    return out


def _run(port, frames_list, npx, M=4):
    import oracle as O

    proc = O.PortProcessor(port, npx, O.color_cfg(M), O.depth_cfg(M))
    fused = []
    for r, g, b, d in frames_list:
        _, _, fu = proc.process(r.ravel(), g.ravel(), b.ravel(), d.ravel())
        fused.append(fu)
    return np.stack(fused), proc.color.planes(), proc.depth.planes()


def _worker(rank, world, port_no, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O

        port = O.Port()
        S, w, h, F = 4, 24, 18, 12
        frames = _frames(port, S, w, h, F)
        if mode == "stream":
            s0, s1 = stream_shard(S, rank, world)
            mine = [tuple(x[s0:s1] for x in fr) for fr in frames]
            npx = (s1 - s0) * w * h
        else:  # row tiles of every stream's frame, flattened
            y0, y1 = row_shard(h, rank, world)
            mine = [tuple(x[:, y0:y1] for x in fr) for fr in frames]
            npx = S * (y1 - y0) * w
        fused, cpl, dpl = _run(port, mine, npx)
        # no data-path collective in the product; gather only to check
        out = [None] * world
        dist.all_gather_object(out, (fused, cpl, dpl))
        if rank == 0:
            full_fused, full_c, full_d = _run(port, frames, S * w * h)
            if mode == "stream":
                got_f = np.concatenate([o[0] for o in out], axis=1)
                got_c = np.concatenate([o[1] for o in out], axis=1)
                got_d = np.concatenate([o[2] for o in out], axis=1)
                ok = (np.array_equal(got_f, full_fused) and got_c.tobytes() == full_c.tobytes()
                      and got_d.tobytes() == full_d.tobytes())
            else:
                def rows(a, k):  # (planes or frames, S*rows*w) -> (.., S, rows, w)
                    y0, y1 = row_shard(h, k, world)
                    return a.reshape(a.shape[0], S, y1 - y0, w)

                got_f = np.concatenate([rows(o[0], k) for k, o in enumerate(out)], axis=2)
                got_c = np.concatenate([rows(o[1], k) for k, o in enumerate(out)], axis=2)
                ok = (np.array_equal(got_f.reshape(F, -1), full_fused)
                      and got_c.reshape(got_c.shape[0], -1).tobytes() == full_c.tobytes())
            q.put(ok)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["stream", "rows"])
def test_sharded_run_is_bit_identical_to_single_rank(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_no, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) is True


def test_bench_timing_uses_max_over_ranks():
    """bench.py reduces each rank's device time with MAX (the slowest GPU
    defines the step), checked here through the same all_reduce on gloo."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_max_worker, args=(r, 2, port_no, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert sorted([q.get(timeout=5), q.get(timeout=5)]) == [7.5, 7.5]


def _max_worker(rank, world, port_no, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = torch.tensor([3.25 if rank == 0 else 7.5], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    q.put(float(t.item()))
    dist.destroy_process_group()
