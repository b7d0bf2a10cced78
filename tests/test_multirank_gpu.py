"""Multi-GPU sharding of the CUDA path, checked on the GPU.

Each rank runs librgbdseg_b200.so on its shard -- a block of camera streams
(BASELINE config 4) or a tile of rows of every frame (config 5) -- exactly as
bench.py's `Shard` assigns them, with no data-path exchange.  The ranks then
gather their fused masks, bank words, flags and fusion state, and rank 0
checks the result is bit-identical to one rank doing the whole job: the
analogue of the reference's worker-count invariance (test_segmenter.cpp:103-130,
acceptance.cpp:206-237).  With one GPU both ranks share cuda:0 (gloo carries
the gather); they never wait on each other's kernels.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from helpers import holes

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _frames(S, w, h, F, start=95):
    import oracle as O

    port = O.Port()
    scenes = [O.PortScene(port, "A", w, h, seed=s + 1) for s in range(S)]
    out = []
    for f in range(F):
        frs = [sc.render(start + f) for sc in scenes]
        d = np.stack([holes(fr.depth, f) for fr in frs])
        out.append((np.stack([fr.r for fr in frs]), np.stack([fr.g for fr in frs]),
                    np.stack([fr.b for fr in frs]), d))
    return out


def _run(R, frames, w, h, S, device, on_device, M=5):
    """The processor over (S, h, w) frames; returns fused masks per frame and
    the final state (colour/depth planes + flags, fusion out/cpt)."""
    import torch

    cfg = R.RunConfig.defaults()
    cfg.color_gmm.components = cfg.depth_gmm.components = M
    proc = R.SequenceProcessor(w, h, cfg, streams=S, device=device)
    fused = []
    for r, g, b, d in frames:
        if on_device:
            dev = torch.device("cuda", device)
            t = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (r, g, b)]
            td = torch.from_numpy(np.ascontiguousarray(d).view(np.int16)).to(dev).view(
                torch.uint16)
            out = torch.empty((S, h, w), dtype=torch.uint8, device=dev)
            proc.submit(*t, td, fused=out)  # ordered after torch's copies
            proc.sync()
            fused.append(out.cpu().numpy())
        else:
            fm = proc.process(np.ascontiguousarray(r), np.ascontiguousarray(g),
                              np.ascontiguousarray(b), np.ascontiguousarray(d), want=("fused",))
            fused.append(fm.fused.reshape(S, h, w))
    cb, db, fs = proc.color_bank(), proc.depth_bank(), proc.fusion_state()
    state = {"color": cb.planes().reshape(-1, S, h, w), "cflags": cb.initialized_plane().reshape(S, h, w),
             "depth": db.planes().reshape(-1, S, h, w), "dflags": db.initialized_plane().reshape(S, h, w),
             "out": fs.out.reshape(S, h, w), "cpt": fs.cpt.reshape(S, h, w)}
    return np.stack(fused), state


def _worker(rank, world, port_no, mode, on_device, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    import paper_2110_14934_b200 as R
    from paper_2110_14934_b200.shard import row_shard, stream_shard

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        device = rank % torch.cuda.device_count()
        torch.cuda.set_device(device)
        S, w, h, F = 5, 64, 46, 14
        frames = _frames(S, w, h, F)
        if mode == "stream":
            s0, s1 = stream_shard(S, rank, world)
            mine = [tuple(x[s0:s1] for x in fr) for fr in frames]
            fused, state = _run(R, mine, w, h, s1 - s0, device, on_device)
        else:
            y0, y1 = row_shard(h, rank, world)
            mine = [tuple(x[:, y0:y1] for x in fr) for fr in frames]
            fused, state = _run(R, mine, w, y1 - y0, S, device, on_device)
        parts = [None] * world
        dist.all_gather_object(parts, (fused, state))
        if rank == 0:
            full_f, full_s = _run(R, frames, w, h, S, device, on_device)
            ax = {"stream": (1, 0), "rows": (2, 1)}[mode]  # (fused axis, state axis) after plane dim
            got_f = np.concatenate([p[0] for p in parts], axis=ax[0])
            ok = np.array_equal(got_f, full_f)
            bad = [] if ok else ["fused"]
            for k, v in full_s.items():
                cat_ax = (ax[1] + 1) if v.ndim == 4 else ax[1]
                got = np.concatenate([p[1][k] for p in parts], axis=cat_ax)
                if got.tobytes() != v.tobytes():
                    bad.append(k)
            q.put(bad)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("on_device", [False, True])
@pytest.mark.parametrize("mode", ["stream", "rows"])
def test_gpu_shards_bit_identical_to_one_rank(cuda, mode, on_device):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_no, mode, on_device, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) == []


def test_bench_launches_n_ranks_itself(cuda):
    """`python bench.py --gpus 2` (no torchrun) re-launches itself with 2
    ranks and reports the whole-job value of both (n_gpus 2, a 2-rank
    communicator; on a 1-GPU box the ranks share it over gloo)."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--preroll", "3", "--no-cpu-baseline", "--traffic", "off",
           "--windows", "", "--e2e-steps", "3"]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["comm"]["nranks"] == 2 and d["comm"]["allreduce_ones"] == 2
    assert d["config"]["pixels_per_step"] == 256 * 640 * 480
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["stats_gather"]["pixels"] == 256 * 640 * 480
    # a mismatched WORLD_SIZE is refused
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"],
                       stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, timeout=300,
                       env=env, cwd=ROOT)
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr
