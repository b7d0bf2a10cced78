"""Round-2 probe: host-fed e2e of the 256 x VGA workload against the number
of H2D/K1/D2H overlap chunks per frame (RunConfig host_chunks; 0 = auto),
pipelined submits over a ring of 6 pinned planar frames, fused masks read
back.  Prints Mpix/s and the implied H2D GB/s per setting."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2110_14934_b200 as R  # noqa: E402

W, H, S = 640, 480, 256
npx = W * H * S
cfg = R.RunConfig.defaults()
cfg.color_gmm.components = cfg.depth_gmm.components = 5
ring, keep = [], []
for f in range(6):
    fr = R.render_scenario("A", W, H, 95 + f, streams=S, device=0)
    buf = torch.empty(5 * npx, dtype=torch.uint8, pin_memory=True)
    for i, k in enumerate("rgb"):
        buf[i * npx:(i + 1) * npx].copy_(fr[k].reshape(-1))
    buf[3 * npx:].view(torch.int16).copy_(fr["depth"].view(torch.int16).reshape(-1))
    del fr
    a = buf.numpy()
    shp = (S, H, W)
    ring.append((a[:npx].reshape(shp), a[npx:2 * npx].reshape(shp), a[2 * npx:3 * npx].reshape(shp),
                 a[3 * npx:].view(np.uint16).reshape(shp)))
    keep.append(buf)
outs = [torch.empty(npx, dtype=torch.uint8, pin_memory=True).numpy().reshape(S, H, W)
        for _ in range(2)]
torch.cuda.synchronize()
steps = 12
for chunks in (0, 2, 4, 8, 16, 32, 0):
    p = R.SequenceProcessor(W, H, cfg, streams=S, host_chunks=chunks)
    for k in range(3):
        p.submit(*ring[k % 6], fused=outs[k % 2])
    p.sync()
    t0 = time.perf_counter()
    for k in range(steps):
        p.submit(*ring[k % 6], fused=outs[k % 2])
    p.sync()
    dt = time.perf_counter() - t0
    t1 = time.perf_counter()
    for k in range(4):
        p.process(*ring[k % 6], want=(), out={"fused": outs[k % 2]})
    ds = time.perf_counter() - t1
    print(f"chunks {chunks:3d}: submit {npx * steps / dt / 1e6:9.1f} Mpix/s "
          f"({5 * npx * steps / dt / 1e9:5.1f} GB/s H2D)   process {npx * 4 / ds / 1e6:9.1f} Mpix/s",
          flush=True)
    del p
