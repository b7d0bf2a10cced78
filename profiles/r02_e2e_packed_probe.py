"""Round-2 probe: host-fed e2e of planar vs interleaved submits (VGA and
1080p), per-call CPU time and end-to-end frame time, same frames, fresh
processors, alternating order to expose drift."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2110_14934_b200 as R  # noqa: E402


def ring(w, h, n, packed):
    out, keep = [], []
    npx = w * h
    for f in range(n):
        src = R.render_scenario("A", w, h, 95 + f)
        buf = torch.empty(5 * npx, dtype=torch.uint8, pin_memory=True)
        if packed:
            buf[:3 * npx].copy_(torch.stack([src["r"], src["g"], src["b"]], dim=-1).reshape(-1))
        else:
            for i, k in enumerate("rgb"):
                buf[i * npx:(i + 1) * npx].copy_(src[k].reshape(-1))
        buf[3 * npx:].view(torch.int16).copy_(src["depth"].view(torch.int16).reshape(-1))
        a = buf.numpy()
        if packed:
            out.append((a[:3 * npx].reshape(h, w, 3), a[3 * npx:].view(np.uint16).reshape(h, w)))
        else:
            out.append((a[:npx].reshape(h, w), a[npx:2 * npx].reshape(h, w),
                        a[2 * npx:3 * npx].reshape(h, w), a[3 * npx:].view(np.uint16).reshape(h, w)))
        keep.append(buf)
    torch.cuda.synchronize()
    return out, keep


for w, h in ((640, 480), (1920, 1080)):
    n = 150
    cfg = R.RunConfig.defaults()
    cfg.color_gmm.components = cfg.depth_gmm.components = 5
    rings = {k: ring(w, h, n, k == "packed") for k in ("planar", "packed")}
    outs = [torch.empty(w * h, dtype=torch.uint8, pin_memory=True).numpy().reshape(h, w)
            for _ in range(2)]
    for rep in range(2):
        for kind in ("planar", "packed") if rep == 0 else ("packed", "planar"):
            p = R.SequenceProcessor(w, h, cfg)
            fr, _ = rings[kind]
            for k in range(5):
                (p.submit(*fr[k], fused=outs[k % 2]) if kind == "planar"
                 else p.submit_interleaved(*fr[k], fused=outs[k % 2]))
            p.sync()
            cpu = 0.0
            t0 = time.perf_counter()
            for k in range(n):
                c0 = time.perf_counter()
                if kind == "planar":
                    p.submit(*fr[k], fused=outs[k % 2])
                else:
                    p.submit_interleaved(*fr[k], fused=outs[k % 2])
                cpu += time.perf_counter() - c0
            p.sync()
            dt = time.perf_counter() - t0
            print(f"{w}x{h} {kind:7s} rep{rep}: {dt / n * 1e6:8.1f} us/frame, "
                  f"submit CPU {cpu / n * 1e6:6.1f} us, {w * h * n / dt / 1e6:8.1f} Mpix/s",
                  flush=True)
            del p
