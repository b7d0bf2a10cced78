"""Round-2 probe: the practical ceilings K1 and the host path run against.

1. HBM at K1's read/write mix.  MEASURED_PEAKS.json's hbm_gbs is a 1:1 copy;
   K1 moves about 2 bytes read per byte written (68.6 R + 32.7 W B/px).  A
   plain elementwise c = a + b over 4 GiB operands (two streams read, one
   written, all 128-byte coalesced) gives the DRAM rate of that mix; a pure
   read (sum) and the 1:1 copy bracket it.
2. PCIe.  pinned H2D of 393 MB (one streams256 frame, 5 B/px) from ONE
   buffer reused vs a ring of 10 distinct buffers, alone and concurrent with
   a 79 MB D2H on another stream (the e2e pattern).
CUDA events, best of 10.  Prints one JSON line."""
import json

import torch

dev = torch.device("cuda", 0)


def best(fn, reps=10):
    out = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        out.append(s.elapsed_time(e))
    return min(out)


res = {}
n = 1 << 30  # 1 Gi f32 = 4 GiB per operand
a = torch.ones(n, device=dev)
b = torch.ones(n, device=dev)
c = torch.empty(n, device=dev)
fn = lambda: torch.add(a, b, out=c)  # noqa: E731
fn()
ms = best(fn)
res["hbm_add_2r1w_gbs"] = round(3 * 4 * n / ms / 1e6, 1)
ms = best(lambda: c.copy_(a))
res["hbm_copy_1r1w_gbs"] = round(2 * 4 * n / ms / 1e6, 1)
s = torch.empty(1, device=dev)
ms = best(lambda: torch.sum(a, dim=0, out=s.view(())))
res["hbm_read_gbs"] = round(4 * n / ms / 1e6, 1)
del a, b, c
torch.cuda.empty_cache()

nb = 393216000
db = torch.empty(nb, dtype=torch.uint8, device=dev)
dout = torch.empty(nb // 5, dtype=torch.uint8, device=dev)
ring = [torch.empty(nb, dtype=torch.uint8, pin_memory=True) for _ in range(10)]
for r in ring:
    r.fill_(1)
hout = torch.empty(nb // 5, dtype=torch.uint8, pin_memory=True)
s2 = torch.cuda.Stream(dev)


def h2d(k):
    db.copy_(ring[k], non_blocking=True)


ms = best(lambda: [h2d(0) for _ in range(10)], reps=3)
res["h2d_one_buffer_gbs"] = round(10 * nb / ms / 1e6, 1)
ms = best(lambda: [h2d(k) for k in range(10)], reps=3)
res["h2d_ring10_gbs"] = round(10 * nb / ms / 1e6, 1)


def both(k):
    db.copy_(ring[k], non_blocking=True)
    with torch.cuda.stream(s2):
        hout.copy_(dout, non_blocking=True)


def bidir(ks):
    for k in ks:
        both(k)
    torch.cuda.current_stream().wait_stream(s2)


ms = best(lambda: bidir([0] * 10), reps=3)
res["h2d_plus_d2h_one_buffer_h2d_gbs"] = round(10 * nb / ms / 1e6, 1)
ms = best(lambda: bidir(range(10)), reps=3)
res["h2d_plus_d2h_ring10_h2d_gbs"] = round(10 * nb / ms / 1e6, 1)
res["note"] = "GB/s = 1e9 B/s; HBM ops over 4 GiB f32 operands; PCIe 393 MB frames"
print(json.dumps(res))
