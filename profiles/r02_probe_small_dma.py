"""Per-frame DMA ceiling of single-VGA host-fed frames (BASELINE configs[1]):
back-to-back pinned H2D copies of one 640x480 RGB-D frame (1.536 MB), alone
and with the 0.3 MB mask read-back on a second stream, vs the e2e rate."""
import json
import torch

n = 640 * 480
reps = 400
src = [torch.empty(5 * n, dtype=torch.uint8, pin_memory=True) for _ in range(4)]
dst = [torch.empty(5 * n, dtype=torch.uint8, device="cuda") for _ in range(2)]
msk = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(2)]
out = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}


def timed(fn):
    for _ in range(20):
        fn(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(reps):
        fn(k)
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps  # us per frame


def h2d(k):
    with torch.cuda.stream(s0 if k % 2 == 0 else s1):
        dst[k % 2].copy_(src[k % 4], non_blocking=True)


def both(k):
    st = s0 if k % 2 == 0 else s1
    with torch.cuda.stream(st):
        dst[k % 2].copy_(src[k % 4], non_blocking=True)
        out[k % 2].copy_(msk[k % 2], non_blocking=True)


res["h2d_1536KB_us"] = round(timed(h2d), 2)
res["h2d_plus_d2h_300KB_us"] = round(timed(both), 2)
res["h2d_gbs"] = round(5 * n / res["h2d_1536KB_us"] / 1e3, 1)
res["vga_fps_dma_bound"] = round(1e6 / res["h2d_plus_d2h_300KB_us"])
res["vga_mpix_s_dma_bound"] = round(n * 1e6 / res["h2d_plus_d2h_300KB_us"] / 1e6, 1)
print(json.dumps(res))
