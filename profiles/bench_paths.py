"""Measure the SURVEY 8(f) rows beside the headline path (one B200).

    python profiles/bench_paths.py [--streams 64] [--steps 20] [--warmup 5]

Prints one JSON line per row, each on S x 640x480 scenario-A streams rendered
on the GPU (frames 95.. after an untimed pre-roll of frames 0..94, like
bench.py), inputs resident in HBM:

* unregistered -- SequenceProcessor(registered=False): K1 without fusion
  (colour + depth masks written), depth->colour registration splat, square
  dilation (radius 1), k_fuse (processor.cpp:175-180).  CUDA events on the
  processor's stream.
* eval_epilogue -- the fused K1 with ground truth: per-stream TP/FP/TN/FN of
  rgb / depth / fused counted in the kernel (eval.cpp:11-31), against the same
  steps without it.  CUDA events on the processor's stream.
* augmented4 -- ModelBank(Augmented4) + segment_augmented (segmenter.cpp:133-147),
  synchronous calls timed on the host (includes ~10 us of API overhead).

`x_dense_roofline_ceiling` = throughput / (measured HBM GB/s / the path's dense
algorithmic bytes per pixel): how the path compares with a kernel moving every
state word at the measured bandwidth.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2110_14934_b200 as R  # noqa: E402
from paper_2110_14934_b200 import _lib  # noqa: E402

W, H, M, START = 640, 480, 5, 95


def peak_gbs() -> float:
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
        return float(json.load(fh)["hbm_gbs"])


def ptr(t):
    return C.c_void_p(t.data_ptr())


def rig() -> R.CameraRig:
    """A fixed Kinect-like rig (25 mm baseline, 1% focal difference)."""
    c = R.CameraRig.identity()
    c.color_cam = [530.0, 530.0, 320.5, 238.0]
    c.translation_mm = [25.0, 0.0, 0.0]
    return c


def frames(S, first, count, with_gt=False):
    return [R.render_scenario("A", W, H, first + f, streams=S, seed0=1, with_gt=with_gt)
            for f in range(count)]


def preroll(proc, S):
    for f in range(0, START):
        fr = R.render_scenario("A", W, H, f, streams=S, seed0=1)
        torch.cuda.synchronize()
        proc.submit(fr["r"], fr["g"], fr["b"], fr["depth"])
        proc.sync()


def timed(proc, steps, warmup, fn):
    ext = torch.cuda.ExternalStream(proc.stream_handle)
    for k in range(warmup):
        fn(k)
    proc.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    for k in range(steps):
        fn(warmup + k)
    e1.record(ext)
    proc.sync()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def line(row, S, ms, dense_bpp, extra):
    npx = S * W * H
    value = npx / (ms / 1e3) / 1e6
    d = {"row": row, "metric": "RGB-D megapixels/s", "value": round(value, 2), "unit": "Mpix/s",
         "ms_per_step": round(ms, 4), "config": {"streams": S, "width": W, "height": H,
                                                  "components": M, "frames": "95.. after pre-roll"},
         "dense_algorithmic_bytes_per_px": dense_bpp,
         "x_dense_roofline_ceiling": round(value * 1e6 * dense_bpp / 1e9 / peak_gbs(), 3)}
    d.update(extra)
    print(json.dumps(d), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=64)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--rows", default="unregistered,eval_epilogue,augmented4,bank_api")
    args = ap.parse_args()
    rows = set(args.rows.split(","))
    S, n = args.streams, args.steps + args.warmup
    cfg = R.RunConfig.defaults()
    cfg.color_gmm.components = cfg.depth_gmm.components = M
    fr = frames(S, START, n, with_gt=True)
    torch.cuda.synchronize()

    # ---- unregistered: K1 (masks) + splat + dilation + fuse ------------------
    if "unregistered" in rows:
        unregistered(args, S, cfg, fr)
    if "eval_epilogue" in rows:
        eval_epilogue(args, S, n, cfg, fr)
    if "augmented4" in rows:
        augmented4(args, S, n, cfg, fr)
    if "bank_api" in rows:
        bank_api(args, S, n, cfg, fr)


def wall(fn, steps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(steps):
        fn(k)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / steps


def bank_api(args, S, n, cfg, fr):
    """The reference's unfused composition through the bank-level drop-in API
    (segment_color / segment_depth / fuse_step, segmenter.cpp:107-131,
    fusion.cpp:17-46), device frames and masks, each call synchronous."""
    cb = R.ModelBank(W, H, "Color3", cfg.color_gmm, streams=S)
    db = R.ModelBank(W, H, "Depth1", cfg.depth_gmm, streams=S)
    fs = R.FusionState(W, H, streams=S)
    rgb = torch.empty((S, H, W), dtype=torch.uint8, device="cuda")
    dep = torch.empty_like(rgb)
    fused = torch.empty_like(rgb)
    for f in range(0, START):  # the same pre-roll as the processor rows
        g = R.render_scenario("A", W, H, f, streams=S, seed0=1)
        R.segment_color(cb, g["r"], g["g"], g["b"], cfg.color_gmm, out=rgb)
        R.segment_depth(db, g["depth"], cfg.depth_gmm, out=dep)
    for f in range(n):
        R.segment_color(cb, fr[f]["r"], fr[f]["g"], fr[f]["b"], cfg.color_gmm, out=rgb)
        R.segment_depth(db, fr[f]["depth"], cfg.depth_gmm, out=dep)
    k0 = args.warmup
    ms_c = wall(lambda k: R.segment_color(cb, fr[k0 + k]["r"], fr[k0 + k]["g"], fr[k0 + k]["b"],
                                          cfg.color_gmm, out=rgb), args.steps)
    ms_d = wall(lambda k: R.segment_depth(db, fr[k0 + k]["depth"], cfg.depth_gmm, out=dep),
                args.steps)
    ms_f = wall(lambda k: fs.step(rgb, dep, out=fused), args.steps)
    line("segment_color", S, ms_c, 3 + 40 * M + 2 + 1,
         {"kernels": "k_bank_color", "timing": "host wall clock around synchronous calls"})
    line("segment_depth", S, ms_d, 2 + 24 * M + 2 + 1,
         {"kernels": "k_bank_depth", "timing": "host wall clock around synchronous calls"})
    line("fuse_step", S, ms_f, 7,
         {"kernels": "k_fuse16", "timing": "host wall clock around synchronous calls"})


def unregistered(args, S, cfg, fr):
    proc = R.SequenceProcessor(W, H, cfg, streams=S, registered=False, rig=rig())
    preroll(proc, S)
    ms = timed(proc, args.steps, args.warmup,
               lambda k: proc.submit(fr[k]["r"], fr[k]["g"], fr[k]["b"], fr[k]["depth"]))
    # dense K1 bytes without fusion state (-2) plus both masks written (+2), then
    # splat (mask 1 + depth 2 read, zeroed colour mask 1), dilation (2 passes of
    # 1 read + 1 write), k_fuse (rgb, registered, out, cpt read; out, cpt written)
    line("unregistered", S, ms, 331 + 3 + 1 + 4 + 6,
         {"kernels": "K1 (no fusion, masks written) + k_register_splat + k_dilate_pass x2 + k_fuse",
          "timing": "CUDA events on the processor stream"})
    del proc


def eval_epilogue(args, S, n, cfg, fr):
    """Fused K1 with and without ground truth."""
    proc = R.SequenceProcessor(W, H, cfg, streams=S)
    preroll(proc, S)
    # pinned, so the per-frame counts read-back stays asynchronous
    counts = [torch.zeros((S, 3, 4), dtype=torch.int64, pin_memory=True) for _ in range(n)]
    base = timed(proc, args.steps, args.warmup,
                 lambda k: proc.submit(fr[k]["r"], fr[k]["g"], fr[k]["b"], fr[k]["depth"]))
    fn = _lib.lib.rgbdseg_processor_submit_eval

    def with_gt(k):
        f = fr[k]
        _lib.check(fn(C.c_void_p(proc._h), ptr(f["r"]), ptr(f["g"]), ptr(f["b"]), ptr(f["depth"]),
                      ptr(f["gt"]), C.c_void_p(counts[k].data_ptr()), None, None, None),
                   "submit_eval")

    ms = timed(proc, args.steps, args.warmup, with_gt)
    line("eval_epilogue", S, ms, 331 + 1,
         {"kernels": "K1 + fused confusion counts (ballots, per-block shared slots, int64 atomics)",
          "ms_without_eval": round(base, 4), "overhead_pct": round(100 * (ms / base - 1), 2),
          "counts_readback": "per step, S x 3 x 4 int64 into pinned host memory",
          "timing": "CUDA events on the processor stream"})
    del proc


def augmented4(args, S, n, cfg, fr):
    """ModelBank(Augmented4) + segment_augmented."""
    bank = R.ModelBank(W, H, "Augmented4", cfg.color_gmm, streams=S)
    resc = R.DepthRescale(0.0, 4000.0)
    mask = torch.empty((S, H, W), dtype=torch.uint8, device="cuda")
    for f in range(n):
        R.segment_augmented(bank, fr[f]["r"], fr[f]["g"], fr[f]["b"], fr[f]["depth"], resc,
                            cfg.color_gmm, out=mask)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for f in range(args.steps):
        g = fr[(f % n)]
        R.segment_augmented(bank, g["r"], g["g"], g["b"], g["depth"], resc, cfg.color_gmm, out=mask)
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    # reads rgb 3 + depth 2 + state 4*(4+2)*M + flag 2; writes state + mask 1 (dense, K1d)
    line("augmented4", S, ms, 5 + 2 * 24 * M + 2 + 1,
         {"kernels": "k_bank_aug (dense read and write-back)",
          "timing": "host wall clock around synchronous calls"})


if __name__ == "__main__":
    main()
