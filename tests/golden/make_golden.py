"""Generate tests/golden/ fixtures from the REFERENCE itself.

Runs the unmodified reference library compiled in place (oracle/_ref, built
by `make -C oracle ref` from /root/reference/proj/src) and records:

* pixel_vectors.npz -- per-pixel known-answer vectors: seeded init values and
  observation sequences, the reference's label after every step_pixel and the
  final PixelMixture bytes (mixture.cpp:58-154), for M in {3,4,5} and
  C in {1,3}, including near-band observations.
* scenarios.json   -- per-frame SHA-1 of the rgb / depth / fused masks and the
  SHA-256 of the final colour / depth banks (all float planes + flags) and of
  the fusion state, for SequenceProcessor::process (processor.cpp:158-184) on
  scenario A and B frames (rendered by render_frame, synthetic.cpp:119-195),
  with and without injected depth holes.

Usage:  python tests/golden/make_golden.py      (needs /root/reference)
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

from helpers import SCENARIOS, holes, sha1, sha256  # noqa: E402


def pixel_vectors(ref: O.Ref):
    rng = np.random.default_rng(20241018)
    recs = []
    for M in (3, 4, 5):
        for C in (1, 3):
            cfg = O.color_cfg(M) if C == 3 else O.depth_cfg(M)
            for trial in range(96):
                steps = 1 + trial % 48
                # quantised to 1/8 so the values are exact in float32 and in uint16
                if trial % 3 == 0:
                    vals = rng.integers(0, 256 * 8, size=(steps + 1, C))
                elif trial % 3 == 1:  # mostly stable with occasional jumps
                    base = rng.integers(0, 256 * 8, size=C)
                    vals = base + rng.integers(-24, 25, size=(steps + 1, C))
                    jump = rng.random(steps + 1) < 0.15
                    vals[jump] = rng.integers(0, 256 * 8, size=(int(jump.sum()), C))
                    vals = np.clip(vals, 0, 256 * 8 - 1)
                else:  # depth-like millimetres
                    base = rng.integers(800 * 8, 4000 * 8, size=C)
                    vals = base + rng.integers(-400, 401, size=(steps + 1, C))
                vals = vals.astype(np.uint16)
                v = vals.astype(np.float32) / 8.0
                m = ref.init_mixture(v[0], cfg)
                labels = [ref.step_pixel(m, v[s], cfg) for s in range(1, steps + 1)]
                recs.append((M, C, vals, labels, bytes(m)))
    n = len(recs)
    L = max(len(r[2]) for r in recs)
    values = np.zeros((n, L, 3), np.uint16)
    lengths = np.zeros(n, np.int32)
    labels = np.zeros((n, L), np.uint8)
    meta = np.zeros((n, 2), np.int32)
    final = np.zeros((n, 128), np.uint8)
    for k, (M, C, vals, labs, mb) in enumerate(recs):
        values[k, : len(vals), :C] = vals
        lengths[k] = len(vals)
        labels[k, 1: len(vals)] = labs
        meta[k] = (M, C)
        final[k] = np.frombuffer(mb, np.uint8)
    np.savez_compressed(os.path.join(HERE, "pixel_vectors.npz"), values=values, lengths=lengths,
                        labels=labels, meta=meta, final=final)
    print("pixel_vectors:", n, "sequences")


def scenario_runs(ref: O.Ref):
    out = {}
    for name, scen, w, h, frames, M, with_holes in SCENARIOS:
        sc = O.RefScene(ref, scen, w, h)
        proc = O.RefProcessor(ref, w, h, O.color_cfg(M), O.depth_cfg(M), workers=0)
        hashes = {"rgb": [], "depth": [], "fused": []}
        for f in range(frames):
            fr = sc.render(f)
            d = holes(fr.depth, f) if with_holes else fr.depth
            rgb, dep, fused = proc.process(fr.r, fr.g, fr.b, d)
            hashes["rgb"].append(sha1(rgb))
            hashes["depth"].append(sha1(dep))
            hashes["fused"].append(sha1(fused))
        out[name] = {
            "scenario": scen, "width": w, "height": h, "frames": frames, "components": M,
            "holes": with_holes, "masks": hashes,
            "color_bank": sha256(proc.bank_planes(0), proc.flags(0)),
            "depth_bank": sha256(proc.bank_planes(1), proc.flags(1)),
            "input_sha1_last": sha1(np.concatenate([fr.r.ravel(), fr.g.ravel(), fr.b.ravel(),
                                                    d.view(np.uint8).ravel()])),
        }
        print(name, "done")
    with open(os.path.join(HERE, "scenarios.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    r = O.Ref()
    pixel_vectors(r)
    scenario_runs(r)
