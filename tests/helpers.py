"""Shared test helpers: golden-scenario table, depth-hole injection, hashes."""
from __future__ import annotations

import hashlib

import numpy as np

# (name, scenario, width, height, frames, M, holes) -- tests/golden/scenarios.json
SCENARIOS = [
    ("A_160x120_M3", "A", 160, 120, 300, 3, False),
    ("A_160x120_M5_holes", "A", 160, 120, 300, 5, True),
    ("B_96x72_M4", "B", 96, 72, 120, 4, False),
    ("A_640x480_M5", "A", 640, 480, 24, 5, True),
]


def holes(depth: np.ndarray, frame: int) -> np.ndarray:
    """Deterministic depth-hole injection (raw 0 = no return, segmenter.cpp:128):
    a rectangle on every 7th frame plus a hashed 1/128 of pixels every frame.
    The synthetic generator never emits 0 (synthetic.cpp:190-191), so parity
    runs need this to exercise the sentinel branch."""
    d = depth.copy()
    h, w = d.shape[-2:]
    if frame % 7 == 3:
        d[..., h // 6: h // 6 + h // 8, w // 5: w // 5 + w // 6] = 0
    n = h * w
    idx = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        key = idx * np.uint64(0x9E3779B97F4A7C15) + np.uint64(frame) * np.uint64(0xBF58476D1CE4E5B9)
    sel = (key >> np.uint64(57)) == 0
    d.reshape(-1, n)[:, sel] = 0
    return d


def sha1(a: np.ndarray) -> str:
    return hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()


def sha256(*arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()
