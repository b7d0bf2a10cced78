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


def random_rig(rng, w, h, big=False):
    """A valid CameraRig as 21 doubles: pinholes near (w/2, h/2), a small
    Rodrigues rotation (orthonormal to ~1e-16) and a translation in mm."""
    fx, fy = rng.uniform(400, 600, 2)
    cfx, cfy = fx * rng.uniform(0.95, 1.05), fy * rng.uniform(0.95, 1.05)
    dcx, dcy = w / 2 + rng.uniform(-3, 3), h / 2 + rng.uniform(-3, 3)
    ccx, ccy = w / 2 + rng.uniform(-3, 3), h / 2 + rng.uniform(-3, 3)
    axis = rng.normal(size=3)
    axis /= np.linalg.norm(axis)
    ang = rng.uniform(0, 0.2 if big else 0.03)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    Rm = np.eye(3) + np.sin(ang) * K + (1 - np.cos(ang)) * (K @ K)
    t = rng.uniform(-60, 60, 3)
    scale = rng.choice([1.0, 0.5, 1.25])
    return np.ascontiguousarray([fx, fy, dcx, dcy, cfx, cfy, ccx, ccy, *Rm.ravel(), *t, scale],
                                np.float64)
