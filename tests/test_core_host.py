"""CPU tests of the product's per-pixel core source (gmm_pixel.cuh) compiled
for the host, against the oracle: random, near-band, tie and non-finite
mixtures.  The GPU tests check the same source compiled for sm_100a."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "native", "core_host.cpp")


@pytest.fixture(scope="module")
def core(tmp_path_factory):
    so = tmp_path_factory.mktemp("core") / "libcore_host.so"
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
                    "-o", str(so), SRC], check=True)
    lib = C.CDLL(str(so))
    lib.core_step.argtypes = [C.POINTER(O.Mix), np.ctypeslib.ndpointer(np.float32),
                              C.POINTER(O.Cfg)]
    return lib


def step_both(core, port, m_core, m_port, v, cfg):
    v = np.ascontiguousarray(v, np.float32)
    a = core.core_step(C.byref(m_core), v, C.byref(cfg))
    b = port.step_pixel(m_port, v, cfg)
    assert a == b
    assert bytes(m_core) == bytes(m_port)


def clone(m):
    n = O.Mix()
    C.memmove(C.byref(n), C.byref(m), C.sizeof(O.Mix))
    return n


def test_core_random_sequences(core, port):
    rng = np.random.default_rng(3)
    for trial in range(4000):
        M = 3 + trial % 3
        Ch = (1, 3, 4)[(trial // 3) % 3]
        cfg = O.color_cfg(M, learning_rate=float(rng.choice([0.05, 0.01, 0.3])),
                          background_threshold=float(rng.choice([0.8, 0.5, 0.95])))
        m = port.init_mixture(rng.uniform(0, 255, Ch), cfg)
        mc = clone(m)
        for s in range(1 + trial % 40):
            if rng.random() < 0.7:
                v = np.array(m.means[:Ch], np.float32) + rng.normal(0, 4, Ch).astype(np.float32)
            else:
                v = rng.uniform(0, 255, Ch).astype(np.float32)
            step_both(core, port, mc, m, v, cfg)


def test_core_ties_and_band_edges(core, port):
    """Equal fitness (ties keep index order), exact band edges, zero weights
    with dark pixels matching an empty component (mean 0)."""
    cfg = O.color_cfg(5)
    rng = np.random.default_rng(9)
    for trial in range(3000):
        m = O.Mix()
        m.components, m.channels = 5, 3
        ws = rng.choice([0.0, 0.2, 0.25, 0.5], 5).astype(np.float32)
        vs = rng.choice([225.0, 100.0, 16.0, 4.0], 5).astype(np.float32)
        for i in range(5):
            m.weights[i] = ws[i]
            m.variances[i] = vs[i]
            for c in range(3):
                m.means[i * 3 + c] = float(rng.choice([0.0, 10.0, 50.0]))
        i = int(rng.integers(0, 5))
        band = np.float32(2.5) * np.sqrt(np.float32(m.variances[i]), dtype=np.float32)
        v = np.array(m.means[i * 3:i * 3 + 3], np.float32)
        v[int(rng.integers(0, 3))] += band * np.float32(rng.choice([-1, 1, 0.999999, 1.000001]))
        step_both(core, port, clone(m), m, v, cfg)


@pytest.mark.parametrize("bad", ["nan_w", "nan_var", "zero_var", "inf_var", "neg_zero"])
def test_core_non_finite_states(core, port, bad):
    """Uploaded states with NaN/inf/0: the NaN fallback replays the literal
    insertion sort, so even a non-order ranks exactly as the reference."""
    cfg = O.color_cfg(5)
    rng = np.random.default_rng(hash(bad) % 2**32)
    for trial in range(400):
        m = O.Mix()
        m.components, m.channels = 5, 1
        for i in range(5):
            m.weights[i] = float(rng.choice([0.0, 0.1, 0.3, 0.6]))
            m.variances[i] = float(rng.choice([4.0, 9.0, 225.0]))
            m.means[i] = float(rng.uniform(0, 255))
        k = int(rng.integers(0, 5))
        if bad == "nan_w":
            m.weights[k] = float("nan")
        elif bad == "nan_var":
            m.variances[k] = float("nan")
        elif bad == "zero_var":
            m.variances[k] = 0.0
            m.weights[k] = float(rng.choice([0.0, 0.5]))
        elif bad == "inf_var":
            m.variances[k] = float("inf")
        else:
            m.weights[k] = -0.0
        v = np.array([rng.uniform(0, 255)], np.float32)
        mc = clone(m)
        a = core.core_step(C.byref(mc), v, C.byref(cfg))
        b = port.step_pixel(m, v, cfg)
        assert a == b, (bad, trial)
        # NaN payloads may differ between x86 and the GPU; compare NaN-aware
        x = np.frombuffer(bytes(mc), np.float32)[2:]
        y = np.frombuffer(bytes(m), np.float32)[2:]
        assert np.array_equal(x, y, equal_nan=True), (bad, trial)


def test_fuse_select_form_equals_list1(core, port):
    """fuse_pixel_sel (K1's branch-free List 1) == fuse_pixel == the oracle's
    fuse step for every (r, d, out, cpt) and counter limits incl. 0 and
    negatives (fusion.cpp:29-44)."""
    f = core.core_fuse
    f.argtypes = [C.c_int, C.c_uint, C.c_uint, C.c_int, C.POINTER(C.c_uint), C.POINTER(C.c_int)]
    for limit in list(range(-3, 8)) + [100, 127, 128, 200]:
        for r in (0, 1):
            for d in (0, 1):
                for out in (0, 1):
                    for cpt in range(-128, 128):
                        res = []
                        for sel in (0, 1):
                            o, c = C.c_uint(out), C.c_int(cpt)
                            f(sel, r, d, limit, C.byref(o), C.byref(c))
                            res.append((o.value, c.value))
                        assert res[0] == res[1], (limit, r, d, out, cpt, res)
    # and against the oracle's List 1 (orc_fuse) on a plane of random states
    rng = np.random.default_rng(5)
    n = 4096
    for limit in (1, 3, 100):
        out = rng.integers(0, 2, n).astype(np.uint8)
        cpt = rng.integers(-limit, limit + 1, n).astype(np.int8)
        rgb = rng.integers(0, 2, n).astype(np.uint8)
        dep = rng.integers(0, 2, n).astype(np.uint8)
        o2, c2 = out.copy(), cpt.copy()
        port.lib.orc_fuse(o2, c2, n, limit, rgb, dep)
        for i in range(n):
            o, c = C.c_uint(int(out[i])), C.c_int(int(cpt[i]))
            f(1, int(rgb[i]), int(dep[i]), limit, C.byref(o), C.byref(c))
            assert (o.value, c.value) == (int(o2[i]), int(c2[i])), (limit, i)
