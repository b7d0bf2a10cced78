"""CPU tests: the oracle restatement pinned against the reference's golden
vectors (tests/golden/, generated from the compiled reference) and against
the reference's own unit-test cases (proj/tests/test_mixture.cpp,
test_fusion.cpp, test_segmenter.cpp) restated on the port."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import oracle as O
from helpers import SCENARIOS, holes, sha1, sha256

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_port_pixel_vectors_match_reference_golden(port):
    """Every label and final mixture of 576 reference sequences, bitwise."""
    z = np.load(os.path.join(GOLD, "pixel_vectors.npz"))
    for k in range(len(z["lengths"])):
        M, Ch = z["meta"][k]
        cfg = O.color_cfg(int(M)) if Ch == 3 else O.depth_cfg(int(M))
        L = int(z["lengths"][k])
        v = z["values"][k, :L, :Ch].astype(np.float32) / 8.0
        m = port.init_mixture(v[0], cfg)
        for s in range(1, L):
            assert port.step_pixel(m, v[s], cfg) == z["labels"][k, s], (k, s)
        assert bytes(m) == z["final"][k].tobytes(), k


@pytest.mark.parametrize("name", [s[0] for s in SCENARIOS])
def test_port_scenarios_match_reference_golden(port, name):
    """SequenceProcessor::process (processor.cpp:158-184) restated: every
    per-frame mask hash and the final banks equal the reference's."""
    gold = json.load(open(os.path.join(GOLD, "scenarios.json")))[name]
    _, scen, w, h, frames, M, with_holes = [s for s in SCENARIOS if s[0] == name][0]
    if w * h * frames > 4_000_000:
        frames = min(frames, 8)  # keep the CPU suite short; hashes are per frame
    sc = O.PortScene(port, scen, w, h)
    proc = O.PortProcessor(port, w * h, O.color_cfg(M), O.depth_cfg(M))
    for f in range(frames):
        fr = sc.render(f)
        d = holes(fr.depth, f) if with_holes else fr.depth
        rgb, dep, fused = proc.process(fr.r, fr.g, fr.b, d)
        assert sha1(rgb) == gold["masks"]["rgb"][f], f
        assert sha1(dep) == gold["masks"]["depth"][f], f
        assert sha1(fused) == gold["masks"]["fused"][f], f
    if frames == gold["frames"]:
        assert sha256(proc.color.planes(), proc.color.flags) == gold["color_bank"]
        assert sha256(proc.depth.planes(), proc.depth.flags) == gold["depth_bank"]


def test_port_render_matches_reference(port, ref):
    for name in "AB":
        ps, rs = O.PortScene(port, name, 200, 150, 7), O.RefScene(ref, name, 200, 150, 7)
        for f in (0, 1, 104, 160, 205, 299):
            a, b = ps.render(f), rs.render(f)
            for k in ("r", "g", "b", "depth", "gt"):
                assert np.array_equal(getattr(a, k), getattr(b, k)), (name, f, k)


def test_port_vs_reference_random_sequences(port, ref):
    """Acceptance criterion 2's generator shape (acceptance.cpp:99-119) run
    through both and compared bitwise, with near-threshold values."""
    rng = np.random.default_rng(7)
    for trial in range(3000):
        M = 3 + trial % 3
        Ch = (1, 3, 4)[trial % 3]
        cfg = O.color_cfg(M, learning_rate=float(rng.uniform(0.005, 0.5)))
        seed = rng.uniform(0, 255, Ch).astype(np.float32)
        a, b = port.init_mixture(seed, cfg), ref.init_mixture(seed, cfg)
        for s in range(1 + trial % 25):
            v = rng.uniform(0, 255, Ch).astype(np.float32)
            if s % 4 == 1:  # land right on a band edge of component 0
                sd = np.sqrt(np.float32(a.variances[0]), dtype=np.float32)
                band = np.float32(cfg.match_lambda) * sd
                v = (np.float32(a.means[0]) + band * np.float32(rng.choice([-1, 1]))
                     ).astype(np.float32) * np.ones(Ch, np.float32)
            assert port.step_pixel(a, v, cfg) == ref.step_pixel(b, v, cfg)
            assert bytes(a) == bytes(b)


# ---- reference unit tests (proj/tests/test_mixture.cpp) restated on the port


def _mix(port, v, cfg):
    return port.init_mixture(np.asarray(v, np.float32), cfg)


def test_mixture_init(port):  # test_mixture.cpp:37-55
    c = O.color_cfg()
    m = _mix(port, [120.0], c)
    assert m.means[0] == 120.0 and list(m.weights[:3]) == [1.0, 0.0, 0.0]
    assert all(m.variances[i] == 225.0 for i in range(3))


def test_mixture_invalid_config(port):  # test_mixture.cpp:57-68
    assert port.cfg_check(O.color_cfg(6)) != 0
    assert port.cfg_check(O.color_cfg(learning_rate=1.5)) != 0
    assert port.cfg_check(O.color_cfg(variance_floor=0.0)) != 0
    assert port.cfg_check(O.color_cfg()) == 0


def test_match_band(port):  # test_mixture.cpp:70-85
    c = O.color_cfg()
    m = _mix(port, [100.0], c)
    m.variances[0] = 100.0
    L = port.lib
    assert L.orc_match(C.byref(m), np.array([120.0], np.float32), C.byref(c)) == 0
    assert L.orc_match(C.byref(m), np.array([130.0], np.float32), C.byref(c)) == -1
    assert L.orc_match(C.byref(m), np.array([100.0], np.float32), C.byref(c)) == 0


def test_matched_weight_update(port):  # test_mixture.cpp:87-102
    c = O.color_cfg(learning_rate=0.1)
    m = _mix(port, [50.0], c)
    m.weights[0], m.weights[1], m.weights[2] = 0.5, 0.3, 0.2
    m.means[1] = m.means[2] = 50.0
    port.lib.orc_update(C.byref(m), np.array([50.0], np.float32), 0, C.byref(c))
    assert np.allclose(list(m.weights[:3]), [0.55, 0.27, 0.18], rtol=1e-5)


def test_classify_prefix(port):  # test_mixture.cpp:121-134
    c = O.color_cfg()
    m = _mix(port, [10.0], c)
    m.weights[0], m.weights[1], m.weights[2] = 0.7, 0.2, 0.1
    for i in range(3):
        m.variances[i] = 25.0
    cl = port.lib.orc_classify
    assert cl(C.byref(m), 2, C.byref(c)) == 1
    assert cl(C.byref(m), 1, C.byref(c)) == 0
    assert cl(C.byref(m), 0, C.byref(c)) == 0
    assert cl(C.byref(m), -1, C.byref(c)) == 1


def test_burn_in(port):  # test_mixture.cpp:212-223, acceptance.cpp:121-128
    c = O.color_cfg()
    m = _mix(port, [77.0], c)
    for _ in range(100):
        last = port.step_pixel(m, np.array([77.0], np.float32), c)
    assert last == 0 and m.weights[0] > 0.99


# ---- fusion (proj/tests/test_fusion.cpp:104-125): exhaustive vs literal List 1

def literal_list1(init, seq, limit=3):
    out, cpt, res = init, 0, []
    for r, d in seq:
        if r == d:
            out, cpt = d, 0
        elif cpt == limit:
            out, cpt = r, 0
        elif cpt == -limit:
            out, cpt = d, 0
        elif out == r:
            cpt += 1
        else:
            cpt -= 1
        res.append((out, cpt))
    return res


def exhaustive_fusion_inputs():
    """All 2 x 4^6 length-6 (r, d) sequences, as 8192 pixels x 6 frames."""
    codes = np.arange(4096)
    steps = [((codes >> (2 * s)) & 1, (codes >> (2 * s + 1)) & 1) for s in range(6)]
    init = np.repeat(np.array([0, 1], np.uint8), 4096)
    rgb = np.stack([np.tile(s[0], 2) for s in steps]).astype(np.uint8)
    dep = np.stack([np.tile(s[1], 2) for s in steps]).astype(np.uint8)
    expect_out = np.zeros((6, 8192), np.uint8)
    expect_cpt = np.zeros((6, 8192), np.int8)
    for p in range(8192):
        res = literal_list1(int(init[p]), list(zip(rgb[:, p], dep[:, p])))
        for s, (o, c) in enumerate(res):
            expect_out[s, p], expect_cpt[s, p] = o, c
    return init, rgb, dep, expect_out, expect_cpt


def test_fusion_exhaustive_port(port):
    init, rgb, dep, eo, ec = exhaustive_fusion_inputs()
    out, cpt = init.copy(), np.zeros(8192, np.int8)
    for s in range(6):
        port.lib.orc_fuse(out, cpt, 8192, 3, np.ascontiguousarray(rgb[s]),
                          np.ascontiguousarray(dep[s]))
        assert np.array_equal(out, eo[s]) and np.array_equal(cpt, ec[s])


# ---- registration (registration.cpp:33-78; test_registration.cpp) ----------

def _port_register(port, mask, depth, rig, cw, ch, radius):
    h, w = mask.shape
    out = np.empty(cw * ch, np.uint8)
    scratch = np.empty(cw * ch, np.uint8)
    port.lib.orc_register(np.ascontiguousarray(mask).ravel(), np.ascontiguousarray(depth).ravel(),
                          w, h, rig, cw, ch, radius, scratch, out)
    return out.reshape(ch, cw)


def _ref_register(ref, mask, depth, rig, cw, ch, radius):
    h, w = mask.shape
    out = np.empty(cw * ch, np.uint8)
    ref.check(ref.lib.rref_register_mask(np.ascontiguousarray(mask).ravel(),
                                         np.ascontiguousarray(depth).ravel(), w, h, rig, cw, ch,
                                         radius, out))
    return out.reshape(ch, cw)


def test_port_registration_reference_cases(port):
    ident = O.rig_array([525, 525, 319.5, 239.5], [525, 525, 319.5, 239.5],
                        [1, 0, 0, 0, 1, 0, 0, 0, 1], [0, 0, 0], 1.0)
    rng = np.random.default_rng(4)
    mask = (rng.integers(0, 5, (48, 64)) == 0).astype(np.uint8)
    depth = (500 + rng.integers(0, 3000, (48, 64))).astype(np.uint16)
    assert np.array_equal(_port_register(port, mask, depth, ident, 64, 48, 0), mask)
    off = O.rig_array([500, 500, 320, 240], [500, 500, 320, 240], [1, 0, 0, 0, 1, 0, 0, 0, 1],
                      [50, 0, 0], 1.0)
    one = np.zeros((480, 640), np.uint8)
    one[240, 320] = 1
    out = _port_register(port, one, np.full((480, 640), 1000, np.uint16), off, 640, 480, 0)
    assert out[240, 345] == 1 and out.sum() == 1  # test_registration.cpp:36-48
    assert not _port_register(port, np.ones((16, 16), np.uint8), np.zeros((16, 16), np.uint16),
                              ident, 16, 16, 1).any()
    far = off.copy()
    far[17] = 100000
    assert not _port_register(port, np.ones((48, 64), np.uint8),
                              np.full((48, 64), 1000, np.uint16), far, 64, 48, 0).any()


def test_port_registration_matches_reference(port, ref):
    from helpers import random_rig

    rng = np.random.default_rng(21)
    for trial in range(60):
        w, h = int(rng.integers(20, 90)), int(rng.integers(16, 70))
        rig = random_rig(rng, w, h, big=trial % 3 == 0)
        mask = (rng.random((h, w)) < 0.3).astype(np.uint8)
        depth = rng.integers(0, 5000, (h, w)).astype(np.uint16)
        depth[rng.random((h, w)) < 0.1] = 0
        radius = int(trial % 4)
        a = _port_register(port, mask, depth, rig, w, h, radius)
        b = _ref_register(ref, mask, depth, rig, w, h, radius)
        assert np.array_equal(a, b), trial


def test_port_unregistered_processor_matches_reference(port, ref):
    """processor.cpp:175-179: registration + dilation between the depth bank
    and fusion; 40 frames of scenario A with a rig, M=4."""
    from helpers import random_rig

    rng = np.random.default_rng(8)
    w, h, M = 96, 72, 4
    rig = random_rig(rng, w, h)
    pp = O.PortProcessor(port, w * h, O.color_cfg(M), O.depth_cfg(M), rig=rig, width=w, height=h,
                         radius=2)
    rp = O.RefProcessor(ref, w, h, O.color_cfg(M), O.depth_cfg(M), workers=2, rig=rig, radius=2)
    sc = O.PortScene(port, "A", w, h)
    for f in range(40):
        fr = sc.render(f)
        d = holes(fr.depth, f)
        for x, y in zip(pp.process(fr.r, fr.g, fr.b, d), rp.process(fr.r, fr.g, fr.b, d)):
            assert np.array_equal(x, y), f


def _ref_bank_planes(ref, bank, M, Ch, n):
    out = np.empty((M * Ch + 2 * M, n), np.float32)
    k = 0
    for i in range(M):
        for c in range(Ch):
            ref.check(ref.lib.rref_bank_get(bank, 0, i, c, out[k].ctypes.data))
            k += 1
    for kind in (1, 2):
        for i in range(M):
            ref.check(ref.lib.rref_bank_get(bank, kind, i, 0, out[k].ctypes.data))
            k += 1
    return out


def test_port_augmented_matches_reference(port, ref):
    """segment_augmented (segmenter.cpp:133-147), Augmented4 bank, against
    the compiled reference: scenario A frames incl. depth 0 (no sentinel)."""
    w, h, M = 64, 48, 4
    cfg = O.color_cfg(M)
    bank = ref.lib.rref_bank_create(w, h, 2, C.byref(cfg))
    pb = O.PortBank(port, w * h, 4, cfg)
    sc = O.PortScene(port, "A", w, h)
    for f in range(30):
        fr = sc.render(f)
        d = holes(fr.depth, f)
        rav = [np.ascontiguousarray(x).ravel() for x in (fr.r, fr.g, fr.b, d)]
        mr = np.empty(w * h, np.uint8)
        ref.check(ref.lib.rref_segment_augmented(bank, *rav, 0.0, 4000.0, C.byref(cfg), 1, mr))
        assert np.array_equal(pb.segment_augmented(fr.r, fr.g, fr.b, d), mr), f
    assert pb.planes().tobytes() == _ref_bank_planes(ref, bank, M, 4, w * h).tobytes()
    ref.lib.rref_bank_destroy(bank)


def test_port_match_classify_update_vs_reference(port, ref):
    """The three pieces of step_pixel on their own (mixture.hpp:45-56) --
    match_component, classify with ANY matched index (incl. none), and
    update_mixture with any matched index -- port vs the compiled reference,
    bitwise, on random mid-sequence mixtures."""
    rng = np.random.default_rng(11)
    L = port.lib
    for trial in range(1500):
        M = 3 + trial % 3
        Ch = (1, 3, 4)[trial % 3]
        cfg = O.color_cfg(M, learning_rate=float(rng.uniform(0.005, 0.5)),
                          background_threshold=float(rng.uniform(0.3, 0.95)))
        m = port.init_mixture(rng.uniform(0, 255, Ch).astype(np.float32), cfg)
        for _ in range(trial % 15):
            port.step_pixel(m, rng.uniform(0, 255, Ch).astype(np.float32), cfg)
        v = rng.uniform(0, 255, Ch).astype(np.float32)
        a = O.Mix.from_buffer_copy(m)
        assert L.orc_match(C.byref(a), v, C.byref(cfg)) == ref.match_component(a, v, cfg)
        for mt in range(-1, M):
            assert L.orc_classify(C.byref(a), mt, C.byref(cfg)) == ref.classify(a, mt, cfg)
            x, y = O.Mix.from_buffer_copy(a), O.Mix.from_buffer_copy(a)
            L.orc_update(C.byref(x), v, mt, C.byref(cfg))
            ref.update_mixture(y, v, mt, cfg)
            assert bytes(x) == bytes(y), (trial, mt)
