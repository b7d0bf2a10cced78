"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every
symbol include/rgbdseg_c.h declares, and validates like the reference
(std::invalid_argument <-> RGBDSEG_EINVAL <-> ValueError) without a GPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rgbdseg_c.h")
LIB = os.path.join(ROOT, "paper_2110_14934_b200", "librgbdseg_b200.so")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rgbdseg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("rgbdseg_segment_color", "rgbdseg_segment_depth", "rgbdseg_fusion_step",
                 "rgbdseg_processor_process", "rgbdseg_step_mixtures", "rgbdseg_bank_download"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(LIB)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_every_declared_symbol():
    from paper_2110_14934_b200 import _lib

    assert set(declared_functions()) <= set(_lib.SIGNATURES)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    arches = set(re.findall(r"sm_\d+a?", out.stdout))
    assert arches == {"sm_100a"}, arches


def _ptx_pair(tmp_path):
    """PTX of the kernels under -fmad=false and -fmad=true (two nvcc runs in
    parallel)."""
    src = os.path.join(ROOT, "paper_2110_14934_b200", "csrc", "rgbdseg_kernels.cu")
    runs = {}
    for fmad in ("false", "true"):
        ptx = tmp_path / f"k_{fmad}.ptx"
        runs[fmad] = (ptx, subprocess.Popen(
            ["nvcc", "-arch=sm_100a", "-ptx", "-std=c++17", f"-fmad={fmad}", "-prec-div=true",
             "-prec-sqrt=true", "-ftz=false", src, "-o", str(ptx)],
            stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    out = []
    for fmad in ("false", "true"):
        ptx, pr = runs[fmad]
        _, err = pr.communicate()
        assert pr.returncode == 0, err
        out.append("\n".join(ln for ln in ptx.read_text().splitlines() if not ln.startswith("//")))
    return out


def test_hot_kernels_have_no_contractible_arithmetic(tmp_path):
    """No FMA contraction may touch the GMM arithmetic (SURVEY Appendix A:
    FMA changes 32% of parameter words).  Every op is an explicit _rn
    intrinsic, so the PTX must be byte-identical under -fmad=false and
    -fmad=true; the only FMAs are the explicit ones inside the exact
    division / square-root sequences of gmm_step_fast."""
    strict, loose = _ptx_pair(tmp_path)

    def gmm_entries(ptx):  # the GMM / fusion kernels (not the scene generator)
        parts = re.split(r"(?=\.(?:visible )?\.?entry )", ptx)
        keep = [p for p in parts if re.match(r"\.(?:visible )?\.?entry ", p)
                and re.search(r"k_(fused_ldg|bank_color|bank_depth|bank_aug|mix_step|mix_op|fuse|near)",
                                 p.split("(")[0])]
        return keep

    a, b = gmm_entries(strict), gmm_entries(loose)
    assert len(a) >= 18 + 6 + 2
    assert a == b
    assert "div.rn.f32" in strict and "sqrt.rn.f32" in strict  # generic replay path
    flush = set(re.findall(r"\b[a-z]+(?:\.[a-z]+)*\.ftz\.f32", strict))
    assert flush <= {"rsqrt.approx.ftz.f32", "rcp.approx.ftz.f32"}, flush


def test_config_validation_messages():
    import paper_2110_14934_b200 as R

    R.MixtureConfig().validate()
    cases = [
        (dict(components=6), "components must be in [3,5]"),
        (dict(components=2), "components must be in [3,5]"),
        (dict(learning_rate=1.5), "learning_rate must be in (0,1)"),
        (dict(background_threshold=0.0), "background_threshold must be in (0,1)"),
        (dict(match_lambda=-1.0), "match_lambda must be positive"),
        (dict(initial_sigma=0.0), "initial_sigma must be positive"),
        (dict(initial_weight=1.0), "initial_weight must be in (0,1)"),
        (dict(variance_floor=0.0), "variance_floor must be positive"),
    ]
    for kw, msg in cases:
        with pytest.raises(ValueError, match=re.escape(msg)):
            R.MixtureConfig(**kw).validate()


def test_invalid_handles_rejected_before_touching_a_gpu():
    import paper_2110_14934_b200 as R

    with pytest.raises(ValueError, match="components"):
        R.ModelBank(8, 8, "Color3", R.MixtureConfig(components=7))
    with pytest.raises(ValueError, match="non-positive"):
        R.ModelBank(0, 8, "Color3", R.MixtureConfig())
    with pytest.raises(ValueError, match="counter_limit"):
        R.FusionState(4, 4, counter_limit=0)
    with pytest.raises(ValueError, match="label must be 0 or 1"):
        R.FusionState(4, 4, initial_label=2)
    with pytest.raises(ValueError, match="dimensionality"):
        R.init_mixture([], R.MixtureConfig())


def test_default_config_json_matches_reference_defaults():
    import json

    import paper_2110_14934_b200 as R

    cfg = json.loads(R.default_config_json())
    assert cfg["color_gmm"]["components"] == 3
    assert cfg["depth_gmm"]["learning_rate"] == pytest.approx(0.01)
    assert cfg["depth_gmm"]["initial_sigma"] == 100.0
    assert cfg["fusion"] == {"counter_limit": 3, "initial_label": 0}


def test_aos_soa_helpers_match_reference_layout():
    """aos_to_soa / soa_to_aos (engine.cpp:39-74, module.cpp:121-131): R,G,B
    interleaved <-> planes, the reference's errors."""
    import numpy as np

    import paper_2110_14934_b200 as R

    rng = np.random.default_rng(1)
    f = rng.integers(0, 256, (7, 5, 3), dtype=np.uint8)
    r, g, b = R.aos_to_soa(f)
    flat = f.reshape(-1)
    assert np.array_equal(r.ravel(), flat[0::3]) and np.array_equal(g.ravel(), flat[1::3])
    assert np.array_equal(b.ravel(), flat[2::3])
    assert np.array_equal(R.soa_to_aos(r, g, b), f)
    with pytest.raises(ValueError, match="HxWx3"):
        R.aos_to_soa(np.zeros((4, 4), np.uint8))
    with pytest.raises(ValueError, match="soa_to_aos: dimension mismatch"):
        R.soa_to_aos(r, g, np.zeros((3, 3), np.uint8))


def test_per_pixel_entry_points_reject_null_buffers_before_touching_a_gpu():
    """init/step/match/classify/update over n > 0 records with a null buffer
    return EINVAL (never dereference it), before any CUDA call."""
    import ctypes as C

    from paper_2110_14934_b200 import _lib

    lib = _lib.lib
    cfg = _lib.MixtureCfg()
    lib.rgbdseg_mixture_defaults(C.byref(cfg))
    rec = (_lib.PixelMixtureRec * 2)()
    vals = (C.c_float * 6)()
    lab = (C.c_uint8 * 2)()
    mt = (C.c_int32 * 2)()
    calls = [
        ("init_mixture", lambda: lib.rgbdseg_init_mixtures(None, 3, 2, C.byref(cfg), rec, 0)),
        ("init_mixture", lambda: lib.rgbdseg_init_mixtures(vals, 3, 2, C.byref(cfg), None, 0)),
        ("step_pixel", lambda: lib.rgbdseg_step_mixtures(None, vals, 3, 2, C.byref(cfg), lab, 0)),
        ("step_pixel", lambda: lib.rgbdseg_step_mixtures(rec, None, 3, 2, C.byref(cfg), lab, 0)),
        ("match_component", lambda: lib.rgbdseg_match_components(rec, vals, 3, 2, C.byref(cfg),
                                                                 None, 0)),
        ("classify", lambda: lib.rgbdseg_classify_mixtures(rec, mt, 2, C.byref(cfg), None, 0)),
        ("update_mixture", lambda: lib.rgbdseg_update_mixtures(rec, None, 3, 2, mt, C.byref(cfg),
                                                               0)),
    ]
    for who, call in calls:
        assert call() == _lib.EINVAL, who
        msg = lib.rgbdseg_last_error().decode()
        assert "null buffer" in msg, (who, msg)


def test_null_handles_and_planes_rejected_before_touching_a_gpu():
    """Every handle-taking entry point returns EINVAL on a null handle (the
    reference's methods cannot be called on no object; a C caller can)."""
    import ctypes as C

    from paper_2110_14934_b200 import _lib

    lib = _lib.lib
    buf = (C.c_uint8 * 16)()
    calls = {
        "bank_download": lambda: lib.rgbdseg_bank_download(None, 0, buf),
        "bank_upload": lambda: lib.rgbdseg_bank_upload(None, 0, buf),
        "fusion_step": lambda: lib.rgbdseg_fusion_step(None, buf, buf, None),
        "fusion_download": lambda: lib.rgbdseg_fusion_download(None, buf, None),
        "fusion_upload": lambda: lib.rgbdseg_fusion_upload(None, buf, None),
        "processor_process": lambda: lib.rgbdseg_processor_process(None, buf, buf, buf, buf,
                                                                   None, None, None),
        "processor_submit": lambda: lib.rgbdseg_processor_submit(None, buf, buf, buf, buf,
                                                                 None, None, None),
        "processor_sync": lambda: lib.rgbdseg_processor_sync(None),
    }
    for who, call in calls.items():
        assert call() == _lib.EINVAL, who
        assert "null handle" in lib.rgbdseg_last_error().decode(), who
    assert lib.rgbdseg_processor_color_bank(None) is None
    assert lib.rgbdseg_bank_planes(None) == 0
