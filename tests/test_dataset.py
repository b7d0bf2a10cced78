"""CPU tests of the I/O edge and the sequence driver (dataset.cpp,
synthetic.cpp spec handling, engine.hpp run_pipeline), after
proj/tests/test_dataset.cpp and test_engine.cpp."""
import json
import os
import threading
import time

import numpy as np
import pytest

import paper_2110_14934_b200 as R
from paper_2110_14934_b200 import dataset as D
from paper_2110_14934_b200 import synthetic as S


def test_png_round_trips(tmp_path):  # test_dataset.cpp:51-91
    rng = np.random.default_rng(1)
    r, g, b = (rng.integers(0, 256, (12, 17), dtype=np.uint8) for _ in range(3))
    D.save_color(r, g, b, tmp_path / "c.png")
    rr, gg, bb = D.load_color(tmp_path / "c.png")
    assert np.array_equal(rr, r) and np.array_equal(gg, g) and np.array_equal(bb, b)
    d = rng.integers(0, 65536, (12, 17)).astype(np.uint16)
    D.save_depth(d, tmp_path / "d.png")
    assert np.array_equal(D.load_depth(tmp_path / "d.png"), d)
    m = (rng.random((12, 17)) < 0.4).astype(np.uint8)
    D.save_mask(m, tmp_path / "m.png")
    assert np.array_equal(D.load_mask_png(tmp_path / "m.png"), m)
    import cv2

    cv2.imwrite(str(tmp_path / "bad.png"), np.full((4, 4), 7, np.uint8))
    with pytest.raises(RuntimeError, match="non-binary mask value 7"):
        D.load_mask(tmp_path / "bad.png")
    with pytest.raises(RuntimeError, match="not 16-bit"):
        D.load_depth(tmp_path / "m.png")


def test_manifest_round_trip_and_errors(tmp_path):  # test_dataset.cpp:135-179
    rig = R.CameraRig.identity(500, 500, 8, 6)
    rig.translation_mm = [10.0, 0.0, 0.0]
    m = D.SequenceManifest(name="x", frame_count=2, depth_scale=1.0, registered=False,
                           frames=[D.FrameRef(0, "color/0.png", "depth/0.png", "gt/0.png"),
                                   D.FrameRef(1, "color/1.png", "depth/1.png")],
                           calibration=rig)
    D.save_manifest(m, tmp_path / "manifest.json")
    back = D.load_manifest(tmp_path / "manifest.json")
    assert back.name == "x" and back.frame_count == 2 and not back.registered
    assert back.frames[0].gt == "gt/0.png" and back.frames[1].gt == ""
    assert back.calibration.translation_mm == [10.0, 0.0, 0.0]
    j = json.loads((tmp_path / "manifest.json").read_text())
    for mutate, msg in [(lambda j: j.update(frame_count=3), "frame_count does not match"),
                        (lambda j: j["frames"][1].update(index=5), "not contiguous"),
                        (lambda j: j.pop("depth_scale"), "malformed manifest"),
                        (lambda j: j["calibration"].update(rotation=[1, 0]), "wrong arity")]:
            jj = json.loads(json.dumps(j))
            mutate(jj)
            (tmp_path / "bad.json").write_text(json.dumps(jj))
            with pytest.raises(RuntimeError, match=msg):
                D.load_manifest(tmp_path / "bad.json")
    (tmp_path / "junk.json").write_text("{not json")
    with pytest.raises(RuntimeError, match="malformed manifest"):
        D.load_manifest(tmp_path / "junk.json")
    with pytest.raises(RuntimeError, match="cannot open manifest"):
        D.load_manifest(tmp_path / "missing.json")


def test_scenario_specs(tmp_path):  # test_dataset.cpp:181-207, synthetic.cpp:85-117
    a = S.builtin_scenario("A")
    a.validate()
    back = S.spec_from_dict(json.loads(S.scenario_spec_json(a)))
    assert back == a
    with pytest.raises(ValueError, match="known: A, B"):
        S.builtin_scenario("Z")
    bad = json.loads(S.scenario_spec_json(a))
    bad["objects"][0]["waypoints"][1]["x"] = 630
    with pytest.raises(ValueError, match="leaves the frame"):
        S.spec_from_dict(bad)
    bad = json.loads(S.scenario_spec_json(a))
    bad["illumination"][0]["end"] = 400
    with pytest.raises(ValueError, match="illumination event range"):
        S.spec_from_dict(bad)
    assert [S._lround(x) for x in (2.5, -2.5, 0.49999999999999994, 3.4999, -0.5)] == \
        [3, -3, 0, 3, -1]


def test_method_set_parse():  # processor.cpp:105-123
    m = D.MethodSet.parse(["fused"])
    assert m.needs_rgb() and m.needs_depth() and not m.augmented
    with pytest.raises(ValueError, match="known: rgb, depth, fused, augmented"):
        D.MethodSet.parse(["edges"])
    with pytest.raises(ValueError, match="no methods requested"):
        D.MethodSet.parse([])


def test_run_pipeline_order_and_in_flight():  # test_engine.cpp:71-97
    for pipelined in (False, True):
        src = iter(range(40))
        in_flight, peak, lock, emitted = [0], [0], threading.Lock(), []

        def source():
            v = next(src, None)
            if v is not None:
                with lock:
                    in_flight[0] += 1
                    peak[0] = max(peak[0], in_flight[0])
                time.sleep(0.001)
            return v

        def sink(v):
            time.sleep(0.001)
            emitted.append(v)
            with lock:
                in_flight[0] -= 1

        stats = D.run_pipeline(source, lambda v: v * 2, sink, pipelined)
        assert emitted == [2 * v for v in range(40)] and stats["frames_processed"] == 40
        assert peak[0] <= 3


def test_run_pipeline_failing_source_drains_then_raises():  # test_engine.cpp:122-140
    for pipelined in (False, True):
        emitted = []

        def source(state={"i": 0}):
            i = state["i"]
            state["i"] += 1
            if i == 5:
                raise D.SourceError(5, "frame 5: boom")
            return i

        with pytest.raises(D.SourceError) as ei:
            D.run_pipeline(source, lambda v: v, emitted.append, pipelined)
        assert ei.value.frame_index == 5
        assert emitted == [0, 1, 2, 3, 4]


def test_source_errors_carry_frame_index(tmp_path):
    m = D.SequenceManifest(name="x", frame_count=1, frames=[D.FrameRef(0, "c.png", "d.png")],
                           root=str(tmp_path))
    with pytest.raises(D.SourceError) as ei:
        D.load_frame(m, 0)
    assert ei.value.frame_index == 0 and "frame 0" in str(ei.value)
