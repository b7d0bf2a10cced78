"""Dataset I/O and the sequence driver: the reference's file-based edge.

* manifest + PNG frames (dataset.hpp:16-70, dataset.cpp:23-213) with the same
  JSON schema, PNG formats (colour 8-bit RGB, depth 16-bit gray, masks 8-bit
  {0,255}; OpenCV with compression level 1 like kPngParams) and errors;
* generate_synthetic / generate_scenario (synthetic.cpp:197-230;
  module.cpp:133-148) rendering on the GPU;
* segment_sequence (module.cpp:150-188): the reference's 3-stage pipeline
  (run_pipeline, engine.hpp:54-139) -- PNG decode of frame k+1 and encode of
  frame k-1 on host threads while frame k runs through SequenceProcessor on
  the GPU; emission order = source order; a failing source drains the frames
  in flight, then re-raises with the frame index (SourceError).
"""
from __future__ import annotations

import json
import os
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import rgbdseg as R
from . import synthetic as S

PNG_PARAMS = None  # resolved lazily: [cv2.IMWRITE_PNG_COMPRESSION, 1]


def _cv2():
    import cv2

    global PNG_PARAMS
    if PNG_PARAMS is None:
        PNG_PARAMS = [cv2.IMWRITE_PNG_COMPRESSION, 1]
    return cv2


class SourceError(RuntimeError):
    """SourceError (engine.hpp:28-32): a frame source failure with its index."""

    def __init__(self, frame_index: int, what: str):
        super().__init__(what)
        self.frame_index = frame_index


@dataclass
class FrameRef:
    index: int = 0
    color: str = ""
    depth: str = ""
    gt: str = ""


@dataclass
class SequenceManifest:
    name: str = ""
    frame_count: int = 0
    depth_scale: float = 1.0
    registered: bool = True
    frames: List[FrameRef] = field(default_factory=list)
    calibration: Optional[R.CameraRig] = None
    root: str = ""


@dataclass
class FrameSet:
    index: int
    r: np.ndarray
    g: np.ndarray
    b: np.ndarray
    depth: np.ndarray
    gt: Optional[np.ndarray] = None


def _fail(path, what):
    raise RuntimeError(f"{path}: {what}")


def load_manifest(path) -> SequenceManifest:
    """load_manifest (dataset.cpp:23-74)."""
    path = str(path)
    try:
        with open(path) as fh:
            j = json.load(fh)
    except OSError:
        _fail(path, "cannot open manifest")
    except json.JSONDecodeError as e:
        _fail(path, f"malformed manifest: {e}")
    m = SequenceManifest(root=os.path.dirname(os.path.abspath(path)))
    try:
        m.name = str(j["name"])
        m.frame_count = int(j["frame_count"])
        m.depth_scale = float(j["depth_scale"])
        m.registered = bool(j["registered"])
        for jf in j["frames"]:
            m.frames.append(FrameRef(int(jf["index"]), str(jf["color"]), str(jf["depth"]),
                                     str(jf.get("gt", ""))))
        if "calibration" in j:
            jc = j["calibration"]
            rig = R.CameraRig()
            rig.depth_cam = [float(jc["depth"][k]) for k in ("fx", "fy", "cx", "cy")]
            rig.color_cam = [float(jc["color"][k]) for k in ("fx", "fy", "cx", "cy")]
            rot, tr = list(jc["rotation"]), list(jc["translation_mm"])
            if len(rot) != 9 or len(tr) != 3:
                _fail(path, "calibration rotation/translation have wrong arity")
            rig.rotation, rig.translation_mm = [float(x) for x in rot], [float(x) for x in tr]
            rig.depth_scale = m.depth_scale
            rig.validate()
            m.calibration = rig
    except (KeyError, TypeError) as e:
        _fail(path, f"malformed manifest: {e}")
    if len(m.frames) != m.frame_count:
        _fail(path, "frame_count does not match frames list")
    for i, f in enumerate(m.frames):
        if f.index != i:
            _fail(path, "frame indices are not contiguous from 0")
    return m


def save_manifest(m: SequenceManifest, path):
    """save_manifest (dataset.cpp:76-101)."""
    j = {"name": m.name, "frame_count": m.frame_count, "depth_scale": m.depth_scale,
         "registered": m.registered,
         "frames": [dict({"index": f.index, "color": f.color, "depth": f.depth},
                         **({"gt": f.gt} if f.gt else {})) for f in m.frames]}
    if m.calibration is not None:
        c = m.calibration
        cam = lambda v: dict(zip(("fx", "fy", "cx", "cy"), map(float, v)))  # noqa: E731
        j["calibration"] = {"depth": cam(c.depth_cam), "color": cam(c.color_cam),
                            "rotation": list(c.rotation), "translation_mm": list(c.translation_mm)}
    with open(path, "w") as fh:
        fh.write(json.dumps(j, indent=2) + "\n")


def save_color(r, g, b, path):
    """save_color (dataset.cpp:103-112): BGR-ordered 8-bit PNG."""
    cv2 = _cv2()
    if not cv2.imwrite(str(path), np.dstack([b, g, r]), PNG_PARAMS):
        _fail(path, "failed to write color PNG")


def load_color(path):
    """load_color (dataset.cpp:114-131) -> (r, g, b)."""
    cv2 = _cv2()
    img = cv2.imread(str(path), cv2.IMREAD_COLOR)
    if img is None:
        _fail(path, "cannot decode color PNG")
    return (np.ascontiguousarray(img[:, :, 2]), np.ascontiguousarray(img[:, :, 1]),
            np.ascontiguousarray(img[:, :, 0]))


def save_depth(depth, path):
    cv2 = _cv2()
    if not cv2.imwrite(str(path), np.ascontiguousarray(depth, np.uint16), PNG_PARAMS):
        _fail(path, "failed to write depth PNG")


def load_depth(path):
    """load_depth (dataset.cpp:139-149): 16-bit single channel only."""
    cv2 = _cv2()
    img = cv2.imread(str(path), cv2.IMREAD_UNCHANGED)
    if img is None:
        _fail(path, "cannot decode depth PNG")
    if img.dtype != np.uint16 or img.ndim != 2:
        _fail(path, "depth PNG is not 16-bit single-channel")
    return np.ascontiguousarray(img)


def save_mask(mask, path):
    """save_mask (dataset.cpp:151-158): {0,1} -> {0,255}."""
    cv2 = _cv2()
    if not cv2.imwrite(str(path), (np.asarray(mask) != 0).astype(np.uint8) * 255, PNG_PARAMS):
        _fail(path, "failed to write mask PNG")


def load_mask(path):
    """load_mask (dataset.cpp:160-177): {0,255} -> {0,1}, rejects other values."""
    cv2 = _cv2()
    img = cv2.imread(str(path), cv2.IMREAD_UNCHANGED)
    if img is None:
        _fail(path, "cannot decode mask PNG")
    if img.dtype != np.uint8 or img.ndim != 2:
        _fail(path, "mask PNG is not 8-bit single-channel")
    bad = (img != 0) & (img != 255)
    if bad.any():
        _fail(path, f"non-binary mask value {int(img[bad][0])}")
    return (img == 255).astype(np.uint8)


load_mask_png = load_mask  # module.cpp:190-191


def load_frame(m: SequenceManifest, index: int, want_gt: bool = True) -> FrameSet:
    """load_frame (dataset.cpp:179-199)."""
    if index < 0 or index >= m.frame_count:
        raise IndexError(f"load_frame: frame {index} out of range")
    ref = m.frames[index]
    try:
        r, g, b = load_color(os.path.join(m.root, ref.color))
        d = load_depth(os.path.join(m.root, ref.depth))
        gt = load_mask(os.path.join(m.root, ref.gt)) if (want_gt and ref.gt) else None
    except Exception as e:  # noqa: BLE001
        raise SourceError(index, f"frame {index}: {e}") from e
    if d.shape != r.shape:
        raise SourceError(index, f"frame {index}: color and depth dimensions differ")
    if gt is not None and gt.shape != r.shape:
        raise SourceError(index, f"frame {index}: ground truth dimensions differ")
    return FrameSet(index, r, g, b, d, gt)


class SequenceSource:
    """SequenceSource (dataset.hpp:51-66): ordered frames, nullopt -> None."""

    def __init__(self, manifest: SequenceManifest, want_gt: bool = True):
        self.manifest, self.want_gt, self.cursor, self.shape = manifest, want_gt, 0, None

    def next(self) -> Optional[FrameSet]:
        if self.cursor >= self.manifest.frame_count:
            return None
        fs = load_frame(self.manifest, self.cursor, self.want_gt)
        if self.shape is None:
            self.shape = fs.r.shape
        elif fs.r.shape != self.shape:
            raise SourceError(self.cursor, f"frame {self.cursor}: dimensions differ from frame 0")
        self.cursor += 1
        return fs


def generate_synthetic(spec: S.ScenarioSpec, out_dir, device: int = 0) -> SequenceManifest:
    """generate_synthetic (synthetic.cpp:197-230): PNG frames + manifest."""
    spec.validate()
    for sub in ("color", "depth", "gt"):
        os.makedirs(os.path.join(out_dir, sub), exist_ok=True)
    m = SequenceManifest(name=spec.name, frame_count=spec.frame_count, depth_scale=1.0,
                         registered=True, root=str(out_dir))
    for f in range(spec.frame_count):
        fr = S.render_frame(spec, f, device=device)
        d = fr["depth"][0].view(__import__("torch").int16).cpu().numpy().view(np.uint16)
        r, g, b, gt = (fr[k][0].cpu().numpy() for k in ("r", "g", "b", "gt"))
        name = f"{f:06d}.png"
        ref = FrameRef(f, f"color/{name}", f"depth/{name}", f"gt/{name}")
        save_color(r, g, b, os.path.join(out_dir, ref.color))
        save_depth(d, os.path.join(out_dir, ref.depth))
        save_mask(gt, os.path.join(out_dir, ref.gt))
        m.frames.append(ref)
    save_manifest(m, os.path.join(out_dir, "manifest.json"))
    return m


def generate_scenario(name: str, seed: int, out_dir) -> str:
    """module.cpp:133-141: builtin scenario with a seed -> manifest path."""
    spec = S.builtin_scenario(name)
    spec.seed = int(seed)
    generate_synthetic(spec, out_dir)
    return os.path.join(str(out_dir), "manifest.json")


def generate_scenario_from_spec(spec_json, out_dir) -> str:
    """module.cpp:142-148."""
    generate_synthetic(S.parse_scenario_spec(spec_json), out_dir)
    return os.path.join(str(out_dir), "manifest.json")


@dataclass
class MethodSet:
    """MethodSet (processor.hpp:35-44, parse processor.cpp:105-123)."""

    rgb: bool = False
    depth: bool = False
    fused: bool = False
    augmented: bool = False

    def needs_rgb(self):
        return self.rgb or self.fused

    def needs_depth(self):
        return self.depth or self.fused

    @staticmethod
    def parse(names) -> "MethodSet":
        m = MethodSet()
        for n in names:
            if n not in ("rgb", "depth", "fused", "augmented"):
                raise ValueError(f"unknown method '{n}' (known: rgb, depth, fused, augmented)")
            setattr(m, n, True)
        if not (m.rgb or m.depth or m.fused or m.augmented):
            raise ValueError("no methods requested")
        return m


def run_pipeline(source, process, sink, pipelined: bool = True) -> dict:
    """run_pipeline (engine.hpp:54-139): ingest f+1 || process f || emit f-1,
    order preserving; a SourceError drains the frames in flight first."""
    t0 = time.perf_counter()
    n = 0
    if not pipelined:
        while True:
            fr = source()
            if fr is None:
                break
            sink(process(fr))
            n += 1
    else:
        failure = None
        with ThreadPoolExecutor(max_workers=2) as pool:
            try:
                current = source()
            except Exception as e:  # noqa: BLE001
                current, failure = None, e
            pending = None
            while current is not None and failure is None:
                ingest = pool.submit(source)
                emit = pool.submit(sink, pending) if pending is not None else None
                result = process(current)
                n += 1
                if emit is not None:
                    emit.result()
                pending = result
                try:
                    current = ingest.result()
                except Exception as e:  # noqa: BLE001
                    current, failure = None, e
            if pending is not None:
                sink(pending)
        if failure is not None:
            raise failure
    wall = time.perf_counter() - t0
    return {"frames_processed": n, "wall_seconds": wall, "fps": n / wall if wall > 0 else 0.0}


def segment_sequence(manifest, methods, out_dir, workers: int = 0, pipeline: bool = True,
                     config: Optional[R.RunConfig] = None, device: int = 0) -> dict:
    """segment_sequence (module.cpp:150-188): masks for every frame of a
    manifest written as out_dir/<method>/%06d.png.  `workers` is accepted
    for signature parity (the GPU grid replaces the CPU row split)."""
    m = load_manifest(manifest)
    config = config or R.RunConfig.defaults()
    ms = MethodSet.parse(methods)
    probe = load_frame(m, 0, False)
    h, w = probe.r.shape
    proc = R.SequenceProcessor(w, h, config, device=device, rig=m.calibration,
                               registered=m.registered)
    aug = None
    if ms.augmented:
        aug = R.ModelBank(w, h, "Augmented4", config.augmented_gmm, device=device)
    outputs = [k for k, on in (("rgb", ms.needs_rgb()), ("depth", ms.needs_depth()),
                               ("fused", ms.fused), ("augmented", ms.augmented)) if on]
    for k in outputs:
        os.makedirs(os.path.join(str(out_dir), k), exist_ok=True)
    src = SequenceSource(m, False)

    def process(fr: FrameSet):
        fm = proc.process(fr.r, fr.g, fr.b, fr.depth)
        res = {"index": fr.index, "rgb": fm.rgb, "depth": fm.depth, "fused": fm.fused}
        if aug is not None:
            res["augmented"] = R.segment_augmented(aug, fr.r, fr.g, fr.b, fr.depth,
                                                   config.augmented_depth_range,
                                                   config.augmented_gmm)
        return res

    def sink(res):
        name = f"{res['index']:06d}.png"
        for k in outputs:
            save_mask(res[k], os.path.join(str(out_dir), k, name))

    return run_pipeline(src.next, process, sink, pipeline)
