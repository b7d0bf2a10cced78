"""Python mirror of the reference ``_rgbdseg`` binding for the hot path.

Names, argument meaning and error behaviour follow the reference pybind11
module (/root/reference/proj/python/module.cpp:40-193) and the C++ API it
wraps (include/rgbdseg/{mixture,segmenter,fusion,processor}.hpp).  Everything
computes on the GPU through the C-ABI (include/rgbdseg_c.h); there is no CPU
path.  Additions beyond the reference binding -- which binds no frame-level
API -- are the device banks (``ModelBank``, ``segment_color``,
``segment_depth``), the fused ``SequenceProcessor`` and batched per-pixel
records, all accepting numpy arrays (host) or CUDA tensors (device).
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import check, lib

# ------------------------------------------------------------------ buffers

PIXEL_MIXTURE_DTYPE = np.dtype(
    [("components", "<i4"), ("channels", "<i4"), ("means", "<f4", 20),
     ("variances", "<f4", 5), ("weights", "<f4", 5)], align=True)
assert PIXEL_MIXTURE_DTYPE.itemsize == C.sizeof(_lib.PixelMixtureRec)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _buf(x, dtype, n: int, what: str, writable=False):
    """Raw pointer of a host numpy array or a CUDA tensor holding n elements."""
    if x is None:
        return None
    if _is_torch(x):
        import torch

        want = {np.uint8: torch.uint8, np.uint16: torch.uint16, np.int8: torch.int8,
                np.float32: torch.float32}[dtype]
        if x.dtype != want:
            raise ValueError(f"{what}: expected dtype {want}, got {x.dtype}")
        if not x.is_contiguous() or x.numel() != n:
            raise ValueError(f"{what}: expected a contiguous tensor of {n} elements")
        return x.data_ptr()
    if not isinstance(x, np.ndarray) or x.dtype != dtype or not x.flags.c_contiguous:
        raise ValueError(f"{what}: expected a C-contiguous numpy array of dtype {np.dtype(dtype)}")
    if x.size != n:
        raise ValueError(f"{what}: dimension mismatch ({x.size} elements, expected {n})")
    if writable and not x.flags.writeable:
        raise ValueError(f"{what}: output array is read-only")
    return x.ctypes.data


def _cuda_tensors(*xs):
    return [x for x in xs if x is not None and _is_torch(x) and x.is_cuda]


def _finish_producers(*xs):
    """Synchronous calls on device tensors: the library's streams are
    non-blocking (not ordered with torch's stream), so the producing work on
    the caller's current stream must be complete before the call reads."""
    ts = _cuda_tensors(*xs)
    if ts:
        import torch

        torch.cuda.current_stream(ts[0].device).synchronize()


def _as_host(x, dtype, shape):
    """numpy input coerced like pybind11's forcecast (module.cpp:17)."""
    if _is_torch(x):
        return x
    a = np.ascontiguousarray(x, dtype=dtype)
    if a.shape != tuple(shape) and a.size == int(np.prod(shape)):
        a = a.reshape(shape)
    if a.shape != tuple(shape):
        raise ValueError(f"dimension mismatch: got {a.shape}, expected {tuple(shape)}")
    return a


def _check_mask(m):
    """mask_from_array (module.cpp:31-36): masks must be {0,1}."""
    if isinstance(m, np.ndarray) and m.size and int(m.max()) > 1:
        raise ValueError("mask values must be 0 or 1")


# ------------------------------------------------------------------ configs

@dataclass
class MixtureConfig:
    """MixtureConfig (mixture.hpp:16-26), defaults mixture.hpp:17-23."""

    components: int = 3
    learning_rate: float = 0.05
    match_lambda: float = 2.5
    background_threshold: float = 0.8
    initial_sigma: float = 15.0
    initial_weight: float = 0.05
    variance_floor: float = 4.0

    def _c(self) -> _lib.MixtureCfg:
        return _lib.MixtureCfg(int(self.components), self.learning_rate, self.match_lambda,
                               self.background_threshold, self.initial_sigma,
                               self.initial_weight, self.variance_floor)

    def validate(self):
        """Raises ValueError like MixtureConfig::validate (mixture.cpp:9-24)."""
        c = self._c()
        check(lib.rgbdseg_mixture_validate(C.byref(c)))

    def to_dict(self):
        return {k: getattr(self, k) for k in (
            "components", "learning_rate", "match_lambda", "background_threshold",
            "initial_sigma", "initial_weight", "variance_floor")}


@dataclass
class RunConfig:
    """The RunConfig fields on the hot path (processor.hpp:17-33)."""

    color_gmm: MixtureConfig = field(default_factory=MixtureConfig)
    depth_gmm: MixtureConfig = field(default_factory=MixtureConfig)
    augmented_gmm: MixtureConfig = field(default_factory=MixtureConfig)
    augmented_depth_range: "DepthRescale" = None
    fusion_counter_limit: int = 3
    fusion_initial_label: int = 0
    dilation_radius: int = 1
    warmup_frames: int = 30

    def __post_init__(self):
        if self.augmented_depth_range is None:
            self.augmented_depth_range = DepthRescale()

    @staticmethod
    def defaults() -> "RunConfig":
        """RunConfig::defaults (processor.cpp:35-43): depth adapts slower."""
        c = RunConfig()
        c.depth_gmm.learning_rate = 0.01
        c.depth_gmm.initial_sigma = 100.0
        return c

    def to_json(self) -> str:
        return json.dumps({
            "color_gmm": self.color_gmm.to_dict(),
            "depth_gmm": self.depth_gmm.to_dict(),
            "augmented_gmm": self.augmented_gmm.to_dict(),
            "augmented_depth_range": {"min_mm": self.augmented_depth_range.min_mm,
                                      "max_mm": self.augmented_depth_range.max_mm},
            "fusion": {"counter_limit": self.fusion_counter_limit,
                       "initial_label": self.fusion_initial_label},
            "registration": {"dilation_radius": self.dilation_radius},
            "evaluation": {"warmup_frames": self.warmup_frames},
        }, indent=2)


def default_config_json() -> str:
    """module.cpp:192 (hot-path subset of RunConfig::to_json)."""
    return RunConfig.defaults().to_json()


# ------------------------------------------------------------------ per pixel

class PixelMixture:
    """PixelMixture (mixture.hpp:30-41); read-only view like module.cpp:55-65."""

    __slots__ = ("_rec",)

    def __init__(self, rec: np.ndarray):
        self._rec = rec  # one PIXEL_MIXTURE_DTYPE record (shape ())

    @property
    def components(self) -> int:
        return int(self._rec["components"])

    @property
    def channels(self) -> int:
        return int(self._rec["channels"])

    @property
    def weights(self):
        return [float(x) for x in self._rec["weights"][: self.components]]

    @property
    def variances(self):
        return [float(x) for x in self._rec["variances"][: self.components]]

    @property
    def means(self):
        m, c = self.components, self.channels
        return self._rec["means"][: m * c].reshape(m, c).tolist()

    def raw(self) -> np.ndarray:
        return self._rec

    def __eq__(self, other):
        return isinstance(other, PixelMixture) and self._rec.tobytes() == other._rec.tobytes()


def init_mixtures(values, cfg: MixtureConfig, device: int = 0) -> np.ndarray:
    """Batched init_mixture (mixture.cpp:58-72) on the GPU: values[n, C] ->
    n PIXEL_MIXTURE_DTYPE records."""
    v = np.ascontiguousarray(values, dtype=np.float32)
    if v.ndim == 1:
        v = v[None, :]
    n, ch = v.shape
    out = np.zeros(n, PIXEL_MIXTURE_DTYPE)
    c = cfg._c()
    check(lib.rgbdseg_init_mixtures(v.ctypes.data, ch, n, C.byref(c), out.ctypes.data, device))
    return out


def step_mixtures(recs: np.ndarray, values, cfg: MixtureConfig, device: int = 0) -> np.ndarray:
    """Batched step_pixel (mixture.cpp:148-154) on the GPU, in place.
    Returns uint8 labels (1 = Foreground)."""
    if recs.dtype != PIXEL_MIXTURE_DTYPE or not recs.flags.c_contiguous:
        raise ValueError("records must be a contiguous PIXEL_MIXTURE_DTYPE array")
    v = np.ascontiguousarray(values, dtype=np.float32)
    n = recs.size
    if v.ndim == 1:
        v = v.reshape(n, -1)
    if v.shape[0] != n:
        raise ValueError("one observation per record expected")
    labels = np.empty(n, np.uint8)
    c = cfg._c()
    check(lib.rgbdseg_step_mixtures(recs.ctypes.data, v.ctypes.data, v.shape[1], n, C.byref(c),
                                    labels.ctypes.data, device))
    return labels


def init_mixture(first_value, cfg: MixtureConfig) -> PixelMixture:
    """init_mixture (module.cpp:67-69): list of 1..4 floats."""
    v = np.asarray(list(first_value), dtype=np.float32)
    if v.size < 1 or v.size > 4:
        raise ValueError("init_mixture: bad observation dimensionality")
    return PixelMixture(init_mixtures(v[None, :], cfg)[0:1].reshape(()))


def step_pixel(mix: PixelMixture, value, cfg: MixtureConfig) -> int:
    """step_pixel (module.cpp:70-73): updates `mix` in place, returns 1 = FG."""
    v = np.asarray(list(value), dtype=np.float32)
    if v.size != mix.channels:
        raise ValueError("step_pixel: observation dimensionality does not match the mixture")
    rec = mix._rec.reshape(1)
    lab = step_mixtures(rec, v[None, :], cfg)
    return int(lab[0])


def _recs_values(recs, values):
    if recs.dtype != PIXEL_MIXTURE_DTYPE or not recs.flags.c_contiguous:
        raise ValueError("records must be a contiguous PIXEL_MIXTURE_DTYPE array")
    n = recs.size
    v = np.ascontiguousarray(values, dtype=np.float32)
    if v.ndim == 1:
        v = v.reshape(n, -1)
    if v.shape[0] != n:
        raise ValueError("one observation per record expected")
    return n, v


def _matched_array(matched, n):
    m = np.ascontiguousarray(
        [-1 if x is None else int(x) for x in matched] if isinstance(matched, (list, tuple))
        else matched, dtype=np.int32).reshape(-1)
    if m.size != n:
        raise ValueError("one matched index per record expected")
    return m


def match_components(recs: np.ndarray, values, cfg: MixtureConfig, device: int = 0) -> np.ndarray:
    """Batched match_component (mixture.cpp:74-92) on the GPU: int32 index of
    each record's matched component, -1 for none (std::nullopt)."""
    n, v = _recs_values(recs, values)
    out = np.empty(n, np.int32)
    c = cfg._c()
    check(lib.rgbdseg_match_components(recs.ctypes.data, v.ctypes.data, v.shape[1], n,
                                       C.byref(c), out.ctypes.data, device))
    return out


def classify_mixtures(recs: np.ndarray, matched, cfg: MixtureConfig, device: int = 0) -> np.ndarray:
    """Batched classify (mixture.cpp:133-146) on the GPU: uint8 labels (1 = FG)."""
    if recs.dtype != PIXEL_MIXTURE_DTYPE or not recs.flags.c_contiguous:
        raise ValueError("records must be a contiguous PIXEL_MIXTURE_DTYPE array")
    n = recs.size
    m = _matched_array(matched, n)
    out = np.empty(n, np.uint8)
    c = cfg._c()
    check(lib.rgbdseg_classify_mixtures(recs.ctypes.data, m.ctypes.data, n, C.byref(c),
                                        out.ctypes.data, device))
    return out


def update_mixtures(recs: np.ndarray, values, matched, cfg: MixtureConfig, device: int = 0):
    """Batched update_mixture (mixture.cpp:94-131) on the GPU, in place."""
    n, v = _recs_values(recs, values)
    m = _matched_array(matched, n)
    c = cfg._c()
    check(lib.rgbdseg_update_mixtures(recs.ctypes.data, v.ctypes.data, v.shape[1], n,
                                      m.ctypes.data, C.byref(c), device))


def match_component(mix: PixelMixture, value, cfg: MixtureConfig) -> Optional[int]:
    """match_component (mixture.hpp:45-48): index of the first component, in
    decreasing w/sigma order, within lambda*sigma in every channel; None if
    there is none."""
    v = np.asarray(list(value), dtype=np.float32)
    if v.size != mix.channels:
        raise ValueError("match_component: observation dimensionality does not match the mixture")
    i = int(match_components(mix._rec.reshape(1), v[None, :], cfg)[0])
    return None if i < 0 else i


def classify(mix: PixelMixture, matched: Optional[int], cfg: MixtureConfig) -> int:
    """classify (mixture.hpp:53-56): 1 = Foreground, 0 = Background."""
    return int(classify_mixtures(mix._rec.reshape(1), [matched], cfg)[0])


def update_mixture(mix: PixelMixture, value, matched: Optional[int], cfg: MixtureConfig) -> None:
    """update_mixture (mixture.hpp:50-51), in place."""
    v = np.asarray(list(value), dtype=np.float32)
    if v.size != mix.channels:
        raise ValueError("update_mixture: observation dimensionality does not match the mixture")
    update_mixtures(mix._rec.reshape(1), v[None, :], [matched], cfg)


# ------------------------------------------------------------------ banks

class BankMode:
    Color3 = _lib.COLOR3
    Depth1 = _lib.DEPTH1
    Augmented4 = _lib.AUGMENTED4


@dataclass
class DepthRescale:
    """DepthRescale (segmenter.hpp:17-21): metric depth onto 0..255."""

    min_mm: float = 0.0
    max_mm: float = 4000.0


class ModelBank:
    """Device-resident ModelBank (segmenter.hpp:25-55) over `streams` frames
    of width x height.  Plane accessors return host copies (the reference
    returns mutable Plane& references; use ``upload_plane`` to write)."""

    def __init__(self, width: int, height: int, mode, cfg: MixtureConfig, streams: int = 1,
                 device: int = 0, _borrowed=None):
        if isinstance(mode, str):
            mode = {"Color3": _lib.COLOR3, "Depth1": _lib.DEPTH1,
                    "Augmented4": _lib.AUGMENTED4}[mode]
        self.width, self.height, self.streams, self.mode = width, height, streams, mode
        self.channels = {_lib.COLOR3: 3, _lib.DEPTH1: 1, _lib.AUGMENTED4: 4}[mode]
        self.device = device
        self._owner = None
        if _borrowed is not None:
            self._h, self._owner = _borrowed
            self.components = lib.rgbdseg_bank_planes(self._h) // (self.channels + 2)
            return
        self.components = int(cfg.components)
        h = C.c_void_p()
        c = cfg._c()
        check(lib.rgbdseg_bank_create(width, height, streams, mode, C.byref(c), device,
                                      C.byref(h)), "ModelBank")
        self._h = h.value

    def __del__(self):
        if getattr(self, "_h", None) and self._owner is None:
            lib.rgbdseg_bank_destroy(self._h)
            self._h = None

    @property
    def npx(self) -> int:
        return self.width * self.height * self.streams

    def _shape(self):
        return (self.height, self.width) if self.streams == 1 else (
            self.streams, self.height, self.width)

    def plane_id_mean(self, i, c):
        return i * self.channels + c

    def plane_id_variance(self, i):
        return self.components * self.channels + i

    def plane_id_weight(self, i):
        return self.components * self.channels + self.components + i

    def download_plane(self, pid: int) -> np.ndarray:
        dt = np.uint8 if pid == _lib.FLAGS_PLANE else np.float32
        out = np.empty(self._shape(), dt)
        check(lib.rgbdseg_bank_download(self._h, pid, out.ctypes.data))
        return out

    def upload_plane(self, pid: int, arr):
        dt = np.uint8 if pid == _lib.FLAGS_PLANE else np.float32
        a = _as_host(arr, dt, self._shape())
        _finish_producers(a)
        check(lib.rgbdseg_bank_upload(self._h, pid, _buf(a, dt, self.npx, "plane")))

    def mean_plane(self, component: int, channel: int) -> np.ndarray:
        return self.download_plane(self.plane_id_mean(component, channel))

    def variance_plane(self, component: int) -> np.ndarray:
        return self.download_plane(self.plane_id_variance(component))

    def weight_plane(self, component: int) -> np.ndarray:
        return self.download_plane(self.plane_id_weight(component))

    def initialized_plane(self) -> np.ndarray:
        return self.download_plane(_lib.FLAGS_PLANE)

    def planes(self) -> np.ndarray:
        """All float planes in ModelBank order, shape (M*C + 2M, npx)."""
        P = lib.rgbdseg_bank_planes(self._h)
        out = np.empty((P, self.npx), np.float32)
        for p in range(P):
            check(lib.rgbdseg_bank_download(self._h, p, out[p].ctypes.data))
        return out

    def gather(self, x: int, y: int, stream: int = 0) -> PixelMixture:
        """ModelBank::gather (segmenter.cpp:36-47)."""
        j = (stream * self.height + y) * self.width + x
        P = self.planes()[:, j]
        rec = np.zeros((), PIXEL_MIXTURE_DTYPE)
        M, Ch = self.components, self.channels
        rec["components"], rec["channels"] = M, Ch
        rec["means"][: M * Ch] = P[: M * Ch]
        rec["variances"][:M] = P[M * Ch: M * Ch + M]
        rec["weights"][:M] = P[M * Ch + M:]
        return PixelMixture(rec)

    def is_initialized(self, x: int, y: int, stream: int = 0) -> bool:
        return bool(self.initialized_plane().reshape(-1)[(stream * self.height + y) * self.width + x])

    def state_equals(self, other: "ModelBank") -> bool:
        """ModelBank::state_equals (segmenter.cpp:58-63), bitwise."""
        return (self.width == other.width and self.height == other.height
                and self.streams == other.streams and self.mode == other.mode
                and self.components == other.components
                and self.planes().tobytes() == other.planes().tobytes()
                and np.array_equal(self.initialized_plane(), other.initialized_plane()))


def _mask_out(out, n, shape):
    if out is None:
        return np.empty(shape, np.uint8), None
    return out, out


def segment_color(bank: ModelBank, r, g, b, cfg: MixtureConfig, workers: int = 1, out=None):
    """segment_color (segmenter.cpp:107-119) on the GPU.  `workers` is
    accepted for signature parity; the CUDA grid replaces the row split."""
    shp = bank._shape()
    r, g, b = (_as_host(x, np.uint8, shp) for x in (r, g, b))
    mask, _ = _mask_out(out, bank.npx, shp)
    c = cfg._c()
    _finish_producers(r, g, b, mask)
    check(lib.rgbdseg_segment_color(bank._h, _buf(r, np.uint8, bank.npx, "segment_color(r)"),
                                    _buf(g, np.uint8, bank.npx, "segment_color(g)"),
                                    _buf(b, np.uint8, bank.npx, "segment_color(b)"), C.byref(c),
                                    _buf(mask, np.uint8, bank.npx, "mask", True)))
    return mask


def segment_depth(bank: ModelBank, depth_mm, cfg: MixtureConfig, workers: int = 1, out=None):
    """segment_depth (segmenter.cpp:121-131) on the GPU; raw 0 = no return."""
    shp = bank._shape()
    d = _as_host(depth_mm, np.uint16, shp)
    mask, _ = _mask_out(out, bank.npx, shp)
    c = cfg._c()
    _finish_producers(d, mask)
    check(lib.rgbdseg_segment_depth(bank._h, _buf(d, np.uint16, bank.npx, "segment_depth"),
                                    C.byref(c), _buf(mask, np.uint8, bank.npx, "mask", True)))
    return mask


def segment_augmented(bank: ModelBank, r, g, b, depth_mm, rescale: DepthRescale,
                      cfg: MixtureConfig, workers: int = 1, out=None):
    """segment_augmented (segmenter.cpp:133-147) on the GPU."""
    shp = bank._shape()
    r, g, b = (_as_host(x, np.uint8, shp) for x in (r, g, b))
    d = _as_host(depth_mm, np.uint16, shp)
    mask, _ = _mask_out(out, bank.npx, shp)
    c = cfg._c()
    _finish_producers(r, g, b, d, mask)
    check(lib.rgbdseg_segment_augmented(
        bank._h, _buf(r, np.uint8, bank.npx, "segment_augmented(r)"),
        _buf(g, np.uint8, bank.npx, "segment_augmented(g)"),
        _buf(b, np.uint8, bank.npx, "segment_augmented(b)"),
        _buf(d, np.uint16, bank.npx, "segment_augmented(depth)"), float(rescale.min_mm),
        float(rescale.max_mm), C.byref(c), _buf(mask, np.uint8, bank.npx, "mask", True)))
    return mask


# ------------------------------------------------------------------ fusion

class FusionState:
    """FusionState + reset_state + fuse_step (fusion.hpp:11-23, module.cpp:75-90)."""

    def __init__(self, width: int, height: int, initial_label: int = 0, counter_limit: int = 3,
                 streams: int = 1, device: int = 0, _borrowed=None):
        self.width, self.height, self.streams = width, height, streams
        self._owner = None
        if _borrowed is not None:
            self._h, self._owner = _borrowed
            return
        h = C.c_void_p()
        check(lib.rgbdseg_fusion_create(width, height, streams, int(initial_label),
                                        int(counter_limit), device, C.byref(h)), "FusionState")
        self._h = h.value

    def __del__(self):
        if getattr(self, "_h", None) and self._owner is None:
            lib.rgbdseg_fusion_destroy(self._h)
            self._h = None

    def _shape(self):
        return (self.height, self.width) if self.streams == 1 else (
            self.streams, self.height, self.width)

    @property
    def npx(self):
        return self.width * self.height * self.streams

    def step(self, rgb, depth, out=None):
        shp = self._shape()
        rgb, depth = _as_host(rgb, np.uint8, shp), _as_host(depth, np.uint8, shp)
        _check_mask(rgb)
        _check_mask(depth)
        res, _ = _mask_out(out, self.npx, shp)
        _finish_producers(rgb, depth, res)
        check(lib.rgbdseg_fusion_step(self._h, _buf(rgb, np.uint8, self.npx, "fuse_step(rgb)"),
                                      _buf(depth, np.uint8, self.npx, "fuse_step(depth)"),
                                      _buf(res, np.uint8, self.npx, "out", True)))
        return res

    @property
    def out(self) -> np.ndarray:
        o = np.empty(self._shape(), np.uint8)
        check(lib.rgbdseg_fusion_download(self._h, o.ctypes.data, None))
        return o

    @property
    def cpt(self) -> np.ndarray:
        c = np.empty(self._shape(), np.int8)
        check(lib.rgbdseg_fusion_download(self._h, None, c.ctypes.data))
        return c

    def upload(self, out=None, cpt=None):
        shp = self._shape()
        o = _as_host(out, np.uint8, shp) if out is not None else None
        c = _as_host(cpt, np.int8, shp) if cpt is not None else None
        check(lib.rgbdseg_fusion_upload(self._h, _buf(o, np.uint8, self.npx, "out"),
                                        _buf(c, np.int8, self.npx, "cpt")))


def fuse_step(state: FusionState, rgb_mask, depth_mask_registered):
    """fuse_step (fusion.cpp:17-46): returns a copy of state.out."""
    return state.step(rgb_mask, depth_mask_registered)


def reset_state(width: int, height: int, initial_label: int = 0, counter_limit: int = 3):
    """reset_state (fusion.cpp:7-15)."""
    return FusionState(width, height, initial_label, counter_limit)


# ------------------------------------------------------------------ registration

class CameraRig:
    """CameraRig (registration.hpp:16-26; module.cpp:92-98): depth and colour
    pinholes, row-major rotation, translation in mm, depth_scale."""

    def __init__(self):
        self.depth_cam = [0.0, 0.0, 0.0, 0.0]  # fx, fy, cx, cy
        self.color_cam = [0.0, 0.0, 0.0, 0.0]
        self.rotation = [1.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0]
        self.translation_mm = [0.0, 0.0, 0.0]
        self.depth_scale = 1.0

    @staticmethod
    def identity(fx=525.0, fy=525.0, cx=319.5, cy=239.5) -> "CameraRig":
        r = CameraRig()
        r.depth_cam = [fx, fy, cx, cy]
        r.color_cam = [fx, fy, cx, cy]
        return r

    def _c(self) -> _lib.CameraRigC:
        c = _lib.CameraRigC()
        c.depth_fx, c.depth_fy, c.depth_cx, c.depth_cy = map(float, self.depth_cam)
        c.color_fx, c.color_fy, c.color_cx, c.color_cy = map(float, self.color_cam)
        for i in range(9):
            c.rotation[i] = float(self.rotation[i])
        for i in range(3):
            c.translation_mm[i] = float(self.translation_mm[i])
        c.depth_scale = float(self.depth_scale)
        return c

    def validate(self):
        c = self._c()
        check(lib.rgbdseg_camera_rig_validate(C.byref(c)))


def register_mask(mask, depth, rig: CameraRig, dilation_radius: int = 1, color_width=None,
                  color_height=None, device: int = 0):
    """register_mask (registration.cpp:50-78; module.cpp:100-110) on the GPU:
    the colour-grid mask of the foreground depth pixels, dilated."""
    _check_mask(mask)
    m = _as_host(mask, np.uint8, np.shape(mask))
    h, w = m.shape[-2:]
    d = _as_host(depth, np.uint16, (h, w))
    cw, ch = color_width or w, color_height or h
    out = np.empty((ch, cw), np.uint8)
    c = rig._c()
    check(lib.rgbdseg_register_mask(_buf(m, np.uint8, w * h, "mask"),
                                    _buf(d, np.uint16, w * h, "depth"), w, h, C.byref(c), cw, ch,
                                    int(dilation_radius), out.ctypes.data, device))
    return out


def dilate_mask(mask, radius: int, device: int = 0):
    """dilate_mask (registration.cpp:33-48) on the GPU."""
    m = _as_host(mask, np.uint8, np.shape(mask))
    h, w = m.shape[-2:]
    out = np.empty((h, w), np.uint8)
    check(lib.rgbdseg_dilate_mask(_buf(m, np.uint8, w * h, "mask"), w, h, int(radius),
                                  out.ctypes.data, device))
    return out


# ------------------------------------------------------------------ processor

@dataclass
class FrameMasks:
    """FrameMasks (processor.hpp:46-53) for the fused method.  `counts`
    (with ground truth): int64 [streams, 3 (rgb, depth, fused), 4 (tp, fp,
    tn, fn)] from the kernel's evaluation epilogue."""

    index: int
    rgb: Optional[object] = None
    depth: Optional[object] = None
    fused: Optional[object] = None
    counts: Optional[np.ndarray] = None


class SequenceProcessor:
    """SequenceProcessor (processor.hpp:60-80) for the fused method on a
    registered sequence, over `streams` independent camera streams batched
    into one fused kernel per step."""

    def __init__(self, width: int, height: int, config: Optional[RunConfig] = None,
                 streams: int = 1, device: int = 0, variant: str = "auto", host_chunks: int = 0,
                 rig: Optional[CameraRig] = None, registered: bool = True):
        config = config or RunConfig.defaults()
        self.width, self.height, self.streams, self.device = width, height, streams, device
        self.config = config
        pc = _lib.ProcessorCfg()
        lib.rgbdseg_processor_defaults(C.byref(pc), width, height)
        pc.streams = streams
        pc.color = config.color_gmm._c()
        pc.depth = config.depth_gmm._c()
        pc.fusion_counter_limit = int(config.fusion_counter_limit)
        pc.fusion_initial_label = int(config.fusion_initial_label)
        pc.device = device
        pc.host_chunks = host_chunks
        pc.registered = 1 if registered else 0
        pc.dilation_radius = int(config.dilation_radius)
        if not registered:
            if rig is None:  # processor.cpp:131-132
                raise ValueError("unregistered sequence requires calibration")
            pc.rig = rig._c()
        h = C.c_void_p()
        check(lib.rgbdseg_processor_create(C.byref(pc), C.byref(h)), "SequenceProcessor")
        self._h = h.value
        self.set_variant(variant)
        self._color = ModelBank(width, height, _lib.COLOR3, None, streams, device,
                                _borrowed=(lib.rgbdseg_processor_color_bank(self._h), self))
        self._depth = ModelBank(width, height, _lib.DEPTH1, None, streams, device,
                                _borrowed=(lib.rgbdseg_processor_depth_bank(self._h), self))
        self._fusion = FusionState(width, height, streams=streams, device=device,
                                   _borrowed=(lib.rgbdseg_processor_fusion(self._h), self))
        self._keep = []

    def __del__(self):
        if getattr(self, "_h", None):
            lib.rgbdseg_processor_destroy(self._h)
            self._h = None

    @property
    def npx(self):
        return self.width * self.height * self.streams

    def _shape(self):
        return (self.height, self.width) if self.streams == 1 else (
            self.streams, self.height, self.width)

    def set_near_threshold(self, rel: float = 1e-5):
        """Turn on (rel > 0) or off (0) the near-threshold report and zero
        its counters (see rgbdseg_processor_set_near_threshold)."""
        check(lib.rgbdseg_processor_set_near_threshold(self._h, float(rel)))

    def near_threshold_counts(self) -> dict:
        """{'color': n, 'depth': n, 'pixel_frames': n} since set_near_threshold."""
        c, d, n = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib.rgbdseg_processor_near_threshold_counts(self._h, C.byref(c), C.byref(d),
                                                          C.byref(n)))
        return {"color": c.value, "depth": d.value, "pixel_frames": n.value}

    def set_variant(self, variant: str):
        check(lib.rgbdseg_processor_set_variant(self._h, _lib.VARIANTS[variant]))

    def color_bank(self) -> ModelBank:
        return self._color

    def depth_bank(self) -> ModelBank:
        return self._depth

    def fusion_state(self) -> FusionState:
        return self._fusion

    @property
    def stream_handle(self) -> int:
        return lib.rgbdseg_processor_stream(self._h) or 0

    @property
    def frames(self) -> int:
        return int(lib.rgbdseg_processor_frames(self._h))

    def _args(self, r, g, b, depth, fused, rgb, dep):
        shp, n = self._shape(), self.npx
        r, g, b = (_as_host(x, np.uint8, shp) for x in (r, g, b))
        depth = _as_host(depth, np.uint16, shp)
        ptrs = [_buf(r, np.uint8, n, "process(r)"), _buf(g, np.uint8, n, "process(g)"),
                _buf(b, np.uint8, n, "process(b)"), _buf(depth, np.uint16, n, "process(depth)"),
                _buf(fused, np.uint8, n, "fused", True), _buf(rgb, np.uint8, n, "rgb", True),
                _buf(dep, np.uint8, n, "depth_mask", True)]
        return ptrs, (r, g, b, depth)

    def process(self, r, g, b, depth, want=("rgb", "depth", "fused"), out=None,
                gt=None) -> FrameMasks:
        """SequenceProcessor::process (processor.cpp:158-184), synchronous.
        `out` may map 'rgb'/'depth'/'fused' to preallocated arrays/tensors.
        With `gt` (ground-truth masks) the kernel also returns the frame's
        confusion counts (eval.cpp:11-31) without the masks leaving the GPU."""
        out = dict(out or {})
        shp = self._shape()
        for k in want:
            if k not in out:
                out[k] = np.empty(shp, np.uint8)
        ptrs, keep = self._args(r, g, b, depth, out.get("fused"), out.get("rgb"), out.get("depth"))
        _finish_producers(*keep, out.get("fused"), out.get("rgb"), out.get("depth"), gt)
        idx = self.frames
        if gt is None:
            check(lib.rgbdseg_processor_process(self._h, *ptrs), "process")
            return FrameMasks(idx, out.get("rgb"), out.get("depth"), out.get("fused"))
        gt = _as_host(gt, np.uint8, shp)
        _check_mask(gt)
        counts = np.zeros((self.streams, 3, 4), np.int64)
        check(lib.rgbdseg_processor_process_eval(self._h, *ptrs[:4],
                                                 _buf(gt, np.uint8, self.npx, "gt"),
                                                 counts.ctypes.data, *ptrs[4:]), "process")
        return FrameMasks(idx, out.get("rgb"), out.get("depth"), out.get("fused"), counts)

    def _packed_args(self, rgb, depth, order, fused, rgbm, depm):
        n = self.npx
        if order not in ("rgb", "bgr"):
            raise ValueError("order must be 'rgb' or 'bgr'")
        shp = self._shape()
        rgb = _as_host(rgb, np.uint8, (*shp, 3))
        depth = _as_host(depth, np.uint16, shp)
        ptrs = [_buf(rgb, np.uint8, 3 * n, "process(rgb interleaved)"),
                _lib.ORDER[order], _buf(depth, np.uint16, n, "process(depth)"),
                _buf(fused, np.uint8, n, "fused", True), _buf(rgbm, np.uint8, n, "rgb", True),
                _buf(depm, np.uint8, n, "depth_mask", True)]
        return ptrs, (rgb, depth)

    def process_interleaved(self, rgb, depth, order: str = "rgb",
                            want=("rgb", "depth", "fused"), out=None) -> FrameMasks:
        """process() from an interleaved colour frame (H, W, 3) or
        (streams, H, W, 3) -- R,G,B (aos_to_soa's layout, engine.cpp:39-56)
        or B,G,R (OpenCV / Kinect order); the kernel deinterleaves it."""
        out = dict(out or {})
        for k in want:
            if k not in out:
                out[k] = np.empty(self._shape(), np.uint8)
        ptrs, keep = self._packed_args(rgb, depth, order, out.get("fused"), out.get("rgb"),
                                       out.get("depth"))
        _finish_producers(*keep, out.get("fused"), out.get("rgb"), out.get("depth"))
        idx = self.frames
        check(lib.rgbdseg_processor_process_interleaved(self._h, *ptrs), "process_interleaved")
        return FrameMasks(idx, out.get("rgb"), out.get("depth"), out.get("fused"))

    def submit_interleaved(self, rgb, depth, order: str = "rgb", fused=None, rgb_mask=None,
                           depth_mask=None):
        """submit() from an interleaved colour frame (see process_interleaved);
        buffers must stay alive until sync()."""
        ptrs, keep = self._packed_args(rgb, depth, order, fused, rgb_mask, depth_mask)
        self._keep.append((keep, fused, rgb_mask, depth_mask))
        _finish_producers(*keep, fused, rgb_mask, depth_mask)
        check(lib.rgbdseg_processor_submit_interleaved(self._h, *ptrs), "submit_interleaved")

    def submit(self, r, g, b, depth, fused=None, rgb=None, depth_mask=None, order=True):
        """Enqueue one step without waiting; buffers must stay alive and
        unmodified until ``sync()``.  With CUDA tensors and ``order`` the step
        is queued after the work on torch's current stream, and that stream
        waits for the step (so torch may consume the outputs directly);
        ``order=False`` leaves ordering to the caller."""
        ptrs, keep = self._args(r, g, b, depth, fused, rgb, depth_mask)
        self._keep.append((keep, fused, rgb, depth_mask))
        ts = _cuda_tensors(*keep, fused, rgb, depth_mask) if order else []
        if ts:
            import torch

            cur = torch.cuda.current_stream(ts[0].device).cuda_stream
            check(lib.rgbdseg_processor_wait_stream(self._h, cur), "submit")
        check(lib.rgbdseg_processor_submit(self._h, *ptrs), "submit")
        if ts:
            check(lib.rgbdseg_processor_signal_stream(self._h, cur), "submit")

    def _planar_ptr(self, frame, what):
        n = self.npx
        if _is_torch(frame):
            import torch

            if frame.dtype != torch.uint8 or not frame.is_contiguous() or frame.numel() != 5 * n:
                raise ValueError(f"{what}: expected a contiguous uint8 tensor of 5*{n} bytes")
            if n % 2:
                raise ValueError(f"{what}: odd pixel count (the depth plane would be "
                                 "misaligned on the device); pass the planes")
            return frame.data_ptr()
        if (not isinstance(frame, np.ndarray) or frame.dtype != np.uint8
                or not frame.flags.c_contiguous or frame.size != 5 * n):
            raise ValueError(f"{what}: expected a C-contiguous uint8 array of 5*{n} bytes")
        return frame.ctypes.data

    def submit_planar(self, frame, fused=None, order=True):
        """submit() of ONE planar frame buffer: r, g, b (npx bytes each) then
        the uint16 depth plane, back to back -- the layout a capture ring of
        pinned buffers uses.  The library moves it in one DMA per chunk; the
        Python side checks one buffer instead of four (~5 us instead of ~20
        per call, which matters for single-VGA frames).  `fused` (npx bytes)
        receives the fused mask at sync()."""
        p = self._planar_ptr(frame, "submit_planar")
        n = self.npx
        fo = _buf(fused, np.uint8, n, "fused", True)
        self._keep.append((frame, fused))
        ts = _cuda_tensors(frame, fused) if order else []
        if ts:
            import torch

            cur = torch.cuda.current_stream(ts[0].device).cuda_stream
            check(lib.rgbdseg_processor_wait_stream(self._h, cur), "submit_planar")
        check(lib.rgbdseg_processor_submit(self._h, p, p + n, p + 2 * n, p + 3 * n, fo, None,
                                           None), "submit_planar")
        if ts:
            check(lib.rgbdseg_processor_signal_stream(self._h, cur), "submit_planar")

    def process_planar(self, frame, fused=None):
        """process() of one planar frame buffer (see submit_planar); returns
        the fused mask (a new array unless `fused` is given)."""
        if fused is None:
            fused = np.empty(self._shape(), np.uint8)
        self.submit_planar(frame, fused)
        self.sync()
        return fused

    def sync(self):
        check(lib.rgbdseg_processor_sync(self._h), "sync")
        self._keep.clear()


# ------------------------------------------------------------------ layout helpers

def aos_to_soa(frame):
    """aos_to_soa (engine.cpp:39-56; module.cpp:121-131): an interleaved
    H x W x 3 uint8 frame -> (r, g, b) planes.  The GPU path does not need
    it (SequenceProcessor.process_interleaved deinterleaves in the kernel)."""
    a = np.asarray(frame)
    if a.ndim != 3 or a.shape[2] != 3:
        raise ValueError("expected an HxWx3 array")
    a = np.ascontiguousarray(a, dtype=np.uint8)
    return tuple(np.ascontiguousarray(a[:, :, c]) for c in range(3))


def soa_to_aos(r, g, b):
    """soa_to_aos (engine.cpp:58-74): three planes -> interleaved H x W x 3."""
    planes = [np.asarray(x, dtype=np.uint8) for x in (r, g, b)]
    for p in planes[1:]:
        if p.shape != planes[0].shape:
            h0, w0 = planes[0].shape[-2:]
            h1, w1 = p.shape[-2:]
            raise ValueError(f"soa_to_aos: dimension mismatch ({w0}x{h0} vs {w1}x{h1})")
    return np.ascontiguousarray(np.stack(planes, axis=-1))


# ------------------------------------------------------------------ evaluation

def confusion_counts(pred, gt, streams: int = 1, device: int = 0):
    """confusion_counts (eval.cpp:11-31; module.cpp:112-116) on the GPU:
    (tp, fp, tn, fn), or an int64 [streams, 4] array when streams > 1."""
    _check_mask(pred)
    _check_mask(gt)
    p = _as_host(pred, np.uint8, np.shape(pred))
    g = _as_host(gt, np.uint8, np.shape(pred))
    n = int(np.prod(np.shape(pred)))
    counts = np.zeros((streams, 4), np.int64)
    check(lib.rgbdseg_confusion_counts(_buf(p, np.uint8, n, "pred"), _buf(g, np.uint8, n, "gt"),
                                       n, streams, counts.ctypes.data, device))
    return tuple(int(x) for x in counts[0]) if streams == 1 else counts


def precision(tp, fp):
    """eval.cpp:33-37: TP / (TP + FP), 0 when the denominator is 0."""
    return tp / (tp + fp) if tp + fp > 0 else 0.0


def recall(tp, fn):
    """eval.cpp:39-43: TP / (TP + FN), 0 when the denominator is 0."""
    return tp / (tp + fn) if tp + fn > 0 else 0.0


def f1_score(tp, fp, fn):
    """f1 (eval.cpp:45-47; module.cpp:117-119): 2PR / (P + R), 0 if P + R = 0."""
    p, r = precision(tp, fp), recall(tp, fn)
    return 2.0 * p * r / (p + r) if p + r > 0.0 else 0.0


# ------------------------------------------------------------------ scenes

def builtin_scenario_names():
    return ["A", "B"]


def render_scenario(name: str, width: int, height: int, frame: int, streams: int = 1,
                    seed0: int = 1, device: int = 0, out=None, stream=None, with_gt=False):
    """Render builtin scenario `name` (synthetic.cpp:234-273, render_frame
    :119-195) for `streams` streams (seeds seed0..seed0+streams-1) straight
    into CUDA tensors (torch is used only as the device allocator)."""
    import torch

    shp = (streams, height, width)
    if out is None:
        dev = torch.device("cuda", device)
        out = {"r": torch.empty(shp, dtype=torch.uint8, device=dev),
               "g": torch.empty(shp, dtype=torch.uint8, device=dev),
               "b": torch.empty(shp, dtype=torch.uint8, device=dev),
               "depth": torch.empty(shp, dtype=torch.uint16, device=dev)}
        if with_gt:
            out["gt"] = torch.empty(shp, dtype=torch.uint8, device=dev)
    gt = out.get("gt")
    check(lib.rgbdseg_render_scenario(name.encode()[:1], width, height, streams, seed0, frame,
                                      out["r"].data_ptr(), out["g"].data_ptr(),
                                      out["b"].data_ptr(), out["depth"].data_ptr(),
                                      gt.data_ptr() if gt is not None else None, device,
                                      stream), "render_scenario")
    return out
