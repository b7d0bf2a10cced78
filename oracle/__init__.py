"""oracle -- CPU parity checkers for the rgbdseg hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this
package, and only as the checker or the CPU baseline.  The product package
(``paper_2110_14934_b200``) never imports it.

Two checkers live here:

* :class:`Port` -- ``liboracle.so``, the plain-C restatement in
  ``rgbdseg_oracle.c`` (each function cites the reference file:line it follows).
* :class:`Ref` -- ``_ref/librgbdseg_ref.so``, the unmodified reference sources
  compiled in place by ``oracle/Makefile`` plus ``ref_shim.cpp``.

Parity of the restatement is pinned against ``Ref`` and against the committed
fixtures in ``tests/golden/`` (generated from ``Ref`` by
``tests/golden/make_golden.py``).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "librgbdseg_ref.so")

_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(dtype=np.uint16, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class Cfg(C.Structure):
    """MixtureConfig (reference mixture.hpp:16-26) as a C struct."""

    _fields_ = [
        ("components", C.c_int),
        ("learning_rate", C.c_float),
        ("match_lambda", C.c_float),
        ("background_threshold", C.c_float),
        ("initial_sigma", C.c_float),
        ("initial_weight", C.c_float),
        ("variance_floor", C.c_float),
    ]


class Mix(C.Structure):
    """PixelMixture (reference mixture.hpp:30-41) as a flat C struct."""

    _fields_ = [
        ("components", C.c_int),
        ("channels", C.c_int),
        ("means", C.c_float * 20),
        ("variances", C.c_float * 5),
        ("weights", C.c_float * 5),
    ]

    def key(self):
        m, ch = self.components, self.channels
        return (
            m,
            ch,
            np.frombuffer(bytes(self.means), np.float32)[: m * ch].tobytes(),
            np.frombuffer(bytes(self.variances), np.float32)[:m].tobytes(),
            np.frombuffer(bytes(self.weights), np.float32)[:m].tobytes(),
        )


def color_cfg(components=3, **kw) -> Cfg:
    """Colour defaults (mixture.hpp:17-23)."""
    c = Cfg(components, 0.05, 2.5, 0.8, 15.0, 0.05, 4.0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def depth_cfg(components=3, **kw) -> Cfg:
    """Depth defaults (RunConfig::defaults, processor.cpp:35-43)."""
    c = color_cfg(components, learning_rate=0.01, initial_sigma=100.0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def n_planes(components: int, channels: int) -> int:
    return components * channels + 2 * components


class Port:
    """ctypes front of liboracle.so (the C restatement)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.orc_cfg_check.argtypes = [C.POINTER(Cfg)]
        L.orc_init.argtypes = [C.POINTER(Mix), _f32p, C.c_int, C.POINTER(Cfg)]
        L.orc_step.argtypes = [C.POINTER(Mix), _f32p, C.POINTER(Cfg)]
        L.orc_match.argtypes = [C.POINTER(Mix), _f32p, C.POINTER(Cfg)]
        L.orc_classify.argtypes = [C.POINTER(Mix), C.c_int, C.POINTER(Cfg)]
        L.orc_update.argtypes = [C.POINTER(Mix), _f32p, C.c_int, C.POINTER(Cfg)]
        L.orc_bank_reset.argtypes = [_f32p, _u8p, C.c_size_t, C.c_int, C.POINTER(Cfg)]
        L.orc_segment_color.argtypes = [_f32p, _u8p, C.c_size_t, _u8p, _u8p, _u8p,
                                        C.POINTER(Cfg), _u8p]
        L.orc_segment_depth.argtypes = [_f32p, _u8p, C.c_size_t, _u16p, C.POINTER(Cfg), _u8p]
        L.orc_segment_augmented.argtypes = [_f32p, _u8p, C.c_size_t, _u8p, _u8p, _u8p, _u16p,
                                            C.c_float, C.c_float, C.POINTER(Cfg), _u8p]
        L.orc_fusion_reset.argtypes = [_u8p, _i8p, C.c_size_t, C.c_uint8]
        L.orc_fuse.argtypes = [_u8p, _i8p, C.c_size_t, C.c_int, _u8p, _u8p]
        L.orc_register.argtypes = [_u8p, _u16p, C.c_int, C.c_int, _f64p, C.c_int, C.c_int,
                                   C.c_int, _u8p, _u8p]
        L.orc_dilate.argtypes = [_u8p, _u8p, C.c_int, C.c_int, C.c_int]
        L.orc_scene_sizeof.restype = C.c_size_t
        L.orc_scene_builtin.argtypes = [C.c_void_p, C.c_char]
        L.orc_render.argtypes = [C.c_void_p, C.c_int, _u8p, _u8p, _u8p, _u16p, C.c_void_p]
        L.orc_hash.restype = C.c_uint64
        L.orc_hash.argtypes = [C.c_uint64] * 5

    # per pixel
    def init_mixture(self, v, cfg: Cfg) -> Mix:
        v = np.ascontiguousarray(v, np.float32)
        m = Mix()
        self.lib.orc_init(C.byref(m), v, len(v), C.byref(cfg))
        return m

    def step_pixel(self, m: Mix, v, cfg: Cfg) -> int:
        return self.lib.orc_step(C.byref(m), np.ascontiguousarray(v, np.float32), C.byref(cfg))

    def cfg_check(self, cfg: Cfg) -> int:
        return self.lib.orc_cfg_check(C.byref(cfg))


@dataclass
class Frame:
    r: np.ndarray
    g: np.ndarray
    b: np.ndarray
    depth: np.ndarray
    gt: np.ndarray | None = None


class PortScene:
    """Builtin scenario 'A'/'B' (synthetic.cpp:234-273) rendered by the port."""

    def __init__(self, port: Port, name="A", width=0, height=0, seed=0):
        self.port = port
        self.buf = C.create_string_buffer(port.lib.orc_scene_sizeof())
        if port.lib.orc_scene_builtin(self.buf, name.encode()[0:1]) != 0:
            raise ValueError(f"unknown scenario {name!r}")
        # orc_scene starts with int width, height, frame_count; uint64 seed
        ints = np.ndarray((3,), np.int32, buffer=self.buf)
        if width:
            ints[0] = width
        if height:
            ints[1] = height
        if seed:
            np.ndarray((1,), np.uint64, buffer=self.buf, offset=16)[0] = seed
        self.width, self.height = int(ints[0]), int(ints[1])

    def render(self, frame: int) -> Frame:
        w, h = self.width, self.height
        r, g, b = (np.empty((h, w), np.uint8) for _ in range(3))
        d = np.empty((h, w), np.uint16)
        gt = np.empty((h, w), np.uint8)
        self.port.lib.orc_render(self.buf, frame, r, g, b, d, gt.ctypes.data)
        return Frame(r, g, b, d, gt)


class PortBank:
    """SoA model bank over the port (segmenter.cpp:24-131)."""

    def __init__(self, port: Port, npx: int, channels: int, cfg: Cfg):
        self.port, self.npx, self.channels, self.cfg = port, npx, channels, cfg
        self.state = np.empty(n_planes(cfg.components, channels) * npx, np.float32)
        self.flags = np.empty(npx, np.uint8)
        port.lib.orc_bank_reset(self.state, self.flags, npx, channels, C.byref(cfg))

    def planes(self) -> np.ndarray:
        return self.state.reshape(-1, self.npx)

    def segment_color(self, r, g, b) -> np.ndarray:
        mask = np.empty(self.npx, np.uint8)
        self.port.lib.orc_segment_color(self.state, self.flags, self.npx,
                                        np.ascontiguousarray(r).ravel(),
                                        np.ascontiguousarray(g).ravel(),
                                        np.ascontiguousarray(b).ravel(),
                                        C.byref(self.cfg), mask)
        return mask

    def segment_augmented(self, r, g, b, d, lo=0.0, hi=4000.0) -> np.ndarray:
        mask = np.empty(self.npx, np.uint8)
        rav = [np.ascontiguousarray(x).ravel() for x in (r, g, b, d)]
        self.port.lib.orc_segment_augmented(self.state, self.flags, self.npx, *rav, lo, hi,
                                            C.byref(self.cfg), mask)
        return mask

    def segment_depth(self, d) -> np.ndarray:
        mask = np.empty(self.npx, np.uint8)
        self.port.lib.orc_segment_depth(self.state, self.flags, self.npx,
                                        np.ascontiguousarray(d).ravel(), C.byref(self.cfg), mask)
        return mask


def rig_array(depth_cam, color_cam, rotation, translation, scale) -> np.ndarray:
    """Pack a CameraRig as the 21 doubles orc_register / rref_register_mask take."""
    return np.ascontiguousarray(list(depth_cam) + list(color_cam) + list(rotation) +
                                list(translation) + [scale], np.float64)


class PortProcessor:
    """Colour bank + depth bank + List-1 fusion, the order of
    SequenceProcessor::process (processor.cpp:158-184).  With `rig` (21
    doubles) and width/height the sequence is unregistered: the depth mask is
    registered and dilated (processor.cpp:175-179) before fusion."""

    def __init__(self, port: Port, npx: int, ccfg: Cfg, dcfg: Cfg, limit=3, initial_label=0,
                 rig=None, width=0, height=0, radius=1):
        self.rig, self.w, self.h, self.radius = rig, width, height, radius
        self.port = port
        self.color = PortBank(port, npx, 3, ccfg)
        self.depth = PortBank(port, npx, 1, dcfg)
        self.limit = limit
        self.out = np.empty(npx, np.uint8)
        self.cpt = np.empty(npx, np.int8)
        port.lib.orc_fusion_reset(self.out, self.cpt, npx, initial_label)

    def process(self, r, g, b, d):
        rgb = self.color.segment_color(r, g, b)
        dep = self.depth.segment_depth(d)
        reg = dep
        if self.rig is not None:
            n = self.w * self.h
            reg = np.empty(n, np.uint8)
            scratch = np.empty(n, np.uint8)
            self.port.lib.orc_register(dep, np.ascontiguousarray(d).ravel(), self.w, self.h,
                                       self.rig, self.w, self.h, self.radius, scratch, reg)
        self.port.lib.orc_fuse(self.out, self.cpt, self.out.size, self.limit, rgb, reg)
        return rgb, dep, self.out.copy()


class Ref:
    """ctypes front of the reference compiled in place (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref`")
        L = self.lib = C.CDLL(path)
        L.rref_last_error.restype = C.c_char_p
        L.rref_cfg_validate.argtypes = [C.POINTER(Cfg)]
        L.rref_init_mixture.argtypes = [_f32p, C.c_int, C.POINTER(Cfg), C.POINTER(Mix)]
        L.rref_step_pixel.argtypes = [C.POINTER(Mix), _f32p, C.POINTER(Cfg), C.POINTER(C.c_int)]
        L.rref_match_component.argtypes = [C.POINTER(Mix), _f32p, C.POINTER(Cfg),
                                           C.POINTER(C.c_int)]
        L.rref_update_mixture.argtypes = [C.POINTER(Mix), _f32p, C.c_int, C.POINTER(Cfg)]
        L.rref_classify.argtypes = [C.POINTER(Mix), C.c_int, C.POINTER(Cfg), C.POINTER(C.c_int)]
        L.rref_bank_create.restype = C.c_void_p
        L.rref_bank_create.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(Cfg)]
        L.rref_bank_destroy.argtypes = [C.c_void_p]
        L.rref_segment_color.argtypes = [C.c_void_p, _u8p, _u8p, _u8p, C.POINTER(Cfg), C.c_int,
                                         _u8p]
        L.rref_segment_depth.argtypes = [C.c_void_p, _u16p, C.POINTER(Cfg), C.c_int, _u8p]
        L.rref_segment_augmented.argtypes = [C.c_void_p, _u8p, _u8p, _u8p, _u16p, C.c_float,
                                             C.c_float, C.POINTER(Cfg), C.c_int, _u8p]
        L.rref_bank_get.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.rref_bank_set.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.rref_fusion_create.restype = C.c_void_p
        L.rref_fusion_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
        L.rref_fusion_destroy.argtypes = [C.c_void_p]
        L.rref_fuse_step.argtypes = [C.c_void_p, _u8p, _u8p, _u8p, _i8p]
        L.rref_register_mask.argtypes = [_u8p, _u16p, C.c_int, C.c_int, _f64p, C.c_int, C.c_int,
                                         C.c_int, _u8p]
        L.rref_scene_create.restype = C.c_void_p
        L.rref_scene_create.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_uint64]
        L.rref_scene_destroy.argtypes = [C.c_void_p]
        L.rref_render.argtypes = [C.c_void_p, C.c_int, _u8p, _u8p, _u8p, _u16p, C.c_void_p]
        L.rref_hash_counter.restype = C.c_uint64
        L.rref_hash_counter.argtypes = [C.c_uint64] * 5
        L.rref_processor_create.restype = C.c_void_p
        L.rref_processor_create.argtypes = [C.c_int, C.c_int, C.POINTER(Cfg), C.POINTER(Cfg),
                                            C.c_int, C.c_int, C.c_int]
        L.rref_processor_destroy.argtypes = [C.c_void_p]
        L.rref_processor_create_rig.restype = C.c_void_p
        L.rref_processor_create_rig.argtypes = [C.c_int, C.c_int, C.POINTER(Cfg), C.POINTER(Cfg),
                                                C.c_int, C.c_int, C.c_int, _f64p, C.c_int]
        L.rref_processor_process.argtypes = [C.c_void_p, _u8p, _u8p, _u8p, _u16p, C.c_void_p,
                                             C.c_void_p, C.c_void_p]
        L.rref_processor_bank_get.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                              C.c_void_p]

    def check(self, rc: int):
        if rc == 1:
            raise ValueError(self.lib.rref_last_error().decode())
        if rc != 0:
            raise RuntimeError(self.lib.rref_last_error().decode())

    def init_mixture(self, v, cfg: Cfg) -> Mix:
        v = np.ascontiguousarray(v, np.float32)
        m = Mix()
        self.check(self.lib.rref_init_mixture(v, len(v), C.byref(cfg), C.byref(m)))
        return m

    def match_component(self, m: Mix, v, cfg: Cfg) -> int:
        mt = C.c_int()
        self.check(self.lib.rref_match_component(C.byref(m), np.ascontiguousarray(v, np.float32),
                                                 C.byref(cfg), C.byref(mt)))
        return mt.value

    def update_mixture(self, m: Mix, v, matched: int, cfg: Cfg) -> None:
        self.check(self.lib.rref_update_mixture(C.byref(m), np.ascontiguousarray(v, np.float32),
                                                matched, C.byref(cfg)))

    def classify(self, m: Mix, matched: int, cfg: Cfg) -> int:
        lab = C.c_int()
        self.check(self.lib.rref_classify(C.byref(m), matched, C.byref(cfg), C.byref(lab)))
        return lab.value

    def step_pixel(self, m: Mix, v, cfg: Cfg) -> int:
        lab = C.c_int()
        self.check(self.lib.rref_step_pixel(C.byref(m), np.ascontiguousarray(v, np.float32),
                                            C.byref(cfg), C.byref(lab)))
        return lab.value


class RefScene:
    def __init__(self, ref: Ref, name="A", width=0, height=0, seed=0, frames=0):
        self.ref = ref
        self.h = ref.lib.rref_scene_create(name.encode(), width, height, frames, seed)
        if not self.h:
            raise ValueError(ref.lib.rref_last_error().decode())
        self.width = width or 640
        self.height = height or 480

    def render(self, frame: int) -> Frame:
        w, h = self.width, self.height
        r, g, b = (np.empty((h, w), np.uint8) for _ in range(3))
        d = np.empty((h, w), np.uint16)
        gt = np.empty((h, w), np.uint8)
        self.ref.check(self.ref.lib.rref_render(self.h, frame, r, g, b, d, gt.ctypes.data))
        return Frame(r, g, b, d, gt)

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.rref_scene_destroy(self.h)


class RefProcessor:
    """The reference SequenceProcessor (fused, registered, SoA)."""

    def __init__(self, ref: Ref, width, height, ccfg: Cfg, dcfg: Cfg, limit=3, initial_label=0,
                 workers=1, rig=None, radius=1):
        self.ref, self.w, self.h = ref, width, height
        self.ccfg, self.dcfg = ccfg, dcfg
        if rig is None:
            self.p = ref.lib.rref_processor_create(width, height, C.byref(ccfg), C.byref(dcfg),
                                                   limit, initial_label, workers)
        else:
            self.p = ref.lib.rref_processor_create_rig(width, height, C.byref(ccfg),
                                                       C.byref(dcfg), limit, initial_label,
                                                       workers, rig, radius)
        if not self.p:
            raise ValueError(ref.lib.rref_last_error().decode())

    def process(self, r, g, b, d, want_masks=True):
        n = self.w * self.h
        rgb = np.empty(n, np.uint8)
        dep = np.empty(n, np.uint8)
        fused = np.empty(n, np.uint8)
        args = [np.ascontiguousarray(x).ravel() for x in (r, g, b)]
        self.ref.check(self.ref.lib.rref_processor_process(
            self.p, *args, np.ascontiguousarray(d).ravel(),
            rgb.ctypes.data if want_masks else None,
            dep.ctypes.data if want_masks else None, fused.ctypes.data))
        return rgb, dep, fused

    def bank_planes(self, which: int) -> np.ndarray:
        """All float planes of bank `which` (0 colour, 1 depth) in ModelBank
        plane order: means[i*C+c], variances[i], weights[i]."""
        cfg = self.ccfg if which == 0 else self.dcfg
        M, Ch = cfg.components, (3 if which == 0 else 1)
        n = self.w * self.h
        out = np.empty((n_planes(M, Ch), n), np.float32)
        k = 0
        for i in range(M):
            for c in range(Ch):
                self.ref.check(self.ref.lib.rref_processor_bank_get(self.p, which, 0, i, c,
                                                                    out[k].ctypes.data))
                k += 1
        for kind in (1, 2):
            for i in range(M):
                self.ref.check(self.ref.lib.rref_processor_bank_get(self.p, which, kind, i, 0,
                                                                    out[k].ctypes.data))
                k += 1
        return out

    def flags(self, which: int) -> np.ndarray:
        f = np.empty(self.w * self.h, np.uint8)
        self.ref.check(self.ref.lib.rref_processor_bank_get(self.p, which, 3, 0, 0, f.ctypes.data))
        return f

    def __del__(self):
        if getattr(self, "p", None):
            self.ref.lib.rref_processor_destroy(self.p)


def fnv1a(buf: np.ndarray) -> int:
    """FNV-1a 64 of a mask (acceptance.cpp:38-46)."""
    h = 1469598103934665603
    data = np.ascontiguousarray(buf).view(np.uint8).ravel()
    # vectorised in chunks is awkward for FNV; masks in tests are small
    for x in data.tobytes():
        h ^= x
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def port_available() -> bool:
    return os.path.exists(PORT_SO)
