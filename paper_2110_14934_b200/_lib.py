"""ctypes binding of librgbdseg_b200.so (include/rgbdseg_c.h).

The product path has no CPU fallback: if the CUDA library is missing this
module raises at import time, and every compute call goes through the C-ABI
into the sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# Always the in-tree library built by `make lib` (no environment override).
LIB_PATH = os.path.join(HERE, "librgbdseg_b200.so")

OK, EINVAL, ECUDA, ENOMEM, ERUNTIME = 0, 1, 2, 3, 4
COLOR3, DEPTH1, AUGMENTED4 = 0, 1, 2
FLAGS_PLANE = -1
VARIANTS = {"auto": 0, "ldg": 1, "ldg_elide": 2, "ldg_elide_l1": 3}
ORDER = {"rgb": 0, "bgr": 1}


class MixtureCfg(C.Structure):
    _fields_ = [
        ("components", C.c_int),
        ("learning_rate", C.c_float),
        ("match_lambda", C.c_float),
        ("background_threshold", C.c_float),
        ("initial_sigma", C.c_float),
        ("initial_weight", C.c_float),
        ("variance_floor", C.c_float),
    ]


class PixelMixtureRec(C.Structure):
    _fields_ = [
        ("components", C.c_int),
        ("channels", C.c_int),
        ("means", C.c_float * 20),
        ("variances", C.c_float * 5),
        ("weights", C.c_float * 5),
    ]


class CameraRigC(C.Structure):
    """rgbdseg_camera_rig = CameraRig (registration.hpp:16-26)."""

    _fields_ = [
        ("depth_fx", C.c_double), ("depth_fy", C.c_double),
        ("depth_cx", C.c_double), ("depth_cy", C.c_double),
        ("color_fx", C.c_double), ("color_fy", C.c_double),
        ("color_cx", C.c_double), ("color_cy", C.c_double),
        ("rotation", C.c_double * 9),
        ("translation_mm", C.c_double * 3),
        ("depth_scale", C.c_double),
    ]


class ProcessorCfg(C.Structure):
    _fields_ = [
        ("width", C.c_int),
        ("height", C.c_int),
        ("streams", C.c_int),
        ("color", MixtureCfg),
        ("depth", MixtureCfg),
        ("fusion_counter_limit", C.c_int),
        ("fusion_initial_label", C.c_int),
        ("device", C.c_int),
        ("host_chunks", C.c_int),
        ("registered", C.c_int),
        ("rig", CameraRigC),
        ("dilation_radius", C.c_int),
    ]


class SceneFrameC(C.Structure):
    """rgbdseg_scene_frame: one frame of a ScenarioSpec, resolved on the host."""

    _fields_ = [
        ("width", C.c_int), ("height", C.c_int), ("streams", C.c_int),
        ("seed0", C.c_uint64), ("frame", C.c_int),
        ("base_depth_mm", C.c_int), ("depth_texture_mm", C.c_int), ("color_texture", C.c_int),
        ("gain", C.c_double),
        ("n_obj", C.c_int), ("obj_rect", (C.c_int * 4) * 4), ("obj_color", (C.c_int * 3) * 4),
        ("obj_depth_offset_mm", C.c_int * 4),
        ("n_shadow", C.c_int), ("shadow_rect", (C.c_int * 4) * 16),
        ("shadow_darken", C.c_double * 16),
        ("n_flicker", C.c_int), ("flicker_rect", (C.c_int * 4) * 16),
        ("flicker_color_sigma", C.c_double * 16), ("flicker_depth_sigma_mm", C.c_double * 16),
        ("noise_color_sigma", C.c_double), ("noise_depth_sigma_mm", C.c_double),
    ]


# Every symbol include/rgbdseg_c.h declares: (restype, argtypes)
_vp, _sz, _i, _u8 = C.c_void_p, C.c_size_t, C.c_int, C.c_uint8
SIGNATURES = {
    "rgbdseg_last_error": (C.c_char_p, []),
    "rgbdseg_version": (C.c_char_p, []),
    "rgbdseg_launch_count": (C.c_uint64, []),
    "rgbdseg_mixture_defaults": (None, [C.POINTER(MixtureCfg)]),
    "rgbdseg_mixture_validate": (_i, [C.POINTER(MixtureCfg)]),
    "rgbdseg_init_mixtures": (_i, [_vp, _i, _sz, C.POINTER(MixtureCfg), _vp, _i]),
    "rgbdseg_step_mixtures": (_i, [_vp, _vp, _i, _sz, C.POINTER(MixtureCfg), _vp, _i]),
    "rgbdseg_match_components": (_i, [_vp, _vp, _i, _sz, C.POINTER(MixtureCfg), _vp, _i]),
    "rgbdseg_classify_mixtures": (_i, [_vp, _vp, _sz, C.POINTER(MixtureCfg), _vp, _i]),
    "rgbdseg_update_mixtures": (_i, [_vp, _vp, _i, _sz, _vp, C.POINTER(MixtureCfg), _i]),
    "rgbdseg_bank_create": (_i, [_i, _i, _i, _i, C.POINTER(MixtureCfg), _i, C.POINTER(_vp)]),
    "rgbdseg_bank_destroy": (None, [_vp]),
    "rgbdseg_bank_planes": (_i, [_vp]),
    "rgbdseg_bank_download": (_i, [_vp, _i, _vp]),
    "rgbdseg_bank_upload": (_i, [_vp, _i, _vp]),
    "rgbdseg_bank_device_ptrs": (_i, [_vp, C.POINTER(_vp), C.POINTER(_sz), C.POINTER(_sz)]),
    "rgbdseg_segment_color": (_i, [_vp, _vp, _vp, _vp, C.POINTER(MixtureCfg), _vp]),
    "rgbdseg_segment_depth": (_i, [_vp, _vp, C.POINTER(MixtureCfg), _vp]),
    "rgbdseg_segment_augmented": (_i, [_vp, _vp, _vp, _vp, _vp, C.c_float, C.c_float,
                                       C.POINTER(MixtureCfg), _vp]),
    "rgbdseg_fusion_create": (_i, [_i, _i, _i, _i, _i, _i, C.POINTER(_vp)]),
    "rgbdseg_fusion_destroy": (None, [_vp]),
    "rgbdseg_fusion_step": (_i, [_vp, _vp, _vp, _vp]),
    "rgbdseg_fusion_download": (_i, [_vp, _vp, _vp]),
    "rgbdseg_fusion_upload": (_i, [_vp, _vp, _vp]),
    "rgbdseg_fusion_set_counter_limit": (_i, [_vp, _i]),
    "rgbdseg_camera_rig_identity": (None, [C.POINTER(CameraRigC), C.c_double, C.c_double,
                                            C.c_double, C.c_double]),
    "rgbdseg_camera_rig_validate": (_i, [C.POINTER(CameraRigC)]),
    "rgbdseg_register_mask": (_i, [_vp, _vp, _i, _i, C.POINTER(CameraRigC), _i, _i, _i, _vp, _i]),
    "rgbdseg_dilate_mask": (_i, [_vp, _i, _i, _i, _vp, _i]),
    "rgbdseg_processor_defaults": (None, [C.POINTER(ProcessorCfg), _i, _i]),
    "rgbdseg_processor_create": (_i, [C.POINTER(ProcessorCfg), C.POINTER(_vp)]),
    "rgbdseg_processor_destroy": (None, [_vp]),
    "rgbdseg_processor_process": (_i, [_vp] * 8),
    "rgbdseg_processor_submit": (_i, [_vp] * 8),
    "rgbdseg_processor_sync": (_i, [_vp]),
    "rgbdseg_processor_submit_interleaved": (_i, [_vp, _vp, _i, _vp, _vp, _vp, _vp]),
    "rgbdseg_processor_process_interleaved": (_i, [_vp, _vp, _i, _vp, _vp, _vp, _vp]),
    "rgbdseg_processor_process_eval": (_i, [_vp] * 10),
    "rgbdseg_processor_submit_eval": (_i, [_vp] * 10),
    "rgbdseg_confusion_counts": (_i, [_vp, _vp, _sz, _i, _vp, _i]),
    "rgbdseg_processor_frames": (C.c_int64, [_vp]),
    "rgbdseg_processor_color_bank": (_vp, [_vp]),
    "rgbdseg_processor_depth_bank": (_vp, [_vp]),
    "rgbdseg_processor_fusion": (_vp, [_vp]),
    "rgbdseg_processor_stream": (_vp, [_vp]),
    "rgbdseg_processor_wait_stream": (_i, [_vp, _vp]),
    "rgbdseg_processor_signal_stream": (_i, [_vp, _vp]),
    "rgbdseg_processor_set_variant": (_i, [_vp, _i]),
    "rgbdseg_processor_set_near_threshold": (_i, [_vp, C.c_float]),
    "rgbdseg_processor_near_threshold_counts": (_i, [_vp, _vp, _vp, _vp]),
    "rgbdseg_render_scenario": (_i, [C.c_char, _i, _i, _i, C.c_uint64, _i, _vp, _vp, _vp, _vp,
                                     _vp, _i, _vp]),
    "rgbdseg_render_frame": (_i, [C.POINTER(SceneFrameC), _vp, _vp, _vp, _vp, _vp, _i, _vp]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the B200 CUDA library is not built "
            "(run `make lib` or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class RgbdsegError(RuntimeError):
    pass


def check(rc: int, what: str = ""):
    """Map a C-ABI status to the reference's exception types:
    EINVAL -> ValueError (std::invalid_argument), others -> RuntimeError."""
    if rc == OK:
        return
    msg = (lib.rgbdseg_last_error() or b"").decode()
    if what:
        msg = f"{what}: {msg}"
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == ENOMEM:
        raise MemoryError(msg)
    raise RgbdsegError(msg)


def launch_count() -> int:
    return int(lib.rgbdseg_launch_count())
