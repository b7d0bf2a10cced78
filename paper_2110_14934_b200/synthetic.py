"""Synthetic RGB-D scenes (synthetic.hpp:13-97, synthetic.cpp): ScenarioSpec,
the builtin scenarios, JSON specs, and GPU rendering.

A spec is resolved per frame on the host exactly as render_frame does
(synthetic.cpp:124-134: illumination gain product, each object's lround'ed
waypoint position, the shadow / flicker events active in that frame) and the
per-pixel counter-hash work runs in the K3 kernel (rgbdseg_render_frame).
K3 evaluates log/cos with CUDA's libdevice, which is not correctly rounded,
so a pixel may very rarely differ from the CPU renderer by one code value;
parity tests always share input bytes, never regenerate them.
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import check, lib


@dataclass
class RegionRect:
    x: int = 0
    y: int = 0
    w: int = 0
    h: int = 0

    def contains(self, px, py):
        return self.x <= px < self.x + self.w and self.y <= py < self.y + self.h


@dataclass
class Waypoint:
    frame: int = 0
    x: float = 0.0
    y: float = 0.0


@dataclass
class ObjectSpec:
    width: int = 0
    height: int = 0
    waypoints: List[Waypoint] = field(default_factory=list)
    depth_offset_mm: int = 0
    color: tuple = (200, 60, 60)


@dataclass
class IlluminationEvent:
    start: int = 0
    end: int = 0
    gain: float = 1.0


@dataclass
class ShadowEvent:
    start: int = 0
    end: int = 0
    region: RegionRect = field(default_factory=RegionRect)
    darken: float = 0.6


@dataclass
class FlickerEvent:
    start: int = 0
    end: int = 0
    region: RegionRect = field(default_factory=RegionRect)
    color_sigma: float = 0.0
    depth_sigma_mm: float = 0.0


@dataclass
class ScenarioSpec:
    """ScenarioSpec (synthetic.hpp:61-74)."""

    name: str = "custom"
    width: int = 640
    height: int = 480
    frame_count: int = 0
    seed: int = 1
    base_depth_mm: int = 2000
    depth_texture_mm: int = 30
    color_texture: int = 8
    objects: List[ObjectSpec] = field(default_factory=list)
    illumination: List[IlluminationEvent] = field(default_factory=list)
    shadows: List[ShadowEvent] = field(default_factory=list)
    flicker: List[FlickerEvent] = field(default_factory=list)
    noise_color_sigma: float = 1.0
    noise_depth_sigma_mm: float = 1.0

    def validate(self):
        """ScenarioSpec::validate (synthetic.cpp:85-117), same messages."""
        if self.width <= 0 or self.height <= 0:
            raise ValueError("scenario: non-positive dimensions")
        if self.frame_count <= 0:
            raise ValueError("scenario: frame_count must be positive")
        if self.base_depth_mm <= self.depth_texture_mm:
            raise ValueError("scenario: base depth must exceed depth texture amplitude")

        def check_range(start, end, what):
            if start < 0 or end > self.frame_count or start >= end:
                raise ValueError(f"scenario: {what} event range outside [0, frame_count)")

        for e in self.illumination:
            check_range(e.start, e.end, "illumination")
            if not e.gain > 0.0:
                raise ValueError("scenario: illumination gain must be > 0")
        for e in self.shadows:
            check_range(e.start, e.end, "shadow")
        for e in self.flicker:
            check_range(e.start, e.end, "flicker")
        for o in self.objects:
            if o.width <= 0 or o.height <= 0:
                raise ValueError("scenario: object with non-positive size")
            if not o.waypoints:
                raise ValueError("scenario: object without waypoints")
            if any(b.frame <= a.frame for a, b in zip(o.waypoints, o.waypoints[1:])):
                raise ValueError("scenario: waypoint frames must increase")
            if o.depth_offset_mm <= 0 or o.depth_offset_mm >= self.base_depth_mm:
                raise ValueError("scenario: object depth offset outside (0, base depth)")
            for f in range(self.frame_count):
                r = object_rect_at(o, f)
                if r.x < 0 or r.y < 0 or r.x + r.w > self.width or r.y + r.h > self.height:
                    raise ValueError(f"scenario: object leaves the frame at frame {f}")


def _lround(x: float) -> int:
    """C lround: nearest, halfway cases away from zero."""
    if x < 0:
        return -_lround(-x)
    f = math.floor(x)
    return int(f) + (1 if x - f >= 0.5 else 0)


def object_rect_at(obj: ObjectSpec, frame: int) -> RegionRect:
    """Piecewise-linear waypoint track, lround'ed corner (synthetic.cpp:37-56)."""
    wp = obj.waypoints
    x, y = wp[0].x, wp[0].y
    if frame >= wp[-1].frame:
        x, y = wp[-1].x, wp[-1].y
    elif frame > wp[0].frame:
        for i in range(1, len(wp)):
            if frame <= wp[i].frame:
                t = float(frame - wp[i - 1].frame) / float(wp[i].frame - wp[i - 1].frame)
                x = wp[i - 1].x + t * (wp[i].x - wp[i - 1].x)
                y = wp[i - 1].y + t * (wp[i].y - wp[i - 1].y)
                break
    return RegionRect(_lround(x), _lround(y), obj.width, obj.height)


def builtin_scenario_names():
    return ["A", "B"]


def builtin_scenario(name: str) -> ScenarioSpec:
    """builtin_scenario (synthetic.cpp:234-273)."""
    spec = ScenarioSpec(width=640, height=480, frame_count=300, seed=1)
    spec.objects.append(ObjectSpec(24, 24, [Waypoint(0, 40, 100), Waypoint(299, 600, 320)], 400,
                                   (230, 40, 220)))
    if name == "A":
        spec.name = "A"
        spec.illumination = [IlluminationEvent(100, 112, 1.5), IlluminationEvent(200, 212, 0.6)]
        spec.shadows = [ShadowEvent(150, 180, RegionRect(300, 300, 200, 120), 0.6)]
        spec.flicker = [FlickerEvent(0, 300, RegionRect(40, 40, 80, 60), 3.0, 30.0)]
        spec.noise_color_sigma, spec.noise_depth_sigma_mm = 1.0, 1.0
        return spec
    if name == "B":
        spec.name = "B"
        gains = [1.4, 0.7, 1.25, 0.8, 1.35, 0.75, 1.2, 0.85, 1.3, 0.9]
        spec.illumination = [IlluminationEvent(30 + 25 * i, 30 + 25 * (i + 1), g)
                             for i, g in enumerate(gains)]
        spec.flicker = [FlickerEvent(0, 300, RegionRect(400, 60, 160, 120), 12.0, 40.0)]
        spec.noise_color_sigma, spec.noise_depth_sigma_mm = 1.5, 2.0
        return spec
    raise ValueError(f"unknown scenario '{name}' (known: {', '.join(builtin_scenario_names())})")


def _region(j):
    return RegionRect(int(j["x"]), int(j["y"]), int(j["w"]), int(j["h"]))


def spec_from_dict(j: dict) -> ScenarioSpec:
    """parse_scenario_spec (synthetic.cpp:286-334) on a parsed JSON object."""
    spec = ScenarioSpec(name=j.get("name", "custom"), width=int(j["width"]),
                        height=int(j["height"]), frame_count=int(j["frame_count"]),
                        seed=int(j.get("seed", 1)))
    bg = j.get("background", {})
    spec.base_depth_mm = int(bg.get("base_depth_mm", 2000))
    spec.depth_texture_mm = int(bg.get("depth_texture_mm", 30))
    spec.color_texture = int(bg.get("color_texture", 8))
    for jo in j.get("objects", []):
        color = (200, 60, 60)
        if "color" in jo:
            if len(jo["color"]) != 3:
                raise RuntimeError("object color must have 3 entries")
            color = tuple(int(c) & 0xFF for c in jo["color"])
        spec.objects.append(ObjectSpec(int(jo["width"]), int(jo["height"]),
                                       [Waypoint(int(w["frame"]), float(w["x"]), float(w["y"]))
                                        for w in jo["waypoints"]],
                                       int(jo["depth_offset_mm"]), color))
    spec.illumination = [IlluminationEvent(int(e["start"]), int(e["end"]), float(e["gain"]))
                         for e in j.get("illumination", [])]
    spec.shadows = [ShadowEvent(int(e["start"]), int(e["end"]), _region(e["region"]),
                                float(e.get("darken", 0.6))) for e in j.get("shadows", [])]
    spec.flicker = [FlickerEvent(int(e["start"]), int(e["end"]), _region(e["region"]),
                                 float(e.get("color_sigma", 0.0)),
                                 float(e.get("depth_sigma_mm", 0.0)))
                    for e in j.get("flicker", [])]
    noise = j.get("noise", {})
    spec.noise_color_sigma = float(noise.get("color_sigma", 1.0))
    spec.noise_depth_sigma_mm = float(noise.get("depth_sigma_mm", 1.0))
    spec.validate()
    return spec


def parse_scenario_spec(path) -> ScenarioSpec:
    try:
        with open(path) as fh:
            j = json.load(fh)
    except OSError:
        raise RuntimeError(f"{path}: cannot open scenario spec")
    return spec_from_dict(j)


def scenario_spec_json(spec: ScenarioSpec) -> str:
    """scenario_spec_json (synthetic.cpp:336-378)."""
    reg = lambda r: {"x": r.x, "y": r.y, "w": r.w, "h": r.h}  # noqa: E731
    return json.dumps({
        "name": spec.name, "width": spec.width, "height": spec.height,
        "frame_count": spec.frame_count, "seed": spec.seed,
        "background": {"base_depth_mm": spec.base_depth_mm,
                       "depth_texture_mm": spec.depth_texture_mm,
                       "color_texture": spec.color_texture},
        "objects": [{"width": o.width, "height": o.height, "depth_offset_mm": o.depth_offset_mm,
                     "color": list(o.color),
                     "waypoints": [{"frame": w.frame, "x": w.x, "y": w.y} for w in o.waypoints]}
                    for o in spec.objects],
        "illumination": [{"start": e.start, "end": e.end, "gain": e.gain}
                         for e in spec.illumination],
        "shadows": [{"start": e.start, "end": e.end, "region": reg(e.region), "darken": e.darken}
                    for e in spec.shadows],
        "flicker": [{"start": e.start, "end": e.end, "region": reg(e.region),
                     "color_sigma": e.color_sigma, "depth_sigma_mm": e.depth_sigma_mm}
                    for e in spec.flicker],
        "noise": {"color_sigma": spec.noise_color_sigma,
                  "depth_sigma_mm": spec.noise_depth_sigma_mm},
    }, indent=2)


SceneFrameC = _lib.SceneFrameC


def resolve_frame(spec: ScenarioSpec, frame: int, streams: int = 1,
                  seed0: Optional[int] = None) -> SceneFrameC:
    """render_frame's per-frame quantities (synthetic.cpp:124-134)."""
    if len(spec.objects) > 4:
        raise ValueError("render: at most 4 objects")
    f = SceneFrameC()
    f.width, f.height, f.streams = spec.width, spec.height, streams
    f.seed0 = spec.seed if seed0 is None else seed0
    f.frame = frame
    f.base_depth_mm, f.depth_texture_mm = spec.base_depth_mm, spec.depth_texture_mm
    f.color_texture = spec.color_texture
    gain = 1.0
    for e in spec.illumination:
        if e.start <= frame < e.end:
            gain *= e.gain
    f.gain = gain
    f.n_obj = len(spec.objects)
    for k, o in enumerate(spec.objects):
        r = object_rect_at(o, frame)
        f.obj_rect[k][0], f.obj_rect[k][1], f.obj_rect[k][2], f.obj_rect[k][3] = r.x, r.y, r.w, r.h
        for c in range(3):
            f.obj_color[k][c] = int(o.color[c])
        f.obj_depth_offset_mm[k] = o.depth_offset_mm
    sh = [e for e in spec.shadows if e.start <= frame < e.end]
    fl = [e for e in spec.flicker if e.start <= frame < e.end]
    if len(sh) > 16 or len(fl) > 16:
        raise ValueError("render: at most 16 active events of each kind")
    f.n_shadow, f.n_flicker = len(sh), len(fl)
    for k, e in enumerate(sh):
        for i, v in enumerate((e.region.x, e.region.y, e.region.w, e.region.h)):
            f.shadow_rect[k][i] = v
        f.shadow_darken[k] = e.darken
    for k, e in enumerate(fl):
        for i, v in enumerate((e.region.x, e.region.y, e.region.w, e.region.h)):
            f.flicker_rect[k][i] = v
        f.flicker_color_sigma[k] = e.color_sigma
        f.flicker_depth_sigma_mm[k] = e.depth_sigma_mm
    f.noise_color_sigma = spec.noise_color_sigma
    f.noise_depth_sigma_mm = spec.noise_depth_sigma_mm
    return f


def render_frame(spec: ScenarioSpec, frame: int, streams: int = 1, seed0: Optional[int] = None,
                 device: int = 0, with_gt: bool = True):
    """render_frame (synthetic.cpp:119-195) for `streams` seeds on the GPU;
    returns CUDA tensors of shape (streams, height, width)."""
    import torch

    f = resolve_frame(spec, frame, streams, seed0)
    shp = (streams, spec.height, spec.width)
    dev = torch.device("cuda", device)
    out = {"r": torch.empty(shp, dtype=torch.uint8, device=dev),
           "g": torch.empty(shp, dtype=torch.uint8, device=dev),
           "b": torch.empty(shp, dtype=torch.uint8, device=dev),
           "depth": torch.empty(shp, dtype=torch.uint16, device=dev)}
    if with_gt:
        out["gt"] = torch.empty(shp, dtype=torch.uint8, device=dev)
    gt = out.get("gt")
    check(lib.rgbdseg_render_frame(C.byref(f), out["r"].data_ptr(), out["g"].data_ptr(),
                                   out["b"].data_ptr(), out["depth"].data_ptr(),
                                   gt.data_ptr() if gt is not None else None, device, None),
          "render_frame")
    return out

