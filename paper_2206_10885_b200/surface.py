"""Primary-visibility renderer on the B200: same interface as the reference
``kilofield.surface`` (surface.py) -- AABB slabs, wavefront sphere tracing with secant
refinement, FD-normal shading, frame buffers.

Only ``FieldSurface`` is traceable here (the grid field is the path being accelerated); handing
any other "traceable" object to these functions raises ``TypeError`` -- there is no CPU tracer
in this package.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import grid as gridmod
from .cameras import CameraPose, camera_struct

PASS_COLOR = "color"
PASS_NORMAL = "normal"
PASS_DEPTH = "depth"
PASSES = (PASS_COLOR, PASS_NORMAL, PASS_DEPTH)

DEPTH_MISS = np.inf


def thread_count() -> int:
    """surface.thread_count (surface.py:32-39).  Kept for callers that size thread pools from it; the
    device renderer does not use host threads."""
    import os

    env = os.environ.get("KNF_THREADS")
    if env:
        try:
            return max(1, int(env))
        except ValueError:
            pass
    return max(1, os.cpu_count() or 1)


class RenderAborted(RuntimeError):
    """Frame rendering stopped early by the abort callback (surface.py:28-29)."""


@dataclass
class Ray:
    origin: np.ndarray
    direction: np.ndarray

    def __post_init__(self):
        self.origin = np.asarray(self.origin, dtype=np.float64)
        self.direction = np.asarray(self.direction, dtype=np.float64)
        if not np.isclose(np.linalg.norm(self.direction), 1.0, atol=1e-6):
            raise ValueError("ray direction must be unit length")


@dataclass
class Hit:
    t: float
    position: np.ndarray
    normal: np.ndarray
    color: np.ndarray
    steps_taken: int


@dataclass
class RenderSettings:
    eps_hit: float = 1e-3
    max_steps: int = 128
    step_scale: float = 0.8
    render_pass: str = PASS_COLOR

    def __post_init__(self):
        if not (0 < self.step_scale <= 1):
            raise ValueError("step_scale must be in (0, 1]")
        if self.render_pass not in PASSES:
            raise ValueError(f"unknown pass {self.render_pass!r}")


def _settings_struct(s) -> N.KnfSettings:
    out = N.KnfSettings()
    out.eps_hit = float(s.eps_hit)
    out.max_steps = int(s.max_steps)
    out.step_scale = float(s.step_scale)
    return out


class FieldSurface:
    """surface.FieldSurface (surface.py:82-99) backed by the device copy of the field.

    Also a drop-in *for the reference's own tracer*: ``kilofield.surface.march_rays`` /
    ``render_frame`` / ``pathtrace.NeuralObject`` accept this object and then run the
    reference's Python loop on GPU SDF evaluations (the lock-step parity harness).
    """

    def __init__(self, kfield, device: int | None = None):
        self.field = kfield
        self._device = device
        self._dev = gridmod.device_field(kfield, device)
        self.bbox_min = np.asarray(self._dev.config.bbox_min, dtype=np.float64)
        self.bbox_max = np.asarray(self._dev.config.bbox_max, dtype=np.float64)

    @property
    def dev(self):
        """The device copy, re-resolved through the cache: after grid.invalidate(field) the next use uploads the
        mutated arrays instead of rendering the stale copy."""
        if not isinstance(self.field, gridmod.DeviceField):
            cur = gridmod.device_field(self.field, self._device if self._device is not None else self._dev.device)
            if cur is not self._dev:
                self._dev = cur
        return self._dev

    def sdf_values(self, pts):
        return gridmod.sdf_values(self.dev, pts).astype(np.float64)

    def shade(self, pts, view_dirs):
        dev = self.dev
        p = _rows3(pts)
        v = _rows3(view_dirs)
        if p.shape != v.shape or p.shape[1] != 3:
            raise ValueError("pts and view_dirs must both be (n,3)")
        colors = np.empty_like(p)
        normals = np.empty_like(p)
        N.check(N.load().knf_shade(dev.handle, N.ptr(p), N.ptr(v), p.shape[0], N.ptr(colors), N.ptr(normals),
                                   N.MEM_HOST, N.current_stream(dev.device)))
        return colors, normals


def _need_field_surface(surface) -> FieldSurface:
    if isinstance(surface, FieldSurface):
        return surface
    raise TypeError(
        "paper_2206_10885_b200 traces FieldSurface objects only (got "
        f"{type(surface).__name__}); analytic teachers stay on the reference's CPU tracer"
    )


# ---------------------------------------------------------------------------------------------
# intersection and marching


def _rows3(a) -> np.ndarray:
    """(n,3) float64 view of a ray array; an empty input is (0,3), as the reference's asarray-and-index code treats it
    (np.atleast_2d([]) would be (1,0))."""
    a = np.asarray(a, dtype=np.float64)
    if a.size == 0:
        return np.zeros((0, 3), dtype=np.float64)
    return np.ascontiguousarray(np.atleast_2d(a))


def ray_aabb_batch(origins, dirs, bbox_min, bbox_max, device: int | None = None):
    """surface.ray_aabb_batch (surface.py:131-149) -> (max(t_enter,0), t_exit, hit)."""
    N.require_gpu()
    device = gridmod._default_device() if device is None else device
    o = _rows3(origins)
    d = _rows3(dirs)
    if o.shape != d.shape or o.shape[1] != 3:
        raise ValueError("origins and dirs must both be (n,3)")
    n = o.shape[0]
    tn = np.empty(n, dtype=np.float64)
    tf = np.empty(n, dtype=np.float64)
    hit = np.empty(n, dtype=np.uint8)
    lo, hi = N.vec3(bbox_min), N.vec3(bbox_max)
    N.check(N.load().knf_ray_aabb(N.ptr(o), N.ptr(d), n, C.byref(lo), C.byref(hi), N.ptr(tn), N.ptr(tf), N.ptr(hit),
                                  device, N.MEM_HOST, N.current_stream(device)))
    return tn, tf, hit.astype(bool)


def ray_aabb(ray: Ray, bbox_min, bbox_max):
    """surface.ray_aabb (surface.py:123-128)."""
    t0, t1, hit = ray_aabb_batch(ray.origin[None, :], ray.direction[None, :], bbox_min, bbox_max)
    if not hit[0]:
        return None
    return float(t0[0]), float(t1[0])


@dataclass
class TraceResult:
    hit: np.ndarray
    t: np.ndarray
    position: np.ndarray
    steps: np.ndarray
    normal: np.ndarray | None = None
    color: np.ndarray | None = None


def march_rays(surface, origins, dirs, t_near, t_far, settings: RenderSettings) -> TraceResult:
    """surface.march_rays (surface.py:162-226): the whole lock-step loop runs on the device as a
    wavefront (route by cell -> tile MLP -> step/secant kernel), one call."""
    fs = _need_field_surface(surface)
    o = _rows3(origins)
    d = _rows3(dirs)
    tn = np.ascontiguousarray(t_near, dtype=np.float64).reshape(-1)
    tf = np.ascontiguousarray(t_far, dtype=np.float64).reshape(-1)
    n = o.shape[0]
    if o.shape != d.shape or o.shape[1] != 3 or tn.shape[0] != n or tf.shape[0] != n:
        raise ValueError("origins/dirs must be (n,3) and t_near/t_far (n,)")
    hit = np.zeros(n, dtype=np.uint8)
    t = np.zeros(n, dtype=np.float64)
    pos = np.empty((n, 3), dtype=np.float64)
    steps = np.zeros(n, dtype=np.int32)
    st = _settings_struct(settings)
    N.check(N.load().knf_march(fs.dev.handle, N.ptr(o), N.ptr(d), N.ptr(tn), N.ptr(tf), n, C.byref(st), N.ptr(hit),
                               N.ptr(t), N.ptr(pos), N.ptr(steps), N.MEM_HOST, N.current_stream(fs.dev.device)))
    if n == 0:
        pos = o.copy()
    return TraceResult(hit=hit.astype(bool), t=t, position=pos, steps=steps)


def trace_and_shade(surface, origins, dirs, settings: RenderSettings) -> TraceResult:
    """surface.trace_and_shade (surface.py:229-241)."""
    fs = _need_field_surface(surface)
    o = _rows3(origins)
    d = _rows3(dirs)
    if o.shape != d.shape or o.shape[1] != 3:
        raise ValueError("origins and dirs must both be (n,3)")
    n = o.shape[0]
    hit = np.zeros(n, dtype=np.uint8)
    t = np.zeros(n, dtype=np.float64)
    pos = np.empty((n, 3), dtype=np.float64)
    steps = np.zeros(n, dtype=np.int32)
    nrm = np.zeros((n, 3), dtype=np.float64)
    col = np.zeros((n, 3), dtype=np.float64)
    st = _settings_struct(settings)
    N.check(N.load().knf_trace_and_shade(fs.dev.handle, N.ptr(o), N.ptr(d), n, C.byref(st), N.ptr(hit), N.ptr(t),
                                         N.ptr(pos), N.ptr(steps), N.ptr(nrm), N.ptr(col), N.MEM_HOST,
                                         N.current_stream(fs.dev.device)))
    return TraceResult(hit=hit.astype(bool), t=t, position=pos, steps=steps, normal=nrm, color=col)


def sphere_trace(surface, ray: Ray, t_near: float, t_far: float, settings: RenderSettings) -> Hit | None:
    """surface.sphere_trace (surface.py:244-258): single-ray march; None on a miss."""
    if not t_near < t_far:
        raise ValueError("need t_near < t_far")
    fs = _need_field_surface(surface)
    res = march_rays(fs, ray.origin[None, :], ray.direction[None, :], np.array([t_near]), np.array([t_far]), settings)
    if not res.hit[0]:
        return None
    colors, normals = fs.shade(res.position[:1], ray.direction[None, :])
    return Hit(t=float(res.t[0]), position=res.position[0], normal=normals[0], color=np.clip(colors[0], 0.0, 1.0),
               steps_taken=int(res.steps[0]))


# ---------------------------------------------------------------------------------------------
# frame rendering


@dataclass
class FrameBuffers:
    color: np.ndarray  # (H, W, 3) float32, background composited
    depth: np.ndarray  # (H, W) float32, +inf at misses
    normal: np.ndarray  # (H, W, 3) float32, zeros at misses
    hit: np.ndarray  # (H, W) bool


def render_rows(surface, pose, settings, background, supersample, row0, row1, out=None, device_out=False):
    """Rows [row0,row1) of a frame through knf_render_frame.  With device_out the buffers are torch
    CUDA tensors and nothing is copied to the host (the resident path bench.py times)."""
    fs = _need_field_surface(surface)
    cam = camera_struct(pose)
    st = _settings_struct(settings)
    bg = N.vec3(background)
    rows, W = row1 - row0, int(pose.width)
    if device_out:
        import torch

        dev = torch.device("cuda", fs.dev.device)
        if out is None:
            out = (torch.empty((rows, W, 3), dtype=torch.float32, device=dev),
                   torch.empty((rows, W), dtype=torch.float32, device=dev),
                   torch.empty((rows, W, 3), dtype=torch.float32, device=dev),
                   torch.empty((rows, W), dtype=torch.uint8, device=dev))
        mem = N.MEM_DEVICE
    else:
        if out is None:
            out = (np.empty((rows, W, 3), dtype=np.float32), np.empty((rows, W), dtype=np.float32),
                   np.empty((rows, W, 3), dtype=np.float32), np.empty((rows, W), dtype=np.uint8))
        mem = N.MEM_HOST
    color, depth, normal, hit = out
    N.check(N.load().knf_render_frame(fs.dev.handle, C.byref(cam), C.byref(st), C.byref(bg), int(supersample),
                                      int(row0), int(row1), N.ptr(color), N.ptr(depth), N.ptr(normal), N.ptr(hit), mem,
                                      N.current_stream(fs.dev.device)))
    return out


def render_frame(surface, pose: CameraPose, settings: RenderSettings | None = None, background=(1.0, 1.0, 1.0),
                 supersample: int = 1, tile_rows: int = 32, abort_check=None) -> FrameBuffers:
    """surface.render_frame (surface.py:273-336).

    Every pixel is a pure function of its ray, so banding does not change the result; without an
    ``abort_check`` the whole frame is one device call, with one the callback is polled before each
    band of ``tile_rows`` rows exactly as the reference polls it (surface.py:303-305).
    """
    settings = settings or RenderSettings()
    if supersample < 1:
        raise ValueError("supersample must be >= 1")
    if tile_rows < 1:
        raise ValueError("tile_rows must be >= 1")
    fs = _need_field_surface(surface)
    H, W = int(pose.height), int(pose.width)
    if abort_check is None:
        color, depth, normal, hit = render_rows(fs, pose, settings, background, supersample, 0, H)
        return FrameBuffers(color=color, depth=depth, normal=normal, hit=hit.astype(bool))
    color = np.empty((H, W, 3), dtype=np.float32)
    depth = np.full((H, W), DEPTH_MISS, dtype=np.float32)
    normal = np.zeros((H, W, 3), dtype=np.float32)
    hit = np.zeros((H, W), dtype=np.uint8)
    for r0 in range(0, H, tile_rows):
        if abort_check():
            raise RenderAborted("camera or settings changed")
        r1 = min(r0 + tile_rows, H)
        render_rows(fs, pose, settings, background, supersample, r0, r1,
                    out=(color[r0:r1], depth[r0:r1], normal[r0:r1], hit[r0:r1]))
    return FrameBuffers(color=color, depth=depth, normal=normal, hit=hit.astype(bool))


def pass_image(buffers: FrameBuffers, render_pass: str, background=(1.0, 1.0, 1.0)) -> np.ndarray:
    """surface.pass_image (surface.py:339-350): displayable float RGB in [0,1]."""
    if render_pass == PASS_COLOR:
        return buffers.color.astype(np.float64)
    if render_pass == PASS_NORMAL:
        img = 0.5 * (buffers.normal.astype(np.float64) + 1.0)
        img[~buffers.hit] = 0.0
        return img
    if render_pass == PASS_DEPTH:
        g = np.where(np.isfinite(buffers.depth), 1.0 / (1.0 + buffers.depth), 0.0)
        return np.repeat(g[:, :, None], 3, axis=2)
    raise ValueError(f"unknown pass {render_pass!r}")
