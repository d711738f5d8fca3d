"""SURVEY 8(f) "next" rows: the callers on either side of the hot path, kept on the device.

* ``render_pass_u8``  -- what ``service.RenderService._render_once`` does for the sphere-traced
  renderer (service.py:279-288): ``to_uint8(pass_image(render_frame(...), render_pass))``, fused on the
  GPU so 3 bytes per pixel cross PCIe instead of 29.
* ``tonemap_u8``      -- ``to_uint8(clip(hdr / spp, 0, 1) ** (1 / 2.2))`` of the progressive path-trace
  branch (service.py:297-299), or plain ``images.to_uint8`` (images.py:15-17).
* ``sample_volume``   -- ``mesh._sample_volume`` (mesh.py:43-57): SDF values on the marching-cubes lattice.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .cameras import camera_struct
from .grid import _default_device, device_field
from .surface import PASSES, RenderAborted, RenderSettings, _need_field_surface, _settings_struct


def render_pass_u8(surface, pose, settings: RenderSettings | None = None, background=(1.0, 1.0, 1.0), supersample: int = 1,
                   tile_rows: int = 32, abort_check=None) -> np.ndarray:
    """(H, W, 3) uint8 image of ``settings.render_pass``; ``abort_check`` is polled per band like render_frame."""
    settings = settings or RenderSettings()
    fs = _need_field_surface(surface)
    cam, st, bg = camera_struct(pose), _settings_struct(settings), N.vec3(background)
    H, W = int(pose.height), int(pose.width)
    out = np.empty((H, W, 3), dtype=np.uint8)
    code = PASSES.index(settings.render_pass)
    bands = [(0, H)] if abort_check is None else [(r, min(r + tile_rows, H)) for r in range(0, H, tile_rows)]
    for r0, r1 in bands:
        if abort_check is not None and abort_check():
            raise RenderAborted("camera or settings changed")
        N.check(N.load().knf_render_pass_u8(fs.dev.handle, C.byref(cam), C.byref(st), C.byref(bg), int(supersample), code, r0, r1,
                                            N.ptr(out[r0:r1]), N.MEM_HOST, N.current_stream(fs.dev.device)))
    return out


def tonemap_u8(img, divisor: float = 1.0, gamma22: bool = False, device: int | None = None) -> np.ndarray:
    a = np.ascontiguousarray(img, dtype=np.float64)
    out = np.empty(a.shape, dtype=np.uint8)
    device = _default_device() if device is None else device
    N.check(N.load().knf_tonemap_u8(N.ptr(a), a.size, float(divisor), int(bool(gamma22)), N.ptr(out), device, N.MEM_HOST,
                                    N.current_stream(device)))
    return out


def to_uint8(img) -> np.ndarray:
    """images.to_uint8 (images.py:15-17)."""
    return tonemap_u8(img)


def sample_volume(field, resolution: int, bbox_min=(-1.0, -1.0, -1.0), bbox_max=(1.0, 1.0, 1.0)) -> np.ndarray:
    """mesh._sample_volume for a KiloField -> (R, R, R) float64 SDF lattice."""
    dev = device_field(field)
    vals = np.empty(int(resolution) ** 3, dtype=np.float32)
    lo, hi = N.vec3(bbox_min), N.vec3(bbox_max)
    N.check(N.load().knf_sample_volume(dev.handle, int(resolution), C.byref(lo), C.byref(hi), N.ptr(vals), N.MEM_HOST,
                                       N.current_stream(dev.device)))
    return vals.astype(np.float64).reshape(resolution, resolution, resolution)


def volume_forward(field, origins, dirs, n_s: int, jitter=None, background=(1.0, 1.0, 1.0), s: float | None = None) -> np.ndarray:
    """training._volume_forward (training.py:330-415), forward only -> (B,3) float64 colours.

    ``s`` defaults to ``exp(field.inv_std_param)`` like the reference.  (Rays that miss the box return the
    background clipped to [0,1]; the reference leaves it unclipped when other rays of the batch are active.)
    """
    dev = device_field(field)
    o = np.ascontiguousarray(np.atleast_2d(origins), dtype=np.float64)
    d = np.ascontiguousarray(np.atleast_2d(dirs), dtype=np.float64)
    if o.shape != d.shape or o.shape[1] != 3:
        raise ValueError("origins and dirs must both be (B,3)")
    B = o.shape[0]
    jit = None
    if jitter is not None:
        jit = np.ascontiguousarray(jitter, dtype=np.float64)
        if jit.shape != (B, n_s):
            raise ValueError("jitter must be (B, n_s)")
    if s is None:
        s = float(np.exp(field.inv_std_param))
    out = np.empty((B, 3), dtype=np.float64)
    bg = N.vec3(background)
    N.check(N.load().knf_volume_forward(dev.handle, N.ptr(o), N.ptr(d), B, int(n_s), N.ptr(jit), C.byref(bg), float(s), N.ptr(out),
                                        N.MEM_HOST, N.current_stream(dev.device)))
    return out


def photometric_loss(field, pose, pixels, target, n_s: int, jitter=None, background=(1.0, 1.0, 1.0)) -> float:
    """training.photometric_loss (training.py:500-517): mean L1 between volume-rendered and target colours.
    ``target`` is the (B,3) colour of each pixel (the reference indexes image.pixels itself)."""
    from .cameras import pixel_rays

    origins, dirs = pixel_rays(pose, pixels)
    colors = volume_forward(field, origins, dirs, n_s, jitter, background)
    return float(np.abs(colors - np.asarray(target, dtype=np.float64)).sum() / len(colors))


class ProgressivePathtracer:
    """The progressive path-trace branch of ``service.RenderService._render_once`` (service.py:289-300) with the
    accumulator kept on the device: every ``add_sample()`` traces ONE more sample per pixel
    (``render_pathtraced(scene, pose, spp=1, seed, sample_offset=k)``), adds it to the running fp64 sum in HBM and
    returns ``to_uint8(clip(sum / k, 0, 1) ** (1 / 2.2))`` -- 3 bytes per pixel cross PCIe per cycle instead of the
    24-byte fp64 radiance the reference's host-side accumulation would need.  ``hdr()`` downloads the running mean
    (== ``render_pathtraced(spp=k).hdr`` up to the summation order: the per-pixel counter RNG makes sample k
    independent of how the samples are batched, pathtrace.py:439-442)."""

    def __init__(self, scene, pose, seed: int = 12345, max_bounces: int = 8):
        import torch

        from . import pathtrace as P

        self._P, self._torch = P, torch
        self.scene, self.pose, self.seed, self.max_bounces = scene, pose, int(seed), int(max_bounces)
        self.device = P._device_index(scene)
        self.accum = torch.zeros((int(pose.height), int(pose.width), 3), dtype=torch.float64, device=torch.device("cuda", self.device))
        self.spp = 0
        self._u8 = torch.empty((int(pose.height), int(pose.width), 3), dtype=torch.uint8, device=self.accum.device)
        self._host = torch.empty((int(pose.height), int(pose.width), 3), dtype=torch.uint8).pin_memory()

    def add_sample(self, abort_check=None) -> np.ndarray:
        if abort_check is not None and abort_check():
            raise RenderAborted("stale path-trace batch")
        H = int(self.pose.height)
        hdr = self._P.pathtrace_rows(self.scene, self.pose, 1, self.seed, self.max_bounces, self.spp, 0, H, device_out=True)
        if abort_check is not None and abort_check():
            raise RenderAborted("stale path-trace batch")  # service.py:294-295: the batch is dropped, the sum untouched
        self.accum.add_(hdr)
        self.spp += 1
        N.check(N.load().knf_tonemap_u8(N.ptr(self.accum), self.accum.numel(), float(self.spp), 1, N.ptr(self._u8), self.device,
                                        N.MEM_DEVICE, N.current_stream(self.device)))
        self._host.copy_(self._u8, non_blocking=False)
        return self._host.numpy().copy()

    def hdr(self) -> np.ndarray:
        return (self.accum / max(self.spp, 1)).cpu().numpy()
