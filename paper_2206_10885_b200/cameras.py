"""Pinhole cameras: same interface as the reference ``kilofield.cameras`` (cameras.py).

``CameraPose`` / ``look_at_pose`` / ``poses_on_sphere`` are host-side bookkeeping;
``pixel_rays`` runs on the GPU (knf_pixel_rays) with the reference's exact fp64 arithmetic.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N


@dataclass
class CameraPose:
    """cameras.py:10-36: rotation columns are the camera's right/up/back axes; looks along -z."""

    position: np.ndarray
    rotation: np.ndarray
    fov_y: float
    width: int
    height: int

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=np.float64)
        self.rotation = np.asarray(self.rotation, dtype=np.float64)
        if self.rotation.shape != (3, 3):
            raise ValueError("rotation must be 3x3")
        if not np.allclose(self.rotation @ self.rotation.T, np.eye(3), atol=1e-6):
            raise ValueError("rotation must be orthonormal")
        if np.linalg.det(self.rotation) < 0:
            raise ValueError("rotation must have determinant +1")
        if not (0 < self.fov_y < np.pi):
            raise ValueError("fov_y must be in (0, pi)")
        if self.width <= 0 or self.height <= 0:
            raise ValueError("image dimensions must be positive")


def look_at_pose(position, target, up, fov_y: float, width: int, height: int) -> CameraPose:
    """cameras.py:39-54."""
    eye = np.asarray(position, dtype=np.float64)
    ahead = np.asarray(target, dtype=np.float64) - eye
    dist = np.linalg.norm(ahead)
    if dist < 1e-12:
        raise ValueError("camera position coincides with target")
    ahead = ahead / dist
    up = np.asarray(up, dtype=np.float64)
    if abs(np.dot(ahead, up) / max(np.linalg.norm(up), 1e-12)) > 0.999:
        up = np.array([1.0, 0.0, 0.0]) if abs(ahead[0]) < 0.9 else np.array([0.0, 0.0, 1.0])
    side = np.cross(ahead, up)
    side /= np.linalg.norm(side)
    return CameraPose(eye, np.stack([side, np.cross(side, ahead), -ahead], axis=1), fov_y, width, height)


def camera_struct(pose) -> N.KnfCamera:
    cam = N.KnfCamera()
    cam.position = N.vec3(pose.position)
    cam.rotation = (C.c_double * 9)(*np.asarray(pose.rotation, dtype=np.float64).reshape(9))
    cam.fov_y = float(pose.fov_y)
    cam.width = int(pose.width)
    cam.height = int(pose.height)
    return cam


def pixel_rays(pose, pixel_xy=None, jitter=None, device: int | None = None):
    """cameras.pixel_rays (cameras.py:57-76) -> (origins (n,3), unit directions (n,3)), fp64.

    pixel_xy: (n,2) integer (column,row) pairs, or None for the full raster in row-major order.
    jitter: (n,2) sub-pixel offsets, or None for pixel centres.
    """
    from .grid import _default_device

    N.require_gpu()
    device = _default_device() if device is None else device
    if pixel_xy is None:
        n = int(pose.width) * int(pose.height)
        px = None
    else:
        px_in = np.asarray(pixel_xy)
        if not np.issubdtype(px_in.dtype, np.integer):
            if not np.all(px_in == np.round(px_in)):
                raise ValueError("pixel_xy must hold integer pixel indices (use jitter for sub-pixel offsets)")
        px = np.ascontiguousarray(px_in, dtype=np.int32).reshape(-1, 2)
        n = px.shape[0]
    jt = None
    if jitter is not None:
        jt = np.ascontiguousarray(jitter, dtype=np.float64).reshape(-1, 2)
        if jt.shape[0] != n:
            raise ValueError("jitter must have one row per pixel")
    origins = np.empty((n, 3), dtype=np.float64)
    dirs = np.empty((n, 3), dtype=np.float64)
    cam = camera_struct(pose)
    N.check(N.load().knf_pixel_rays(C.byref(cam), N.ptr(px), N.ptr(jt), n, N.ptr(origins), N.ptr(dirs), device,
                                    N.MEM_HOST, N.current_stream(device)))
    return origins, dirs


def poses_on_sphere(n_views: int, radius: float, fov_y: float, width: int, height: int, seed):
    """cameras.py:79-87."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_views):
        v = rng.normal(size=3)
        v /= np.linalg.norm(v)
        out.append(look_at_pose(radius * v, (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), fov_y, width, height))
    return out


def orbit_pose(k: int, n_views: int, radius: float, elevation: float, fov_y: float, width: int, height: int):
    """The viewer's orbit parametrisation (frontend orbit.ts:36-53), used by BASELINE config 2."""
    az = 2.0 * np.pi * k / n_views
    pos = radius * np.array([np.cos(elevation) * np.sin(az), np.sin(elevation), np.cos(elevation) * np.cos(az)])
    return look_at_pose(pos, (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), fov_y, width, height)
