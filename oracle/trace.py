"""Oracle part 2: cameras, ray/AABB slabs, sphere tracing, shading, frame render
(TEST INFRASTRUCTURE ONLY).  Restates reference ``cameras.py`` and ``surface.py``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import field as F

MISS_DEPTH = np.inf  # surface.py:25


# ---------------------------------------------------------------------------
# camera (reference cameras.py:10-76)


@dataclass
class Camera:
    """cameras.py:10-36: rotation columns = right / up / back; looks along -z."""

    position: np.ndarray
    rotation: np.ndarray
    fov_y: float
    width: int
    height: int

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=np.float64)
        self.rotation = np.asarray(self.rotation, dtype=np.float64)


def camera_look_at(position, target, up, fov_y, width, height) -> Camera:
    """cameras.py:39-54."""
    position = np.asarray(position, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - position
    length = np.linalg.norm(fwd)
    if length < 1e-12:
        raise ValueError("camera position coincides with target")
    fwd = fwd / length
    up = np.asarray(up, dtype=np.float64)
    if abs(np.dot(fwd, up) / max(np.linalg.norm(up), 1e-12)) > 0.999:
        up = np.array([1.0, 0.0, 0.0]) if abs(fwd[0]) < 0.9 else np.array([0.0, 0.0, 1.0])
    right = np.cross(fwd, up)
    right /= np.linalg.norm(right)
    up2 = np.cross(right, fwd)
    return Camera(position, np.stack([right, up2, -fwd], axis=1), fov_y, width, height)


def camera_rays(cam: Camera, pixels=None, jitter=None):
    """cameras.py:57-76.  pixels: (n,2) (col,row).  fp64 throughout.

    px = (col + off_x - W/2) * s ; py = (H/2 - row - off_y) * s ; s = 2 tan(fov/2) / H
    dir = normalise([px, py, -1] @ R^T); origin broadcast.
    """
    if pixels is None:
        cc, rr = np.meshgrid(np.arange(cam.width), np.arange(cam.height))
        pixels = np.stack([cc.ravel(), rr.ravel()], axis=1)
    pixels = np.asarray(pixels, dtype=np.float64)
    off = np.full_like(pixels, 0.5) if jitter is None else jitter
    s = 2.0 * np.tan(cam.fov_y / 2) / cam.height
    px = (pixels[:, 0] + off[:, 0] - cam.width / 2) * s
    py = (cam.height / 2 - pixels[:, 1] - off[:, 1]) * s
    local = np.stack([px, py, -np.ones_like(px)], axis=1)
    world = local @ cam.rotation.T
    world /= np.linalg.norm(world, axis=1, keepdims=True)
    origins = np.ascontiguousarray(np.broadcast_to(cam.position, world.shape))
    return origins, world


# ---------------------------------------------------------------------------
# settings + traceable adapter (reference surface.py:64-99)


@dataclass
class MarchSettings:
    """surface.py:64-75."""

    eps_hit: float = 1e-3
    max_steps: int = 128
    step_scale: float = 0.8
    render_pass: str = "color"

    def __post_init__(self):
        if not (0 < self.step_scale <= 1):
            raise ValueError("step_scale must be in (0, 1]")
        if self.render_pass not in ("color", "normal", "depth"):
            raise ValueError(f"unknown pass {self.render_pass!r}")


class FieldTraceable:
    """surface.py:82-99: bbox + sdf_values + shade on an OracleField."""

    def __init__(self, field: F.OracleField):
        self.field = field
        self.bbox_min = field.spec.lo
        self.bbox_max = field.spec.hi

    def sdf_values(self, pts):
        return F.query_sdf_values(self.field, pts).astype(np.float64)

    def shade(self, pts, view_dirs):
        # surface.py:93-99: FD normals (fallback: face the ray), a SECOND sdf query for
        # the features, then the colour MLP.
        nrm, ok = F.fd_normals(self.field, pts)
        nrm[~ok] = -view_dirs[~ok]
        _, feats = F.query_sdf(self.field, pts)
        rgb = F.query_color(self.field, pts, view_dirs, nrm, feats)
        return rgb.astype(np.float64), nrm


# ---------------------------------------------------------------------------
# slabs + march (reference surface.py:131-241)


def slab_intersect(origins, dirs, lo, hi):
    """surface.py:131-149 -> (max(t_enter,0), t_exit, hit)."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / dirs
        ta = (lo - origins) * inv
        tb = (hi - origins) * inv
    t_in = np.minimum(ta, tb)
    t_out = np.maximum(ta, tb)
    flat = dirs == 0.0
    if np.any(flat):
        within = (origins >= lo) & (origins <= hi)
        t_in = np.where(flat, np.where(within, -np.inf, np.inf), t_in)
        t_out = np.where(flat, np.where(within, np.inf, -np.inf), t_out)
    enter = t_in.max(axis=1)
    leave = t_out.min(axis=1)
    return np.maximum(enter, 0.0), leave, (leave >= enter) & (leave >= 0)


@dataclass
class MarchOutput:
    hit: np.ndarray
    t: np.ndarray
    position: np.ndarray
    steps: np.ndarray
    normal: np.ndarray | None = None
    color: np.ndarray | None = None


def march(surface, origins, dirs, t_near, t_far, cfg: MarchSettings, trace_log=None) -> MarchOutput:
    """surface.py:162-226.  Lock-step sphere tracing.

    Per ray (fp64 state): t starts at t_near, live while t_near < t_far.  Each round
    evaluates d = sdf(o + t dir) for every live ray and counts a step.
      |d| <= eps  -> converged.  If a previous sample exists and |d - d_prev| > 1e-12,
                     try the secant root clipped to [lo, hi + (hi - lo)] with
                     lo/hi = min/max(t, t_prev); keep it only if |sdf| there is not larger.
      otherwise   -> remember (t, d), advance t += scale * max(d, eps/2); retire if t > t_far.
    ``trace_log`` (a list) receives per-round (ray indices, t, d) for lock-step parity tests.
    """
    n = len(origins)
    eps = cfg.eps_hit
    t = t_near.copy()
    live = t_near < t_far
    hit = np.zeros(n, dtype=bool)
    steps = np.zeros(n, dtype=np.int32)
    t_final = np.zeros(n)
    t_last = np.full(n, np.nan)
    d_last = np.full(n, np.nan)

    for _ in range(cfg.max_steps):
        rays = np.flatnonzero(live)
        if rays.size == 0:
            break
        d = surface.sdf_values(origins[rays] + t[rays, None] * dirs[rays])
        steps[rays] += 1
        if trace_log is not None:
            trace_log.append((rays.copy(), t[rays].copy(), d.copy()))

        close = np.abs(d) <= eps
        done = rays[close]
        if done.size:
            tc, dc = t[done], d[close]
            tp, dp = t_last[done], d_last[done]
            root = tc.copy()
            usable = np.isfinite(tp) & (np.abs(dc - dp) > 1e-12)
            root[usable] = tc[usable] - dc[usable] * (tc[usable] - tp[usable]) / (dc[usable] - dp[usable])
            a = np.minimum(tc, tp)
            b = np.maximum(tc, tp)
            root[usable] = np.clip(root[usable], a[usable], b[usable] + (b[usable] - a[usable]))
            if np.any(usable):
                probe = origins[done[usable]] + root[usable, None] * dirs[done[usable]]
                d_probe = surface.sdf_values(probe)
                if trace_log is not None:
                    trace_log.append((done[usable].copy(), root[usable].copy(), d_probe.copy()))
                reject = np.abs(d_probe) > np.abs(dc[usable])
                back = np.flatnonzero(usable)[reject]
                root[back] = tc[back]
            hit[done] = True
            t_final[done] = root
            live[done] = False

        moving = rays[~close]
        if moving.size:
            dm = d[~close]
            t_last[moving] = t[moving]
            d_last[moving] = dm
            t[moving] = t[moving] + cfg.step_scale * np.maximum(dm, eps / 2)
            live[moving[t[moving] > t_far[moving]]] = False

    return MarchOutput(hit=hit, t=t_final, position=origins + t_final[:, None] * dirs, steps=steps)


def trace_shade(surface, origins, dirs, cfg: MarchSettings) -> MarchOutput:
    """surface.py:229-241: box test (miss => t_near=1, t_far=0), march, shade the hits."""
    tn, tf, inside = slab_intersect(origins, dirs, surface.bbox_min, surface.bbox_max)
    tn = np.where(inside, tn, 1.0)
    tf = np.where(inside, tf, 0.0)
    out = march(surface, origins, dirs, tn, tf, cfg)
    out.normal = np.zeros_like(origins)
    out.color = np.zeros_like(origins)
    if np.any(out.hit):
        m = out.hit
        rgb, nrm = surface.shade(out.position[m], dirs[m])
        out.color[m] = np.clip(rgb, 0.0, 1.0)
        out.normal[m] = nrm
    return out


# ---------------------------------------------------------------------------
# frame driver (reference surface.py:265-350)


@dataclass
class Frame:
    color: np.ndarray
    depth: np.ndarray
    normal: np.ndarray
    hit: np.ndarray


def render(surface, cam: Camera, cfg: MarchSettings | None = None, background=(1.0, 1.0, 1.0),
           supersample: int = 1, tile_rows: int = 32) -> Frame:
    """surface.py:273-336, single-threaded (the reference proves thread-count invariance).

    Bands of ``tile_rows`` rows; with supersample=k each pixel owns k*k sub-rays on a
    (kH x kW) raster: colour = mean over sub-rays (background composited per sub-ray);
    depth/normal/hit = those of the sub-ray with the smallest depth (first on ties,
    sub-rays ordered row-major inside the pixel).
    """
    cfg = cfg or MarchSettings()
    if supersample < 1:
        raise ValueError("supersample must be >= 1")
    bg = np.asarray(background, dtype=np.float64)
    W, H, k = cam.width, cam.height, supersample
    fine = Camera(cam.position, cam.rotation, cam.fov_y, W * k, H * k)
    color = np.empty((H, W, 3), dtype=np.float32)
    depth = np.full((H, W), MISS_DEPTH, dtype=np.float32)
    normal = np.zeros((H, W, 3), dtype=np.float32)
    hitmap = np.zeros((H, W), dtype=bool)

    for r0 in range(0, H, tile_rows):
        r1 = min(r0 + tile_rows, H)
        cc, rr = np.meshgrid(np.arange(W * k), np.arange(r0 * k, r1 * k))
        o, d = camera_rays(fine, np.stack([cc.ravel(), rr.ravel()], axis=1))
        res = trace_shade(surface, o, d, cfg)
        rows = r1 - r0
        rgb = np.where(res.hit[:, None], res.color, bg[None, :]).reshape(rows, k, W, k, 3)
        dep = np.where(res.hit, res.t, MISS_DEPTH).reshape(rows, k, W, k)
        nrm = res.normal.reshape(rows, k, W, k, 3)
        hh = res.hit.reshape(rows, k, W, k)
        color[r0:r1] = rgb.mean(axis=(1, 3))
        dep_px = dep.transpose(0, 2, 1, 3).reshape(rows, W, k * k)
        pick = np.argmin(dep_px, axis=2)[:, :, None]
        depth[r0:r1] = np.take_along_axis(dep_px, pick, axis=2)[:, :, 0]
        nrm_px = nrm.transpose(0, 2, 1, 3, 4).reshape(rows, W, k * k, 3)
        normal[r0:r1] = np.take_along_axis(nrm_px, pick[:, :, :, None], axis=2)[:, :, 0, :]
        hit_px = hh.transpose(0, 2, 1, 3).reshape(rows, W, k * k)
        hitmap[r0:r1] = np.take_along_axis(hit_px, pick, axis=2)[:, :, 0]
    return Frame(color, depth, normal, hitmap)


def pass_image(frame: Frame, which: str) -> np.ndarray:
    """surface.py:339-350."""
    if which == "color":
        return frame.color.astype(np.float64)
    if which == "normal":
        img = 0.5 * (frame.normal.astype(np.float64) + 1.0)
        img[~frame.hit] = 0.0
        return img
    if which == "depth":
        g = np.where(np.isfinite(frame.depth), 1.0 / (1.0 + frame.depth), 0.0)
        return np.repeat(g[:, :, None], 3, axis=2)
    raise ValueError(f"unknown pass {which!r}")
