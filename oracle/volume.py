"""Oracle part 4: forward pass of the S-density volume renderer (TEST INFRASTRUCTURE ONLY).
Restates reference ``training._volume_forward`` (training.py:330-415) without the backward cache."""

from __future__ import annotations

import numpy as np

from . import field as F
from .trace import slab_intersect

PHI_MIN = 1e-12  # training.py:23


def _logistic64(x):
    # training.py:418-424
    out = np.empty_like(x, dtype=np.float64)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def volume_forward(field: F.OracleField, origins, dirs, n_s: int, jitter=None, background=(1.0, 1.0, 1.0), s=None):
    """(B,3) float64 colours.  s defaults to exp(log_s)."""
    spec = field.spec
    B = len(origins)
    bg = np.asarray(background, dtype=np.float64)
    t0, t1, inside = slab_intersect(origins, dirs, spec.lo, spec.hi)
    live = inside & (t0 < t1)
    colors = np.tile(bg, (B, 1))
    if not live.any():
        return np.clip(colors, 0.0, 1.0)
    A = int(live.sum())
    o, d = origins[live], dirs[live]
    if jitter is None:
        jitter = np.full((B, n_s), 0.5)
    dt = ((t1 - t0)[live] / n_s)[:, None]
    ts = t0[live][:, None] + (np.arange(n_s)[None, :] + jitter[live]) * dt  # training.py:362-363
    pts = (o[:, None, :] + ts[..., None] * d[:, None, :]).reshape(-1, 3)
    value, feats = F.query_sdf(field, pts)
    dvals = value.astype(np.float64).reshape(A, n_s)
    z = feats.reshape(A, n_s, -1)
    m = n_s - 1
    pts_m = pts.reshape(A, n_s, 3)[:, :m].reshape(-1, 3)
    s = float(np.exp(field.log_s)) if s is None else float(s)
    view = np.repeat(d, m, axis=0)
    normals = -view.copy()
    near = np.abs(dvals[:, :m].reshape(-1)) <= 20.0 / s  # training.py:373-383
    if near.any():
        nrm, ok = F.fd_normals(field, pts_m[near])
        nrm[~ok] = -view[near][~ok]
        normals[near] = nrm
    rgb = F.query_color(field, pts_m.astype(np.float32), view, normals, z[:, :m].reshape(-1, z.shape[-1]))
    cvals = rgb.astype(np.float64).reshape(A, m, 3)
    phi = _logistic64(s * dvals)
    lead = np.maximum(phi[:, :m], PHI_MIN)
    alpha = np.clip((phi[:, :m] - phi[:, 1:]) / lead, 0.0, 1.0)
    T_full = np.cumprod(1.0 - alpha, axis=1)
    T = np.concatenate([np.ones((A, 1)), T_full[:, :-1]], axis=1)
    raw = ((T * alpha)[..., None] * cvals).sum(axis=1) + T_full[:, -1][:, None] * bg[None, :]
    colors[live] = np.clip(raw, 0.0, 1.0)
    return colors
