"""Oracle part 1: the grid-of-MLPs field queries (TEST INFRASTRUCTURE ONLY).

NumPy restatement of reference ``nn.py`` (encode + activations) and
``grid.py`` (container, routing, grouped forward, FD normals).  See
``oracle/__init__.py`` for the usage rules.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence

import numpy as np

# reference grid.py:25 -- below this many points per occupied cell the padded path is taken
PADDED_CUTOFF = 48.0
# reference grid.py:21
DEGENERATE_NORM = 1e-8

ACT_IDENTITY, ACT_RELU, ACT_SOFTPLUS, ACT_SIGMOID = 0, 1, 2, 3  # nn.py:22 codes
SDF_ACTS = (ACT_SOFTPLUS, ACT_SOFTPLUS, ACT_IDENTITY)  # grid.py:67
COLOR_ACTS = (ACT_RELU, ACT_RELU, ACT_SIGMOID)  # grid.py:68


# ---------------------------------------------------------------------------
# containers (reference grid.py:32-154)


@dataclass
class FieldSpec:
    """Geometry + widths of a field; mirrors GridConfig (grid.py:32-64)."""

    resolution: int = 16
    lo: Sequence[float] = (-1.0, -1.0, -1.0)
    hi: Sequence[float] = (1.0, 1.0, 1.0)
    pos_octaves: int = 6
    dir_octaves: int = 4
    n_features: int = 8
    fd_step: float = 1e-3

    def __post_init__(self):
        self.lo = np.asarray(self.lo, dtype=np.float64)
        self.hi = np.asarray(self.hi, dtype=np.float64)

    @property
    def n_cells(self) -> int:
        return self.resolution**3

    def sdf_widths(self) -> List[int]:
        # grid.py:60-61
        return [3 + 6 * self.pos_octaves, 32, 32, 1 + self.n_features]

    def color_widths(self) -> List[int]:
        # grid.py:63-64 : x(3) | enc(v) | n(3) | z(F)
        return [3 + (3 + 6 * self.dir_octaves) + 3 + self.n_features, 32, 32, 3]


@dataclass
class FieldParams:
    """One MLP family: per layer a (cells,out,in) weight stack and (cells,out) bias stack."""

    widths: List[int]
    acts: Sequence[int]
    W: List[np.ndarray]
    b: List[np.ndarray]


@dataclass
class OracleField:
    spec: FieldSpec
    sdf: FieldParams
    color: FieldParams
    log_s: np.ndarray


def _draw_family(n_cells, widths, acts, rng, dtype):
    # grid.py:110-116: per layer, U(+-sqrt(6/fan_in)) drawn in fp64 then cast; zero biases
    Ws, bs = [], []
    for fin, fout in zip(widths[:-1], widths[1:]):
        lim = np.sqrt(6.0 / fin)
        Ws.append(rng.uniform(-lim, lim, size=(n_cells, fout, fin)).astype(dtype))
        bs.append(np.zeros((n_cells, fout), dtype=dtype))
    return FieldParams(list(widths), tuple(acts), Ws, bs)


def make_random_field(spec: FieldSpec, seed: int, dtype=np.float32, init_s: float = 20.0) -> OracleField:
    """grid.py:150-154: one generator; the SDF family is drawn before the colour family."""
    rng = np.random.default_rng(seed)
    sdf = _draw_family(spec.n_cells, spec.sdf_widths(), SDF_ACTS, rng, dtype)
    col = _draw_family(spec.n_cells, spec.color_widths(), COLOR_ACTS, rng, dtype)
    return OracleField(spec, sdf, col, np.array(np.log(init_s), dtype=dtype))


def field_from_stacks(spec: FieldSpec, sdf_W, sdf_b, col_W, col_b, log_s=None) -> OracleField:
    """Wrap existing stacked arrays (e.g. those of a reference KiloField) without copying."""
    sdf = FieldParams(spec.sdf_widths(), SDF_ACTS, list(sdf_W), list(sdf_b))
    col = FieldParams(spec.color_widths(), COLOR_ACTS, list(col_W), list(col_b))
    if log_s is None:
        log_s = np.array(np.log(20.0), dtype=np.float32)
    return OracleField(spec, sdf, col, np.asarray(log_s))


# ---------------------------------------------------------------------------
# encode + activations (reference nn.py:26-93)


def positional_features(x: np.ndarray, octaves: int) -> np.ndarray:
    """nn.py:66-93.  [x | sin(pi x) | cos(pi x) | sin(2 pi x) | cos(2 pi x) | ...].

    Octave 0 uses sin/cos of (pi * x) evaluated in the array's own dtype; higher
    octaves follow by the double-angle recurrence in that dtype (nn.py:88-92),
    NOT by fresh sin/cos calls -- the recurrence's rounding is part of the function.
    """
    x = np.asarray(x)
    flat = x.ndim == 1
    p = x.reshape(1, -1) if flat else x
    rows, d = p.shape
    feats = np.empty((rows, d * (1 + 2 * octaves)), dtype=p.dtype)
    feats[:, 0:d] = p
    if octaves > 0:
        angle = np.pi * p  # python scalar: stays in p.dtype (nn.py:82)
        s = np.sin(angle)
        c = np.cos(angle)
        col = d
        for _ in range(octaves):
            feats[:, col : col + d] = s
            feats[:, col + d : col + 2 * d] = c
            col += 2 * d
            s, c = (2.0 * s) * c, 1.0 - (2.0 * s) * s  # nn.py:89
    return feats[0] if flat else feats


def softplus32(x: np.ndarray) -> np.ndarray:
    """nn.py:26-33: log1p(exp(-|x|)) + max(x, 0), each step in x.dtype."""
    u = np.exp(-np.abs(x))
    return np.log1p(u) + np.maximum(x, 0.0)


def logistic32(x: np.ndarray) -> np.ndarray:
    """nn.py:36-38: sign-split sigmoid."""
    u = np.exp(-np.abs(x))
    return np.where(x >= 0, 1.0 / (1.0 + u), u / (1.0 + u))


def _activate(code: int, z: np.ndarray) -> np.ndarray:
    # nn.py:41-50
    if code == ACT_IDENTITY:
        return z
    if code == ACT_RELU:
        return np.maximum(z, 0.0)
    if code == ACT_SOFTPLUS:
        return softplus32(z)
    if code == ACT_SIGMOID:
        return logistic32(z)
    raise ValueError(f"activation code {code}")


# ---------------------------------------------------------------------------
# routing (reference grid.py:161-213)


def cell_triples(spec: FieldSpec, pts: np.ndarray) -> np.ndarray:
    """grid.py:176-179.  fp64 arithmetic on whatever dtype pts carries (fp32 from
    sdf_query): scaled = (p - lo) / (hi - lo) * N ; floor ; clamp to [0, N-1]."""
    n = spec.resolution
    scaled = (pts - spec.lo) / (spec.hi - spec.lo) * n
    return np.clip(np.floor(scaled).astype(np.int64), 0, n - 1)


def cell_ids(spec: FieldSpec, pts: np.ndarray) -> np.ndarray:
    """grid.py:182-185: flat = (i*N + j)*N + k."""
    t = cell_triples(spec, pts)
    n = spec.resolution
    return (t[:, 0] * n + t[:, 1]) * n + t[:, 2]


@dataclass
class CellGroups:
    """grid.py:188-204: stable sort permutation plus occupied-cell segments."""

    count: int
    perm: np.ndarray  # perm[r] = original row of sorted row r
    cells: np.ndarray
    seg_lo: np.ndarray
    seg_hi: np.ndarray

    def gather(self, a):
        return np.ascontiguousarray(a[self.perm])

    def scatter(self, a_sorted):
        out = np.empty_like(a_sorted)
        out[self.perm] = a_sorted
        return out


def group_by_cell(spec: FieldSpec, pts: np.ndarray) -> CellGroups:
    """grid.py:207-213."""
    ids = cell_ids(spec, pts)
    perm = np.argsort(ids, kind="stable")
    cells, seg_lo = np.unique(ids[perm], return_index=True)
    seg_hi = np.append(seg_lo[1:], len(pts))
    return CellGroups(len(pts), perm, cells, seg_lo, seg_hi)


# ---------------------------------------------------------------------------
# grouped forward (reference grid.py:232-294)


def grouped_forward(fam: FieldParams, rows_sorted: np.ndarray, groups: CellGroups) -> np.ndarray:
    """Run each occupied cell's three layers on its contiguous block of rows.

    Two numerically-equivalent strategies, chosen exactly as grid.py:249-266 does:
    avg rows per occupied cell >= 48 -> per-cell ``h @ W.T + b`` (grid.py:253-265);
    otherwise power-of-two padded size classes through one batched matmul per
    class (grid.py:266-290).
    """
    n = groups.count
    dtype = fam.W[0].dtype
    depth = len(fam.W)
    avg = n / max(len(groups.cells), 1)
    if avg >= PADDED_CUTOFF:
        h = rows_sorted
        for k in range(depth):
            Wk, bk = fam.W[k], fam.b[k]
            z = np.empty((n, Wk.shape[1]), dtype=dtype)
            for c, a, e in zip(groups.cells, groups.seg_lo, groups.seg_hi):
                z[a:e] = h[a:e] @ Wk[c].T + bk[c]
            h = _activate(fam.acts[k], z)
        return h

    out = np.empty((n, fam.W[-1].shape[1]), dtype=dtype)
    sizes = groups.seg_hi - groups.seg_lo
    klass = np.maximum(0, np.ceil(np.log2(sizes)).astype(np.int64))  # grid.py:232-238
    for kc in np.unique(klass):
        pad = 1 << int(kc)
        members = np.nonzero(klass == kc)[0]
        a = groups.seg_lo[members]
        e = groups.seg_hi[members]
        slot = a[:, None] + np.arange(pad)[None, :]
        live = slot < e[:, None]
        slot = np.where(live, slot, a[:, None])  # padding rows replay the first row
        cells = groups.cells[members]
        h = rows_sorted[slot]
        for k in range(depth):
            z = np.matmul(h, fam.W[k][cells].transpose(0, 2, 1))
            z += fam.b[k][cells][:, None, :]
            h = _activate(fam.acts[k], z)
        out[slot[live]] = h[live]
    return out


# ---------------------------------------------------------------------------
# field queries (reference grid.py:365-409)


def query_sdf(field: OracleField, points: np.ndarray):
    """grid.py:373-380 -> (value (n,), features (n,F)), both in the field dtype."""
    dtype = field.sdf.W[0].dtype
    pts = np.ascontiguousarray(np.atleast_2d(points), dtype=dtype)
    g = group_by_cell(field.spec, pts)
    enc = positional_features(g.gather(pts), field.spec.pos_octaves)
    out = g.scatter(grouped_forward(field.sdf, enc, g))
    return out[:, 0], out[:, 1:]


def query_sdf_values(field: OracleField, points: np.ndarray) -> np.ndarray:
    """grid.py:383-384."""
    return query_sdf(field, points)[0]


def query_color(field: OracleField, x, v, n, z) -> np.ndarray:
    """grid.py:387-400: input row = [x | enc_L4(v) | n | z]; routed by x."""
    dtype = field.sdf.W[0].dtype
    x = np.atleast_2d(np.asarray(x, dtype=dtype))
    v = np.atleast_2d(np.asarray(v, dtype=dtype))
    n = np.atleast_2d(np.asarray(n, dtype=dtype))
    z = np.atleast_2d(np.asarray(z, dtype=dtype))
    rows = np.concatenate([x, positional_features(v, field.spec.dir_octaves), n, z], axis=1)
    g = group_by_cell(field.spec, x)
    return g.scatter(grouped_forward(field.color, g.gather(rows), g))


def grouped_query(field: OracleField, points, kind: str, **aux):
    """grid.py:403-409."""
    if kind == "sdf":
        return query_sdf(field, points)
    if kind == "color":
        return query_color(field, points, aux["v"], aux["n"], aux["z"])
    raise ValueError(f"unknown query kind {kind!r}")


# ---------------------------------------------------------------------------
# finite-difference normals (reference grid.py:416-469)


def fd_probe_points(spec: FieldSpec, pts: np.ndarray):
    """grid.py:416-437.  For axis a the +h/-h probes differ from the point only in
    coordinate a.  If that coordinate lies inside [lo_a, hi_a] the probes are clamped
    to the box (one-sided at the wall); otherwise they are left unclamped.
    Returns (plus (n,3,3), minus (n,3,3), span (n,3)) with span = plus_a - minus_a."""
    h = spec.fd_step
    plus = np.repeat(pts[:, None, :], 3, axis=1)
    minus = plus.copy()
    span = np.empty((len(pts), 3), dtype=np.float64)
    for a in range(3):
        coord = pts[:, a]
        inside = (coord >= spec.lo[a]) & (coord <= spec.hi[a])
        up = coord + h
        dn = coord - h
        plus[:, a, a] = np.where(inside, np.minimum(up, spec.hi[a]), up)
        minus[:, a, a] = np.where(inside, np.maximum(dn, spec.lo[a]), dn)
        span[:, a] = plus[:, a, a] - minus[:, a, a]
    return plus, minus, span


def fd_gradient(field: OracleField, x: np.ndarray) -> np.ndarray:
    """grid.py:440-451: all 6n probes go through ONE sdf query ([plus...; minus...])."""
    pts = np.atleast_2d(np.asarray(x, dtype=np.float64))
    plus, minus, span = fd_probe_points(field.spec, pts)
    batch = np.concatenate([plus.reshape(-1, 3), minus.reshape(-1, 3)], axis=0)
    d = query_sdf_values(field, batch).astype(np.float64)
    m = len(pts)
    g = (d[: 3 * m].reshape(m, 3) - d[3 * m :].reshape(m, 3)) / span
    return g[0] if np.asarray(x).ndim == 1 else g


def fd_normals(field: OracleField, x: np.ndarray, eps: float = DEGENERATE_NORM):
    """grid.py:454-461 -> (unit normals or zeros, ok mask)."""
    g = np.atleast_2d(fd_gradient(field, x))
    length = np.linalg.norm(g, axis=1)
    ok = length > eps
    nrm = np.zeros_like(g)
    nrm[ok] = g[ok] / length[ok, None]
    return nrm, ok
