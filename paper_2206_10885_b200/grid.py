"""Grid-of-MLPs field queries on the B200: same names and signatures as the reference
``kilofield.grid`` (grid.py), backed by libknf_b200's routing + fused tile-MLP kernels.

Drop-in notes
  * Every function accepts the reference's own ``KiloField`` (anything exposing ``.config``,
    ``.sdf.weights/.biases`` and ``.color.weights/.biases``) as well as this module's.
  * NumPy in -> NumPy out (host buffers are staged through the C-ABI, KNF_MEM_HOST).  torch CUDA
    tensors in -> torch CUDA tensors out, nothing leaves the device (KNF_MEM_DEVICE).
  * A field is uploaded once and cached (the reference treats fields as immutable while
    rendering); call ``invalidate(field)`` after mutating its arrays.
  * No CPU fallback: without the built library or a CUDA device these functions raise.
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native as N

NORMAL_EPS = 1e-8  # grid.py:21

SOFTPLUS, RELU, SIGMOID, IDENTITY = "softplus", "relu", "sigmoid", "identity"
SDF_ACTIVATIONS = [SOFTPLUS, SOFTPLUS, IDENTITY]  # grid.py:67
COLOR_ACTIVATIONS = [RELU, RELU, SIGMOID]  # grid.py:68


class DegenerateGradientError(ValueError):
    """FD gradient too small to normalize into a surface normal (grid.py:28-29)."""


# ---------------------------------------------------------------------------------------------
# containers (grid.py:32-154) -- plain host-side data, kept so the package stands alone


@dataclass
class GridConfig:
    resolution: int = 16
    bbox_min: tuple = (-1.0, -1.0, -1.0)
    bbox_max: tuple = (1.0, 1.0, 1.0)
    sdf_freqs: int = 6
    dir_freqs: int = 4
    feature_dim: int = 8
    fd_step: float = 1e-3

    def __post_init__(self):
        self.bbox_min = np.asarray(self.bbox_min, dtype=np.float64)
        self.bbox_max = np.asarray(self.bbox_max, dtype=np.float64)
        if self.resolution < 1:
            raise ValueError("resolution must be >= 1")
        if not np.all(self.bbox_min < self.bbox_max):
            raise ValueError("bbox_min must be < bbox_max componentwise")
        if self.fd_step <= 0:
            raise ValueError("fd_step must be > 0")

    @property
    def n_cells(self) -> int:
        return self.resolution**3

    @property
    def cell_size(self) -> np.ndarray:
        return (self.bbox_max - self.bbox_min) / self.resolution

    def sdf_layer_dims(self):
        return [3 + 6 * self.sdf_freqs, 32, 32, 1 + self.feature_dim]

    def color_layer_dims(self):
        return [3 + (3 + 6 * self.dir_freqs) + 3 + self.feature_dim, 32, 32, 3]


@dataclass
class MlpGrid:
    layer_dims: list
    activations: list
    weights: list  # per layer (n_cells, out, in)
    biases: list  # per layer (n_cells, out)

    @property
    def n_cells(self) -> int:
        return self.weights[0].shape[0]

    @property
    def dtype(self):
        return self.weights[0].dtype

    def param_count(self) -> int:
        return sum(w.size + b.size for w, b in zip(self.weights, self.biases))


@dataclass
class KiloField:
    config: GridConfig
    sdf: MlpGrid
    color: MlpGrid
    inv_std_param: np.ndarray

    @property
    def s(self) -> float:
        return float(np.exp(self.inv_std_param))

    @property
    def dtype(self):
        return self.sdf.dtype

    def param_count(self) -> int:
        return self.sdf.param_count() + self.color.param_count() + 1


def _init_family(n_cells, dims, acts, rng, dtype):
    ws, bs = [], []
    for k in range(len(dims) - 1):
        bound = np.sqrt(6.0 / dims[k])
        ws.append(rng.uniform(-bound, bound, size=(n_cells, dims[k + 1], dims[k])).astype(dtype))
        bs.append(np.zeros((n_cells, dims[k + 1]), dtype=dtype))
    return MlpGrid(list(dims), list(acts), ws, bs)


def field_init(cfg: GridConfig, seed: int, dtype=np.float32, init_s: float = 20.0) -> KiloField:
    """Same random stream as the reference (grid.py:150-154): SDF stacks first, then colour."""
    rng = np.random.default_rng(seed)
    sdf = _init_family(cfg.n_cells, cfg.sdf_layer_dims(), SDF_ACTIVATIONS, rng, dtype)
    col = _init_family(cfg.n_cells, cfg.color_layer_dims(), COLOR_ACTIVATIONS, rng, dtype)
    return KiloField(cfg, sdf, col, np.array(np.log(init_s), dtype=dtype))


def refine_field(field: KiloField, factor: int = 2) -> KiloField:
    """The same field on a grid `factor` times finer per axis: every child cell inherits its parent's networks, which
    take GLOBAL coordinates (grid.py:373-380 encodes the point, not a cell-local offset), so the SDF / colour functions
    are unchanged -- bit for bit, since a point is evaluated by identical weights with identical arithmetic.  Gives a
    trained 16^3-cell (4096-MLP) workload from the committed 8^3 fixture without shipping an 84 MB model file."""
    if factor < 1:
        raise ValueError("factor must be >= 1")
    cfg = field.config
    n, m = int(cfg.resolution), int(cfg.resolution) * int(factor)
    idx = np.arange(m) // factor
    parent = ((idx[:, None, None] * n + idx[None, :, None]) * n + idx[None, None, :]).reshape(-1)
    fine = GridConfig(m, tuple(cfg.bbox_min), tuple(cfg.bbox_max), cfg.sdf_freqs, cfg.dir_freqs, cfg.feature_dim, cfg.fd_step)

    def fam(g):
        return MlpGrid(list(g.layer_dims), list(g.activations), [np.ascontiguousarray(w[parent]) for w in g.weights],
                       [np.ascontiguousarray(b[parent]) for b in g.biases])

    return KiloField(fine, fam(field.sdf), fam(field.color), np.array(field.inv_std_param))


KERNEL_SDF_FREQS, KERNEL_DIR_FREQS, KERNEL_FEATURE_DIM = 6, 4, 8  # the widths the kernels are compiled for (grid.py:32-68 defaults)


def _embed_layer(name, k, w, b, lx, lv, nf):
    """A field with fewer encoding octaves or features than the compiled widths, embedded EXACTLY: the missing inputs get
    zero weight columns at the positions the wide layout gives them (the Fourier octaves are ordered ascending, so a
    narrower encoding is a prefix; colour inputs are [x(3), enc(v), n(3), z(F)], grid.py:387-400) and the missing
    outputs zero rows.  A zero column adds fma(x, 0, acc) = acc to the k-ordered chain and the nonzero terms keep their
    order, so every value the reference computes is reproduced bit for bit; the extra feature outputs are 0 and are
    sliced off by the host API."""
    w = np.ascontiguousarray(w, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    n = w.shape[0]
    if name == "sdf" and k == 0 and lx < KERNEL_SDF_FREQS:
        wide = np.zeros((n, 32, 3 + 6 * KERNEL_SDF_FREQS), np.float32)
        wide[:, :, : 3 + 6 * lx] = w
        w = wide
    elif name == "sdf" and k == 2 and nf < KERNEL_FEATURE_DIM:
        wide = np.zeros((n, 1 + KERNEL_FEATURE_DIM, 32), np.float32)
        wide[:, : 1 + nf] = w
        bw = np.zeros((n, 1 + KERNEL_FEATURE_DIM), np.float32)
        bw[:, : 1 + nf] = b
        w, b = wide, bw
    elif name == "color" and k == 0 and (lv < KERNEL_DIR_FREQS or nf < KERNEL_FEATURE_DIM):
        ev, evw = 3 + 6 * lv, 3 + 6 * KERNEL_DIR_FREQS
        wide = np.zeros((n, 32, 3 + evw + 3 + KERNEL_FEATURE_DIM), np.float32)
        wide[:, :, 0:3] = w[:, :, 0:3]                                       # x
        wide[:, :, 3 : 3 + ev] = w[:, :, 3 : 3 + ev]                          # enc(v): a prefix of the wider encoding
        wide[:, :, 3 + evw : 3 + evw + 3] = w[:, :, 3 + ev : 3 + ev + 3]      # n
        wide[:, :, 3 + evw + 3 : 3 + evw + 3 + nf] = w[:, :, 3 + ev + 3 :]    # z
        w = wide
    return np.ascontiguousarray(w), np.ascontiguousarray(b)


# ---------------------------------------------------------------------------------------------
# device residency


class DeviceField:
    """Owns a knf_field_t: the field's cell-major weight blobs on one GPU."""

    def __init__(self, handle, device: int, config):
        self._handle = handle
        self.device = device
        self.config = config
        self._finalizer = weakref.finalize(self, DeviceField._destroy, handle)

    @staticmethod
    def _destroy(handle):
        try:
            N.load().knf_field_destroy(handle)
        except Exception:
            pass

    @property
    def handle(self):
        if self._handle is None:
            raise ValueError("device field already closed")
        return self._handle

    def close(self):
        if self._handle is not None:
            self._finalizer()
            self._handle = None

    @classmethod
    def upload(cls, field, device: int | None = None) -> "DeviceField":
        lib = N.load()
        N.require_gpu()
        device = _default_device() if device is None else int(device)
        cfg = field.config
        desc = N.KnfFieldDesc()
        desc.resolution = int(cfg.resolution)
        desc.bbox_min = N.vec3(cfg.bbox_min)
        desc.bbox_max = N.vec3(cfg.bbox_max)
        lx, lv, nf = int(cfg.sdf_freqs), int(cfg.dir_freqs), int(cfg.feature_dim)
        if lx > KERNEL_SDF_FREQS or lv > KERNEL_DIR_FREQS or nf > KERNEL_FEATURE_DIM or min(lx, lv, nf) < 0:
            raise N.KnfUnsupported(f"sdf_freqs={lx}, dir_freqs={lv}, feature_dim={nf}: the kernels are compiled for the reference widths "
                                   f"({KERNEL_SDF_FREQS}, {KERNEL_DIR_FREQS}, {KERNEL_FEATURE_DIM}); narrower fields are embedded exactly, wider ones are not supported")
        desc.sdf_freqs, desc.dir_freqs, desc.feature_dim = KERNEL_SDF_FREQS, KERNEL_DIR_FREQS, KERNEL_FEATURE_DIM
        desc.fd_step = float(cfg.fd_step)
        expect_sdf = [(32, 3 + 6 * lx), (32, 32), (1 + nf, 32)]
        expect_col = [(32, 3 + 3 + 6 * lv + 3 + nf), (32, 32), (3, 32)]
        n_cells = int(cfg.resolution) ** 3
        # Everything the C side memcpy's is validated here first: it reads n_cells * out * in weights and
        # n_cells * out biases per layer without looking at shapes.
        for name, fam, expect, acts in (("sdf", field.sdf, expect_sdf, SDF_ACTIVATIONS), ("color", field.color, expect_col, COLOR_ACTIVATIONS)):
            if len(fam.weights) != 3 or len(fam.biases) != 3:
                raise N.KnfUnsupported("only 3-layer MLP families are supported")
            for k in range(3):
                w, b = np.asarray(fam.weights[k]), np.asarray(fam.biases[k])
                if w.ndim != 3 or tuple(w.shape[1:]) != expect[k]:
                    raise N.KnfUnsupported(f"{name} layer {k} has shape {tuple(w.shape[1:])}, kernels need {expect[k]}")
                if w.shape[0] != n_cells:
                    raise ValueError(f"{name} weight stack {k} does not match resolution^3 = {n_cells} cells")
                if tuple(b.shape) != (n_cells, expect[k][0]):
                    raise ValueError(f"{name} bias stack {k} has shape {tuple(b.shape)}, expected {(n_cells, expect[k][0])}")
                # the reference evaluates in the field's own dtype (grid.py:253-290, tiny_field64 in its tests); these
                # kernels reproduce its float32 arithmetic only -- narrowing a float64 field silently would be a
                # different function, so refuse it
                if w.dtype != np.float32 or b.dtype != np.float32:
                    raise N.KnfUnsupported(f"{name} layer {k} is {w.dtype}/{b.dtype}: only float32 fields are supported "
                                           "(cast explicitly with astype(np.float32) if narrowing is intended)")
            # an empty activation list marks the internal geometry-only field (_geometry_field); anything else must be
            # the reference's activations, which are what the kernels are compiled for (nn.py:41-50)
            if len(fam.activations) and [str(a) for a in fam.activations] != [str(a) for a in acts]:
                raise N.KnfUnsupported(f"{name} activations {list(fam.activations)} differ from the reference's {list(acts)}")
        keep = []
        for name, fam in (("sdf", field.sdf), ("color", field.color)):
            for k in range(3):
                w, b = _embed_layer(name, k, fam.weights[k], fam.biases[k], lx, lv, nf)
                keep += [w, b]
                getattr(desc, f"{name}_w")[k] = w.ctypes.data
                getattr(desc, f"{name}_b")[k] = b.ctypes.data
        handle = C.c_void_p()
        N.check(lib.knf_field_create(C.byref(desc), device, C.byref(handle)))
        return cls(handle, device, cfg)

    @classmethod
    def from_knf(cls, path, device: int | None = None) -> "DeviceField":
        """.knf file straight to the device layout (modelio.load_model checks kept)."""
        lib = N.load()
        N.require_gpu()
        device = _default_device() if device is None else int(device)
        handle = C.c_void_p()
        N.check(lib.knf_field_create_from_knf(str(path).encode(), device, C.byref(handle)))
        desc = N.KnfFieldDesc()
        N.check(lib.knf_field_describe(handle, C.byref(desc)))
        cfg = GridConfig(desc.resolution, tuple(desc.bbox_min), tuple(desc.bbox_max), desc.sdf_freqs, desc.dir_freqs,
                         desc.feature_dim, desc.fd_step)
        return cls(handle, device, cfg)

    def stats(self) -> dict:
        st = N.KnfStats()
        N.check(N.load().knf_field_stats(self.handle, C.byref(st)))
        return {k: getattr(st, k) for k, _ in N.KnfStats._fields_}

    def reset_stats(self):
        N.check(N.load().knf_field_stats_reset(self.handle))

    def set_profiling(self, enable: bool):
        N.check(N.load().knf_field_set_profiling(self.handle, int(bool(enable))))

    PRECISIONS = {"fp32_chain": 0, "tensor_bf16x3": 1, "tensor_fp16x2": 2}

    def set_precision(self, mode):
        """Arithmetic of the SDF hidden layers: "fp32_chain" (the reference's k-ordered FMA chain, FP32 pipe) or
        "tensor_bf16x3" (exact 3-way bf16 split on the tensor cores; include/knf_b200.h KNF_PRECISION_*)."""
        code = self.PRECISIONS[mode] if isinstance(mode, str) else int(mode)
        N.check(N.load().knf_field_set_precision(self.handle, code))

    FILTERS = {"off": 0, "on": 1, "auto": 2}

    def set_filter(self, mode):
        """Decision filter of the exact march (include/knf_b200.h knf_field_set_filter): "off" | "on" | "auto".
        Results are bit-identical either way; it only changes which kernel answers the d < -eps predicates."""
        code = self.FILTERS[mode] if isinstance(mode, str) else int(mode)
        N.check(N.load().knf_field_set_filter(self.handle, code))

    def filter_delta(self) -> float:
        return float(N.load().knf_field_filter_delta(self.handle))

    def filter_kernel(self) -> str:
        """Which decision-filter kernel this handle launches (include/knf_b200.h knf_field_filter_kernel)."""
        return N.load().knf_field_filter_kernel(self.handle).decode()

    def filter_cells_off(self) -> int:
        """Cells whose activations could leave the fp16 range: the decision filter leaves them to the exact kernel."""
        n = int(N.load().knf_field_filter_cells_off(self.handle))
        if n < 0:
            N.check(n)
        return n

    def lipschitz(self):
        """Per-cell, per-axis Lipschitz bounds behind the decision filter's certified skipping
        (include/knf_b200.h knf_field_lipschitz): (closed_form, refined, refine_ms), two (n_cells, 3) float32 arrays.
        Runs the sub-box refinement (csrc/knf_bounds.cuh) if no march has triggered it yet."""
        n = int(self.config.resolution) ** 3
        closed = np.empty((n, 3), dtype=np.float32)
        refined = np.empty((n, 3), dtype=np.float32)
        ms = C.c_float(0.0)
        N.check(N.load().knf_field_lipschitz(self.handle, closed.ctypes.data, refined.ctypes.data, C.addressof(ms), N.current_stream(self.device)))
        return closed, refined, float(ms.value)

    def get_precision(self) -> str:
        code = N.load().knf_field_get_precision(self.handle)
        N.check(min(code, 0))
        return {v: k for k, v in self.PRECISIONS.items()}[code]


def _default_device() -> int:
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # pragma: no cover
        pass
    return 0


_CACHE: dict = {}


def device_field(field, device: int | None = None) -> DeviceField:
    """The cached device copy of `field` (uploaded on first use)."""
    if isinstance(field, DeviceField):
        return field
    device = _default_device() if device is None else int(device)
    key = (id(field), device)
    hit = _CACHE.get(key)
    if hit is not None:
        return hit
    dev = DeviceField.upload(field, device)
    _CACHE[key] = dev
    try:
        weakref.finalize(field, _CACHE.pop, key, None)
    except TypeError:  # object without weakref support: keep until invalidate()
        pass
    return dev


def invalidate(field):
    """Drop cached device copies after mutating a field's arrays: the next query uploads the field again.

    The old handle is NOT destroyed here -- a FieldSurface or an uploaded path-trace scene may still hold it (the
    scene stores the raw knf_field_t); it is freed by its finaliser once nothing references the DeviceField."""
    for key in [k for k in _CACHE if k[0] == id(field)]:
        _CACHE.pop(key)


# ---------------------------------------------------------------------------------------------
# argument plumbing


class _Args:
    """Uniform view over NumPy (host staging) and torch-CUDA (device resident) arguments."""

    def __init__(self, dev: DeviceField, *arrays):
        self.dev = dev
        self.torch = any(N._is_torch(a) for a in arrays if a is not None)
        if self.torch:
            import torch

            self.t = torch
            self.mem = N.MEM_DEVICE
            self.device = torch.device("cuda", dev.device)
        else:
            self.mem = N.MEM_HOST
        self.stream = N.current_stream(dev.device)

    def inp(self, x, dtype, cols):
        if self.torch:
            t = self.t.as_tensor(x, device=self.device).to(_TORCH_DTYPES(self.t)[dtype]).contiguous()
            if t.dim() == 1 and cols is not None:
                t = t.reshape(1, -1)
        else:
            t = np.ascontiguousarray(np.atleast_2d(x) if cols is not None else x, dtype=dtype)
        if cols is not None and (t.ndim != 2 or t.shape[1] != cols):
            raise ValueError(f"expected an (n,{cols}) array, got shape {tuple(t.shape)}")
        return t

    def out(self, shape, dtype):
        if self.torch:
            return self.t.empty(shape, dtype=_TORCH_DTYPES(self.t)[dtype], device=self.device)
        return np.empty(shape, dtype=dtype)


def _TORCH_DTYPES(t):
    return {np.float32: t.float32, np.float64: t.float64, np.int32: t.int32, np.uint8: t.uint8, np.int64: t.int64,
            np.uint64: t.int64}


# ---------------------------------------------------------------------------------------------
# routing (grid.py:161-213)


def flat_cell(cfg, i: int, j: int, k: int) -> int:
    n = cfg.resolution
    return (i * n + j) * n + k


def cell_index_flat(cfg_or_field, pts):
    """grid.cell_index_flat on the GPU: fp64 arithmetic on the points' own precision (fp32 on the
    hot path -- sdf_query casts first, grid.py:375 -- or fp64), int64 result, bit-exact with the
    reference.  The first argument may be a field (device copy reused) or a bare GridConfig."""
    dev = _geometry_field(cfg_or_field)
    a = _Args(dev, pts)
    is64 = (pts.dtype == a.t.float64) if a.torch else (np.asarray(pts).dtype != np.float32)
    p = a.inp(pts, np.float64 if is64 else np.float32, 3)
    out = a.out((p.shape[0],), np.int32)
    fn = N.load().knf_cell_index_f64 if is64 else N.load().knf_cell_index
    N.check(fn(dev.handle, N.ptr(p), p.shape[0], N.ptr(out), a.mem, a.stream))
    return out.long() if a.torch else out.astype(np.int64)


def cell_index(cfg, x):
    """grid.cell_index (grid.py:166-173) for one fp64 point -> (i, j, k)."""
    flat = int(cell_index_flat(cfg, np.asarray(x, dtype=np.float64)[None, :])[0])
    n = _config_of(cfg).resolution
    return flat // (n * n), (flat // n) % n, flat % n


@dataclass
class Routing:
    """grid.Routing (grid.py:188-204).  `order` groups rows by cell (ascending cells); the order of
    rows inside one cell is unspecified (the reference's is stable) -- results do not depend on it."""

    n: int
    order: np.ndarray
    cells: np.ndarray
    starts: np.ndarray
    ends: np.ndarray

    def sort(self, arr):
        return np.ascontiguousarray(arr[self.order])

    def unsort(self, arr_sorted):
        out = np.empty_like(arr_sorted)
        out[self.order] = arr_sorted
        return out


def route(cfg_or_field, pts) -> Routing:
    dev = _geometry_field(cfg_or_field)
    p = np.ascontiguousarray(np.atleast_2d(pts), dtype=np.float32)
    n = p.shape[0]
    n_seg_cap = max(1, min(n, dev.config.resolution**3))
    order = np.empty(n, dtype=np.int32)
    seg_cell = np.empty(n_seg_cap, dtype=np.int32)
    seg_start = np.empty(n_seg_cap + 1, dtype=np.int32)
    n_seg = np.zeros(1, dtype=np.int32)
    N.check(N.load().knf_route(dev.handle, N.ptr(p), n, None, N.ptr(order), N.ptr(seg_cell), N.ptr(seg_start),
                               N.ptr(n_seg), N.MEM_HOST, N.current_stream(dev.device)))
    k = int(n_seg[0])
    return Routing(n, order.astype(np.int64), seg_cell[:k].astype(np.int64), seg_start[:k].astype(np.int64),
                   seg_start[1 : k + 1].astype(np.int64))


_GEOM_FIELDS: dict = {}


def _config_of(x):
    return x.config if hasattr(x, "config") else x


def _geometry_field(cfg_or_field) -> DeviceField:
    """A device field for geometry-only calls.  Given a bare GridConfig, a zero-weight field of the
    same geometry is created once per (resolution, bbox) and cached."""
    if isinstance(cfg_or_field, DeviceField):
        return cfg_or_field
    if hasattr(cfg_or_field, "sdf") and hasattr(cfg_or_field, "config"):
        return device_field(cfg_or_field)
    cfg = cfg_or_field
    key = (int(cfg.resolution), tuple(np.asarray(cfg.bbox_min, float)), tuple(np.asarray(cfg.bbox_max, float)),
           float(getattr(cfg, "fd_step", 1e-3)), _default_device())
    dev = _GEOM_FIELDS.get(key)
    if dev is None:
        gc = GridConfig(int(cfg.resolution), tuple(cfg.bbox_min), tuple(cfg.bbox_max), fd_step=float(getattr(cfg, "fd_step", 1e-3)))
        n = gc.n_cells
        zeros = lambda dims: MlpGrid(dims, [], [np.zeros((n, dims[k + 1], dims[k]), np.float32) for k in range(3)],
                                     [np.zeros((n, dims[k + 1]), np.float32) for k in range(3)])
        dev = DeviceField.upload(KiloField(gc, zeros(gc.sdf_layer_dims()), zeros(gc.color_layer_dims()), np.zeros(())))
        _GEOM_FIELDS[key] = dev
    return dev


# ---------------------------------------------------------------------------------------------
# field queries (grid.py:365-409)


@dataclass
class SdfSample:
    value: np.ndarray
    features: np.ndarray


def sdf_query(field, points) -> SdfSample:
    """grid.sdf_query: signed distance + features at each point."""
    dev = device_field(field)
    a = _Args(dev, points)
    p = a.inp(points, np.float32, 3)
    out = a.out((p.shape[0], 1 + KERNEL_FEATURE_DIM), np.float32)
    N.check(N.load().knf_sdf_forward(dev.handle, N.ptr(p), p.shape[0], N.ptr(out), a.mem, a.stream))
    return SdfSample(value=out[:, 0], features=out[:, 1 : 1 + int(dev.config.feature_dim)])  # (embedded narrower fields: the rest is 0)


def sdf_values(field, points):
    dev = device_field(field)
    a = _Args(dev, points)
    p = a.inp(points, np.float32, 3)
    out = a.out((p.shape[0],), np.float32)
    N.check(N.load().knf_sdf_values(dev.handle, N.ptr(p), p.shape[0], N.ptr(out), a.mem, a.stream))
    return out


def color_query(field, x, v, n, z):
    """grid.color_query: RGB in (0,1) from the colour MLP of the cell that owns x."""
    dev = device_field(field)
    a = _Args(dev, x, v, n, z)
    xs = a.inp(x, np.float32, 3)
    vs = a.inp(v, np.float32, 3)
    ns = a.inp(n, np.float32, 3)
    nf = int(dev.config.feature_dim)
    zs = a.inp(z, np.float32, nf)
    if nf < KERNEL_FEATURE_DIM:  # embedded narrower field: the missing features meet zero weights
        wide = a.out((zs.shape[0], KERNEL_FEATURE_DIM), np.float32)
        wide[:, :nf] = zs
        wide[:, nf:] = 0
        zs = wide
    m = xs.shape[0]
    if not (vs.shape[0] == ns.shape[0] == zs.shape[0] == m):
        raise ValueError("x, v, n, z must have the same number of rows")
    out = a.out((m, 3), np.float32)
    N.check(N.load().knf_color_forward(dev.handle, N.ptr(xs), N.ptr(vs), N.ptr(ns), N.ptr(zs), m, N.ptr(out), a.mem,
                                       a.stream))
    return out


def grouped_query(field, points, kind: str, **aux):
    """grid.grouped_query (grid.py:403-409)."""
    if kind == "sdf":
        return sdf_query(field, points)
    if kind == "color":
        return color_query(field, points, aux["v"], aux["n"], aux["z"])
    raise ValueError(f"unknown query kind {kind!r}")


# ---------------------------------------------------------------------------------------------
# finite-difference gradients (grid.py:416-469)


def grad_fd(field, x):
    dev = device_field(field)
    a = _Args(dev, x)
    single = (x.dim() if a.torch else np.asarray(x).ndim) == 1
    p = a.inp(x, np.float64, 3)
    out = a.out((p.shape[0], 3), np.float64)
    N.check(N.load().knf_fd_gradient(dev.handle, N.ptr(p), p.shape[0], N.ptr(out), a.mem, a.stream))
    return out[0] if single else out


def grad_analytic(field, x, return_distance: bool = False):
    """Analytic gradient of the owning cell's SDF network at each point (fp32, forward-mode differentiation on the
    device; include/knf_b200.h knf_sdf_gradient).  Not a reference function: the reference's normals are the global
    finite differences of ``grad_fd`` / ``normal_batch``, which also see the jumps between neighbouring cells."""
    dev = device_field(field)
    a = _Args(dev, x)
    p = a.inp(x, np.float32, 3)
    grad = a.out((p.shape[0], 3), np.float32)
    dist = a.out((p.shape[0],), np.float32)
    N.check(N.load().knf_sdf_gradient(dev.handle, N.ptr(p), p.shape[0], N.ptr(dist), N.ptr(grad), a.mem, a.stream))
    return (grad, dist) if return_distance else grad


def normal_batch(field, x, eps: float = NORMAL_EPS):
    dev = device_field(field)
    a = _Args(dev, x)
    p = a.inp(x, np.float64, 3)
    nrm = a.out((p.shape[0], 3), np.float64)
    ok = a.out((p.shape[0],), np.uint8)
    N.check(N.load().knf_fd_normals(dev.handle, N.ptr(p), p.shape[0], float(eps), N.ptr(nrm), N.ptr(ok), a.mem,
                                    a.stream))
    return nrm, (ok.bool() if a.torch else ok.astype(bool))


def normal(field, x):
    """grid.normal (grid.py:464-469): raises DegenerateGradientError on a flat spot."""
    nrm, ok = normal_batch(field, np.asarray(x, dtype=np.float64)[None, :])
    if not ok[0]:
        raise DegenerateGradientError(f"gradient norm <= {NORMAL_EPS} at {x}")
    return nrm[0]
