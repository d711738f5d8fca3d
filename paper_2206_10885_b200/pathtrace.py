"""Monte Carlo path tracer over mixed scenes on the B200: same interface as the reference
``kilofield.pathtrace`` (pathtrace.py) -- analytic primitives plus neural grid objects treated as
Lambertian surfaces, counter-hash RNG, Russian roulette, cosine sampling.

The whole bounce loop runs on the device (libknf_b200: knf_trace_paths / knf_pathtrace); the
classes here are plain scene descriptions.  ``LatLongEnvMap`` is out of scope (no BASELINE config
uses it); scenes must use ``ConstantEnv``.
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .cameras import CameraPose, camera_struct
from .grid import _default_device
from .surface import FieldSurface, RenderSettings, _settings_struct

RR_START_BOUNCE = 3  # pathtrace.py:25-27
RR_MIN, RR_MAX = 0.05, 0.95
_PRIMARY_SLOT = 1 << 20


@dataclass
class Rng:
    """pathtrace.Rng (pathtrace.py:37-49): value = hash(seed, pixel, sample, slot), bit-exact."""

    seed: int

    def uniform(self, pixel, sample, slot, device: int | None = None):
        device = _default_device() if device is None else device
        shape = np.broadcast(np.asarray(pixel), np.asarray(sample), np.asarray(slot)).shape
        px = np.ascontiguousarray(np.broadcast_to(np.asarray(pixel, dtype=np.uint64), shape)).reshape(-1)
        sm = np.ascontiguousarray(np.broadcast_to(np.asarray(sample, dtype=np.uint64), shape)).reshape(-1)
        sl = np.ascontiguousarray(np.broadcast_to(np.asarray(slot, dtype=np.uint64), shape)).reshape(-1)
        out = np.empty(px.shape[0], dtype=np.float64)
        N.check(N.load().knf_rng_uniform(C.c_uint64(self.seed & 0xFFFFFFFFFFFFFFFF), N.ptr(px), N.ptr(sm), N.ptr(sl),
                                         px.shape[0], N.ptr(out), device, N.MEM_HOST, N.current_stream(device)))
        return out.reshape(shape) if shape else float(out[0])


# ---------------------------------------------------------------------------------------------
# materials, environments, objects (pathtrace.py:56-280)


@dataclass
class Lambertian:
    albedo: tuple = (0.5, 0.5, 0.5)

    def __post_init__(self):
        self.albedo = np.asarray(self.albedo, dtype=np.float64)
        if np.any(self.albedo < 0) or np.any(self.albedo > 1):
            raise ValueError("albedo must lie in [0, 1]")


@dataclass
class Emissive:
    radiance: tuple = (1.0, 1.0, 1.0)

    def __post_init__(self):
        self.radiance = np.asarray(self.radiance, dtype=np.float64)
        if np.any(self.radiance < 0):
            raise ValueError("radiance must be non-negative")


@dataclass
class ConstantEnv:
    rgb: tuple = (1.0, 1.0, 1.0)

    def __post_init__(self):
        self.rgb = np.asarray(self.rgb, dtype=np.float64)

    def radiance(self, dirs):
        return np.broadcast_to(self.rgb, np.shape(dirs)).copy()


@dataclass
class SphereObj:
    center: tuple
    radius: float
    material: object

    def __post_init__(self):
        self.center = np.asarray(self.center, dtype=np.float64)
        if self.radius <= 0:
            raise ValueError("radius must be > 0")


@dataclass
class QuadObj:
    """Parallelogram: corner + s*edge_u + t*edge_v for s, t in [0, 1]."""

    corner: tuple
    edge_u: tuple
    edge_v: tuple
    material: object

    def __post_init__(self):
        self.corner = np.asarray(self.corner, dtype=np.float64)
        self.edge_u = np.asarray(self.edge_u, dtype=np.float64)
        self.edge_v = np.asarray(self.edge_v, dtype=np.float64)
        if np.linalg.norm(np.cross(self.edge_u, self.edge_v)) < 1e-12:
            raise ValueError("degenerate quad")


@dataclass
class BoxObj:
    bmin: tuple
    bmax: tuple
    material: object

    def __post_init__(self):
        self.bmin = np.asarray(self.bmin, dtype=np.float64)
        self.bmax = np.asarray(self.bmax, dtype=np.float64)
        if not np.all(self.bmin < self.bmax):
            raise ValueError("bmin must be < bmax")


@dataclass
class NeuralObject:
    """A grid field placed in the scene by a rigid + uniform-scale map (pathtrace.py:225-274)."""

    surface: FieldSurface
    translation: tuple = (0.0, 0.0, 0.0)
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    scale: float = 1.0
    settings: RenderSettings = field(default_factory=RenderSettings)

    def __post_init__(self):
        self.translation = np.asarray(self.translation, dtype=np.float64)
        self.rotation = np.asarray(self.rotation, dtype=np.float64)
        if not np.allclose(self.rotation @ self.rotation.T, np.eye(3), atol=1e-6):
            raise ValueError("rotation must be orthonormal")
        if self.scale <= 0:
            raise ValueError("scale must be > 0")
        if not isinstance(self.surface, FieldSurface):
            raise TypeError("NeuralObject needs a paper_2206_10885_b200.surface.FieldSurface")

    def to_local(self, o, d):
        return (o - self.translation) @ self.rotation / self.scale, d @ self.rotation


@dataclass
class Scene:
    objects: list
    environment: object = field(default_factory=ConstantEnv)


# ---------------------------------------------------------------------------------------------
# device scene


class _DeviceScene:
    def __init__(self, handle, keep):
        self.handle = handle
        self._keep = keep  # fields must outlive the scene handle
        self._fin = weakref.finalize(self, _DeviceScene._destroy, handle)

    @staticmethod
    def _destroy(handle):
        try:
            N.load().knf_scene_destroy(handle)
        except Exception:
            pass


def _material(obj, mat):
    if isinstance(mat, Lambertian):
        obj.material = N.MAT_LAMBERTIAN
        obj.rgb = N.vec3(mat.albedo)
    elif isinstance(mat, Emissive):
        obj.material = N.MAT_EMISSIVE
        obj.rgb = N.vec3(mat.radiance)
    else:
        raise TypeError(f"unsupported material {type(mat).__name__}")


def invalidate_scene(scene: Scene) -> None:
    """Forget the cached device copy of `scene` (device_scene notices edits by itself; this is for callers that
    mutate arrays in place in ways a value comparison cannot see, e.g. after grid.invalidate(field))."""
    if hasattr(scene, "_knf_device_scene"):
        del scene._knf_device_scene


def _device_index(scene: Scene) -> int:
    for o in scene.objects:
        if isinstance(o, NeuralObject):
            return o.surface.dev.device
    return _default_device()


def _scene_fingerprint(scene: Scene):
    """Everything knf_scene_create reads, as a hashable value: the reference re-reads the Python objects on every call
    (and service.py mutates and reuses scenes across frames), so the cached upload is only valid while this is unchanged."""
    vec = lambda v: tuple(np.asarray(v, dtype=np.float64).ravel().tolist())
    mat = lambda m: (type(m).__name__, vec(m.albedo if isinstance(m, Lambertian) else getattr(m, "radiance", ())))
    items = []
    for o in scene.objects:
        if isinstance(o, SphereObj):
            items.append(("sphere", vec(o.center), float(o.radius), mat(o.material)))
        elif isinstance(o, QuadObj):
            items.append(("quad", vec(o.corner), vec(o.edge_u), vec(o.edge_v), mat(o.material)))
        elif isinstance(o, BoxObj):
            items.append(("box", vec(o.bmin), vec(o.bmax), mat(o.material)))
        elif isinstance(o, NeuralObject):
            st = o.settings
            items.append(("neural", vec(o.translation), vec(o.rotation), float(o.scale), int(o.surface.dev.handle.value or 0),
                          (float(st.eps_hit), int(st.max_steps), float(st.step_scale))))
        else:
            raise TypeError(f"unsupported scene object {type(o).__name__}")
    env = scene.environment
    return tuple(items), (type(env).__name__, vec(getattr(env, "rgb", ())))


def device_scene(scene: Scene) -> _DeviceScene:
    """The uploaded scene description, cached on the Scene instance and rebuilt whenever anything the device copy
    holds has changed (objects, geometry, materials, transforms, settings, field handles, environment)."""
    if not isinstance(scene.environment, ConstantEnv):
        raise N.KnfUnsupported("only ConstantEnv environments are supported on the device path")
    fp = _scene_fingerprint(scene)
    cached = getattr(scene, "_knf_device_scene", None)
    if cached is not None and cached[0] == fp:
        return cached[1]
    N.require_gpu()
    n = len(scene.objects)
    arr = (N.KnfObject * max(n, 1))()
    keep = []
    for i, o in enumerate(scene.objects):
        k = arr[i]
        k.rot = (C.c_double * 9)(1, 0, 0, 0, 1, 0, 0, 0, 1)
        k.s = 1.0
        if isinstance(o, SphereObj):
            k.kind = N.OBJ_SPHERE
            k.a = N.vec3(o.center)
            k.s = float(o.radius)
            _material(k, o.material)
        elif isinstance(o, QuadObj):
            k.kind = N.OBJ_QUAD
            k.a, k.b, k.c = N.vec3(o.corner), N.vec3(o.edge_u), N.vec3(o.edge_v)
            _material(k, o.material)
        elif isinstance(o, BoxObj):
            k.kind = N.OBJ_BOX
            k.a, k.b = N.vec3(o.bmin), N.vec3(o.bmax)
            _material(k, o.material)
        elif isinstance(o, NeuralObject):
            k.kind = N.OBJ_NEURAL
            k.a = N.vec3(o.translation)
            k.rot = (C.c_double * 9)(*np.asarray(o.rotation, dtype=np.float64).reshape(9))
            k.s = float(o.scale)
            k.field = o.surface.dev.handle
            k.settings = _settings_struct(o.settings)
            keep.append(o.surface.dev)
        else:
            raise TypeError(f"unsupported scene object {type(o).__name__}")
    env = N.vec3(scene.environment.rgb)
    handle = C.c_void_p()
    N.check(N.load().knf_scene_create(arr, n, C.byref(env), _device_index(scene), C.byref(handle)))
    dev = _DeviceScene(handle, keep)
    scene._knf_device_scene = (fp, dev)
    return dev


# ---------------------------------------------------------------------------------------------
# sampling + tracing


def sample_lambertian(n, rng_pair):
    """pathtrace.sample_lambertian (pathtrace.py:287-304): cosine-weighted direction(s) about n."""
    u1, u2 = rng_pair
    scalar = np.asarray(u1).ndim == 0
    nn = np.ascontiguousarray(np.atleast_2d(np.asarray(n, dtype=np.float64)))
    a = np.ascontiguousarray(np.atleast_1d(np.asarray(u1, dtype=np.float64)))
    b = np.ascontiguousarray(np.atleast_1d(np.asarray(u2, dtype=np.float64)))
    m = nn.shape[0]
    if a.shape[0] != m or b.shape[0] != m:
        raise ValueError("need one (u1, u2) pair per normal")
    d = np.empty((m, 3), dtype=np.float64)
    pdf = np.empty(m, dtype=np.float64)
    dev = _default_device()
    N.check(N.load().knf_sample_lambertian(N.ptr(nn), N.ptr(a), N.ptr(b), m, N.ptr(d), N.ptr(pdf), dev, N.MEM_HOST,
                                           N.current_stream(dev)))
    if m == 1 and scalar:
        return d[0], float(pdf[0])
    return d, pdf


def intersect_scene(scene: Scene, origins, dirs, t_max: float = np.inf):
    """pathtrace.intersect_scene (pathtrace.py:311-330) -> (t, obj_index, None).  The third slot held
    per-object march results in the reference; the device keeps those internally."""
    ds = device_scene(scene)
    o = np.ascontiguousarray(np.atleast_2d(origins), dtype=np.float64)
    d = np.ascontiguousarray(np.atleast_2d(dirs), dtype=np.float64)
    n = o.shape[0]
    t = np.empty(n, dtype=np.float64)
    obj = np.empty(n, dtype=np.int32)
    dev = _device_index(scene)
    N.check(N.load().knf_intersect_scene(ds.handle, N.ptr(o), N.ptr(d), n, float(t_max), N.ptr(t), N.ptr(obj), N.MEM_HOST,
                                         N.current_stream(dev)))
    return t, obj.astype(int), None


def _trace_batch(scene: Scene, origins, dirs, pixel_ids, sample_idx, rng: Rng, max_bounces: int):
    """pathtrace._trace_batch (pathtrace.py:340-420) -> (n,3) radiance."""
    ds = device_scene(scene)
    o = np.ascontiguousarray(np.atleast_2d(origins), dtype=np.float64)
    d = np.ascontiguousarray(np.atleast_2d(dirs), dtype=np.float64)
    pix = np.ascontiguousarray(pixel_ids, dtype=np.uint64).reshape(-1)
    n = o.shape[0]
    rad = np.empty((n, 3), dtype=np.float64)
    dev = _device_index(scene)
    N.check(N.load().knf_trace_paths(ds.handle, N.ptr(o), N.ptr(d), N.ptr(pix), n, C.c_uint64(int(sample_idx)),
                                     C.c_uint64(rng.seed & 0xFFFFFFFFFFFFFFFF), int(max_bounces), N.ptr(rad), N.MEM_HOST,
                                     N.current_stream(dev)))
    return rad


def trace_path(scene: Scene, ray, rng: Rng, max_bounces: int = 8, pixel: int = 0, sample: int = 0) -> np.ndarray:
    """pathtrace.trace_path (pathtrace.py:423-427): radiance along one camera ray."""
    o = np.asarray(ray.origin, dtype=np.float64)[None, :]
    d = np.asarray(ray.direction, dtype=np.float64)[None, :]
    return _trace_batch(scene, o, d, np.array([pixel]), sample, rng, max_bounces)[0]


@dataclass
class PathtraceResult:
    hdr: np.ndarray  # (H, W, 3) float64 mean radiance
    ldr: np.ndarray  # (H, W, 3) float64 in [0, 1], gamma 2.2


def pathtrace_rows(scene: Scene, pose: CameraPose, spp: int, seed: int, max_bounces: int, sample_offset: int, row0: int,
                   row1: int, device_out: bool = False):
    """Rows [row0,row1) of render_pathtraced's hdr buffer (the unit multi-GPU sharding splits on)."""
    ds = device_scene(scene)
    cam = camera_struct(pose)
    rows, W = row1 - row0, int(pose.width)
    dev = _device_index(scene)
    if device_out:
        import torch

        hdr = torch.empty((rows, W, 3), dtype=torch.float64, device=torch.device("cuda", dev))
        mem = N.MEM_DEVICE
    else:
        hdr = np.empty((rows, W, 3), dtype=np.float64)
        mem = N.MEM_HOST
    N.check(N.load().knf_pathtrace(ds.handle, C.byref(cam), int(spp), C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), int(max_bounces),
                                   int(sample_offset), int(row0), int(row1), N.ptr(hdr), mem, N.current_stream(dev)))
    return hdr


def render_pathtraced(scene: Scene, pose: CameraPose, spp: int, seed: int, max_bounces: int = 8, tile_rows: int = 64,
                      sample_offset: int = 0) -> PathtraceResult:
    """pathtrace.render_pathtraced (pathtrace.py:436-471).  Per-pixel counter RNG makes the result
    independent of banding, so ``tile_rows`` is accepted for compatibility and the device picks its
    own band size."""
    if spp < 1:
        raise ValueError("spp must be >= 1")
    hdr = pathtrace_rows(scene, pose, spp, seed, max_bounces, sample_offset, 0, int(pose.height))
    return PathtraceResult(hdr=hdr, ldr=np.clip(hdr, 0.0, 1.0) ** (1.0 / 2.2))
