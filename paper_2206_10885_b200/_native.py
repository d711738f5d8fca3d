"""ctypes binding of libknf_b200.so (include/knf_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_2206_10885_b200/csrc``).  There is no CPU fallback: if the library is missing, or no
CUDA device is visible, every compute entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KNF_B200_LIB") or os.path.join(_HERE, "libknf_b200.so")  # env override: kernel A/B experiments

KNF_OK = 0
KNF_E_INVALID = -1
KNF_E_UNSUPPORTED = -2
KNF_E_CUDA = -3
KNF_E_IO = -4
KNF_E_NOMEM = -5

MEM_DEVICE = 0
MEM_HOST = 1

OBJ_SPHERE, OBJ_QUAD, OBJ_BOX, OBJ_NEURAL = 0, 1, 2, 3
MAT_LAMBERTIAN, MAT_EMISSIVE = 0, 1


class NativeLibraryMissing(RuntimeError):
    """libknf_b200.so has not been built (run ``python -c 'import __graft_entry__ as g; g.build()'``)."""


class KnfError(RuntimeError):
    """A libknf_b200 call failed for a non-contract reason (CUDA, memory, IO)."""


class KnfUnsupported(KnfError):
    pass


class KnfFieldDesc(C.Structure):
    _fields_ = [
        ("resolution", C.c_int32),
        ("bbox_min", C.c_double * 3),
        ("bbox_max", C.c_double * 3),
        ("sdf_freqs", C.c_int32),
        ("dir_freqs", C.c_int32),
        ("feature_dim", C.c_int32),
        ("fd_step", C.c_double),
        ("sdf_w", C.c_void_p * 3),
        ("sdf_b", C.c_void_p * 3),
        ("color_w", C.c_void_p * 3),
        ("color_b", C.c_void_p * 3),
    ]


class KnfCamera(C.Structure):
    _fields_ = [
        ("position", C.c_double * 3),
        ("rotation", C.c_double * 9),
        ("fov_y", C.c_double),
        ("width", C.c_int32),
        ("height", C.c_int32),
    ]


class KnfSettings(C.Structure):
    _fields_ = [("eps_hit", C.c_double), ("max_steps", C.c_int32), ("step_scale", C.c_double)]


class KnfStats(C.Structure):
    _fields_ = [
        ("sdf_evals", C.c_int64),
        ("color_evals", C.c_int64),
        ("rays", C.c_int64),
        ("hits", C.c_int64),
        ("wavefronts", C.c_int64),
        ("kernel_launches", C.c_int64),
        ("sdf_mlp_launches", C.c_int64),
        ("route_launches", C.c_int64),
        ("sdf_mlp_ms", C.c_double),
        ("route_ms", C.c_double),
        ("color_mlp_ms", C.c_double),
        ("other_ms", C.c_double),
        ("march_lane_slots", C.c_int64),
        ("march_routed_requests", C.c_int64),
        ("filter_evals", C.c_int64),
        ("filter_deferred", C.c_int64),
        ("filter_skipped", C.c_int64),
        ("filter_lane_slots", C.c_int64),
        ("filter_launches", C.c_int64),
        ("filter_ms", C.c_double),
    ]


class KnfObject(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("material", C.c_int32),
        ("rgb", C.c_double * 3),
        ("a", C.c_double * 3),
        ("b", C.c_double * 3),
        ("c", C.c_double * 3),
        ("rot", C.c_double * 9),
        ("s", C.c_double),
        ("field", C.c_void_p),
        ("settings", KnfSettings),
    ]


_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int

# name -> argtypes (every function returns int unless noted)
_SIGNATURES = {
    "knf_abi_version": [],
    "knf_device_count": [],
    "knf_field_create": [C.POINTER(KnfFieldDesc), _I32, C.POINTER(_P)],
    "knf_field_create_from_knf": [C.c_char_p, _I32, C.POINTER(_P)],
    "knf_field_destroy": [_P],
    "knf_field_describe": [_P, C.POINTER(KnfFieldDesc)],
    "knf_field_stats": [_P, C.POINTER(KnfStats)],
    "knf_field_stats_reset": [_P],
    "knf_field_set_profiling": [_P, _I32],
    "knf_field_set_precision": [_P, _I32],
    "knf_field_get_precision": [_P],
    "knf_field_set_filter": [_P, _I32],
    "knf_field_filter_delta": [_P],
    "knf_field_filter_cells_off": [_P],
    "knf_field_filter_kernel": [_P],
    "knf_field_lipschitz": [_P, _P, _P, _P, _P],
    "knf_cell_index": [_P, _P, _I64, _P, _I32, _P],
    "knf_cell_index_f64": [_P, _P, _I64, _P, _I32, _P],
    "knf_route": [_P, _P, _I64, _P, _P, _P, _P, _P, _I32, _P],
    "knf_sdf_forward": [_P, _P, _I64, _P, _I32, _P],
    "knf_sdf_values": [_P, _P, _I64, _P, _I32, _P],
    "knf_sdf_gradient": [_P, _P, _I64, _P, _P, _I32, _P],
    "knf_color_forward": [_P, _P, _P, _P, _P, _I64, _P, _I32, _P],
    "knf_fourier_encode": [_P, _I64, C.c_int32, _P, _I32, _I32, _P],
    "knf_softplus": [_P, _I64, _P, _I32, _I32, _P],
    "knf_sigmoid": [_P, _I64, _P, _I32, _I32, _P],
    "knf_fd_gradient": [_P, _P, _I64, _P, _I32, _P],
    "knf_fd_normals": [_P, _P, _I64, C.c_double, _P, _P, _I32, _P],
    "knf_pixel_rays": [C.POINTER(KnfCamera), _P, _P, _I64, _P, _P, _I32, _I32, _P],
    "knf_ray_aabb": [_P, _P, _I64, C.POINTER(C.c_double * 3), C.POINTER(C.c_double * 3), _P, _P, _P, _I32, _I32, _P],
    "knf_march": [_P, _P, _P, _P, _P, _I64, C.POINTER(KnfSettings), _P, _P, _P, _P, _I32, _P],
    "knf_shade": [_P, _P, _P, _I64, _P, _P, _I32, _P],
    "knf_trace_and_shade": [_P, _P, _P, _I64, C.POINTER(KnfSettings), _P, _P, _P, _P, _P, _P, _I32, _P],
    "knf_render_frame": [_P, C.POINTER(KnfCamera), C.POINTER(KnfSettings), C.POINTER(C.c_double * 3), _I32, _I32,
                         _I32, _P, _P, _P, _P, _I32, _P],
    "knf_render_pass_u8": [_P, C.POINTER(KnfCamera), C.POINTER(KnfSettings), C.POINTER(C.c_double * 3), _I32, _I32, _I32, _I32, _P, _I32, _P],
    "knf_tonemap_u8": [_P, _I64, C.c_double, _I32, _P, _I32, _I32, _P],
    "knf_sample_volume": [_P, C.c_int32, C.POINTER(C.c_double * 3), C.POINTER(C.c_double * 3), _P, _I32, _P],
    "knf_volume_forward": [_P, _P, _P, _I64, C.c_int32, _P, C.POINTER(C.c_double * 3), C.c_double, _P, _I32, _P],
    "knf_scene_create": [C.POINTER(KnfObject), C.c_int32, C.POINTER(C.c_double * 3), _I32, C.POINTER(_P)],
    "knf_scene_destroy": [_P],
    "knf_rng_uniform": [C.c_uint64, _P, _P, _P, _I64, _P, _I32, _I32, _P],
    "knf_sample_lambertian": [_P, _P, _P, _I64, _P, _P, _I32, _I32, _P],
    "knf_intersect_scene": [_P, _P, _P, _I64, C.c_double, _P, _P, _I32, _P],
    "knf_pathtrace": [_P, C.POINTER(KnfCamera), C.c_int32, C.c_uint64, C.c_int32, C.c_int32, _I32, _I32, _P, _I32, _P],
    "knf_trace_paths": [_P, _P, _P, _P, _I64, C.c_uint64, C.c_uint64, C.c_int32, _P, _I32, _P],
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES) + ("knf_last_error",)

_lib = None
_lock = threading.Lock()


def load():
    """Load (once) and return the ctypes handle; raises NativeLibraryMissing if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} not found: the CUDA extension must be built first "
                "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback"
            )
        lib = C.CDLL(LIB_PATH)
        for name, args in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = C.c_int
        lib.knf_field_filter_delta.restype = C.c_double
        lib.knf_field_filter_kernel.restype = C.c_char_p
        lib.knf_last_error.argtypes = []
        lib.knf_last_error.restype = C.c_char_p
        if lib.knf_abi_version() != 2:
            raise KnfError("libknf_b200 ABI version mismatch")
        _lib = lib
    return _lib


def last_error() -> str:
    msg = load().knf_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int):
    """Map a return code onto the reference's exception conventions."""
    if rc == KNF_OK:
        return
    msg = last_error()
    if rc == KNF_E_INVALID:
        raise ValueError(msg)
    if rc == KNF_E_UNSUPPORTED:
        raise KnfUnsupported(msg)
    if rc == KNF_E_NOMEM:
        raise MemoryError(msg)
    if rc == KNF_E_IO:
        raise OSError(msg)
    raise KnfError(msg)


def device_count() -> int:
    n = load().knf_device_count()
    if n < 0:
        raise KnfError(last_error())
    return n


def require_gpu():
    if device_count() < 1:
        raise KnfError("no CUDA device visible: paper_2206_10885_b200 has no CPU fallback")


# ---- argument helpers ----------------------------------------------------------------------------

def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def host_array(x, dtype, shape_tail=None):
    """C-contiguous NumPy view/copy of x with the given dtype."""
    a = np.ascontiguousarray(x, dtype=dtype)
    if shape_tail is not None and a.shape[1:] != tuple(shape_tail):
        raise ValueError(f"expected trailing shape {tuple(shape_tail)}, got {a.shape}")
    return a


def ptr(a):
    """void* of a NumPy array, a torch tensor, or None."""
    if a is None:
        return None
    if _is_torch(a):
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(a.ctypes.data)


def vec3(v):
    return (C.c_double * 3)(*[float(t) for t in np.asarray(v, dtype=np.float64).reshape(3)])


def current_stream(device_index: int):
    """cudaStream_t of torch's current stream on that device (0 if torch has no CUDA)."""
    try:
        import torch

        if torch.cuda.is_available():
            return C.c_void_p(torch.cuda.current_stream(device_index).cuda_stream)
    except Exception:  # pragma: no cover - torch optional for the pure-ctypes path
        pass
    return C.c_void_p(0)
