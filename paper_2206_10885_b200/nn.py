"""Encoder and activations as stand-alone operators: same names as the reference ``kilofield.nn``
(nn.py:26-93) for the pieces that sit on the render path.  They run the exact device routines the
fused MLP kernels use, so they double as a direct parity probe of the device math.
(``mlp_forward`` / backward / Adam are training-side and not provided.)"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .grid import _default_device

SOFTPLUS, RELU, SIGMOID, IDENTITY = "softplus", "relu", "sigmoid", "identity"
ACTIVATIONS = (IDENTITY, RELU, SOFTPLUS, SIGMOID)


def encoded_dim(n: int, L: int) -> int:
    return n + 2 * n * L


def fourier_encode(x, L: int):
    """nn.fourier_encode for 3-vectors ((3,) or (batch,3)), fp32: [x | sin(pi x) | cos(pi x) | ...]."""
    if L < 0:
        raise ValueError("L must be >= 0")
    a = np.asarray(x)
    single = a.ndim == 1
    p = np.ascontiguousarray(np.atleast_2d(a), dtype=np.float32)
    if p.shape[1] != 3:
        raise N.KnfUnsupported("the device encoder handles 3-vectors (positions / directions) only")
    out = np.empty((p.shape[0], 3 + 6 * L), dtype=np.float32)
    dev = _default_device()
    N.check(N.load().knf_fourier_encode(N.ptr(p), p.shape[0], int(L), N.ptr(out), dev, N.MEM_HOST, N.current_stream(dev)))
    return out[0] if single else out


def _unary(fn_name, x):
    a = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty_like(a)
    dev = _default_device()
    N.check(getattr(N.load(), fn_name)(N.ptr(a), a.size, N.ptr(out), dev, N.MEM_HOST, N.current_stream(dev)))
    return out


def softplus(x):
    """nn.softplus (nn.py:26-33): ln(1 + e^x), overflow-safe."""
    return _unary("knf_softplus", x)


def sigmoid(x):
    """nn.sigmoid (nn.py:36-38)."""
    return _unary("knf_sigmoid", x)


def apply_activation(name: str, x):
    """nn.apply_activation (nn.py:41-50)."""
    if name == IDENTITY:
        return np.asarray(x)
    if name == RELU:
        return np.maximum(x, 0.0)
    if name == SOFTPLUS:
        return softplus(x)
    if name == SIGMOID:
        return sigmoid(x)
    raise ValueError(f"unknown activation {name!r}")
