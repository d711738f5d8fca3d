"""Degree-5 near-minimax polynomial for ln(1 + e) on [0, 1] (softplus_fast_poly_f2xN, knf_common.cuh): weighted least
squares iterated towards equal ripple, then the error of the fp32 Horner evaluation on a 200 001-point grid."""
import numpy as np
deg = 5
x = np.linspace(0, 1, 200001)
V = np.vander(x, deg + 1)
w = np.ones_like(x)
best, best_err = None, np.inf
for it in range(60):
    c, *_ = np.linalg.lstsq(V * w[:, None], np.log1p(x) * w, rcond=None)
    err = np.abs(V @ c - np.log1p(x))
    if err.max() < best_err:
        best, best_err = c, err.max()
    w = w * (1 + 3 * err / err.max())
    w /= w.mean()
xf = x.astype(np.float32)
acc = np.full_like(xf, np.float32(best[0]))
for cc in best[1:]:
    acc = (acc * xf + np.float32(cc)).astype(np.float32)
print("coefficients (highest first):", [float(np.float32(v)) for v in best])
print("max |error| float64:", best_err, " fp32 Horner:", np.abs(acc.astype(np.float64) - np.log1p(x)).max())
