"""Sub-box refinement of the per-cell Lipschitz bounds (csrc/knf_bounds.cuh): tightening factor, device time, a float64
NumPy restatement on a few cells, a soundness check against sampled gradients, and the frame-time effect."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2206_10885_b200 import grid
res = int(sys.argv[1]) if len(sys.argv) > 1 else 16
field = grid.field_init(grid.GridConfig(resolution=res), seed=0)
dev = grid.device_field(field)
t0 = time.time()
closed, refined, ms = dev.lipschitz()
print(f"resolution {res}: refinement {ms:.1f} ms on the device ({time.time() - t0:.2f} s wall); closed-form mean {closed.mean():.1f}, refined mean {refined.mean():.1f}, "
      f"ratio mean {np.mean(closed / refined):.2f} min {np.min(closed / refined):.2f} max {np.max(closed / refined):.2f}")
# soundness: sampled |d d / d x_a| (float64 central differences of the float64 network) never exceeds the bound
W = [np.asarray(w, np.float64) for w in field.sdf.weights]; B = [np.asarray(b, np.float64) for b in field.sdf.biases]
lo, hi = np.asarray(field.config.bbox_min, float), np.asarray(field.config.bbox_max, float)
rng = np.random.default_rng(0)
worst = 0.0
for c in rng.integers(0, res ** 3, 24):
    ci = np.array([c // (res * res), (c // res) % res, c % res])
    clo = lo + (hi - lo) * ci / res
    x = clo + rng.uniform(0, 1, (40000, 3)) * (hi - lo) / res
    def fwd(x):
        f = [x]
        for o in range(6):
            f += [np.sin(2 ** o * np.pi * x), np.cos(2 ** o * np.pi * x)]
        e = np.concatenate(f, -1)
        h = np.logaddexp(0, e @ W[0][c].T + B[0][c]); h = np.logaddexp(0, h @ W[1][c].T + B[1][c])
        return h @ W[2][c][0] + B[2][c][0]
    h = 1e-6
    g = np.stack([np.abs(fwd(x + h * np.eye(3)[a]) - fwd(x - h * np.eye(3)[a])) / (2 * h) for a in range(3)], 1).max(0)
    worst = max(worst, float((g / refined[c]).max()))
    assert (g <= refined[c] * (1 + 1e-6)).all(), (c, g, refined[c])
print(f"sampled gradient / refined bound: worst {worst:.3f} over 24 cells x 40000 points (must stay below 1)")
