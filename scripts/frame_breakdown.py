"""Per-kernel-class time of the 1080p random-init frame (library event profiling)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2206_10885_b200 import grid, surface
from bench import orbit_view
W, H = 1920, 1080
args = [a for a in sys.argv[1:] if a not in ("distilled", "trained16", "trained8")]
if "trained16" in sys.argv[1:]:
    from paper_2206_10885_b200.modelio import load_model
    fs = surface.FieldSurface(grid.refine_field(load_model(os.path.join(ROOT, "tests", "golden", "sphere_stripes_r8_distilled.knf")), 2))
elif "trained8" in sys.argv[1:]:
    from paper_2206_10885_b200.modelio import load_model
    fs = surface.FieldSurface(load_model(os.path.join(ROOT, "tests", "golden", "sphere_stripes_r8_distilled.knf")))
elif "distilled" in sys.argv[1:]:
    from paper_2206_10885_b200.modelio import load_model
    fs = surface.FieldSurface(load_model(os.path.join(ROOT, "tests", "golden", "sphere_r4_distilled.knf")))
else:
    fs = surface.FieldSurface(grid.field_init(grid.GridConfig(resolution=16), seed=0))
for a in args:
    k, v = a.split("=")
    getattr(fs.dev, "set_" + k)(v)
dev = torch.device("cuda", 0)
bufs = (torch.empty((H, W, 3), dtype=torch.float32, device=dev), torch.empty((H, W), dtype=torch.float32, device=dev),
        torch.empty((H, W, 3), dtype=torch.float32, device=dev), torch.empty((H, W), dtype=torch.uint8, device=dev))
st = surface.RenderSettings()
def loop(n):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for s in range(n):
        surface.render_rows(fs, orbit_view(s, W, H), st, (1.0, 1.0, 1.0), 1, 0, H, out=bufs, device_out=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / n
loop(30)
fs.dev.set_profiling(True); fs.dev.reset_stats()
n = 10
ms = loop(n)
s = fs.dev.stats()
print("filter fill %.3f exact fill %.3f" % (s["filter_evals"] / max(s["filter_lane_slots"], 1), s["sdf_evals"] / max(s["march_lane_slots"], 1)))
print("frame %.2f ms | exact kernel %.2f ms (%d launches, %.1f M evals) | filter %.2f ms (%d launches, %.1f M evals, %.2f M deferred) | route %.2f ms (%d) | colour %.2f | other %.2f | wavefronts %d launches %d"
      % (ms, s["sdf_mlp_ms"] / n, s["sdf_mlp_launches"] / n, s["sdf_evals"] / n / 1e6, s["filter_ms"] / n, s["filter_launches"] / n, s["filter_evals"] / n / 1e6,
         s["filter_deferred"] / n / 1e6, s["route_ms"] / n, s["route_launches"] / n, s["color_mlp_ms"] / n, s["other_ms"] / n, s["wavefronts"] / n, s["kernel_launches"] / n))
