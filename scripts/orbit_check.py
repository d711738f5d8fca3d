"""Config 2 (800x800, 100-view orbit) on the distilled field: total ms, twice."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2206_10885_b200 import grid, surface, cameras
from paper_2206_10885_b200.modelio import load_model
name = sys.argv[1] if len(sys.argv) > 1 else "distilled"
field = load_model(os.path.join(ROOT, "tests", "golden", "sphere_r4_distilled.knf")) if name == "distilled" else grid.field_init(grid.GridConfig(resolution=16), seed=0)
fs = surface.FieldSurface(field)
st = surface.RenderSettings()
for rep in range(3):
    fs.dev.reset_stats()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for k in range(100):
        surface.render_rows(fs, cameras.orbit_pose(k, 100, 2.5, 0.2, np.deg2rad(40), 800, 800), st, (1, 1, 1), 1, 0, 800, device_out=True)
    torch.cuda.synchronize(); ms = (time.perf_counter() - t0) * 1e3
    s = fs.dev.stats()
    print(f"{name} orbit: {ms:.0f} ms ({100e3/ms:.0f} FPS) wavefronts/frame {s['wavefronts']/100:.1f} launches/frame {s['kernel_launches']/100:.0f} exact evals/frame {s['sdf_evals']/100/1e6:.2f} M filter {s['filter_evals']/100/1e6:.2f} M", flush=True)
