"""Tiny driver for ncu: render 1080p frames (device resident) of the random-init field, or of the trained 16^3 field (argv 2 = trained16)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2206_10885_b200 import grid, surface, cameras
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
if len(sys.argv) > 2 and sys.argv[2] == "trained16":
    from paper_2206_10885_b200.modelio import load_model
    field = grid.refine_field(load_model(os.path.join(ROOT, "tests", "golden", "sphere_stripes_r8_distilled.knf")), 2)
else:
    field = grid.field_init(grid.GridConfig(resolution=16), seed=0)
fs = surface.FieldSurface(field)
pose = cameras.orbit_pose(3, 100, 2.5, 0.2, np.deg2rad(40), 1920, 1080)
for _ in range(n):
    surface.render_rows(fs, pose, surface.RenderSettings(), (1, 1, 1), 1, 0, 1080, device_out=True)
torch.cuda.synchronize()
