"""Tiny driver for ncu: render 1080p frames of the random-init field (device resident)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_10885_b200 import grid, surface, cameras
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
fs = surface.FieldSurface(grid.field_init(grid.GridConfig(resolution=16), seed=0))
pose = cameras.orbit_pose(3, 100, 2.5, 0.2, np.deg2rad(40), 1920, 1080)
for _ in range(n):
    surface.render_rows(fs, pose, surface.RenderSettings(), (1, 1, 1), 1, 0, 1080, device_out=True)
torch.cuda.synchronize()
