import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2206_10885_b200 import grid, surface
from bench import orbit_view
W, H = 1920, 1080
fs = surface.FieldSurface(grid.field_init(grid.GridConfig(resolution=16), seed=0))
dev = torch.device("cuda", 0)
bufs = (torch.empty((H, W, 3), dtype=torch.float32, device=dev), torch.empty((H, W), dtype=torch.float32, device=dev),
        torch.empty((H, W, 3), dtype=torch.float32, device=dev), torch.empty((H, W), dtype=torch.uint8, device=dev))
st = surface.RenderSettings()
for s in range(int(sys.argv[1])):
    surface.render_rows(fs, orbit_view(3, W, H), st, (1.0, 1.0, 1.0), 1, 0, H, out=bufs, device_out=True)
torch.cuda.synchronize()
