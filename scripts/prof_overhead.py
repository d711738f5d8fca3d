"""1080p random-init frame time with and without the library's per-launch event profiling."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2206_10885_b200 import grid, surface
from bench import orbit_view
W, H = 1920, 1080
fs = surface.FieldSurface(grid.field_init(grid.GridConfig(resolution=16), seed=0))
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
loop(40)
for rep in range(2):
    fs.dev.set_profiling(False); a = loop(20)
    fs.dev.set_profiling(True); b = loop(20); fs.dev.stats()
    print(f"profiling off {a:.2f} ms/frame, on {b:.2f} ms/frame")
