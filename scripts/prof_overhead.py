"""Times the device-resident 1080p frame loop with the per-launch event profiling on and off."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_10885_b200 import grid, surface
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import orbit_view
W, H = 1920, 1080
field = grid.field_init(grid.GridConfig(resolution=16), seed=0)
fs = surface.FieldSurface(field, device=0)
st = surface.RenderSettings()
dev = torch.device("cuda", 0)
bufs = (torch.empty((H, W, 3), dtype=torch.float32, device=dev), torch.empty((H, W), dtype=torch.float32, device=dev),
        torch.empty((H, W, 3), dtype=torch.float32, device=dev), torch.empty((H, W), dtype=torch.uint8, device=dev))
def loop(n, s0=0):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); t0 = time.perf_counter(); e0.record()
    for s in range(n):
        surface.render_rows(fs, orbit_view(s0 + s, W, H), st, (1.0, 1.0, 1.0), 1, 0, H, out=bufs, device_out=True)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, (time.perf_counter() - t0) * 1e3 / n
print("warm", loop(3))
for rep in range(3):
    for prof in (True, False):
        fs.dev.set_profiling(prof)
        if prof: fs.dev.reset_stats()
        print("profiling", prof, "ms/frame (events, wall): %.2f %.2f" % loop(20, 3))
        if prof: fs.dev.stats()
