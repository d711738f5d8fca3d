"""Decision filter on vs off in the exact mode: bit-identical frames?  timing, filter statistics."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2206_10885_b200 import grid, surface, cameras
from paper_2206_10885_b200.modelio import load_model
from bench import orbit_view
W, H = 1920, 1080
for name, field in (("random_init_16", grid.field_init(grid.GridConfig(resolution=16), seed=0)),
                    ("distilled_4", load_model(os.path.join(ROOT, "tests", "golden", "sphere_r4_distilled.knf")))):
    fs = surface.FieldSurface(field)
    print(name, "filter delta max", fs.dev.filter_delta(), flush=True)
    frames = {}
    for mode in ("off", "on", "auto"):
        fs.dev.set_filter(mode)
        fs.dev.reset_stats()
        frames[mode] = surface.render_frame(fs, orbit_view(3, W, H))
        st = fs.dev.stats()
        print(" ", mode, "hits", int(frames[mode].hit.sum()), "exact evals", st["sdf_evals"], "filter evals", st["filter_evals"], "deferred", st["filter_deferred"], "skipped", st["filter_skipped"],
              "wavefronts", st["wavefronts"], "launches", st["kernel_launches"], flush=True)
    for mode in ("on", "auto"):
        same = all(np.array_equal(getattr(frames["off"], k), getattr(frames[mode], k)) for k in ("color", "depth", "normal", "hit"))
        print("  filter", mode, "== off bit for bit:", same, flush=True)
    dev = torch.device("cuda", 0)
    bufs = (torch.empty((H, W, 3), dtype=torch.float32, device=dev), torch.empty((H, W), dtype=torch.float32, device=dev),
            torch.empty((H, W, 3), dtype=torch.float32, device=dev), torch.empty((H, W), dtype=torch.uint8, device=dev))
    stt = surface.RenderSettings()
    def loop(n):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for s in range(n):
            surface.render_rows(fs, orbit_view(s, W, H), stt, (1.0, 1.0, 1.0), 1, 0, H, out=bufs, device_out=True)
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3 / n
    loop(30)
    for mode in ("off", "on", "auto"):
        fs.dev.set_filter(mode); loop(3)
        print("  1080p filter", mode, "%.2f ms/frame" % loop(20), flush=True)
