"""Soak test of the decision filter: filter on vs off, bit-for-bit, over several random-init fields (seeds, grid
resolutions) and views at full 1920x1080 -> gpurun_out/filter_soak.json."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2206_10885_b200 import grid, surface
from bench import orbit_view
W, H = 1920, 1080
out = []
for res, seed in ((16, 0), (16, 1), (16, 2), (8, 5), (32, 7)):
    field = grid.field_init(grid.GridConfig(resolution=res), seed=seed)
    fs = surface.FieldSurface(field)
    for view in (0, 17, 58):
        fs.dev.set_filter("off"); a = surface.render_frame(fs, orbit_view(view, W, H))
        fs.dev.set_filter("on"); fs.dev.reset_stats(); b = surface.render_frame(fs, orbit_view(view, W, H)); st = fs.dev.stats()
        same = all(np.array_equal(getattr(a, k), getattr(b, k)) for k in ("color", "depth", "normal", "hit"))
        rec = {"resolution": res, "seed": seed, "view": view, "identical": bool(same), "hits": int(a.hit.sum()), "exact_evals": int(st["sdf_evals"]),
               "filter_evals": int(st["filter_evals"]), "undecided": int(st["filter_deferred"]), "certified": int(st["filter_skipped"]), "delta_max": fs.dev.filter_delta()}
        print(rec, flush=True)
        out.append(rec)
    fs.dev.close() if hasattr(fs.dev, "close") else None
print("ALL IDENTICAL:", all(r["identical"] for r in out))
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "filter_soak.json"), "w"), indent=1)
