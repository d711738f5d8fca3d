import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2206_10885_b200 import grid, surface
from paper_2206_10885_b200.modelio import load_model
from bench import orbit_view
W, H = 1920, 1080
for name in ("trained8", "trained16"):
    f = load_model("/root/repo/tests/golden/sphere_stripes_r8_distilled.knf")
    if name == "trained16": f = grid.refine_field(f, 2)
    fs = surface.FieldSurface(f)
    for s in range(3): surface.render_frame(fs, orbit_view(s, W, H))
    fs.dev.reset_stats()
    surface.render_frame(fs, orbit_view(3, W, H))
    st = fs.dev.stats()
    print(name, {k: st[k] for k in ("sdf_evals", "march_routed_requests", "march_lane_slots", "wavefronts", "rays", "hits")})
