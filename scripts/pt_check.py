"""Config 5 (4K path tracing, floor + neural object) timing on the random-init field, filter modes."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2206_10885_b200 import grid, surface, cameras, pathtrace
f16 = grid.field_init(grid.GridConfig(resolution=16), seed=0)
fs = surface.FieldSurface(f16)
scene16 = pathtrace.Scene([pathtrace.QuadObj((-3, -1.0, -3), (6, 0, 0), (0, 0, 6), pathtrace.Lambertian((0.7, 0.7, 0.7))),
                           pathtrace.NeuralObject(fs)], pathtrace.ConstantEnv((1, 1, 1)))
pose = cameras.look_at_pose((0.5, 0.8, 3.2), (0, -0.2, 0), (0, 1, 0), np.deg2rad(45), 3840, 2160)
ref = None
for mode in sys.argv[1:] or ["auto", "off", "on", "auto"]:
    fs.dev.set_filter(mode)
    for rep in range(2):
        fs.dev.reset_stats()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        out = pathtrace.pathtrace_rows(scene16, pose, 1, 0, 8, 0, 0, 2160, device_out=True)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t0) * 1e3
        st = fs.dev.stats()
        hdr = out[0] if isinstance(out, (tuple, list)) else out
        same = None if ref is None else bool(torch.equal(hdr, ref))
        if ref is None: ref = hdr.clone()
        print(f"filter {mode}: {dt:.1f} ms  exact {st['sdf_evals']/1e6:.1f} M filter {st['filter_evals']/1e6:.1f} M skipped {st['filter_skipped']/1e6:.1f} M wavefronts {st['wavefronts']} launches {st['kernel_launches']} same_as_first={same}", flush=True)
