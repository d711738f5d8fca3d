"""Quick device-side timings (CUDA events) of the hot path; prints one line per workload."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_10885_b200 import grid, surface, cameras
from paper_2206_10885_b200.modelio import load_model

def timed(fn, warm=2, it=5):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(it):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts)), float(np.min(ts))

print(torch.cuda.get_device_name(0))
f16 = grid.field_init(grid.GridConfig(resolution=16), seed=0)
dev = grid.device_field(f16)
for M in (1 << 16, 1_000_000, 1 << 22):
    pts = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, (M, 3)).astype(np.float32), device="cuda")
    med, best = timed(lambda: grid.sdf_query(dev, pts))
    print(f"sdf_query M={M}: {med:.3f} ms median ({best:.3f} best) -> {M/med/1e3:.1f} Mq/s ; {M*5120/med/1e9:.2f} TFLOP/s")
    z = grid.sdf_query(dev, pts).features.contiguous()
    v = torch.nn.functional.normalize(torch.randn(M, 3, device="cuda"), dim=1)
    med, best = timed(lambda: grid.color_query(dev, pts, v, v, z))
    print(f"color_query M={M}: {med:.3f} ms -> {M/med/1e3:.1f} Mq/s")
# clustered: all points in one cell / 64 cells
for ncell in (1, 64):
    M = 1 << 20
    rng = np.random.default_rng(1)
    base = rng.integers(0, 16, size=(ncell, 3))
    pick = base[rng.integers(0, ncell, M)]
    p = ((pick + rng.uniform(0.01, 0.99, (M, 3))) / 8.0 - 1.0).astype(np.float32)
    pts = torch.as_tensor(p, device="cuda")
    med, best = timed(lambda: grid.sdf_query(dev, pts))
    print(f"sdf_query clustered in {ncell} cells M={M}: {med:.3f} ms -> {M/med/1e3:.1f} Mq/s")

fd = load_model(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "sphere_r4_distilled.knf"))
for name, field in (("random16", f16), ("distilled4", fd)):
    fs = surface.FieldSurface(field)
    for (w, h) in ((256, 256), (800, 800), (1920, 1080)):
        pose = cameras.look_at_pose((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), w, h)
        med, best = timed(lambda: surface.render_rows(fs, pose, surface.RenderSettings(), (1, 1, 1), 1, 0, h, device_out=True), warm=1, it=3)
        fs.dev.set_profiling(True); fs.dev.reset_stats()
        surface.render_rows(fs, pose, surface.RenderSettings(), (1, 1, 1), 1, 0, h, device_out=True)
        st = fs.dev.stats(); fs.dev.set_profiling(False)
        t0 = time.perf_counter(); fb = surface.render_frame(fs, pose); e2e = (time.perf_counter() - t0) * 1e3
        print(f"render {name} {w}x{h}: {med:.2f} ms device ({1e3/med:.1f} FPS, {w*h/med/1e3:.1f} Mrays/s), e2e host {e2e:.1f} ms; "
              f"sdf evals {st['sdf_evals']} ({st['sdf_evals']/(w*h):.1f}/ray, {st['sdf_evals']/med/1e6:.2f} Gevals/s), hits {st['hits']}, launches {st['kernel_launches']}, wavefronts {st['wavefronts']}, mlp {st['sdf_mlp_ms']:.2f} ms, route {st['route_ms']:.2f} ms, tile fill {st['sdf_evals']/max(st['march_lane_slots'],1):.3f}")
