"""Timings of the other BASELINE.json configs (2, 4, 5) -> gpurun_out/configs_r1.json.  Device-side CUDA events."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2206_10885_b200 import grid, surface, cameras, pathtrace
from paper_2206_10885_b200.modelio import load_model

def ev_time(fn, warm=1, it=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize(); ts = []
    for _ in range(it):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))

out = {}
f16 = grid.field_init(grid.GridConfig(resolution=16), seed=0)
fd = load_model(os.path.join(ROOT, "tests", "golden", "sphere_r4_distilled.knf"))
# config 2: 800x800 100-view orbit
for name, field in (("random_init_16", f16), ("distilled_4", fd)):
    fs = surface.FieldSurface(field)
    def orbit():
        for k in range(100):
            surface.render_rows(fs, cameras.orbit_pose(k, 100, 2.5, 0.2, np.deg2rad(40), 800, 800), surface.RenderSettings(), (1, 1, 1), 1, 0, 800, device_out=True)
    ms = ev_time(orbit, warm=1, it=1)
    out[f"config2_orbit_800x800_100views_{name}"] = {"ms_total": ms, "fps": 100e3 / ms, "mrays_per_s": 100 * 640000 / ms / 1e3}
# config 4: batched forward sweep
dev = grid.device_field(f16)
sweep = {}
for M in [1 << 14, 1 << 16, 1 << 18, 1_000_000, 1 << 22, 1 << 24]:
    pts = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, (M, 3)).astype(np.float32), device="cuda")
    ms = ev_time(lambda: grid.sdf_query(dev, pts))
    z = grid.sdf_query(dev, pts).features.contiguous()
    v = torch.nn.functional.normalize(torch.randn(M, 3, device="cuda"), dim=1)
    msc = ev_time(lambda: grid.color_query(dev, pts, v, v, z))
    sweep[str(M)] = {"sdf_ms": ms, "sdf_Mq_per_s": M / ms / 1e3, "sdf_tflops": M * 5120 / ms / 1e9, "color_ms": msc, "color_Mq_per_s": M / msc / 1e3}
    del pts, z, v
out["config4_forward_sweep"] = sweep
# the same 1e6 / 2^24-point SDF forward in the tensor-core precision modes
modes = {}
for mode in ("fp32_chain", "tensor_bf16x3", "tensor_fp16x2"):
    dev.set_precision(mode)
    for M in (1_000_000, 1 << 24):
        pts = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, (M, 3)).astype(np.float32), device="cuda")
        ms = ev_time(lambda: grid.sdf_query(dev, pts))
        modes[f"{mode}_{M}"] = {"sdf_ms": ms, "sdf_Mq_per_s": M / ms / 1e3, "sdf_tflops": M * 5120 / ms / 1e9}
        del pts
dev.set_precision("fp32_chain")
out["config4_precision_modes"] = modes
for ncell in (1, 8, 64):
    M = 1 << 20
    rng = np.random.default_rng(1); base = rng.integers(0, 16, size=(ncell, 3)); pick = base[rng.integers(0, ncell, M)]
    pts = torch.as_tensor(((pick + rng.uniform(0.01, 0.99, (M, 3))) / 8.0 - 1.0).astype(np.float32), device="cuda")
    ms = ev_time(lambda: grid.sdf_query(dev, pts))
    out[f"config4_clustered_{ncell}_cells_1Mi"] = {"sdf_ms": ms, "sdf_Mq_per_s": M / ms / 1e3}
# config 5: 3840x2160 path traced, floor quad + neural object, spp 1 (row band of the frame per rank; full frame here)
scene = pathtrace.Scene([pathtrace.QuadObj((-3, -1.0, -3), (6, 0, 0), (0, 0, 6), pathtrace.Lambertian((0.7, 0.7, 0.7))),
                         pathtrace.NeuralObject(surface.FieldSurface(fd))], pathtrace.ConstantEnv((1, 1, 1)))
pose = cameras.look_at_pose((0.5, 0.8, 3.2), (0, -0.2, 0), (0, 1, 0), np.deg2rad(45), 3840, 2160)
ms = ev_time(lambda: pathtrace.pathtrace_rows(scene, pose, 1, 0, 8, 0, 0, 2160, device_out=True), warm=1, it=2)
out["config5_pathtrace_3840x2160_spp1_distilled"] = {"ms": ms, "Mpaths_per_s": 3840 * 2160 / ms / 1e3}
scene16 = pathtrace.Scene([pathtrace.QuadObj((-3, -1.0, -3), (6, 0, 0), (0, 0, 6), pathtrace.Lambertian((0.7, 0.7, 0.7))),
                           pathtrace.NeuralObject(surface.FieldSurface(f16))], pathtrace.ConstantEnv((1, 1, 1)))
ms = ev_time(lambda: pathtrace.pathtrace_rows(scene16, pose, 1, 0, 8, 0, 0, 2160, device_out=True), warm=1, it=2)
out["config5_pathtrace_3840x2160_spp1_random_init"] = {"ms": ms, "Mpaths_per_s": 3840 * 2160 / ms / 1e3}
print(json.dumps(out, indent=1))
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "configs_r1.json"), "w"), indent=1)
