"""fp32_chain vs tensor_bf16x3: forward error against the oracle, 256^2 frame parity, 1080p frame time."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import oracle
from conftest import oracle_from_product
from paper_2206_10885_b200 import grid, surface, cameras
from bench import orbit_view

out = {}
from paper_2206_10885_b200 import nn as knn
xs = np.concatenate([np.random.default_rng(5).normal(0, 1.5, 3_000_000), np.random.default_rng(6).uniform(-30, 30, 1_000_000)]).astype(np.float32)
sp_dev, sp_ref = knn.softplus(xs), oracle.softplus32(xs)
out["softplus_vs_numpy"] = {"n": int(xs.size), "mismatches": int((sp_dev != sp_ref).sum()), "max_abs": float(np.abs(sp_dev - sp_ref).max())}
print("softplus device vs numpy on this host:", out["softplus_vs_numpy"], flush=True)
f42 = grid.field_init(grid.GridConfig(resolution=16), seed=42)
pts = np.random.default_rng(42).uniform(-1.1, 1.1, (100_000, 3)).astype(np.float32)
ref = oracle.query_sdf(oracle_from_product(f42), pts)
ref_full = np.concatenate([np.asarray(ref[0])[:, None], np.asarray(ref[1])], axis=1)
fs = surface.FieldSurface(f42)
for mode in ("fp32_chain", "tensor_bf16x3", "tensor_fp16x2"):
    fs.dev.set_precision(mode)
    s = grid.sdf_query(fs.dev, pts)
    full = np.concatenate([np.asarray(s.value)[:, None], np.asarray(s.features)], axis=1)
    err = np.abs(full - ref_full)
    out["forward_" + mode] = {"max_abs": float(err.max()), "mean_abs": float(err.mean()), "dist_mean_abs": float(err[:, 0].mean()),
                              "dist_max_abs": float(err[:, 0].max())}
    print(mode, out["forward_" + mode], flush=True)

def compare(a, b):
    both = a.hit & b.hit
    rel = np.abs(a.depth[both] - b.depth[both]) / b.depth[both]
    nerr = np.abs(a.normal - b.normal)[both].max(axis=1); cerr = np.abs(a.color - b.color)[both].max(axis=1)
    return {"hit_agreement": float((a.hit == b.hit).mean()), "flips": int((a.hit != b.hit).sum()),
            "depth_frac_le_1e-4": float((rel <= 1e-4).mean()), "normal_frac_le_1e-3": float((nerr <= 1e-3).mean()),
            "rgb_frac_le_1e-3": float((cerr <= 1e-3).mean())}

f0 = grid.field_init(grid.GridConfig(resolution=16), seed=0)
fs0 = surface.FieldSurface(f0)
sizes = [(256, 256)] + ([(1920, 1080)] if "--full" in sys.argv else [])
for (w, h) in sizes:
    pose = cameras.look_at_pose((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), w, h)
    ocam = oracle.camera_look_at((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), w, h)
    t0 = time.perf_counter(); ref = oracle.render(oracle.FieldTraceable(oracle_from_product(f0)), ocam, oracle.MarchSettings()); cpu = time.perf_counter() - t0
    frames = {}
    for mode in ("fp32_chain", "tensor_bf16x3", "tensor_fp16x2"):
        fs0.dev.set_precision(mode)
        frames[mode] = surface.render_frame(fs0, pose)
        out[f"frame_{w}x{h}_{mode}_vs_oracle"] = compare(frames[mode], ref)
        print(w, h, mode, out[f"frame_{w}x{h}_{mode}_vs_oracle"], flush=True)
    out[f"frame_{w}x{h}_chain_vs_tensor"] = compare(frames["fp32_chain"], frames["tensor_bf16x3"])
    print(w, h, "chain vs tensor", out[f"frame_{w}x{h}_chain_vs_tensor"], "oracle s", cpu, flush=True)

W, H = 1920, 1080
dev = torch.device("cuda", 0)
bufs = (torch.empty((H, W, 3), dtype=torch.float32, device=dev), torch.empty((H, W), dtype=torch.float32, device=dev),
        torch.empty((H, W, 3), dtype=torch.float32, device=dev), torch.empty((H, W), dtype=torch.uint8, device=dev))
st = surface.RenderSettings()
def loop(n):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for s in range(n):
        surface.render_rows(fs0, orbit_view(s, W, H), st, (1.0, 1.0, 1.0), 1, 0, H, out=bufs, device_out=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / n
loop(30)
for rep in range(2):
    for mode in ("fp32_chain", "tensor_bf16x3", "tensor_fp16x2"):
        fs0.dev.set_precision(mode)
        loop(3)
        out[f"ms_1080p_{mode}"] = loop(20)
        print("1080p", mode, "%.2f ms/frame" % out[f"ms_1080p_{mode}"], flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "precision_check.json"), "w"), indent=1)
