"""GPU vs oracle end-to-end parity at 256^2 on the random-init and the distilled field -> JSON."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle
from conftest import oracle_from_product
from paper_2206_10885_b200 import grid, surface, cameras
from paper_2206_10885_b200.modelio import load_model

def compare(a, b):
    both = a.hit & b.hit
    rel = np.abs(a.depth[both] - b.depth[both]) / b.depth[both]
    nerr = np.abs(a.normal - b.normal)[both].max(axis=1); cerr = np.abs(a.color - b.color)[both].max(axis=1)
    return {"hit_agreement": float((a.hit == b.hit).mean()), "hits_gpu": int(a.hit.sum()), "hits_ref": int(b.hit.sum()),
            "depth_rel_max": float(rel.max()), "depth_frac_le_1e-4": float((rel <= 1e-4).mean()),
            "normal_max": float(nerr.max()), "normal_frac_le_1e-3": float((nerr <= 1e-3).mean()),
            "rgb_max": float(cerr.max()), "rgb_frac_le_1e-3": float((cerr <= 1e-3).mean())}

out = {}
pose = cameras.look_at_pose((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 256, 256)
ocam = oracle.camera_look_at((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 256, 256)
for name, field in (("random_init_16", grid.field_init(grid.GridConfig(resolution=16), seed=0)),
                    ("distilled_4", load_model(os.path.join(ROOT, "tests", "golden", "sphere_r4_distilled.knf")))):
    t0 = time.perf_counter(); ref = oracle.render(oracle.FieldTraceable(oracle_from_product(field)), ocam, oracle.MarchSettings()); cpu_s = time.perf_counter() - t0
    got = surface.render_frame(surface.FieldSurface(field), pose)
    out[name + "_256x256_gpu_vs_oracle"] = dict(compare(got, ref), oracle_seconds=cpu_s)
if "--full" in sys.argv:
    # the headline frame: 1920x1080, random-init 16^3, bench camera (about 2 minutes of oracle time)
    f16 = grid.field_init(grid.GridConfig(resolution=16), seed=0)
    pose = cameras.look_at_pose((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 1920, 1080)
    ocam = oracle.camera_look_at((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 1920, 1080)
    t0 = time.perf_counter(); ref = oracle.render(oracle.FieldTraceable(oracle_from_product(f16)), ocam, oracle.MarchSettings()); cpu_s = time.perf_counter() - t0
    got = surface.render_frame(surface.FieldSurface(f16), pose)
    out["random_init_16_1920x1080_gpu_vs_oracle"] = dict(compare(got, ref), oracle_seconds=cpu_s)
print(json.dumps(out, indent=1))
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "parity_r1.json"), "w"), indent=1)
