#!/usr/bin/env python3
"""Measures how far the UNMODIFIED reference disagrees with ITSELF when only its band size changes
(OpenBLAS picks different sgemm kernels for different per-cell batch sizes, so last-ulp SDF values
depend on how many rays share a cell).  This is the parity noise floor quoted in DESIGN.md.
Build container only: KNF_THREADS=1 python tests/golden/measure_reference_noise.py"""
import json, os, sys
import numpy as np
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("KNF_THREADS", "1")
from kilofield import grid as G, surface as S
from kilofield.cameras import look_at_pose
from kilofield.modelio import load_model

HERE = os.path.dirname(os.path.abspath(__file__))
out = {}


def compare(a, b):
    both = a.hit & b.hit
    return {
        "hit_agreement": float((a.hit == b.hit).mean()), "hits_a": int(a.hit.sum()), "hits_b": int(b.hit.sum()),
        "depth_rel_max": float((np.abs(a.depth[both] - b.depth[both]) / a.depth[both]).max()) if both.any() else 0.0,
        "depth_rel_frac_le_1e-4": float(((np.abs(a.depth[both] - b.depth[both]) / a.depth[both]) <= 1e-4).mean()) if both.any() else 1.0,
        "normal_max": float(np.abs(a.normal - b.normal)[both].max()) if both.any() else 0.0,
        "normal_frac_le_1e-3": float((np.abs(a.normal - b.normal)[both].max(axis=1) <= 1e-3).mean()) if both.any() else 1.0,
        "rgb_max": float(np.abs(a.color - b.color)[both].max()) if both.any() else 0.0,
        "rgb_frac_le_1e-3": float((np.abs(a.color - b.color)[both].max(axis=1) <= 1e-3).mean()) if both.any() else 1.0,
    }


pose = look_at_pose((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 256, 256)
f0 = G.field_init(G.GridConfig(resolution=16), seed=0)
a = S.render_frame(S.FieldSurface(f0), pose, S.RenderSettings(), tile_rows=32)
b = S.render_frame(S.FieldSurface(f0), pose, S.RenderSettings(), tile_rows=256)
out["random_init_16_256x256_tile32_vs_tile256"] = compare(a, b)
fd = load_model(os.path.join(HERE, "sphere_r4_distilled.knf"))
a = S.render_frame(S.FieldSurface(fd), pose, S.RenderSettings(), tile_rows=32)
b = S.render_frame(S.FieldSurface(fd), pose, S.RenderSettings(), tile_rows=256)
out["distilled_4_256x256_tile32_vs_tile256"] = compare(a, b)
json.dump(out, open(os.path.join(HERE, "reference_noise.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
