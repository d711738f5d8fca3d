#!/usr/bin/env python3
"""Generate the golden fixtures in this directory from the UNMODIFIED reference.

Run in the build container only (the reference is mounted read-only at
/root/reference and does not exist on the GPU box):

    KNF_THREADS=1 python tests/golden/make_golden.py

Everything written here is a small .npz / .knf / .json produced by importing
``kilofield`` from /root/reference/pkg/src and calling its public functions on
seeded inputs.  ``tests/test_oracle_golden.py`` pins ``oracle/`` to these files;
the ``-m gpu`` parity tests compare the CUDA path with them as well.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    if not os.path.isdir(REF_SRC):
        raise SystemExit("reference not mounted; golden fixtures can only be regenerated in the build container")
    os.environ.setdefault("KNF_THREADS", "1")
    sys.path.insert(0, REF_SRC)
    from kilofield import grid as G
    from kilofield import nn as NN
    from kilofield import pathtrace as PT
    from kilofield import surface as S
    from kilofield.cameras import look_at_pose, pixel_rays
    from kilofield.modelio import save_model
    from kilofield.teacher import AnalyticTeacher, PositionStripes, Sphere
    from kilofield.training import DistillConfig, distill_run

    meta = {"numpy": np.__version__, "generated_unix": int(time.time()), "files": {}}

    def put(name, **arrays):
        path = os.path.join(HERE, name)
        np.savez_compressed(path, **arrays)
        meta["files"][name] = {k: [list(np.shape(v)), str(np.asarray(v).dtype)] for k, v in arrays.items()}
        print(f"wrote {name}: {os.path.getsize(path) / 1024:.1f} KiB")

    # -- 1. encode + activations --------------------------------------------------------------
    rng = np.random.default_rng(101)
    x = rng.uniform(-1.2, 1.2, size=(4096, 3)).astype(np.float32)
    z = rng.normal(0, 3, size=8192).astype(np.float32)
    put(
        "encode_act.npz",
        x=x,
        enc6=NN.fourier_encode(x, 6),
        enc4=NN.fourier_encode(x, 4),
        z=z,
        softplus=NN.softplus(z),
        sigmoid=NN.sigmoid(z),
    )

    # -- 2. cell routing: uniform + adversarial (faces +- ulps, corners, outside) ---------------
    def adversarial_points(n_res, lo, hi, rng):
        faces = lo + (hi - lo) * np.arange(n_res + 1) / n_res
        vals = []
        for f in faces:
            f32 = np.float32(f)
            v = f32
            ring = [f32]
            for _ in range(2):
                v = np.nextafter(v, np.float32(np.inf), dtype=np.float32)
                ring.append(v)
            v = f32
            for _ in range(2):
                v = np.nextafter(v, np.float32(-np.inf), dtype=np.float32)
                ring.append(v)
            vals.extend(ring)
        vals = np.array(vals + [lo - 0.5, hi + 0.5, lo - 1e-7, hi + 1e-7, 0.0, -0.0], dtype=np.float32)
        pts = np.stack([rng.choice(vals, 6000), rng.choice(vals, 6000), rng.choice(vals, 6000)], axis=1)
        return pts.astype(np.float32)

    rng = np.random.default_rng(202)
    cells = {}
    for n_res in (1, 4, 16):
        cfg = G.GridConfig(resolution=n_res)
        pts = np.concatenate(
            [adversarial_points(n_res, -1.0, 1.0, rng), rng.uniform(-1.3, 1.3, size=(6000, 3)).astype(np.float32)]
        )
        cells[f"pts_{n_res}"] = pts
        cells[f"ids_{n_res}"] = G.cell_index_flat(cfg, pts).astype(np.int64)
    cfg_odd = G.GridConfig(resolution=5, bbox_min=(-0.7, -1.1, 0.2), bbox_max=(0.9, 0.4, 1.7))
    pts = rng.uniform(-1.5, 2.0, size=(8000, 3)).astype(np.float32)
    cells["pts_odd"] = pts
    cells["ids_odd"] = G.cell_index_flat(cfg_odd, pts).astype(np.int64)
    put("cells.npz", **cells)

    # -- 3. forward queries, 4^3 seed 7 (the reference tests' small_field) ----------------------
    f4 = G.field_init(G.GridConfig(resolution=4), seed=7)
    rng = np.random.default_rng(303)
    pts = rng.uniform(-1.1, 1.1, size=(3000, 3)).astype(np.float32)  # avg 47 per cell: per-cell-loop/padded boundary
    v = rng.normal(size=(3000, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    nrm = rng.normal(size=(3000, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    smp = G.sdf_query(f4, pts)
    rgb = G.color_query(f4, pts, v, nrm, smp.features)
    few = pts[:150]  # avg < 48 -> padded path
    smp_few = G.sdf_query(f4, few)
    put(
        "forward_r4_seed7.npz",
        pts=pts, v=v, n=nrm, value=smp.value, features=smp.features, rgb=rgb,
        value_few=smp_few.value, features_few=smp_few.features,
    )

    # -- 4. forward queries, A1's field and point stream (16^3 seed 42), first 20000 points -----
    f16 = G.field_init(G.GridConfig(resolution=16), seed=42)
    pts = np.random.default_rng(0).uniform(-1.1, 1.1, size=(100_000, 3)).astype(np.float32)
    smp = G.sdf_query(f16, pts)  # full batch, as test_acceptance.py:113-127 does
    put("forward_r16_seed42.npz", pts=pts[:20000], value=smp.value[:20000], features=smp.features[:20000])
    del f16

    # -- 5. FD normals incl. boundary / outside points ------------------------------------------
    rng = np.random.default_rng(404)
    p = rng.uniform(-0.999, 0.999, size=(600, 3))
    p[:100, 0] = 1.0
    p[100:200, 1] = -1.0
    p[200:260, 2] = 1.0 - 4e-4
    p[260:300] *= 1.3
    grad = G.grad_fd(f4, p)
    nb, ok = G.normal_batch(f4, p)
    put("fd_normals_r4.npz", pts=p, grad=grad, normals=nb, ok=ok)

    # -- 6. distilled (well-conditioned) 4^3 field ----------------------------------------------
    teacher = AnalyticTeacher(Sphere((0.0, 0.0, 0.0), 0.5), PositionStripes(0, 0.4, (0.9, 0.6, 0.2), (0.2, 0.3, 0.8)))
    fd = G.field_init(G.GridConfig(resolution=4), seed=0)
    t0 = time.perf_counter()
    hist = distill_run(fd, teacher, DistillConfig(steps=1500, seed=0))
    meta["distill"] = {"steps": 1500, "seconds": time.perf_counter() - t0, "final": hist[-1]}
    save_model(fd, os.path.join(HERE, "sphere_r4_distilled.knf"))
    print("wrote sphere_r4_distilled.knf")

    # -- 7. frames ------------------------------------------------------------------------------
    def frame_arrays(prefix, fb):
        return {f"{prefix}color": fb.color, f"{prefix}depth": fb.depth, f"{prefix}normal": fb.normal, f"{prefix}hit": fb.hit}

    pose96 = look_at_pose((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 96, 96)
    fb = S.render_frame(S.FieldSurface(fd), pose96, S.RenderSettings())
    o, d = pixel_rays(pose96)
    res = S.trace_and_shade(S.FieldSurface(fd), o, d, S.RenderSettings())  # one band = whole frame
    put("frame_distilled_96.npz", **frame_arrays("", fb), steps=res.steps, t=res.t, trace_hit=res.hit)

    pose_ss = look_at_pose((1.2, 0.9, 2.0), (0, 0, 0), (0, 1, 0), np.deg2rad(35), 40, 30)
    fb = S.render_frame(S.FieldSurface(fd), pose_ss, S.RenderSettings(), background=(0.2, 0.4, 0.6), supersample=2, tile_rows=8)
    put("frame_distilled_ss2.npz", **frame_arrays("", fb))

    f0 = G.field_init(G.GridConfig(resolution=16), seed=0)
    pose64 = look_at_pose((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 64, 64)
    fb = S.render_frame(S.FieldSurface(f0), pose64, S.RenderSettings())
    o, d = pixel_rays(pose64)
    res = S.trace_and_shade(S.FieldSurface(f0), o, d, S.RenderSettings())
    put("frame_random16_64.npz", **frame_arrays("", fb), steps=res.steps, t=res.t, trace_hit=res.hit)
    del f0

    # -- 8. counter RNG -------------------------------------------------------------------------
    rng = np.random.default_rng(505)
    pix = rng.integers(0, 3840 * 2160, size=512).astype(np.uint64)
    smp_i = rng.integers(0, 64, size=512)
    slot = rng.integers(0, 30, size=512)
    slot[:64] = PT._PRIMARY_SLOT + (np.arange(64) % 2)
    us = {}
    for seed in (0, 12345, 2**63 + 17):
        us[f"u_{seed}"] = np.array([PT.Rng(seed).uniform(pix[i], int(smp_i[i]), int(slot[i])) for i in range(512)])
    put("rng.npz", pixel=pix, sample=smp_i, slot=slot, **us)

    # -- 9. path tracing ------------------------------------------------------------------------
    floor = PT.QuadObj((-3, -1.0, -3), (6, 0, 0), (0, 0, 6), PT.Lambertian((0.7, 0.7, 0.7)))
    # edge order chosen so the quad normal points up (+y): u x v = (6,0,0)x(0,0,6) = (0,-36,0) -> flipped at shading
    lamp = PT.SphereObj((1.5, 1.2, 0.5), 0.4, PT.Emissive((6.0, 5.0, 4.0)))
    crate = PT.BoxObj((-1.9, -1.0, -0.6), (-1.2, -0.3, 0.1), PT.Lambertian((0.2, 0.6, 0.3)))
    neural = PT.NeuralObject(S.FieldSurface(fd), translation=(0.1, -0.2, 0.0), rotation=np.eye(3), scale=1.0)
    scene = PT.Scene([floor, lamp, crate, neural], PT.ConstantEnv((0.6, 0.7, 0.9)))
    pose_pt = look_at_pose((0.5, 0.8, 3.2), (0, -0.2, 0), (0, 1, 0), np.deg2rad(45), 32, 24)
    out = PT.render_pathtraced(scene, pose_pt, spp=2, seed=7, max_bounces=8)
    put("pathtrace_scene.npz", hdr=out.hdr, ldr=out.ldr)
    analytic = PT.Scene([floor, lamp, crate], PT.ConstantEnv((0.6, 0.7, 0.9)))
    out = PT.render_pathtraced(analytic, pose_pt, spp=3, seed=11, max_bounces=8, sample_offset=2)
    put("pathtrace_analytic.npz", hdr=out.hdr, ldr=out.ldr)

    # -- 10. volume-render forward (training._volume_forward), distilled field -------------------------------
    from kilofield import training as T

    rng = np.random.default_rng(606)
    pose_v = look_at_pose((0.3, 0.5, 2.4), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 64, 64)
    pix = np.stack([rng.integers(0, 64, 400), rng.integers(0, 64, 400)], axis=1)
    vo, vd = pixel_rays(pose_v, pix)
    vo[:20] += [3.0, 0.0, 0.0]  # a few rays that miss the box
    jit = rng.uniform(size=(400, 24))
    col, _ = T._volume_forward(fd, vo, vd, 24, jit, (1.0, 1.0, 1.0))
    col_mid, _ = T._volume_forward(fd, vo, vd, 16, None, (0.2, 0.4, 0.6))
    put("volume_forward.npz", origins=vo, dirs=vd, jitter=jit, colors=col, colors_nojitter=col_mid, s=np.float64(fd.s))

    with open(os.path.join(HERE, "golden_meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1, default=float)
    print("done")


if __name__ == "__main__":
    main()
