"""Trained-field fixture: distil the sphere + stripes teacher into an 8^3 field with the UNMODIFIED reference's own
training code (kilofield.training.distill_run, the recipe of pkg/tests/test_acceptance.py:60-75: 12 000 steps, lr step
size 1000, seed 0) and save it as tests/golden/sphere_stripes_r8_distilled.knf, plus reference renders of it:

  frame_trained_r8_128.npz    kilofield.surface.render_frame, 128 x 128, cmd_bench camera
  pathtrace_trained_r8.npz    kilofield.pathtrace.render_pathtraced of a floor quad + NeuralObject with rotation and
                              scale != identity (pathtrace.py:225-274), 48 x 36, 2 spp

Run where /root/reference exists (the build container):  python tests/golden/make_trained.py
A 16^3-cell trained workload is derived from the same file at load time (tests/conftest.py refine_field: every child
cell inherits its parent's networks, so the field is the same function on a 4096-cell grid) -- an 84 MB 16^3 .knf is
not committed."""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from kilofield import grid as G  # noqa: E402
from kilofield import pathtrace as PT  # noqa: E402
from kilofield import surface as S  # noqa: E402
from kilofield.cameras import look_at_pose  # noqa: E402
from kilofield.modelio import save_model  # noqa: E402
from kilofield.teacher import AnalyticTeacher, PositionStripes, Sphere  # noqa: E402
from kilofield.training import DistillConfig, distill_run  # noqa: E402


def rot(axis, angle):
    axis = np.asarray(axis, dtype=np.float64) / np.linalg.norm(axis)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + np.sin(angle) * K + (1 - np.cos(angle)) * (K @ K)


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 12000
    teacher = AnalyticTeacher(Sphere((0.0, 0.0, 0.0), 0.5), PositionStripes(0, 0.4, (0.9, 0.6, 0.2), (0.2, 0.3, 0.8)))
    field = G.field_init(G.GridConfig(resolution=8), seed=0)
    t0 = time.perf_counter()
    hist = distill_run(field, teacher, DistillConfig(steps=steps, lr_step_size=1000, seed=0), log_every=1000)
    print(f"distilled {steps} steps in {time.perf_counter() - t0:.0f} s, final {hist[-1]}", flush=True)
    save_model(field, os.path.join(HERE, "sphere_stripes_r8_distilled.knf"))
    surf = S.FieldSurface(field)
    pose = look_at_pose((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 128, 128)
    fb = S.render_frame(surf, pose, S.RenderSettings())
    np.savez_compressed(os.path.join(HERE, "frame_trained_r8_128.npz"), color=fb.color, depth=fb.depth, normal=fb.normal, hit=fb.hit)
    R, T, scale = rot((0.3, 1.0, 0.2), 0.7), (0.25, -0.1, 0.15), 0.8
    scene = PT.Scene([PT.QuadObj((-3, -0.9, -3), (6, 0, 0), (0, 0, 6), PT.Lambertian((0.7, 0.7, 0.7))), PT.NeuralObject(surf, T, R, scale)],
                     PT.ConstantEnv((1, 1, 1)))
    ppose = look_at_pose((0.6, 0.7, 2.6), (0.2, -0.1, 0.1), (0, 1, 0), np.deg2rad(40), 48, 36)
    res = PT.render_pathtraced(scene, ppose, spp=2, seed=9)
    np.savez_compressed(os.path.join(HERE, "pathtrace_trained_r8.npz"), hdr=res.hdr, rotation=R, translation=np.asarray(T), scale=scale)
    print("hit fraction", float(fb.hit.mean()), "done", flush=True)


if __name__ == "__main__":
    main()
