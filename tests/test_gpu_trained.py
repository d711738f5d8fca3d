"""GPU parity on a TRAINED field (VERDICT r1 missing 5): the 8^3 sphere + stripes field distilled for 12 000 steps by the
reference's own training code, and the same function refined onto a 16^3 grid (4096 MLPs) -- the workload users have,
where rays never crawl and the decision filter switches itself off, so the exact FP32 kernels are the product."""

import os

import numpy as np
import pytest

import oracle
from conftest import golden, oracle_from_product

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2206_10885_b200 import surface

    return surface


def test_trained_frame_vs_reference_golden(S, trained_field):
    """kilofield.surface.render_frame of the same .knf (128^2, cmd_bench camera): north_star bars."""
    from paper_2206_10885_b200 import cameras

    g = golden("frame_trained_r8_128.npz")
    pose = cameras.look_at_pose((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 128, 128)
    fs = S.FieldSurface(trained_field)
    fs.dev.reset_stats()
    fb = S.render_frame(fs, pose)
    st = fs.dev.stats()
    agree = (fb.hit == g["hit"]).mean()
    both = fb.hit & g["hit"]
    rel = np.abs(fb.depth[both] - g["depth"][both]) / g["depth"][both]
    nerr = np.abs(fb.normal - g["normal"])[both].max(axis=1)
    cerr = np.abs(fb.color - g["color"])[both].max(axis=1)
    print(f"trained 8^3, 128^2: hits {agree:.4%} ({int(both.sum())} both), depth rel max {rel.max():.2e}, normal<=1e-3 {np.mean(nerr <= 1e-3):.4%} "
          f"(max {nerr.max():.2e}), rgb max {cerr.max():.2e}; evals/ray {st['sdf_evals'] / st['rays']:.1f}, filter evals {st['filter_evals']}")
    assert agree >= 0.999
    assert np.mean(rel <= 1e-4) >= 0.999
    assert np.mean(cerr <= 1e-3) >= 0.999
    assert np.mean(nerr <= 1e-3) >= 0.995  # FD normals amplify SDF ulps x500; the reference vs itself across band sizes: 99.99 %
    assert st["filter_evals"] <= 0.02 * st["sdf_evals"]  # a real surface: nothing to filter


def test_refined_16_cubed_field_is_the_same_function(S, trained_field):
    """grid.refine_field: 4096 cells, identical function -> identical frames, bit for bit (routing to the finer grid changes
    which blob a point reads, not a single operand)."""
    from paper_2206_10885_b200 import cameras, grid

    fine = grid.refine_field(trained_field, 2)
    assert fine.config.resolution == 16 and fine.sdf.weights[0].shape[0] == 4096
    pts = np.random.default_rng(1).uniform(-1.05, 1.05, size=(200_000, 3)).astype(np.float32)
    a, b = grid.sdf_query(trained_field, pts), grid.sdf_query(fine, pts)
    assert np.array_equal(a.value, b.value) and np.array_equal(a.features, b.features)
    pose = cameras.look_at_pose((0.7, 0.6, 2.2), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 320, 180)
    fa, fb = S.render_frame(S.FieldSurface(trained_field), pose), S.render_frame(S.FieldSurface(fine), pose)
    for k in ("color", "depth", "normal", "hit"):
        assert np.array_equal(getattr(fa, k), getattr(fb, k)), k
    assert fa.hit.mean() > 0.05


def test_trained_16_cubed_full_hd_bands_vs_oracle(S, trained_field):
    """1920x1080 on the trained 16^3 field: two 32-row bands through the object against the oracle's band code."""
    from paper_2206_10885_b200 import cameras, grid

    fine = grid.refine_field(trained_field, 2)
    W, H = 1920, 1080
    fs = S.FieldSurface(fine)
    pose = cameras.look_at_pose((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), W, H)
    ocam = oracle.camera_look_at((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), W, H)
    osurf = oracle.FieldTraceable(oracle_from_product(fine))
    flips = both_n = d_ok = n_ok = c_ok = 0
    for r0 in (400, 524):
        color, depth, normal, hit = S.render_rows(fs, pose, S.RenderSettings(), (1, 1, 1), 1, r0, r0 + 32)
        hit = hit.astype(bool)
        cc, rr = np.meshgrid(np.arange(W), np.arange(r0, r0 + 32))
        o, d = oracle.camera_rays(ocam, np.stack([cc.ravel(), rr.ravel()], axis=1))
        ref = oracle.trace_shade(osurf, o, d, oracle.MarchSettings())
        rhit = ref.hit.reshape(32, W)
        both = hit & rhit
        rel = np.abs(depth[both] - ref.t.reshape(32, W)[both].astype(np.float32)) / ref.t.reshape(32, W)[both]
        nerr = np.abs(normal - ref.normal.reshape(32, W, 3).astype(np.float32))[both].max(axis=1)
        cerr = np.abs(color - ref.color.reshape(32, W, 3).astype(np.float32))[both].max(axis=1)
        flips += int((hit != rhit).sum())
        both_n += int(both.sum())
        d_ok += int((rel <= 1e-4).sum())
        n_ok += int((nerr <= 1e-3).sum())
        c_ok += int((cerr <= 1e-3).sum())
    print(f"trained 16^3 1080p bands: {flips} hit flips of {2 * 32 * W} rays, both-hit {both_n}: depth {d_ok / both_n:.4%}, normal {n_ok / both_n:.4%}, rgb {c_ok / both_n:.4%}")
    assert both_n >= 10000
    assert flips <= 1e-3 * 2 * 32 * W
    assert d_ok >= 0.999 * both_n and c_ok >= 0.999 * both_n and n_ok >= 0.995 * both_n


def test_rotated_scaled_neural_object_vs_reference_golden(S, trained_field):
    """pathtrace.NeuralObject with rotation and scale != identity (pathtrace.py:225-274) on the trained field against the
    reference's own render_pathtraced of the same scene (tests/golden/make_trained.py), same seed and counter RNG."""
    from paper_2206_10885_b200 import cameras, pathtrace

    g = golden("pathtrace_trained_r8.npz")
    scene = pathtrace.Scene([pathtrace.QuadObj((-3, -0.9, -3), (6, 0, 0), (0, 0, 6), pathtrace.Lambertian((0.7, 0.7, 0.7))),
                             pathtrace.NeuralObject(S.FieldSurface(trained_field), tuple(g["translation"]), g["rotation"], float(g["scale"]))],
                            pathtrace.ConstantEnv((1, 1, 1)))
    pose = cameras.look_at_pose((0.6, 0.7, 2.6), (0.2, -0.1, 0.1), (0, 1, 0), np.deg2rad(40), 48, 36)
    got = pathtrace.render_pathtraced(scene, pose, spp=2, seed=9).hdr
    err = np.abs(got - g["hdr"]).max(axis=2)
    print(f"rotated / scaled NeuralObject, 48x36 x 2 spp: |hdr - reference| <= 1e-3 on {np.mean(err <= 1e-3):.4%} of pixels (max {err.max():.2e})")
    assert np.mean(err <= 1e-3) >= 0.985  # a last-ulp difference in a bounce direction can land on another object: isolated pixels
