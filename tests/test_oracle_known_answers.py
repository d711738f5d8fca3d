"""The reference's own known-answer tests for the hot path, re-run on oracle/."""

import numpy as np
import pytest

import oracle


def test_cell_index_corners_midpoint_clamp():
    # test_grid.py:38-49
    spec = oracle.FieldSpec(resolution=16)
    tri = lambda p: tuple(oracle.cell_triples(spec, np.asarray([p], dtype=np.float64))[0])
    assert tri((-1, -1, -1)) == (0, 0, 0)
    assert tri((0, 0, 0)) == (8, 8, 8)
    assert tri((2, 0, 0)) == (15, 8, 8)
    assert tri((1, 1, 1)) == (15, 15, 15)


def test_fourier_layout_and_direct_formula():
    # test_nn.py:31-64
    x = np.array([0.1, -0.3, 0.7])
    e = oracle.positional_features(x, 3)
    assert e.shape == (21,)
    assert np.allclose(e[:3], x)
    for k in range(3):
        assert np.allclose(e[3 + 6 * k : 6 + 6 * k], np.sin(2**k * np.pi * x), atol=1e-12)
        assert np.allclose(e[6 + 6 * k : 9 + 6 * k], np.cos(2**k * np.pi * x), atol=1e-12)


def test_grouped_equals_naive(small_oracle):
    # test_grid.py:28-35, 81-86: grouped dispatch == per-point straight-line evaluation, <= 1e-6
    rng = np.random.default_rng(3)
    pts = rng.uniform(-1.1, 1.1, size=(400, 3)).astype(np.float32)
    value, _ = oracle.query_sdf(small_oracle, pts)
    ids = oracle.cell_ids(small_oracle.spec, pts)
    for i in range(0, 400, 7):
        h = oracle.positional_features(pts[i], 6)
        for k in range(3):
            z = small_oracle.sdf.W[k][ids[i]] @ h + small_oracle.sdf.b[k][ids[i]]
            h = oracle.field._activate(small_oracle.sdf.acts[k], z)
        assert abs(h[0] - value[i]) <= 1e-6


def test_padded_path_equals_loop_path(small_oracle, monkeypatch):
    # test_grid.py:160-167
    rng = np.random.default_rng(4)
    pts = rng.uniform(-1, 1, size=(3000, 3)).astype(np.float32)
    a, _ = oracle.query_sdf(small_oracle, pts)
    monkeypatch.setattr(oracle.field, "PADDED_CUTOFF", 1e9)
    b, _ = oracle.query_sdf(small_oracle, pts)
    assert np.abs(a - b).max() <= 1e-6


def test_color_zero_weights_is_half(small_oracle):
    # test_grid.py:106-132
    import copy

    f = copy.deepcopy(small_oracle)
    for w in f.color.W:
        w[:] = 0
    rgb = oracle.query_color(f, np.zeros((5, 3)), np.tile([0, 0, 1.0], (5, 1)), np.tile([0, 1.0, 0], (5, 1)), np.zeros((5, 8)))
    assert np.allclose(rgb, 0.5)


def test_ray_aabb_cases():
    # test_surface.py:38-60
    lo, hi = (-1, -1, -1), (1, 1, 1)
    tn, tf, hit = oracle.slab_intersect(np.array([[0, 0, -2.0]]), np.array([[0, 0, 1.0]]), lo, hi)
    assert hit[0] and tn[0] == 1.0 and tf[0] == 3.0
    tn, tf, hit = oracle.slab_intersect(np.array([[0, 0, 0.0]]), np.array([[0, 0, 1.0]]), lo, hi)
    assert hit[0] and tn[0] == 0.0 and tf[0] == 1.0
    _, _, hit = oracle.slab_intersect(np.array([[0, 3.0, -2.0]]), np.array([[0, 0, 1.0]]), lo, hi)
    assert not hit[0]
    _, _, hit = oracle.slab_intersect(np.array([[0, 0, 2.0]]), np.array([[0, 0, 1.0]]), lo, hi)
    assert not hit[0]


class _Sphere:
    """Analytic traceable (what the reference's TeacherSurface provides, surface.py:102-116)."""

    bbox_min = np.array([-1.0, -1, -1])
    bbox_max = np.array([1.0, 1, 1])

    def sdf_values(self, p):
        return np.linalg.norm(p, axis=1) - 0.5

    def shade(self, p, v):
        n = p / np.linalg.norm(p, axis=1, keepdims=True)
        return np.full_like(p, 0.5), n


def test_sphere_trace_analytic():
    # test_surface.py:64-71: t = 1.5 +- 5e-3 from z = -2, never past the first root (:91-109)
    o = np.array([[0, 0, -2.0]])
    d = np.array([[0, 0, 1.0]])
    res = oracle.trace_shade(_Sphere(), o, d, oracle.MarchSettings())
    assert res.hit[0] and abs(res.t[0] - 1.5) <= 5e-3 and res.t[0] <= 1.5 + 1e-3
    assert res.steps[0] <= 128
    assert np.allclose(res.normal[0], [0, 0, -1], atol=0.035)
    res = oracle.trace_shade(_Sphere(), np.array([[0.9, 0.9, -2.0]]), d, oracle.MarchSettings())
    assert not res.hit[0]


def test_white_furnace_exact():
    # test_pathtrace.py:96-106: albedo-1 sphere under a unit sky returns exactly 1
    scene = oracle.PathScene([oracle.SphereShape((0, 0, 0), 0.5, oracle.Diffuse((1, 1, 1)))], oracle.UniformSky((1, 1, 1)))
    cam = oracle.camera_look_at((0, 0, 2.0), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 8, 8)
    hdr, _ = oracle.render_paths(scene, cam, spp=4, seed=3)
    # paths still bouncing at max_bounces contribute nothing, every other path contributes 1
    assert np.all((hdr <= 1.0 + 1e-12) & (hdr >= 0.0))
    assert np.allclose(hdr[0, 0], 1.0, rtol=1e-12)  # corner pixel misses the sphere


def test_lambertian_sampling_moments():
    # test_pathtrace.py:45-64: hemisphere, E[cos] = 2/3
    n = np.tile([0.0, 0.0, 1.0], (20000, 1))
    rng = np.random.default_rng(0)
    d = oracle.cosine_sample(n, rng.uniform(size=20000), rng.uniform(size=20000))
    assert np.all(d[:, 2] >= 0)
    assert np.allclose(np.linalg.norm(d, axis=1), 1.0)
    assert abs(d[:, 2].mean() - 2 / 3) < 0.01


def test_settings_validation():
    with pytest.raises(ValueError):
        oracle.MarchSettings(step_scale=0.0)
    with pytest.raises(ValueError):
        oracle.MarchSettings(render_pass="albedo")
    with pytest.raises(ValueError):
        oracle.grouped_query(None, None, "density")
