"""GPU parity, part 2: ray generation, slabs, the wavefront sphere trace, shading and frames
(BASELINE configs 1-3 in miniature), through the C-ABI."""

import numpy as np
import pytest

import oracle
from conftest import golden, oracle_from_product

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2206_10885_b200 import surface

    return surface


@pytest.fixture(scope="module")
def cams():
    from paper_2206_10885_b200 import cameras

    return cameras


def test_pixel_rays_bit_exact(cams):
    for (w, h, pos) in [(64, 48, (1.2, 0.9, 2.0)), (7, 5, (0, 0, 2.5)), (33, 65, (-2, 0.3, 0.4))]:
        pose = cams.look_at_pose(pos, (0, 0, 0), (0, 1, 0), np.deg2rad(35), w, h)
        ocam = oracle.camera_look_at(pos, (0, 0, 0), (0, 1, 0), np.deg2rad(35), w, h)
        assert np.array_equal(pose.rotation, ocam.rotation)
        o, d = cams.pixel_rays(pose)
        oo, od = oracle.camera_rays(ocam)
        assert np.array_equal(o, oo) and np.array_equal(d, od)
    rng = np.random.default_rng(0)
    pix = np.stack([rng.integers(0, 33, 500), rng.integers(0, 65, 500)], axis=1)
    jit = rng.uniform(size=(500, 2))
    o, d = cams.pixel_rays(pose, pix, jit)
    oo, od = oracle.camera_rays(ocam, pix, jit)
    assert np.array_equal(d, od)


def test_ray_aabb(S):
    rng = np.random.default_rng(1)
    o = rng.uniform(-3, 3, size=(20000, 3))
    d = rng.normal(size=(20000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d[:500, 0] = 0.0  # axis-parallel rays
    d[200:700, 1] = 0.0
    o[:100, 0] = 1.0  # on the slab boundary
    tn, tf, hit = S.ray_aabb_batch(o, d, (-1, -1, -1), (1, 1, 1))
    otn, otf, ohit = oracle.slab_intersect(o, d, (-1, -1, -1), (1, 1, 1))
    assert np.array_equal(hit, ohit)
    assert np.array_equal(tn, otn) and np.array_equal(tf, otf)
    assert S.ray_aabb(S.Ray((0, 0, -2), (0, 0, 1)), (-1, -1, -1), (1, 1, 1)) == (1.0, 3.0)
    assert S.ray_aabb(S.Ray((0, 3, -2), (0, 0, 1)), (-1, -1, -1), (1, 1, 1)) is None


def _rays(w, h, pos=(0, 0, 2.5), fov=40):
    cam = oracle.camera_look_at(pos, (0, 0, 0), (0, 1, 0), np.deg2rad(fov), w, h)
    o, d = oracle.camera_rays(cam)
    tn, tf, inside = oracle.slab_intersect(o, d, (-1, -1, -1), (1, 1, 1))
    return o, d, np.where(inside, tn, 1.0), np.where(inside, tf, 0.0)


def test_lockstep_march_random_init(S):
    """SURVEY 8c protocol (3): the reference's own march loop (oracle.march) driven by GPU SDF
    evaluations, compared round by round with the pure-CPU march.  While both marches hold the
    same ray set the per-round distances must agree to forward tolerance; this proves the
    kernels independent of the chaos that a random-init SDF adds to end-to-end frames."""
    from paper_2206_10885_b200 import grid

    field = grid.field_init(grid.GridConfig(resolution=16), seed=0)
    ofield = oracle_from_product(field)
    o, d, tn, tf = _rays(40, 40)
    log_cpu = []
    cfg = oracle.MarchSettings(max_steps=32)
    oracle.march(oracle.FieldTraceable(ofield), o, d, tn, tf, cfg, trace_log=log_cpu)
    gpu = S.FieldSurface(field)
    compared, worst, flips = 0, 0.0, 0
    for rays, t, d_cpu in log_cpu:
        # same fp64 point arithmetic as surface.py:184, evaluated by the GPU at the CPU's t
        d_gpu = gpu.sdf_values(o[rays] + t[:, None] * d[rays])
        worst = max(worst, float(np.abs(d_gpu - d_cpu).max()))
        flips += int(((np.abs(d_gpu) <= cfg.eps_hit) != (np.abs(d_cpu) <= cfg.eps_hit)).sum())
        compared += len(rays)
    print(f"lock-step: {compared} evaluations over {len(log_cpu)} rounds, worst |d_gpu - d_cpu| = {worst:.2e}, "
          f"convergence-decision flips {flips}")
    assert compared >= 30000
    assert worst <= 5e-6
    assert flips <= max(2, compared // 20000)


def test_march_distilled_matches_oracle(S, distilled_field, distilled_oracle):
    o, d, tn, tf = _rays(96, 96)
    res = S.march_rays(S.FieldSurface(distilled_field), o, d, tn, tf, S.RenderSettings())
    ref = oracle.march(oracle.FieldTraceable(distilled_oracle), o, d, tn, tf, oracle.MarchSettings())
    agree = (res.hit == ref.hit).mean()
    both = res.hit & ref.hit
    drel = np.abs(res.t[both] - ref.t[both]) / ref.t[both]
    print(f"march distilled: hit agreement {agree:.4%}, depth rel max {drel.max():.2e}, steps equal {(res.steps == ref.steps).mean():.4%}")
    assert agree >= 0.999
    # A ray whose |d| lands within ~1e-6 of eps_hit converges one step earlier/later on the GPU than
    # on the CPU and then refines from a different bracket (~1e-4 of the reference's rays, DESIGN.md
    # Numerics); everything else must sit inside the 1e-4 bar, and the outliers inside one step.
    assert (drel <= 1e-4).mean() >= 0.999 and drel.max() <= 2e-3
    assert (res.steps == ref.steps).mean() >= 0.995
    perr = np.abs(res.position[both] - ref.position[both]).max(axis=1)
    assert (perr <= 1e-4).mean() >= 0.999
    assert np.all(res.steps <= 128)
    # misses keep t = 0 and position = origin, like the reference
    assert np.all(res.t[~res.hit] == 0) and np.array_equal(res.position[~res.hit], o[~res.hit])


def test_frame_distilled_vs_golden(S, cams, distilled_field):
    """End-to-end FrameBuffers vs the reference's render of the same field + camera
    (north_star bar: hit >= 99.9 %, depth <= 1e-4 rel, normal & RGB <= 1e-3)."""
    g = golden("frame_distilled_96.npz")
    pose = cams.look_at_pose((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 96, 96)
    fb = S.render_frame(S.FieldSurface(distilled_field), pose, S.RenderSettings())
    assert fb.color.dtype == np.float32 and fb.color.shape == (96, 96, 3)
    assert fb.depth.dtype == np.float32 and fb.hit.dtype == bool
    agree = (fb.hit == g["hit"]).mean()
    both = fb.hit & g["hit"]
    drel = (np.abs(fb.depth[both] - g["depth"][both]) / g["depth"][both]).max()
    nerr = np.abs(fb.normal - g["normal"])[both]
    cerr = np.abs(fb.color - g["color"])[both]
    print(f"frame distilled 96^2: hit {agree:.4%}, depth rel {drel:.2e}, normal max {nerr.max():.2e} "
          f"(>1e-3 on {(nerr.max(axis=1) > 1e-3).mean():.3%}), rgb max {cerr.max():.2e}")
    drel_all = np.abs(fb.depth[both] - g["depth"][both]) / g["depth"][both]
    assert agree >= 0.999
    assert (drel_all <= 1e-4).mean() >= 0.999 and drel <= 2e-3
    assert (cerr.max(axis=1) <= 1e-3).mean() >= 0.999
    # FD normals amplify SDF ulps by 500/|g|: the reference disagrees with ITSELF by 1.0e-3 between
    # tile_rows=32 and 128 on this field (DESIGN.md Numerics).  Pixels whose depth is a convergence-
    # flip outlier (see test_march_distilled_matches_oracle) carry a different hit point; the rest
    # must be inside 2e-3, and 99.9 % of all both-hit pixels inside the 1e-3 bar.
    same_point = drel_all <= 1e-4
    assert nerr[same_point].max() <= 2e-3 and (nerr.max(axis=1) <= 1e-3).mean() >= 0.999
    assert np.all(np.isinf(fb.depth[~fb.hit])) and np.all(fb.normal[~fb.hit] == 0)
    assert np.all(fb.color[~fb.hit] == 1.0)
    nn = np.linalg.norm(fb.normal[fb.hit], axis=1)
    assert np.allclose(nn, 1.0, atol=1e-6)


def test_frame_supersampled_vs_golden(S, cams, distilled_field):
    g = golden("frame_distilled_ss2.npz")
    pose = cams.look_at_pose((1.2, 0.9, 2.0), (0, 0, 0), (0, 1, 0), np.deg2rad(35), 40, 30)
    fb = S.render_frame(S.FieldSurface(distilled_field), pose, S.RenderSettings(), background=(0.2, 0.4, 0.6), supersample=2)
    agree = (fb.hit == g["hit"]).mean()
    both = fb.hit & g["hit"]
    print(f"frame ss2: hit {agree:.4%}, rgb max {np.abs(fb.color - g['color'])[both].max():.2e}")
    assert agree >= 0.995
    assert ((np.abs(fb.depth[both] - g["depth"][both]) / g["depth"][both]) <= 1e-4).mean() >= 0.995
    assert (np.abs(fb.color - g["color"])[both].max(axis=1) <= 2e-3).mean() >= 0.995
    bgpix = ~fb.hit & ~g["hit"]
    assert np.abs(fb.color[bgpix] - g["color"][bgpix]).max() <= 1e-6


def test_frame_banding_and_abort(S, cams, distilled_field):
    pose = cams.look_at_pose((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 50, 37)
    fs = S.FieldSurface(distilled_field)
    whole = S.render_frame(fs, pose)
    polls = []
    banded = S.render_frame(fs, pose, tile_rows=8, abort_check=lambda: polls.append(1) and False)
    assert len(polls) == 5
    for k in ("color", "depth", "normal", "hit"):
        assert np.array_equal(getattr(whole, k), getattr(banded, k)), k  # banding-invariant, like thread count in the reference
    with pytest.raises(S.RenderAborted):
        S.render_frame(fs, pose, tile_rows=8, abort_check=lambda: True)
    with pytest.raises(ValueError):
        S.render_frame(fs, pose, supersample=0)
    img = S.pass_image(whole, "normal")
    assert img.shape == (37, 50, 3) and np.all(img[~whole.hit] == 0)
    with pytest.raises(ValueError):
        S.pass_image(whole, "albedo")


def test_frame_random_init_reported(S, cams):
    """BASELINE config 1 in miniature (64^2).  A random-init SDF makes t <- t + 0.8 d an expanding map, so
    1-ulp SDF differences flip hit decisions (the reference flips against itself, DESIGN.md
    Numerics).  Parity here is statistical; the strict bar is carried by the distilled field and
    by the lock-step test above."""
    from paper_2206_10885_b200 import grid

    g = golden("frame_random16_64.npz")
    field = grid.field_init(grid.GridConfig(resolution=16), seed=0)
    pose = cams.look_at_pose((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 64, 64)
    fb = S.render_frame(S.FieldSurface(field), pose)
    agree = (fb.hit == g["hit"]).mean()
    both = fb.hit & g["hit"]
    print(f"frame random-init 64^2: hit agreement {agree:.4%}; hits gpu {fb.hit.sum()} ref {g['hit'].sum()}; both {both.sum()}")
    assert agree >= 0.985
    assert abs(int(fb.hit.sum()) - int(g["hit"].sum())) <= 0.25 * int(g["hit"].sum()) + 5


def test_shade_matches_oracle(S, distilled_field, distilled_oracle):
    o, d, tn, tf = _rays(64, 64)
    ref = oracle.march(oracle.FieldTraceable(distilled_oracle), o, d, tn, tf, oracle.MarchSettings())
    pts, dirs = ref.position[ref.hit], d[ref.hit]
    col, nrm = S.FieldSurface(distilled_field).shade(pts, dirs)
    ocol, onrm = oracle.FieldTraceable(distilled_oracle).shade(pts, dirs)
    print(f"shade: normal max {np.abs(nrm - onrm).max():.2e}, rgb max {np.abs(col - ocol).max():.2e} on {len(pts)} hits")
    assert np.abs(col - ocol).max() <= 1e-3
    assert (np.abs(nrm - onrm).max(axis=1) <= 1e-3).mean() >= 0.999


def test_sphere_trace_single_ray(S, distilled_field, distilled_oracle):
    fs = S.FieldSurface(distilled_field)
    # (a ray exactly on the x = y = 0 cell faces overshoots the seam of this briefly-distilled field
    # in the reference too, so aim slightly off-axis)
    o, d = np.array([[0.13, 0.21, -2.0]]), np.array([[0.0, 0.0, 1.0]])
    ref = oracle.march(oracle.FieldTraceable(distilled_oracle), o, d, np.array([1.0]), np.array([3.0]), oracle.MarchSettings())
    assert ref.hit[0]
    hit = S.sphere_trace(fs, S.Ray(o[0], d[0]), 1.0, 3.0, S.RenderSettings())
    assert hit is not None and abs(hit.t - ref.t[0]) <= 1e-4 and hit.steps_taken == ref.steps[0]
    assert abs(hit.t - (2.0 - np.sqrt(0.25 - 0.13**2 - 0.21**2))) <= 3e-2
    assert abs(np.linalg.norm(hit.normal) - 1) <= 1e-9 and hit.normal[2] < -0.5  # 1500-step distillation: rough sphere
    assert np.all((hit.color >= 0) & (hit.color <= 1))
    # a grazing ray: whatever the oracle decides, the GPU decides the same
    o, d = np.array([[0.95, 0.95, -2.0]]), np.array([[0.0, 0.0, 1.0]])
    ref = oracle.march(oracle.FieldTraceable(distilled_oracle), o, d, np.array([1.0]), np.array([3.0]), oracle.MarchSettings())
    got = S.sphere_trace(fs, S.Ray(o[0], d[0]), 1.0, 3.0, S.RenderSettings())
    assert (got is not None) == bool(ref.hit[0])
    if got is not None:
        assert abs(got.t - ref.t[0]) <= 1e-4 and got.steps_taken == ref.steps[0]
    with pytest.raises(ValueError):
        S.sphere_trace(fs, S.Ray((0, 0, -2.0), (0, 0, 1.0)), 3.0, 1.0, S.RenderSettings())
    with pytest.raises(TypeError):
        S.march_rays(object(), np.zeros((1, 3)), np.zeros((1, 3)), np.zeros(1), np.ones(1), S.RenderSettings())


def test_reference_tracer_accepts_gpu_surface(S, distilled_field, distilled_oracle):
    """The drop-in boundary is the traceable-surface protocol (surface.py:1-7): the reference-style
    CPU loop (here: the oracle's) must run unmodified on our FieldSurface."""
    o, d, tn, tf = _rays(32, 32)
    a = oracle.trace_shade(S.FieldSurface(distilled_field), o, d, oracle.MarchSettings())
    b = oracle.trace_shade(oracle.FieldTraceable(distilled_oracle), o, d, oracle.MarchSettings())
    assert (a.hit == b.hit).mean() >= 0.999
    both = a.hit & b.hit
    assert (np.abs(a.t[both] - b.t[both]) <= 1e-4).mean() >= 0.995


def test_decision_filter_is_exact(S, cams, distilled_field):
    """The decision filter (tensor-core predicate + certified skipping, include/knf_b200.h knf_field_set_filter) may
    only change WHICH kernel looks at a sample, never a result: frames and march outputs with the filter forced on
    must equal the filter-off ones bit for bit, on the chaotic random-init field (98 % of evaluations filtered) and
    on a real surface (nothing to filter)."""
    from paper_2206_10885_b200 import grid

    for name, field, size in (("random-init 16^3", grid.field_init(grid.GridConfig(resolution=16), seed=0), 160),
                              ("random-init 8^3 seed 3", grid.field_init(grid.GridConfig(resolution=8), seed=3), 112),
                              ("distilled 4^3", distilled_field, 96)):
        # a fresh handle: what the auto mode learnt from other tests' marches on a shared (cached) handle must not decide here
        fs = S.FieldSurface(grid.DeviceField.upload(field))
        pose = cams.look_at_pose((0.3, 0.4, 2.4), (0, 0, 0), (0, 1, 0), np.deg2rad(40), size, size)
        o, d, tn, tf = _rays(size // 2, size // 2)
        out = {}
        try:
            for mode in ("off", "on", "auto"):
                fs.dev.set_filter(mode)
                fs.dev.reset_stats()
                fb = S.render_frame(fs, pose)
                st = fs.dev.stats()
                out[mode] = (fb, S.march_rays(fs, o, d, tn, tf, S.RenderSettings()), st)
        finally:
            fs.dev.set_filter("auto")
        fb0, m0, st0 = out["off"]
        assert st0["filter_evals"] == 0 and st0["filter_skipped"] == 0
        for mode in ("on", "auto"):
            fb, m, st = out[mode]
            for k in ("color", "depth", "normal", "hit"):
                assert np.array_equal(getattr(fb, k), getattr(fb0, k)), (name, mode, k)
            assert np.array_equal(m.hit, m0.hit) and np.array_equal(m.t, m0.t) and np.array_equal(m.steps, m0.steps)
            assert np.array_equal(m.position, m0.position)
        st = out["on"][2]
        print(f"{name}: filter on -> exact {st['sdf_evals']}, filter {st['filter_evals']}, undecided {st['filter_deferred']}, "
              f"certified {st['filter_skipped']} (delta {fs.dev.filter_delta():.3g}); off -> exact {st0['sdf_evals']}")
        if name.startswith("random-init 16"):
            assert st["filter_evals"] + st["filter_skipped"] > 5 * st["sdf_evals"]  # the filter carries the crawl (evaluated or certified)
            assert out["auto"][2]["filter_evals"] > 0
        elif name.startswith("distilled"):
            assert out["auto"][2]["filter_evals"] == 0        # auto switches itself off on a real surface
    with pytest.raises(ValueError):
        fs.dev.set_filter(5)


def test_frame_random_init_256_parity(S, cams):
    """BASELINE config 1 at full size (256^2, random-init 16^3, the cmd_bench camera) against the oracle run on this
    host: north_star bars -- hit masks >= 99.9 %, depth 1e-4, normals / RGB 1e-3 on the both-hit pixels."""
    from paper_2206_10885_b200 import grid

    field = grid.field_init(grid.GridConfig(resolution=16), seed=0)
    pose = cams.look_at_pose((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 256, 256)
    ocam = oracle.camera_look_at((0, 0, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 256, 256)
    ref = oracle.render(oracle.FieldTraceable(oracle_from_product(field)), ocam, oracle.MarchSettings())
    fb = S.render_frame(S.FieldSurface(field), pose)
    agree = (fb.hit == ref.hit).mean()
    both = fb.hit & ref.hit
    rel = np.abs(fb.depth[both] - ref.depth[both]) / ref.depth[both]
    nerr = np.abs(fb.normal - ref.normal)[both].max(axis=1)
    cerr = np.abs(fb.color - ref.color)[both].max(axis=1)
    print(f"256^2 random-init: hit agreement {agree:.4%} ({int((fb.hit != ref.hit).sum())} flips), depth<=1e-4 {np.mean(rel <= 1e-4):.4%}, "
          f"normal<=1e-3 {np.mean(nerr <= 1e-3):.4%}, rgb<=1e-3 {np.mean(cerr <= 1e-3):.4%}")
    # north_star bars, asserted at what is achieved: hit masks >= 99.9 % (measured 99.963 %: 24 flips; the
    # reference against itself across band sizes flips 6, tests/golden/reference_noise.json); EVERY both-hit pixel inside the
    # depth 1e-4 and RGB 1e-3 bars; normals (FD: SDF ulps x 500) inside 1e-3 on >= 99.95 % (measured 100 %)
    assert agree >= 0.9995
    assert np.all(rel <= 1e-4) and np.all(cerr <= 1e-3) and np.mean(nerr <= 1e-3) >= 0.9995
