"""GPU: the decision filter under attack (VERDICT r1 "what's weak" 2) and the host-side hazards ADVICE r1 listed.

The decision filter (knf_march.cuh) may only change WHICH kernel looks at a sample.  Every test here renders / marches
the same rays with the filter forced off and forced on and demands bit-identical results, on inputs chosen to break
the assumptions behind the per-cell error bound: samples outside the box (caller-supplied t ranges), weights scaled
until hidden activations leave the fp16 range, non-zero biases, fine grids, cameras inside the object, tiny step
budgets.  Each case is also compared with the CPU oracle's march of the same rays."""

import copy

import numpy as np
import pytest

import oracle
from conftest import oracle_from_product

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2206_10885_b200 import surface

    return surface


@pytest.fixture(scope="module")
def G():
    from paper_2206_10885_b200 import grid

    return grid


def _camera_rays(w, h, pos=(0, 0, 2.5), fov=40):
    cam = oracle.camera_look_at(pos, (0, 0, 0), (0, 1, 0), np.deg2rad(fov), w, h)
    o, d = oracle.camera_rays(cam)
    tn, tf, inside = oracle.slab_intersect(o, d, (-1, -1, -1), (1, 1, 1))
    return o, d, np.where(inside, tn, 1.0), np.where(inside, tf, 0.0)


def _march_on_off(S, field, o, d, tn, tf, settings):
    """march_rays with the filter off / on / auto; asserts bit-identity, returns (result, stats_on)."""
    fs = S.FieldSurface(field)
    out = {}
    try:
        for mode in ("off", "on", "auto"):
            fs.dev.set_filter(mode)
            fs.dev.reset_stats()
            out[mode] = (S.march_rays(fs, o, d, tn, tf, settings), fs.dev.stats())
    finally:
        fs.dev.set_filter("auto")
    r0, st0 = out["off"]
    assert st0["filter_evals"] == 0 and st0["filter_skipped"] == 0
    for mode in ("on", "auto"):
        r = out[mode][0]
        assert np.array_equal(r.hit, r0.hit), mode
        assert np.array_equal(r.t, r0.t), mode
        assert np.array_equal(r.steps, r0.steps), mode
        assert np.array_equal(r.position, r0.position), mode
    return r0, out["on"][1], fs


def _vs_oracle(name, res, field, o, d, tn, tf, cfg, hit_bar, step_bar):
    ref = oracle.march(oracle.FieldTraceable(oracle_from_product(field)), o, d, tn, tf, cfg)
    agree = float((res.hit == ref.hit).mean())
    steps_eq = float((res.steps == ref.steps).mean())
    both = res.hit & ref.hit
    drel = np.abs(res.t[both] - ref.t[both]) / np.maximum(np.abs(ref.t[both]), 1e-12) if both.any() else np.zeros(1)
    print(f"{name}: vs oracle hit agreement {agree:.4%}, steps equal {steps_eq:.4%}, depth rel <= 1e-4 on {np.mean(drel <= 1e-4):.4%} "
          f"of {int(both.sum())} both-hit rays")
    assert agree >= hit_bar, name
    assert steps_eq >= step_bar, name
    # depth on the both-hit rays: the chaotic fields here flip a convergence step on a handful of rays (the reference
    # does so against itself, tests/golden/reference_noise.json), so allow that many outliers
    assert int((drel > 1e-4).sum()) <= max(3, int((1.0 - hit_bar) * both.sum())), name
    return ref


def test_filter_with_t_ranges_that_leave_the_box(S, G):
    """march_rays accepts caller-supplied [t_near, t_far] (surface.py:162-178): samples outside the box clamp to
    boundary cells with raw coordinates beyond what the filter's bound was derived for.  They must go to the exact
    kernel; results stay bit-identical and agree with the oracle."""
    field = G.field_init(G.GridConfig(resolution=16), seed=0)
    rng = np.random.default_rng(5)
    n = 6000
    o = rng.uniform(-2.5, 2.5, size=(n, 3))
    o[: n // 3] = rng.uniform(-0.9, 0.9, size=(n // 3, 3))  # a third start inside the box
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    tn = np.zeros(n)
    tf = rng.uniform(0.5, 6.0, size=n)  # far beyond the box for most rays
    res, st, _ = _march_on_off(S, field, o, d, tn, tf, S.RenderSettings())
    assert st["filter_evals"] > 0  # the crawl inside the box still runs on the filter
    # outside the box a random-init network of sin/cos features keeps crawling too, so most rays burn the 128 steps
    _vs_oracle("t ranges leaving the box", res, field, o, d, tn, tf, oracle.MarchSettings(), 0.995, 0.99)


@pytest.mark.parametrize("scale,expect_filter", [(10.0, True), (100.0, False)])
def test_filter_with_scaled_weights_and_biases(S, G, scale, expect_filter):
    """Weights x10 / x100 with non-zero biases: activations grow until fp16 operand pieces overflow (x100).  The bound
    must either still hold (x10, larger delta) or switch the filter off for the cell (delta = +inf)."""
    field = G.field_init(G.GridConfig(resolution=8), seed=11)
    rng = np.random.default_rng(12)
    for k in range(2):  # hidden layers
        field.sdf.weights[k] *= np.float32(scale)
    for k in range(3):
        field.sdf.biases[k] += rng.normal(scale=0.5, size=field.sdf.biases[k].shape).astype(np.float32)
    field.sdf.biases[2][:, 0] -= np.float32(2.0 * scale)  # keep a negative region so rays crawl
    o, d, tn, tf = _camera_rays(72, 72)
    res, st, fs = _march_on_off(S, field, o, d, tn, tf, S.RenderSettings())
    off = fs.dev.filter_cells_off()
    print(f"weights x{scale:g}: delta {fs.dev.filter_delta():.3g}, cells off {off}/{8**3}, filter evals {st['filter_evals']}, "
          f"undecided {st['filter_deferred']}, exact {st['sdf_evals']}")
    if expect_filter:
        assert off == 0 and st["filter_evals"] > 0
    else:
        assert off == 8**3 and st["filter_evals"] == 0  # every cell's activation bound exceeds the fp16 range
    # scaled fields are far more chaotic than random-init (|grad d| grows with scale^2): the oracle comparison is a
    # sanity bar, bit-identity above is the proof
    _vs_oracle(f"weights x{scale:g}", res, field, o, d, tn, tf, oracle.MarchSettings(), 0.97, 0.95)


def test_filter_with_some_cells_beyond_fp16(S, G):
    """Only a slab of cells gets x200 weights: those cells carry delta = +inf and are served by the exact kernel while
    their neighbours keep the filter."""
    field = G.field_init(G.GridConfig(resolution=8), seed=4)
    big = np.zeros((8, 8, 8), dtype=bool)
    big[:, :, 3:5] = True
    big = big.reshape(-1)
    for k in range(2):
        field.sdf.weights[k][big] *= np.float32(200.0)
    o, d, tn, tf = _camera_rays(64, 64)
    res, st, fs = _march_on_off(S, field, o, d, tn, tf, S.RenderSettings())
    assert fs.dev.filter_cells_off() == int(big.sum())
    assert st["filter_evals"] > 0 and st["filter_deferred"] > 0
    _vs_oracle("x200 slab", res, field, o, d, tn, tf, oracle.MarchSettings(), 0.97, 0.95)


def test_filter_on_a_32_cubed_field(S, G):
    field = G.field_init(G.GridConfig(resolution=32), seed=2)
    o, d, tn, tf = _camera_rays(96, 96, pos=(0.4, 0.3, 2.4))
    res, st, _ = _march_on_off(S, field, o, d, tn, tf, S.RenderSettings())
    assert st["filter_evals"] + st["filter_skipped"] > st["sdf_evals"]  # most samples are decided or certified by the filter
    _vs_oracle("32^3", res, field, o, d, tn, tf, oracle.MarchSettings(), 0.995, 0.99)


def test_filter_with_camera_inside_the_object(S, distilled_field):
    """Camera inside the distilled sphere: every ray starts in the negative region and crawls outwards."""
    o, d, _, _ = _camera_rays(80, 80, pos=(0.05, 0.02, 0.1), fov=70)
    tn, tf, inside = oracle.slab_intersect(o, d, (-1, -1, -1), (1, 1, 1))
    assert inside.all()
    res, st, _ = _march_on_off(S, distilled_field, o, d, tn, tf, S.RenderSettings())
    assert st["filter_evals"] > 0
    _vs_oracle("camera inside", res, distilled_field, o, d, tn, tf, oracle.MarchSettings(), 0.999, 0.995)


@pytest.mark.parametrize("max_steps", [1, 7, 128])
def test_filter_with_step_budgets(S, G, max_steps):
    field = G.field_init(G.GridConfig(resolution=16), seed=0)
    o, d, tn, tf = _camera_rays(64, 64)
    settings = S.RenderSettings(max_steps=max_steps)
    res, st, _ = _march_on_off(S, field, o, d, tn, tf, settings)
    assert res.steps.max() <= max_steps
    _vs_oracle(f"max_steps={max_steps}", res, field, o, d, tn, tf, oracle.MarchSettings(max_steps=max_steps), 0.995, 0.99)


def test_frames_identical_filter_on_off_vs_oracle(S, G):
    """Whole frames (march + refinement + FD normals + colour), filter off / on, and against oracle.render."""
    from paper_2206_10885_b200 import cameras

    field = G.field_init(G.GridConfig(resolution=16), seed=0)
    pose = cameras.look_at_pose((0.3, 0.4, 2.4), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 128, 128)
    fs = S.FieldSurface(field)
    frames = {}
    try:
        for mode in ("off", "on"):
            fs.dev.set_filter(mode)
            frames[mode] = S.render_frame(fs, pose)
    finally:
        fs.dev.set_filter("auto")
    for k in ("color", "depth", "normal", "hit"):
        assert np.array_equal(getattr(frames["on"], k), getattr(frames["off"], k)), k
    ocam = oracle.camera_look_at((0.3, 0.4, 2.4), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 128, 128)
    ref = oracle.render(oracle.FieldTraceable(oracle_from_product(field)), ocam, oracle.MarchSettings())
    fb = frames["on"]
    agree = (fb.hit == ref.hit).mean()
    both = fb.hit & ref.hit
    rel = np.abs(fb.depth[both] - ref.depth[both]) / ref.depth[both]
    print(f"128^2 filtered frame vs oracle: hits {agree:.4%}, depth<=1e-4 {np.mean(rel <= 1e-4):.4%}")
    assert agree >= 0.998 and np.mean(rel <= 1e-4) >= 0.998


# ---- certified skipping: the per-cell Lipschitz bounds (csrc/knf_bounds.cuh) -----------------------------------------


def test_lipschitz_refinement_matches_restatement_and_is_sound(G, monkeypatch):
    """The device refinement against its float64 NumPy restatement (tests/lip_restatement.py) on a coarse setting the
    restatement finishes in seconds, the closed form against its restatement, and soundness: on thousands of random
    points per cell the true |d d / d x_a| stays below the bound the filter kernels read."""
    import lip_restatement as L

    monkeypatch.setenv("KNF_LIP_WIDTH", "0.02")  # 8^3 grid: k = 13 sub-boxes per axis
    monkeypatch.setenv("KNF_LIP_FINE", "3")
    field = G.field_init(G.GridConfig(resolution=8, bbox_min=(-1.0, -1.2, -0.8), bbox_max=(1.0, 0.8, 1.2)), seed=5)
    rng = np.random.default_rng(1)
    field.sdf.biases[0] += rng.normal(scale=0.3, size=field.sdf.biases[0].shape).astype(np.float32)
    field.sdf.biases[1] += rng.normal(scale=0.3, size=field.sdf.biases[1].shape).astype(np.float32)
    dev = G.DeviceField.upload(field)
    try:
        closed, refined, ms = dev.lipschitz()
        again = dev.lipschitz()[1]
    finally:
        dev.close()
    assert np.array_equal(again, refined) and (refined <= closed).all() and (refined > 0).all()
    for c in (0, 77, 300, 511):
        W1, W2, w3 = (np.asarray(field.sdf.weights[k][c], np.float64) for k in range(3))
        want_closed = L.closed_form(W1, W2, w3[0])
        assert np.allclose(closed[c], want_closed, rtol=1e-5), (c, closed[c], want_closed)
        want = np.minimum(L.refine_cell(field, c, 0.02, 3), want_closed)
        assert np.allclose(refined[c], want, rtol=2e-6), (c, refined[c], want)
        assert (refined[c] >= want * (1 - 1e-7)).all()  # stored rounded UP
    print(f"8^3 odd box, width 0.02: closed-form / refined = {np.mean(closed / refined):.2f} (mean), refinement {ms:.1f} ms")
    monkeypatch.delenv("KNF_LIP_WIDTH")
    monkeypatch.delenv("KNF_LIP_FINE")
    field = G.field_init(G.GridConfig(resolution=16), seed=0)
    dev = G.DeviceField.upload(field)
    try:
        closed, refined, ms = dev.lipschitz()
    finally:
        dev.close()
    worst = 0.0
    for c in np.random.default_rng(2).integers(0, 16 ** 3, 12):
        g = L.sampled_gradient_max(field, int(c), n=20000, seed=int(c))
        assert (g <= refined[c]).all(), (c, g, refined[c])
        worst = max(worst, float((g / refined[c]).max()))
    ratio = closed / refined
    print(f"16^3 default width: closed-form / refined mean {ratio.mean():.2f} (min {ratio.min():.2f}, max {ratio.max():.2f}), "
          f"refinement {ms:.0f} ms, sampled gradient reaches {worst:.3f} of the bound")
    assert ratio.mean() > 5.0  # the refinement is what makes certified skipping pay


def test_lipschitz_accessor_without_filter_blobs(G):
    """A field whose hidden-layer weights leave the fp16 range has no decision-filter blobs and therefore no Lipschitz bounds to
    report: knf_field_lipschitz says so (KNF_E_UNSUPPORTED) instead of returning stale or zero bounds."""
    from paper_2206_10885_b200 import _native as N

    field = G.field_init(G.GridConfig(resolution=4), seed=3)
    field.sdf.weights[1][0, 0, 0] = np.float32(7.0e4)  # beyond the fp16 operand pieces
    dev = G.DeviceField.upload(field)
    try:
        with pytest.raises(N.KnfUnsupported):
            dev.lipschitz()
    finally:
        dev.close()


@pytest.mark.parametrize("eps,step_scale,bars", [(1e-3, 0.8, (0.99, 0.98)), (0.02, 1.0, (0.97, 0.95)), (1e-4, 0.5, (0.99, 0.98))])
def test_skipping_on_an_off_centre_box_and_other_step_sizes(S, G, eps, step_scale, bars):
    """Certified skipping with the refined bounds on a non-cubic, off-centre box, rays that start outside it (samples clamped
    into boundary cells must not start a skip run) and crawl steps from 2.5e-5 to 0.02: filter off / on / auto bit-identical,
    closed-form run (KNF_FILTER_SKIP=2, the default) and per-sample skipping alike."""
    cfg = G.GridConfig(resolution=8, bbox_min=(-1.5, -1.0, -0.5), bbox_max=(1.0, 1.2, 0.8))
    field = G.field_init(cfg, seed=21)
    rng = np.random.default_rng(22)
    n = 5000
    o = rng.uniform(-2.0, 2.0, size=(n, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    tn = np.zeros(n)
    tf = rng.uniform(0.3, 3.0, size=n)
    settings = S.RenderSettings(eps_hit=eps, step_scale=step_scale, max_steps=160)
    res, st, _ = _march_on_off(S, field, o, d, tn, tf, settings)
    assert st["filter_evals"] > 0 and st["filter_skipped"] > 0
    print(f"eps {eps:g} step_scale {step_scale:g}: filter evals {st['filter_evals']}, certified {st['filter_skipped']}, exact {st['sdf_evals']}")
    # (bit-identity above is the proof; against the oracle a coarse eps lets more rays of this chaotic field flip a
    # convergence step on the reference's own small-batch BLAS order, hence the wider sanity bar there)
    _vs_oracle(f"off-centre box eps={eps:g}", res, field, o, d, tn, tf,
               oracle.MarchSettings(eps_hit=eps, step_scale=step_scale, max_steps=160), *bars)


# ---- host-side hazards ------------------------------------------------------------------------------


def test_degenerate_gradient_raises(G):
    """pkg/tests/test_grid.py:255-267: an all-zero SDF family has no gradient anywhere."""
    field = G.field_init(G.GridConfig(resolution=4), seed=7)
    for w in field.sdf.weights:
        w[...] = 0
    for b in field.sdf.biases:
        b[...] = 0
    with pytest.raises(G.DegenerateGradientError):
        G.normal(field, np.array([0.2, 0.2, 0.2]))
    nrm, ok = G.normal_batch(field, np.array([[0.2, 0.2, 0.2], [-0.5, 0.1, 0.9]]))
    assert not ok.any() and np.all(np.isfinite(nrm))  # never NaN (the reference's test name says as much)


def test_empty_march_and_trace(S, small_field):
    fs = S.FieldSurface(small_field)
    r = S.march_rays(fs, [], [], [], [], S.RenderSettings())
    assert r.hit.shape == (0,) and r.t.shape == (0,) and r.position.shape == (0, 3) and r.steps.shape == (0,)
    r = S.trace_and_shade(fs, np.zeros((0, 3)), np.zeros((0, 3)), S.RenderSettings())
    assert r.hit.shape == (0,) and r.color.shape == (0, 3)


def test_upload_rejects_what_it_cannot_reproduce(G, small_field):
    from paper_2206_10885_b200._native import KnfUnsupported

    f64 = G.field_init(G.GridConfig(resolution=2), seed=1, dtype=np.float64)
    with pytest.raises(KnfUnsupported):
        G.sdf_values(f64, np.zeros((4, 3), np.float32))  # the reference evaluates a float64 field in float64
    bad = copy.deepcopy(small_field)
    bad.sdf.biases[1] = bad.sdf.biases[1][:, :16]
    with pytest.raises(ValueError):
        G.sdf_values(bad, np.zeros((4, 3), np.float32))
    bad = copy.deepcopy(small_field)
    bad.sdf.activations = [G.RELU, G.SOFTPLUS, G.IDENTITY]
    with pytest.raises(KnfUnsupported):
        G.sdf_values(bad, np.zeros((4, 3), np.float32))


def test_invalidate_reuploads_and_keeps_live_handles_valid(S, G):
    """grid.invalidate() after mutating a field: the next query sees the new weights, a FieldSurface built earlier
    follows, and a path-trace scene that captured the old handle keeps rendering (no use-after-free)."""
    from paper_2206_10885_b200 import cameras, pathtrace

    field = G.field_init(G.GridConfig(resolution=4), seed=3)
    pts = np.random.default_rng(0).uniform(-1, 1, size=(512, 3)).astype(np.float32)
    fs = S.FieldSurface(field)
    before = G.sdf_values(field, pts)
    scene = pathtrace.Scene([pathtrace.QuadObj((-2, -1.01, -2), (4, 0, 0), (0, 0, 4), pathtrace.Lambertian((0.7, 0.7, 0.7))),
                             pathtrace.NeuralObject(fs)], pathtrace.ConstantEnv((1, 1, 1)))
    pose = cameras.look_at_pose((0, 0.5, 2.8), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 24, 24)
    img0 = pathtrace.render_pathtraced(scene, pose, spp=1, seed=1).hdr
    field.sdf.biases[2][:, 0] += np.float32(0.25)
    G.invalidate(field)
    after = G.sdf_values(field, pts)
    assert np.allclose(after - before, 0.25, atol=1e-6)
    assert np.allclose(fs.sdf_values(pts.astype(np.float64)) - before, 0.25, atol=1e-6)  # the surface re-resolved its device copy
    img1 = pathtrace.render_pathtraced(scene, pose, spp=1, seed=1).hdr  # scene notices the new handle and rebuilds
    assert np.all(np.isfinite(img1)) and img1.shape == img0.shape
    fresh = pathtrace.Scene(list(scene.objects), scene.environment)
    assert np.array_equal(pathtrace.render_pathtraced(fresh, pose, spp=1, seed=1).hdr, img1)


def test_scene_cache_follows_edits(S, distilled_field):
    """pathtrace.device_scene caches the upload on the Scene; the reference re-reads the Python objects on every call
    (service.py mutates and reuses scenes), so edits must show."""
    from paper_2206_10885_b200 import cameras, pathtrace

    quad = pathtrace.QuadObj((-2, -0.8, -2), (4, 0, 0), (0, 0, 4), pathtrace.Lambertian((0.7, 0.7, 0.7)))
    ball = pathtrace.SphereObj((0.0, 0.0, 0.0), 0.5, pathtrace.Lambertian((0.9, 0.2, 0.2)))
    scene = pathtrace.Scene([quad, ball], pathtrace.ConstantEnv((1, 1, 1)))
    pose = cameras.look_at_pose((0, 0.6, 3.0), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 32, 32)
    a = pathtrace.render_pathtraced(scene, pose, spp=2, seed=3).hdr
    scene.objects[1] = pathtrace.SphereObj((0.4, 0.0, 0.0), 0.5, pathtrace.Lambertian((0.2, 0.9, 0.2)))  # same count, new object
    b = pathtrace.render_pathtraced(scene, pose, spp=2, seed=3).hdr
    ref = pathtrace.render_pathtraced(pathtrace.Scene([quad, scene.objects[1]], pathtrace.ConstantEnv((1, 1, 1))), pose, spp=2, seed=3).hdr
    assert not np.array_equal(a, b) and np.array_equal(b, ref)
    scene.environment = pathtrace.ConstantEnv((0.2, 0.3, 0.9))
    c = pathtrace.render_pathtraced(scene, pose, spp=2, seed=3).hdr
    assert not np.array_equal(b, c)


def test_two_streams_share_a_handle(S, G):
    """KNF_MEM_DEVICE calls return while their kernels run; a call on ANOTHER stream must wait for them instead of
    reusing the handle's workspace underneath (CallScope, knf_engine.cu).  Also: a call must not change the caller's
    current device."""
    import torch

    field = G.field_init(G.GridConfig(resolution=8), seed=9)
    dev = G.device_field(field)
    pts = torch.rand((400_000, 3), device="cuda", dtype=torch.float32) * 2 - 1
    want = G.sdf_query(dev, pts).value.clone()
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for rep in range(6):
        with torch.cuda.stream(s1 if rep % 2 == 0 else s2):
            outs.append(G.sdf_query(dev, pts).value)
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, want)
    assert torch.cuda.current_device() == 0
