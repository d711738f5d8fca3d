"""GPU parity, part 1: routing and the batched multi-network forward (BASELINE config 4),
through the C-ABI, against the oracle and the reference-generated golden vectors."""

import numpy as np
import pytest

import oracle
from conftest import golden, oracle_from_product

pytestmark = pytest.mark.gpu

FWD_TOL = 2e-6  # reference's own grouped-vs-naive bound is 1e-6 (test_grid.py:81-86); see DESIGN.md Numerics


@pytest.fixture(scope="module")
def G():
    from paper_2206_10885_b200 import grid

    return grid


def test_device_math_against_reference_golden():
    """The device routines behind the MLP kernels, probed directly: the encoder (NumPy's SIMD sin/cos
    + the fp32 double-angle recurrence) and the sigmoid (NumPy's exp + IEEE division) must be
    BIT-EXACT with the reference; so must softplus (NumPy's exp + Intel SVML's log1p restated, oracle/np_softplus.c),
    up to the one-in-millions argument where the Markstein division rounds differently from IEEE."""
    from paper_2206_10885_b200 import nn

    g = golden("encode_act.npz")
    assert np.array_equal(nn.fourier_encode(g["x"], 6), g["enc6"])
    assert np.array_equal(nn.fourier_encode(g["x"], 4), g["enc4"])
    assert nn.fourier_encode(g["x"][0], 6).shape == (39,)
    assert np.array_equal(nn.sigmoid(g["z"]), g["sigmoid"])
    sp = nn.softplus(g["z"])
    ulp = np.spacing(np.abs(g["softplus"]))
    print(f"softplus vs NumPy: identical {np.mean(sp == g['softplus']):.3f}, max {np.abs(sp - g['softplus']).max():.2e}, max ulps {(np.abs(sp - g['softplus']) / ulp).max():.1f}")
    assert np.abs(sp - g["softplus"]).max() <= 5e-7 and (np.abs(sp - g["softplus"]) / ulp).max() <= 4
    assert np.mean(sp == g["softplus"]) >= 0.9999
    with pytest.raises(ValueError):
        nn.fourier_encode(g["x"], -1)


def test_cell_ids_bit_exact_golden(G):
    g = golden("cells.npz")
    for n in (1, 4, 16):
        cfg = G.GridConfig(resolution=n)
        assert np.array_equal(G.cell_index_flat(cfg, g[f"pts_{n}"]), g[f"ids_{n}"])
    cfg = G.GridConfig(resolution=5, bbox_min=(-0.7, -1.1, 0.2), bbox_max=(0.9, 0.4, 1.7))
    assert np.array_equal(G.cell_index_flat(cfg, g["pts_odd"]), g["ids_odd"])


def test_cell_ids_bit_exact_million(G):
    # SURVEY 8c protocol (1): 1e6 uniform points + every face coordinate +-{0,1,2} ulp
    rng = np.random.default_rng(0)
    pts = rng.uniform(-1.05, 1.05, size=(1_000_000, 3)).astype(np.float32)
    faces = (-1.0 + 2.0 * np.arange(17) / 16).astype(np.float32)
    ring = [faces]
    up, dn = faces, faces
    for _ in range(2):
        up = np.nextafter(up, np.float32(np.inf))
        dn = np.nextafter(dn, np.float32(-np.inf))
        ring += [up, dn]
    vals = np.concatenate(ring)
    pts[:60000] = rng.choice(vals, size=(60000, 3))
    cfg = G.GridConfig(resolution=16)
    want = oracle.cell_ids(oracle.FieldSpec(resolution=16), pts)
    assert np.array_equal(G.cell_index_flat(cfg, pts), want)
    # fp64 points keep their precision (grid.cell_index passes fp64 straight through)
    p64 = pts[:5000].astype(np.float64) + 1e-12
    assert np.array_equal(G.cell_index_flat(cfg, p64), oracle.cell_ids(oracle.FieldSpec(resolution=16), p64))
    assert G.cell_index(cfg, (0.0, 0.0, 0.0)) == (8, 8, 8)
    assert G.cell_index(cfg, (2.0, 0.0, 0.0)) == (15, 8, 8)
    assert G.cell_index(cfg, (-1.0, -1.0, -1.0)) == (0, 0, 0)


def test_route_groups_by_cell(G, small_field):
    rng = np.random.default_rng(5)
    pts = rng.uniform(-1.2, 1.2, size=(5000, 3)).astype(np.float32)
    r = G.route(small_field, pts)
    ids = oracle.cell_ids(oracle.FieldSpec(resolution=4), pts)
    assert sorted(r.order.tolist()) == list(range(5000))  # a permutation
    assert np.all(np.diff(ids[r.order]) >= 0)  # sorted by cell
    cells, starts = np.unique(ids[r.order], return_index=True)
    assert np.array_equal(r.cells, cells) and np.array_equal(r.starts, starts)
    assert np.array_equal(r.ends, np.append(starts[1:], 5000))
    assert np.array_equal(r.unsort(r.sort(pts)), pts)


def test_sdf_forward_matches_golden_and_oracle(G, small_field, small_oracle):
    g = golden("forward_r4_seed7.npz")
    got = G.sdf_query(small_field, g["pts"])
    assert got.value.dtype == np.float32 and got.features.shape == (3000, 8)
    assert np.abs(got.value - g["value"]).max() <= FWD_TOL
    assert np.abs(got.features - g["features"]).max() <= FWD_TOL
    v, f = oracle.query_sdf(small_oracle, g["pts"])
    assert np.abs(got.value - v).max() <= FWD_TOL
    few = G.sdf_query(small_field, g["pts"][:150])
    assert np.abs(few.value - g["value_few"]).max() <= FWD_TOL
    assert np.abs(G.sdf_values(small_field, g["pts"]) - g["value"]).max() <= FWD_TOL


def test_sdf_forward_a1_field(G):
    # A1 (test_acceptance.py:113-127): 16^3 seed 42, U(-1.1,1.1) points
    g = golden("forward_r16_seed42.npz")
    field = G.field_init(G.GridConfig(resolution=16), seed=42)
    got = G.sdf_query(field, g["pts"])
    err_v = np.abs(got.value - g["value"])
    err_f = np.abs(got.features - g["features"])
    print(f"A1 parity: value max {err_v.max():.2e} mean {err_v.mean():.2e}; features max {err_f.max():.2e}")
    assert err_v.max() <= FWD_TOL and err_f.max() <= FWD_TOL


def test_color_forward(G, small_field):
    g = golden("forward_r4_seed7.npz")
    rgb = G.color_query(small_field, g["pts"], g["v"], g["n"], g["features"])
    assert rgb.shape == (3000, 3) and rgb.dtype == np.float32
    err = np.abs(rgb - g["rgb"]).max()
    print(f"colour parity: max {err:.2e}")
    assert err <= 1e-6
    assert np.all((rgb > 0) & (rgb < 1))
    one = G.color_query(small_field, g["pts"][7], g["v"][7], g["n"][7], g["features"][7])
    assert np.abs(one[0] - rgb[7]).max() <= 1e-6  # batch == single (test_grid.py:106-132)
    assert np.array_equal(G.grouped_query(small_field, g["pts"], "color", v=g["v"], n=g["n"], z=g["features"]), rgb)
    with pytest.raises(ValueError):
        G.grouped_query(small_field, g["pts"], "density")


def test_permutation_equivariance_exact(G, small_field):
    # test_grid.py:136-142 (array_equal): every point is evaluated with a fixed FMA order
    rng = np.random.default_rng(9)
    pts = rng.uniform(-1, 1, size=(4000, 3)).astype(np.float32)
    perm = rng.permutation(4000)
    a = G.sdf_query(small_field, pts)
    b = G.sdf_query(small_field, pts[perm])
    assert np.array_equal(a.value[perm], b.value)
    assert np.array_equal(a.features[perm], b.features)
    # ... and independent of how many points share the cell (the reference is not: OpenBLAS
    # switches kernels with batch size)
    c = G.sdf_query(small_field, pts[:37])
    assert np.array_equal(c.value, a.value[:37])


def test_ragged_and_empty_batches(G, small_field, small_oracle):
    assert G.sdf_query(small_field, np.zeros((0, 3), np.float32)).value.shape == (0,)
    for n in (1, 2, 63, 64, 65, 255, 256, 257, 1000):
        pts = np.random.default_rng(n).uniform(-1, 1, size=(n, 3)).astype(np.float32)
        pts[:, :] = pts[:, :] * 0.2 + 0.3  # all in one or two cells: exercises partial warps/tiles
        v, _ = oracle.query_sdf(small_oracle, pts)
        assert np.abs(G.sdf_values(small_field, pts) - v).max() <= FWD_TOL


def test_outside_points_clamp_to_boundary_cells(G, small_field, small_oracle):
    pts = np.random.default_rng(1).uniform(-3, 3, size=(2000, 3)).astype(np.float32)
    v, f = oracle.query_sdf(small_oracle, pts)
    got = G.sdf_query(small_field, pts)
    assert np.abs(got.value - v).max() <= 1e-5  # |enc| arguments up to 3*pi*32: still the same algorithm


def test_torch_device_path(G, small_field):
    import torch

    g = golden("forward_r4_seed7.npz")
    t = torch.as_tensor(g["pts"], device="cuda")
    out = G.sdf_query(small_field, t)
    assert out.value.is_cuda
    assert np.array_equal(out.value.cpu().numpy(), G.sdf_query(small_field, g["pts"]).value)


def test_fd_normals(G, small_field):
    g = golden("fd_normals_r4.npz")
    grad = G.grad_fd(small_field, g["pts"])
    err = np.abs(grad - g["grad"]).max()
    print(f"FD gradient parity: max {err:.2e} (SDF ulps x 500)")
    assert err <= 2 * 500 * FWD_TOL  # two SDF evaluations per difference
    nrm, ok = G.normal_batch(small_field, g["pts"])
    assert np.array_equal(ok, g["ok"])
    assert np.abs(nrm - g["normals"]).max() <= 1e-3
    assert np.allclose(np.linalg.norm(nrm[ok], axis=1), 1.0, atol=1e-12)
    assert np.abs(G.normal(small_field, g["pts"][5]) - g["normals"][5]).max() <= 1e-3
    assert G.grad_fd(small_field, g["pts"][0]).shape == (3,)


def test_unsupported_architecture_is_loud(G):
    """Widths beyond the compiled ones cannot be embedded: refuse loudly."""
    from paper_2206_10885_b200 import _native as N

    for cfg in (G.GridConfig(resolution=2, feature_dim=12), G.GridConfig(resolution=2, sdf_freqs=7), G.GridConfig(resolution=2, dir_freqs=5)):
        with pytest.raises(N.KnfUnsupported):
            G.sdf_query(G.field_init(cfg, seed=0), np.zeros((3, 3), np.float32))


@pytest.mark.parametrize("lx,lv,nf", [(4, 2, 5), (6, 4, 3), (0, 0, 1), (5, 4, 8)])
def test_narrower_widths_are_embedded_exactly(G, lx, lv, nf):
    """GridConfig.sdf_freqs / dir_freqs / feature_dim below the defaults (grid.py:32-64).  Such a field is embedded
    into the compiled 39-32-32-9 / 41-32-32-3 networks with zero weights at the missing inputs / outputs, which leaves every
    k-ordered FMA chain unchanged -- so parity with the oracle is the same as for the default widths."""
    import oracle
    from paper_2206_10885_b200 import cameras, surface

    cfg = G.GridConfig(resolution=4, sdf_freqs=lx, dir_freqs=lv, feature_dim=nf)
    field = G.field_init(cfg, seed=5)
    spec = oracle.FieldSpec(resolution=4, pos_octaves=lx, dir_octaves=lv, n_features=nf)
    ofield = oracle.field.field_from_stacks(spec, field.sdf.weights, field.sdf.biases, field.color.weights, field.color.biases)
    rng = np.random.default_rng(8)
    pts = rng.uniform(-1.05, 1.05, size=(20000, 3)).astype(np.float32)
    got = G.sdf_query(field, pts)
    ov, of = oracle.query_sdf(ofield, pts)
    assert got.features.shape == (20000, nf)
    assert np.abs(got.value - ov).max() <= 2e-6 and (nf == 0 or np.abs(got.features - of).max() <= 2e-6)
    v = rng.normal(size=(20000, 3)).astype(np.float32)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    rgb = G.color_query(field, pts, v, v, got.features)
    assert np.abs(rgb - oracle.query_color(ofield, pts, v, v, got.features)).max() <= 1e-6
    assert np.array_equal(G.cell_index_flat(field, pts), oracle.cell_ids(spec, pts))
    # a whole frame through the march, FD normals and the colour pass
    pose = cameras.look_at_pose((0.2, 0.3, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 48, 40)
    fb = surface.render_frame(surface.FieldSurface(field), pose)
    ref = oracle.render(oracle.FieldTraceable(ofield), oracle.camera_look_at((0.2, 0.3, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 48, 40),
                        oracle.MarchSettings())
    assert (fb.hit == ref.hit).mean() >= 0.995
    both = fb.hit & ref.hit
    if both.any():
        assert np.mean(np.abs(fb.depth[both] - ref.depth[both]) / ref.depth[both] <= 1e-4) >= 0.99
        assert np.mean(np.abs(fb.color - ref.color)[both].max(axis=1) <= 2e-3) >= 0.99


def test_knf_straight_to_device(G, distilled_field, golden_dir):
    import os

    from paper_2206_10885_b200.modelio import load_model_to_device

    dev = load_model_to_device(os.path.join(golden_dir, "sphere_r4_distilled.knf"))
    pts = np.random.default_rng(2).uniform(-1, 1, size=(3000, 3)).astype(np.float32)
    assert np.array_equal(G.sdf_query(dev, pts).value, G.sdf_query(distilled_field, pts).value)
    with pytest.raises(OSError):
        load_model_to_device(os.path.join(golden_dir, "rng.npz"))


def test_handle_is_thread_safe(G, small_field, small_oracle):
    """SPEC.md:190-191 / service.py:253-255: pure functions on an immutable field, callable from many
    host threads (ctypes releases the GIL; the handle serialises calls internally)."""
    from concurrent.futures import ThreadPoolExecutor

    rng = np.random.default_rng(11)
    batches = [rng.uniform(-1, 1, size=(2000 + 37 * k, 3)).astype(np.float32) for k in range(12)]
    want = [G.sdf_query(small_field, b).value for b in batches]
    with ThreadPoolExecutor(max_workers=6) as pool:
        got = list(pool.map(lambda b: G.sdf_query(small_field, b).value, batches * 3))
    for k, g in enumerate(got):
        assert np.array_equal(g, want[k % 12])


@pytest.mark.parametrize("mode", ["tensor_bf16x3", "tensor_fp16x2"])
def test_tensor_precision_modes(G, mode):
    """KNF_PRECISION_TENSOR_*: the hidden layers as exact-split mma.sync products.  Same API, same routing, distances
    within the forward tolerance of the oracle (bf16x3 is closer to exact arithmetic than the fp32 chain itself)."""
    g = golden("forward_r16_seed42.npz")
    field = G.field_init(G.GridConfig(resolution=16), seed=42)
    dev = G.device_field(field)
    ref = G.sdf_query(dev, g["pts"])
    try:
        dev.set_precision(mode)
        assert dev.get_precision() == mode
        got = G.sdf_query(dev, g["pts"])
        dv, df = np.abs(got.value - g["value"]), np.abs(got.features - g["features"])
        print(f"{mode}: |d - reference| max {dv.max():.2e} mean {dv.mean():.2e}; features max {df.max():.2e}; vs fp32 chain max {np.abs(got.value - ref.value).max():.2e}")
        assert dv.max() <= 4e-6 and df.max() <= 4e-6 and dv.mean() <= 4e-7
        # order independence holds in every mode
        perm = np.random.default_rng(3).permutation(len(g["pts"]))
        again = G.sdf_query(dev, g["pts"][perm])
        assert np.array_equal(again.value, got.value[perm]) and np.array_equal(again.features, got.features[perm])
        # ragged tile sizes (1..70 points in one cell) and the distance-only entry point
        few = g["pts"][:70]
        assert np.array_equal(G.sdf_values(dev, few), G.sdf_query(dev, few).value)
    finally:
        dev.set_precision("fp32_chain")
    with pytest.raises(ValueError):
        dev.set_precision(7)


def _analytic_gradient_f64(ofield, pts):
    """float64 forward-mode gradient of the owning cell's SDF network (nn.fourier_encode + two softplus layers)."""
    spec = ofield.spec
    cells = oracle.cell_ids(spec, pts.astype(np.float32))
    W = [w.astype(np.float64) for w in ofield.sdf.W]
    b = [v.astype(np.float64) for v in ofield.sdf.b]
    L = spec.pos_octaves
    out_d, out_g = np.empty(len(pts)), np.empty((len(pts), 3))
    for i, (x, c) in enumerate(zip(pts.astype(np.float64), cells)):
        feats, J = [x[0], x[1], x[2]], [np.eye(3)[0], np.eye(3)[1], np.eye(3)[2]]
        for o in range(L):
            f = (2.0 ** o) * np.pi
            for a in range(3):
                feats.append(np.sin(f * x[a])); J.append(f * np.cos(f * x[a]) * np.eye(3)[a])
            for a in range(3):
                feats.append(np.cos(f * x[a])); J.append(-f * np.sin(f * x[a]) * np.eye(3)[a])
        h, dh = np.array(feats), np.array(J)  # (39,), (39,3)
        for k in range(2):
            z = W[k][c] @ h + b[k][c]
            dz = W[k][c] @ dh
            sg = 1.0 / (1.0 + np.exp(-z))
            h, dh = np.log1p(np.exp(-np.abs(z))) + np.maximum(z, 0), sg[:, None] * dz
        out_d[i] = W[2][c][0] @ h + b[2][c][0]
        out_g[i] = W[2][c][0] @ dh
    return out_d, out_g


def test_analytic_gradient(G, distilled_field, distilled_oracle):
    """knf_sdf_gradient (north_star: the fused MLP also emits the SDF gradient): forward-mode analytic gradient of the
    owning cell's network against a float64 evaluation of the same derivative; its deviation from the reference's
    global finite-difference normals is REPORTED (the reference renders with FD, and so does the parity path)."""
    rng = np.random.default_rng(9)
    for name, field, ofield in (("distilled 4^3", distilled_field, distilled_oracle),
                                ("random-init 16^3", G.field_init(G.GridConfig(resolution=16), seed=0), None)):
        if ofield is None:
            ofield = oracle_from_product(field)
        pts = rng.uniform(-0.98, 0.98, size=(1500, 3)).astype(np.float32)
        grad, dist = G.grad_analytic(field, pts, return_distance=True)
        d64, g64 = _analytic_gradient_f64(ofield, pts)
        scale = np.abs(g64).max()
        print(f"{name}: analytic gradient vs float64: max |err| {np.abs(grad - g64).max():.2e} (|grad| up to {scale:.1f}), distance max |err| {np.abs(dist - d64).max():.2e}")
        assert np.abs(grad - g64).max() <= 2e-5 * max(scale, 1.0)
        assert np.abs(dist - d64).max() <= 5e-6
        assert np.allclose(dist, G.sdf_values(field, pts), atol=3e-6)
        # deviation from the reference's FD normals (grid.normal_batch): reported, and loosely bounded on the smooth field
        na = grad / np.maximum(np.linalg.norm(grad, axis=1, keepdims=True), 1e-30)
        nf, ok = G.normal_batch(field, pts.astype(np.float64))
        dev = np.abs(na - nf)[ok].max(axis=1)
        print(f"{name}: analytic vs FD normals: median {np.median(dev):.2e}, p99 {np.quantile(dev, 0.99):.2e}, max {dev.max():.2e}")
        if name.startswith("distilled"):
            assert np.median(dev) <= 5e-3
    # ragged / empty
    assert G.grad_analytic(distilled_field, np.zeros((0, 3), np.float32)).shape == (0, 3)
    assert G.grad_analytic(distilled_field, pts[:1]).shape == (1, 3)


def test_chunked_scan_equals_single_cta_scan(G, monkeypatch):
    """Grids beyond 65 536 cells scan their per-cell counts in chunks over many CTAs (route_scan_part / _apply); forcing
    that path on a 16^3 grid (KNF_SCAN_SPLIT, read when a handle is created) must reproduce the single-CTA scan: same
    routing segments, bit-identical queries and frames."""
    import copy

    from paper_2206_10885_b200 import cameras, surface

    field = G.field_init(G.GridConfig(resolution=16), seed=3)
    pts = np.random.default_rng(2).uniform(-1.05, 1.05, size=(300_000, 3)).astype(np.float32)
    pose = cameras.look_at_pose((0.3, 0.2, 2.5), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 160, 120)
    ref_route = G.route(field, pts[:50_000])
    ref_q = G.sdf_query(field, pts)
    ref_f = surface.render_frame(surface.FieldSurface(field), pose)
    monkeypatch.setenv("KNF_SCAN_SPLIT", "64")
    chunked = copy.deepcopy(field)  # a new object -> a new device handle, created under the environment variable
    r = G.route(chunked, pts[:50_000])
    assert np.array_equal(r.cells, ref_route.cells) and np.array_equal(r.starts, ref_route.starts) and np.array_equal(r.ends, ref_route.ends)
    assert np.array_equal(np.sort(r.order), np.arange(50_000))
    q = G.sdf_query(chunked, pts)
    assert np.array_equal(q.value, ref_q.value) and np.array_equal(q.features, ref_q.features)
    f = surface.render_frame(surface.FieldSurface(chunked), pose)
    for k in ("color", "depth", "normal", "hit"):
        assert np.array_equal(getattr(f, k), getattr(ref_f, k)), k
