"""GPU parity of the SURVEY 8(f) "next" rows: the service's uint8 frame hook and the mesh lattice sampler."""

import numpy as np
import pytest

import oracle
from conftest import oracle_from_product

pytestmark = pytest.mark.gpu


def _to_uint8(img):  # images.py:15-17
    return (np.clip(np.asarray(img, dtype=np.float64), 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)


def test_render_pass_u8_equals_host_pipeline(distilled_field):
    from paper_2206_10885_b200 import cameras, hooks, surface

    fs = surface.FieldSurface(distilled_field)
    pose = cameras.look_at_pose((1.0, 0.7, 2.2), (0, 0, 0), (0, 1, 0), np.deg2rad(40), 70, 45)
    for which in ("color", "normal", "depth"):
        st = surface.RenderSettings(render_pass=which)
        want = _to_uint8(surface.pass_image(surface.render_frame(fs, pose, st, background=(0.1, 0.5, 0.9)), which))
        got = hooks.render_pass_u8(fs, pose, st, background=(0.1, 0.5, 0.9))
        assert got.dtype == np.uint8 and got.shape == (45, 70, 3)
        assert np.array_equal(got, want), which
    polls = []
    banded = hooks.render_pass_u8(fs, pose, surface.RenderSettings(), tile_rows=16, abort_check=lambda: polls.append(1) and False)
    assert len(polls) == 3 and np.array_equal(banded, hooks.render_pass_u8(fs, pose))
    with pytest.raises(surface.RenderAborted):
        hooks.render_pass_u8(fs, pose, abort_check=lambda: True)


def test_tonemap_u8():
    from paper_2206_10885_b200 import hooks

    rng = np.random.default_rng(0)
    hdr = rng.uniform(-0.2, 3.0, size=(40, 30, 3))
    assert np.array_equal(hooks.to_uint8(hdr), _to_uint8(hdr))
    want = _to_uint8(np.clip(hdr / 3.0, 0.0, 1.0) ** (1.0 / 2.2))
    got = hooks.tonemap_u8(hdr, divisor=3.0, gamma22=True)
    assert (got != want).mean() <= 1e-4 and np.abs(got.astype(int) - want.astype(int)).max() <= 1  # pow() last-ulp at a .5 boundary


def test_sample_volume(distilled_field, distilled_oracle):
    from paper_2206_10885_b200 import grid, hooks

    R = 33
    vol = hooks.sample_volume(distilled_field, R, (-1, -1, -1), (1, 1, 1))
    xs = [np.linspace(-1.0, 1.0, R) for _ in range(3)]
    gx, gy, gz = np.meshgrid(*xs, indexing="ij")
    pts = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
    assert vol.shape == (R, R, R) and vol.dtype == np.float64
    # same lattice points as NumPy's: bit-identical to evaluating the host-built lattice
    assert np.array_equal(vol.ravel(), grid.sdf_values(distilled_field, pts).astype(np.float64))
    want = oracle.query_sdf_values(distilled_oracle, pts).astype(np.float64)
    assert np.abs(vol.ravel() - want).max() <= 4e-6
    off = hooks.sample_volume(distilled_field, 9, (-0.7, -1.2, 0.1), (0.9, 0.3, 1.4))
    xs = [np.linspace(a, b, 9) for a, b in ((-0.7, 0.9), (-1.2, 0.3), (0.1, 1.4))]
    gx, gy, gz = np.meshgrid(*xs, indexing="ij")
    p2 = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
    assert np.array_equal(off.ravel(), grid.sdf_values(distilled_field, p2).astype(np.float64))


def test_volume_forward_matches_reference_golden(distilled_field, distilled_oracle):
    """training._volume_forward, forward only."""
    from conftest import golden
    from paper_2206_10885_b200 import hooks

    g = golden("volume_forward.npz")
    assert abs(float(np.exp(distilled_field.inv_std_param)) - float(g["s"])) < 1e-12
    col = hooks.volume_forward(distilled_field, g["origins"], g["dirs"], 24, g["jitter"], (1.0, 1.0, 1.0))
    err = np.abs(col - g["colors"]).max()
    print(f"volume forward vs reference: max err {err:.2e}")
    assert err <= 2e-4  # colours integrate alpha = f(s * d) with s = 20: SDF ulps are amplified ~x20, FD normals feed the colour MLP
    assert (np.abs(col - g["colors"]).max(axis=1) <= 1e-5).mean() >= 0.99
    assert np.all(col[:20] == 1.0)  # rays that miss the box: background
    col2 = hooks.volume_forward(distilled_field, g["origins"], g["dirs"], 16, None, (0.2, 0.4, 0.6))
    assert np.abs(col2 - g["colors_nojitter"]).max() <= 2e-4
    o = oracle.volume_forward(distilled_oracle, g["origins"], g["dirs"], 16, None, (0.2, 0.4, 0.6), s=float(g["s"]))
    assert np.abs(col2 - o).max() <= 2e-4
    with pytest.raises(ValueError):
        hooks.volume_forward(distilled_field, g["origins"], g["dirs"], 1)
