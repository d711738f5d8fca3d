"""CPU-side checks of the drop-in boundary: the C-ABI library builds, loads, exports every symbol
include/knf_b200.h declares, and fails loudly (no CPU fallback) when there is no GPU."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "knf_b200.h")


def _declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(knf_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as g
    from paper_2206_10885_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        g.build()
    return _native.load()


def test_header_symbols_all_exported(lib):
    from paper_2206_10885_b200 import _native

    declared = _declared_symbols()
    assert len(declared) >= 26
    raw = ctypes.CDLL(_native.LIB_PATH)
    for name in declared:
        assert hasattr(raw, name), f"{name} declared in knf_b200.h but not exported"
    assert set(declared) == set(_native.EXPORTED_SYMBOLS), "ctypes binding and header disagree"


def test_abi_version(lib):
    assert lib.knf_abi_version() == 2


def test_struct_sizes_match_c_layout():
    from paper_2206_10885_b200 import _native as N

    assert ctypes.sizeof(N.KnfCamera) == 3 * 8 + 9 * 8 + 8 + 4 + 4
    assert ctypes.sizeof(N.KnfSettings) == 24
    assert ctypes.sizeof(N.KnfStats) == 112 + 6 * 8  # + filter_evals, filter_deferred, filter_skipped, filter_lane_slots, filter_launches, filter_ms
    assert ctypes.sizeof(N.KnfFieldDesc) == 8 + 48 + 16 + 8 + 12 * 8


def _has_gpu():
    from paper_2206_10885_b200 import _native as N

    try:
        return N.device_count() > 0
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="only meaningful on a box without a GPU")
def test_no_cpu_fallback(lib):
    from paper_2206_10885_b200 import _native as N
    from paper_2206_10885_b200 import grid

    field = grid.field_init(grid.GridConfig(resolution=2), seed=0)
    with pytest.raises(N.KnfError):
        grid.sdf_query(field, np.zeros((4, 3), np.float32))


def test_missing_library_is_loud(monkeypatch, tmp_path):
    from paper_2206_10885_b200 import _native as N

    monkeypatch.setattr(N, "_lib", None)
    monkeypatch.setattr(N, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(N.NativeLibraryMissing):
        N.load()


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2206_10885_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "/root/reference" not in text or f.endswith((".cu", ".cuh", ".h")), f


def test_host_side_containers_match_reference_init(small_field, small_oracle):
    for a, b in zip(small_field.sdf.weights + small_field.color.weights, small_oracle.sdf.W + small_oracle.color.W):
        assert np.array_equal(a, b)


def test_knf_roundtrip(tmp_path, small_field):
    from paper_2206_10885_b200 import modelio

    p = tmp_path / "m.knf"
    modelio.save_model(small_field, p)
    back = modelio.load_model(p)
    assert np.array_equal(back.sdf.weights[0], small_field.sdf.weights[0])
    assert np.array_equal(back.color.biases[2], small_field.color.biases[2])
    raw = bytearray(open(p, "rb").read())
    raw[200] ^= 0xFF
    open(p, "wb").write(bytes(raw))
    with pytest.raises(modelio.ChecksumError):
        modelio.load_model(p)
    open(p, "wb").write(bytes(raw[:1000]))
    with pytest.raises(modelio.TruncatedPayloadError):
        modelio.load_model(p)
    open(p, "wb").write(b"XXXX" + bytes(raw[4:]))
    with pytest.raises(modelio.BadMagicError):
        modelio.load_model(p)


def test_settings_and_pose_validation():
    from paper_2206_10885_b200 import cameras, surface

    with pytest.raises(ValueError):
        surface.RenderSettings(step_scale=1.5)
    with pytest.raises(ValueError):
        surface.RenderSettings(render_pass="albedo")
    with pytest.raises(ValueError):
        cameras.look_at_pose((0, 0, 0), (0, 0, 0), (0, 1, 0), 0.5, 4, 4)
    with pytest.raises(ValueError):
        cameras.CameraPose((0, 0, 0), np.eye(3), 4.0, 4, 4)
