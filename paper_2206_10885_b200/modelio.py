""".knf model files: same format as the reference ``kilofield.modelio`` (modelio.py:1-14).

``load_model`` / ``save_model`` are the host-side forms (NumPy stacks in a KiloField);
``load_model_to_device`` is SURVEY 8(f).1 -- the file goes straight to the GPU's cell-major
blob layout through knf_field_create_from_knf, with the same magic / version / truncation /
CRC32 checks.
"""

from __future__ import annotations

import struct
import zlib

import numpy as np

from .grid import COLOR_ACTIVATIONS, SDF_ACTIVATIONS, DeviceField, GridConfig, KiloField, MlpGrid

MAGIC = b"KNSF"
FORMAT_VERSION = 1
_ACT_CODE = {"identity": 0, "relu": 1, "softplus": 2, "sigmoid": 3}
_ACT_NAME = {v: k for k, v in _ACT_CODE.items()}


class ModelIOError(Exception):
    pass


class BadMagicError(ModelIOError):
    pass


class VersionMismatchError(ModelIOError):
    pass


class TruncatedPayloadError(ModelIOError):
    pass


class ChecksumError(ModelIOError):
    pass


def _spec_bytes(fam: MlpGrid) -> bytes:
    k = len(fam.weights)
    return struct.pack(f"<I{k + 1}I{k}I", k, *fam.layer_dims, *[_ACT_CODE[a] for a in fam.activations])


def _header(field: KiloField) -> bytes:
    c = field.config
    return b"".join([MAGIC, struct.pack("<II", FORMAT_VERSION, c.resolution), struct.pack("<6f", *c.bbox_min, *c.bbox_max),
                     struct.pack("<III", c.feature_dim, c.sdf_freqs, c.dir_freqs), _spec_bytes(field.sdf),
                     _spec_bytes(field.color)])


def _rows(fam: MlpGrid) -> np.ndarray:
    # one row per cell: W1 | b1 | W2 | b2 | W3 | b3 (modelio.py:72-78)
    parts = []
    for w, b in zip(fam.weights, fam.biases):
        parts += [np.asarray(w, "<f4").reshape(fam.n_cells, -1), np.asarray(b, "<f4").reshape(fam.n_cells, -1)]
    return np.concatenate(parts, axis=1)


def save_model(field: KiloField, path):
    payload = np.asarray(field.inv_std_param, "<f4").tobytes() + _rows(field.sdf).tobytes() + _rows(field.color).tobytes()
    with open(path, "wb") as fh:
        fh.write(_header(field))
        fh.write(payload)
        fh.write(struct.pack("<I", zlib.crc32(payload) & 0xFFFFFFFF))


def _read_spec(buf, off):
    (k,) = struct.unpack_from("<I", buf, off)
    dims = list(struct.unpack_from(f"<{k + 1}I", buf, off + 4))
    codes = struct.unpack_from(f"<{k}I", buf, off + 4 + 4 * (k + 1))
    try:
        acts = [_ACT_NAME[c] for c in codes]
    except KeyError as e:
        raise ModelIOError(f"unknown activation code {e}") from None
    return dims, acts, off + 4 + 4 * (k + 1) + 4 * k


def _split(flat, n_cells, dims, acts) -> MlpGrid:
    rows = flat.reshape(n_cells, -1)
    ws, bs, col = [], [], 0
    for fin, fout in zip(dims[:-1], dims[1:]):
        ws.append(np.ascontiguousarray(rows[:, col : col + fin * fout].reshape(n_cells, fout, fin), dtype=np.float32))
        col += fin * fout
        bs.append(np.ascontiguousarray(rows[:, col : col + fout], dtype=np.float32))
        col += fout
    return MlpGrid(dims, acts, ws, bs)


def load_model(path) -> KiloField:
    with open(path, "rb") as fh:
        buf = fh.read()
    if buf[:4] != MAGIC:
        raise BadMagicError(f"expected {MAGIC!r}, found {buf[:4]!r}")
    version, n = struct.unpack_from("<II", buf, 4)
    if version != FORMAT_VERSION:
        raise VersionMismatchError(f"format version {version}, supported {FORMAT_VERSION}")
    bbox = struct.unpack_from("<6f", buf, 12)
    feat, lx, lv = struct.unpack_from("<III", buf, 36)
    sdf_dims, sdf_acts, off = _read_spec(buf, 48)
    col_dims, col_acts, off = _read_spec(buf, off)
    cfg = GridConfig(resolution=n, bbox_min=bbox[:3], bbox_max=bbox[3:], sdf_freqs=lx, dir_freqs=lv, feature_dim=feat)
    per = lambda d: sum(a * b + b for a, b in zip(d[:-1], d[1:]))
    n_sdf, n_col = per(sdf_dims) * cfg.n_cells, per(col_dims) * cfg.n_cells
    size = 4 * (1 + n_sdf + n_col)
    if len(buf) < off + size + 4:
        raise TruncatedPayloadError(f"file has {len(buf)} bytes, needs {off + size + 4}")
    payload = buf[off : off + size]
    if zlib.crc32(payload) & 0xFFFFFFFF != struct.unpack_from("<I", buf, off + size)[0]:
        raise ChecksumError("payload CRC32 mismatch")
    vals = np.frombuffer(payload, dtype="<f4")
    return KiloField(cfg, _split(vals[1 : 1 + n_sdf], cfg.n_cells, sdf_dims, sdf_acts),
                     _split(vals[1 + n_sdf :], cfg.n_cells, col_dims, col_acts), np.array(vals[0], dtype=np.float32))


def load_model_to_device(path, device: int | None = None) -> DeviceField:
    """File -> device blobs without building the stacked host arrays in Python."""
    return DeviceField.from_knf(path, device)
