"""BASELINE config 4: batched SDF forward throughput per precision mode (device resident, CUDA events)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2206_10885_b200 import grid
import oracle
from bench import _event_ms
f16 = grid.field_init(grid.GridConfig(resolution=16), seed=0)
dev = grid.device_field(f16)
of = oracle.make_random_field(oracle.FieldSpec(resolution=16), seed=0)
for M in (1_000_000, 1 << 24):
    pts_np = np.random.default_rng(0).uniform(-1, 1, (M, 3)).astype(np.float32)
    pts = torch.as_tensor(pts_np, device="cuda")
    for mode in ("fp32_chain", "tensor_bf16x3", "tensor_fp16x2"):
        dev.set_precision(mode)
        ms = _event_ms(lambda: grid.sdf_query(dev, pts), warm=2, it=5)
        line = f"M={M} {mode:14s} {ms:8.3f} ms  {M / ms / 1e6:6.2f} Gq/s  {M * 5120 / ms / 1e9:6.1f} TFLOP/s"
        if M == 1_000_000:
            got = grid.sdf_query(dev, pts[:200000])
            ov, ofe = oracle.query_sdf(of, pts_np[:200000])
            line += f"  max|value - oracle| {np.abs(got.value.cpu().numpy() - ov).max():.2e} features {np.abs(got.features.cpu().numpy() - ofe).max():.2e}"
        print(line, flush=True)
dev.set_precision("fp32_chain")
