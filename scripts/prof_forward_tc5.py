import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_10885_b200 import grid
dev = grid.device_field(grid.field_init(grid.GridConfig(resolution=16), seed=0))
dev.set_precision(sys.argv[1] if len(sys.argv) > 1 else "tensor_fp16x2")
pts = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, (1 << 22, 3)).astype(np.float32), device="cuda")
for _ in range(3):
    grid.sdf_query(dev, pts)
torch.cuda.synchronize()
