"""Exhaustive measurement of |fp32 feature - true feature| of nn.fourier_encode (nn.py:66-93) as the kernels evaluate it
(NumPy's float32 sin / cos at octave 0, then the rounded double-angle recurrence): EVERY float32 x with |x| <= 1.001 goes
through knf_fourier_encode on the device and is compared with sin / cos(2^o pi x) in float64.  The per-octave maxima are the
constants kFeatureErr in csrc/knf_api.cu (certified skipping compares the exact kernel's distances at two points through a
Lipschitz bound of the REAL-arithmetic network, so the features' own error enters the filter bound delta twice)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2206_10885_b200 import _native as N
lib = N.load()
dev = torch.device("cuda", 0)
L = 6
hi_bits = int(np.float32(1.001).view(np.int32))
CH = 3 << 22  # values per chunk (3 per point)
worst = torch.zeros((L, 2), dtype=torch.float64, device=dev)
worst_x = torch.zeros((L, 2), dtype=torch.float64, device=dev)
n_total = 0
for sign in (0, 1):
    for b0 in range(0, hi_bits + 1, CH):
        b1 = min(b0 + CH, hi_bits + 1)
        bits = torch.arange(b0, b1, dtype=torch.int64, device=dev)
        pad = (-len(bits)) % 3
        if pad:
            bits = torch.cat([bits, bits[-1:].repeat(pad)])
        bits = (bits | (sign << 31)).to(torch.int32) if sign == 0 else (bits - (1 << 31)).to(torch.int32)
        x = bits.view(torch.float32).reshape(-1, 3).contiguous()
        out = torch.empty((x.shape[0], 3 + 6 * L), dtype=torch.float32, device=dev)
        N.check(lib.knf_fourier_encode(x.data_ptr(), x.shape[0], L, out.data_ptr(), 0, N.MEM_DEVICE, N.current_stream(0)))
        xd = x.double()
        for o in range(L):
            ang = (2.0 ** o) * np.pi * xd
            es = (out[:, 3 + 6 * o : 6 + 6 * o].double() - torch.sin(ang)).abs()
            ec = (out[:, 6 + 6 * o : 9 + 6 * o].double() - torch.cos(ang)).abs()
            for j, e in enumerate((es, ec)):
                m = e.max()
                if m > worst[o, j]:
                    worst[o, j] = m
                    worst_x[o, j] = xd.reshape(-1)[e.reshape(-1).argmax()]
        n_total += b1 - b0
        assert torch.equal(out[:, 0:3], x)
u = 2.0 ** -24
res = {"inputs": n_total, "range": 1.001, "max_abs_error": worst.cpu().tolist(), "in_units_of_2^-24": (worst / u).cpu().tolist(), "at_x": worst_x.cpu().tolist()}
print(json.dumps(res))
for o in range(L):
    print(f"octave {o}: sin {worst[o,0].item():.3e} ({worst[o,0].item()/u:.1f} u)  cos {worst[o,1].item():.3e} ({worst[o,1].item()/u:.1f} u)")
