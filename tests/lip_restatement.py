"""float64 NumPy restatement of csrc/knf_bounds.cuh (sub-box refinement of the per-cell Lipschitz bounds behind the decision
filter's certified skipping) -- test infrastructure.  There is no reference counterpart: the reference evaluates every crawl
sample (surface.py:217-223); the bound only decides which of those evaluations the product may skip, and every result stays
bit-identical to evaluating them all (tests/test_gpu_filter.py).  The restatement follows the header comment of
knf_bounds.cuh step by step, vectorised over the sub-boxes of one cell."""

import numpy as np

K_LIP_SLACK = 1.0e-5  # knf_common.cuh kLipSlack


def _sig(z):
    return 1.0 / (1.0 + np.exp(-z))


def _trig_range(lo, hi):
    def rng(fn, peak):
        a, b = fn(lo), fn(hi)
        mn, mx = np.minimum(a, b), np.maximum(a, b)
        has_max = (peak + 2 * np.pi * np.ceil((lo - peak) / (2 * np.pi))) <= hi
        has_min = (peak + np.pi + 2 * np.pi * np.ceil((lo - peak - np.pi) / (2 * np.pi))) <= hi
        mx = np.where(has_max, 1.0, mx)
        mn = np.where(has_min, -1.0, mn)
        return (mn + mx) / 2, (mx - mn) / 2

    return rng(np.sin, np.pi / 2) + rng(np.cos, 0.0)


def spectral_norm_bound(W2):
    """The closed-form code's upper bound on |W2|_2: Gershgorin on (W2^T W2)^16 (knf_api.cu lipschitz_bound)."""
    G = W2.T @ W2
    log_scale = 0.0
    for _ in range(4):
        mx = np.abs(G).max()
        if mx > 0:
            G = G / mx
            log_scale = 2.0 * (log_scale + np.log(mx))
        else:
            log_scale *= 2.0
        G = G @ G
    row = np.abs(G).sum(1).max()
    return np.exp((np.log(row) + log_scale) / 32.0) if row > 0 else 0.0


def closed_form(W1, W2, w3):
    n3, n2 = np.linalg.norm(w3), spectral_norm_bound(W2)
    out = np.zeros(3)
    for a in range(3):
        m = np.linalg.norm(W1[:, a])
        for o in range(6):
            m += 2.0 ** o * np.pi * np.linalg.norm(np.stack([W1[:, 3 + 6 * o + a], W1[:, 6 + 6 * o + a]], 1), 2)
        out[a] = 1.001 * n3 * n2 * m + 1e-12
    return out


def refine_cell(field, c, width, fine, chunk=32768):
    """Refined bounds (3,) of cell c for target sub-box width `width` and `fine` Taylor samples -- what lip_store_kernel
    writes, before the minimum with the closed form and the fp32 round-up."""
    cfg = field.config
    N = int(cfg.resolution)
    W1, W2 = (np.asarray(field.sdf.weights[k][c], np.float64) for k in range(2))
    w3 = np.asarray(field.sdf.weights[2][c][0], np.float64)
    b1, b2 = (np.asarray(field.sdf.biases[k][c], np.float64) for k in range(2))
    A1, A2 = np.abs(W1), np.abs(W2)
    lo, hi = np.asarray(cfg.bbox_min, np.float64), np.asarray(cfg.bbox_max, np.float64)
    ext = hi - lo
    cell_w = (ext / N).max()
    coord = max(np.abs(lo).max(), np.abs(hi).max())
    k = int(max(1.0, min(64.0, np.ceil(cell_w / width))))
    margin = 4.0 * K_LIP_SLACK * cell_w + 4e-7 * coord
    ci = np.array([c // (N * N), (c // N) % N, c % N])
    elo = lo + ext * ci / N - margin
    ehi = lo + ext * (ci + 1) / N + margin
    wsub = (ehi - elo) / k
    n3, n2, n2f = np.linalg.norm(w3), spectral_norm_bound(W2) * 1.0001, np.linalg.norm(W2)
    k3 = np.zeros(3)
    for a in range(3):
        for o in range(6):
            k3[a] += (2.0 ** o * np.pi) ** 3 * np.linalg.norm(np.stack([W1[:, 3 + 6 * o + a], W1[:, 6 + 6 * o + a]], 1), 2)
    # Taylor samples of g_a and g_a' along each axis: (k * fine, 32)
    g, gp = [], []
    for a in range(3):
        xs = elo[a] + wsub[a] * (np.arange(k * fine) + 0.5) / fine
        ga = np.tile(W1[:, a], (k * fine, 1))
        gpa = np.zeros((k * fine, 32))
        for o in range(6):
            f = 2.0 ** o * np.pi
            ws, wc = W1[:, 3 + 6 * o + a], W1[:, 6 + 6 * o + a]
            ga = ga + f * (np.outer(np.cos(f * xs), ws) - np.outer(np.sin(f * xs), wc))
            gpa = gpa - f * f * (np.outer(np.sin(f * xs), ws) + np.outer(np.cos(f * xs), wc))
        g.append(ga)
        gp.append(gpa)
    best = np.zeros(3)
    idx = np.arange(k ** 3)
    for s0 in range(0, k ** 3, chunk):
        s = idx[s0 : s0 + chunk]
        si = np.stack([s // (k * k), (s // k) % k, s % k], 1)
        n = len(s)
        xlo, xhi = elo + wsub * si, elo + wsub * (si + 1)
        pc, pr = np.zeros((n, 39)), np.zeros((n, 39))
        pc[:, :3] = elo + wsub * (si + 0.5)
        pr[:, :3] = 0.5 * wsub * (1 + 1e-12) + 1e-13
        for o in range(6):
            f = 2.0 ** o * np.pi
            sc, sr, cc, cr = _trig_range(f * xlo, f * xhi)
            pc[:, 3 + 6 * o : 6 + 6 * o], pr[:, 3 + 6 * o : 6 + 6 * o] = sc, sr + 1e-12
            pc[:, 6 + 6 * o : 9 + 6 * o], pr[:, 6 + 6 * o : 9 + 6 * o] = cc, cr + 1e-12
        z1c = pc @ W1.T + b1
        z1r = pr @ A1.T
        z1r = z1r + 1e-12 * (np.abs(z1c) + z1r) + 1e-13
        s1l, s1u = _sig(z1c - z1r), _sig(z1c + z1r)
        c1, r1 = (s1l + s1u) / 2, (s1u - s1l) / 2 + 1e-13
        h1l, h1u = np.logaddexp(0, z1c - z1r), np.logaddexp(0, z1c + z1r)
        h1c, h1r = (h1l + h1u) / 2, (h1u - h1l) / 2 * (1 + 1e-12) + 1e-13
        z2c = h1c @ W2.T + b2
        z2r = h1r @ A2.T
        z2r = z2r + 1e-12 * (np.abs(z2c) + z2r) + 1e-13
        s2l, s2u = _sig(z2c - z2r), _sig(z2c + z2r)
        c2, r2 = (s2l + s2u) / 2, (s2u - s2l) / 2 + 1e-13
        rw = r2 * np.abs(w3)
        vt = (c2 * w3) @ W2
        q = rw @ A2
        nrw = np.linalg.norm(rw, axis=1)
        for a in range(3):
            h = 0.5 * wsub[a] / fine
            rem_a = 2.0 * n3 * n2 * (0.5 * h * h * k3[a])
            rem_b = (2.0 * n3 * n2 + n3 * n2f) * (0.5 * h * h * k3[a])
            for i in range(fine):
                gg, ggp = g[a][si[:, a] * fine + i], gp[a][si[:, a] * fine + i]
                cg, cgp = c1 * gg, c1 * ggp
                u, up = cg @ W2.T, cgp @ W2.T
                rg, rgp = r1 * np.abs(gg), r1 * np.abs(ggp)
                base = (np.abs((vt * cg).sum(1)) + h * np.abs((vt * cgp).sum(1))
                        + (rw * np.abs(u) + np.abs(vt) * rg).sum(1) + h * (rw * np.abs(up) + np.abs(vt) * rgp).sum(1))
                tot_a = base + nrw * n2 * (np.linalg.norm(rg, axis=1) + h * np.linalg.norm(rgp, axis=1)) + rem_a
                tot_b = base + (q * (rg + h * rgp)).sum(1) + rem_b
                best[a] = max(best[a], np.minimum(tot_a, tot_b).max())
    return 1.001 * best + 1e-12


def sampled_gradient_max(field, c, n=40000, seed=0):
    """max over n random points of the cell of |d d / d x_a| (float64 network, central differences)."""
    cfg = field.config
    N = int(cfg.resolution)
    W = [np.asarray(field.sdf.weights[k][c], np.float64) for k in range(3)]
    B = [np.asarray(field.sdf.biases[k][c], np.float64) for k in range(3)]
    lo, hi = np.asarray(cfg.bbox_min, np.float64), np.asarray(cfg.bbox_max, np.float64)
    ci = np.array([c // (N * N), (c // N) % N, c % N])
    x = lo + (hi - lo) * (ci + np.random.default_rng(seed).uniform(0, 1, (n, 3))) / N

    def fwd(x):
        f = [x]
        for o in range(6):
            f += [np.sin(2.0 ** o * np.pi * x), np.cos(2.0 ** o * np.pi * x)]
        h = np.logaddexp(0, np.concatenate(f, -1) @ W[0].T + B[0])
        h = np.logaddexp(0, h @ W[1].T + B[1])
        return h @ W[2][0] + B[2][0]

    e = 1e-6
    return np.stack([np.abs(fwd(x + e * np.eye(3)[a]) - fwd(x - e * np.eye(3)[a])) / (2 * e) for a in range(3)], 1).max(0)
