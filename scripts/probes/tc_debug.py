"""Bring-up probe: tensor-core Hermitian of small inputs, compared with numpy."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1603_03820_b200 import alskit as A
from paper_1603_03820_b200.session import PREC_TF32X2, DeviceCsr, dev_hermitian
np.set_printoptions(linewidth=220, precision=4, suppress=True)
dev = torch.device('cuda')
for f in (16, 32, 33, 36, 40, 100):
    n = 500
    thf = A.random_factor(n, f, 5)
    th = thf.entries.reshape(n, f)
    for lengths in ([1], [1, 1], [3, 1, 40], [0, 1, 2, 3]):
        rng = np.random.default_rng(1)
        rp = np.zeros(len(lengths) + 1, np.int64); rp[1:] = np.cumsum(lengths)
        cols = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lengths]).astype(np.int32)
        vals = rng.uniform(1, 5, len(cols)).astype(np.float32)
        m = len(lengths)
        r = A.CsrMatrix(m, n, 0, rp, cols, vals)
        R = DeviceCsr.from_host(r, dev)
        T = torch.from_numpy(thf.entries).to(dev)
        a = torch.zeros(m * f * f, dtype=torch.float32, device=dev)
        b = torch.zeros(m * f, dtype=torch.float32, device=dev)
        dev_hermitian(R, T, n, f, 0.0, PREC_TF32X2, a, b)
        a = a.cpu().numpy().reshape(m, f, f); b = b.cpu().numpy().reshape(m, f)
        for u in range(m):
            c = cols[rp[u]:rp[u + 1]]; v = vals[rp[u]:rp[u + 1]]
            g = th[c].astype(np.float64).T @ th[c]
            bb = (v[:, None] * th[c]).sum(0)
            ea, eb = np.abs(a[u] - g).max(), np.abs(b[u] - bb).max()
            print(f"f={f} lengths={lengths} u={u} errA={ea:.2e} errB={eb:.2e}")
            if ea > 1e-4:
                bad = np.argwhere(np.abs(a[u] - g) > 1e-4)
                print("  bad entries (first 10):", bad[:10].tolist(), "count", len(bad))
                i, j = bad[0]
                print("  dev", a[u][i, :8], "\n  exp", g[i, :8])
