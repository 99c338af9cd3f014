"""Time rld_dense_eigh at the preconditioner sizes on several spectra; with RLD_TRI_EIG_DEBUG=1 the
library reports fallbacks to DSYEVD."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_03474_b200._session import session  # noqa: E402

s = session()
for spec in ("decaying", "wishart", "degenerate"):
    for n in (74, 266, 288):
        g = np.random.default_rng(n)
        Q, _ = np.linalg.qr(g.standard_normal((n, n)))
        if spec == "decaying":
            lam = np.logspace(4, -2, n)
        elif spec == "degenerate":
            lam = np.repeat([5.0, 2.0, 2.0, 0.5], -(-n // 4))[:n]
        else:
            X = g.standard_normal((n + 5, n))
            lam = None
        An = X.T @ X if lam is None else (Q * lam) @ Q.T
        An = (An + An.T) / 2
        A0 = torch.from_numpy(An).cuda()
        A = A0.clone()
        w = torch.empty(n, dtype=torch.float64, device="cuda")
        best = 1e9
        for _ in range(6):
            A.copy_(A0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s.handle.check(s.lib.rld_dense_eigh(s.handle.ptr, n, A.data_ptr(), w.data_ptr()), "eigh")
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        V = A.cpu().numpy().T
        wv = w.cpu().numpy()
        err = np.linalg.norm((V * wv) @ V.T - An) / np.linalg.norm(An)
        orth = np.linalg.norm(V.T @ V - np.eye(n))
        print(f"{spec:10s} n={n}: {best * 1e3:.3f} ms  recon {err:.1e} orth {orth:.1e}", flush=True)
