"""Time rld_dense_eigh (tri_eig.cu, or DSYEVD with RLD_TRI_EIG=0) at the preconditioner sizes (argv: sizes)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_03474_b200._session import session  # noqa: E402

s = session()
for n in [int(a) for a in sys.argv[1:]] or (74, 256, 266, 288, 512, 522, 544, 1034, 2058):
    g = np.random.default_rng(n)
    Q, _ = np.linalg.qr(g.standard_normal((n, n)))
    A0 = torch.from_numpy((Q * np.logspace(4, -2, n)) @ Q.T).cuda()
    A = A0.clone()
    w = torch.empty(n, dtype=torch.float64, device="cuda")
    best = 1e9
    for _ in range(6):
        A.copy_(A0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.handle.check(s.lib.rld_dense_eigh(s.handle.ptr, n, A.data_ptr(), w.data_ptr()), "eigh")
        best = min(best, time.perf_counter() - t0)
    print(f"n={n}: {best * 1e3:.3f} ms", flush=True)
