"""Time rld_dense_cholesky (one-cluster kernel, or cuSOLVER with RLD_SMALL_CHOL=0) at the CholQR sizes."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_03474_b200._session import session  # noqa: E402

s = session()
for n in [int(a) for a in sys.argv[1:]] or (74, 256, 266, 512, 522, 640, 1024, 2048):
    g = np.random.default_rng(n)
    X = g.standard_normal((n + 8, n))
    G0 = torch.from_numpy(X.T @ X).cuda()
    G = G0.clone()
    info = C.c_int32(0)
    best = 1e9
    for r in range(8):
        G.copy_(G0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.handle.check(s.lib.rld_dense_cholesky(s.handle.ptr, n, G.data_ptr(), C.byref(info)), "chol")
        best = min(best, time.perf_counter() - t0)
    print(f"n={n} info={info.value} best wall {best * 1e6:.1f} us", flush=True)
