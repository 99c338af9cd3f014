import os, sys, subprocess
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2405_03474_b200 as rld
from oracle import rstar_oracle as O
n, m, d = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
g = np.random.default_rng(n + m)
pts = g.standard_normal((n, d))
spec = rld.KernelSpec("rbf", 1.0, 1.5, 1e-3)
R = rld.ResidentMatrix(rld.KernelMatrix(spec, pts), dtype="fp32", path=sys.argv[4])
V = g.standard_normal((m, n))
Y = R.kv_apply(torch.from_numpy(V).cuda()).cpu().numpy()
rows = g.choice(n, 8, replace=False)
err = 0
for i in rows:
    k = O.covariance_block("rbf", 1.0, 1.5, 1e-3, pts, rows=slice(i, i + 1))[0].astype(np.float32).astype(np.float64)
    err = max(err, float(np.max(np.abs(Y[:, i] - V @ k) / (np.abs(V) @ np.abs(k)))))
print("ok", err)
'''
for env, n, m, path in [({}, 19968, 128, "stored"), ({}, 65536, 128, "stored"), ({}, 24960, 300, "stored"),
                        ({}, 39936, 522, "stored"), ({}, 4099, 70, "stored")]:
    r = subprocess.run([sys.executable, "-c", code, str(n), str(m), "4", path], capture_output=True, text=True, timeout=300,
                       env={**os.environ, **env})
    print(env, n, m, path, (r.stdout.strip().splitlines() or ["?"])[-1], flush=True)
