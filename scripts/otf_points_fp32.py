import numpy as np, sys, time
sys.path.insert(0,'/root/repo')
from oracle import rstar_oracle as O
def run(pts, fam, ell, jit, order, s, k):
    K = O.covariance_block(fam, 1.0, ell, jit, pts)
    return O.rstar_dense(K, order=order, s=s, t=20, k=k, q=5, seed=0).value
rng = np.random.default_rng(0)
n = 8192
# config-5 style: spacing ~0.01 with ell=0.02, coordinates rounded as fp32 at magnitude ~0.5
p = rng.uniform(0, 0.2, (n, 3)) + 0.4
for name, pts in [("c5", p)]:
    v64 = run(pts, "matern52", 0.02, 1e-1, 3, 16, 16)
    p32 = pts.astype(np.float32).astype(np.float64)
    v32 = run(p32, "matern52", 0.02, 1e-1, 3, 16, 16)
    print(name, v64, v32, abs(v32-v64)/abs(v64), flush=True)
# config-4 style: clusters std scaled so density matches, ell=0.1, RBF jitter 1e-2
cent = rng.uniform(0.2, 0.8, (16, 3)); lab = rng.integers(0, 16, n)
p = cent[lab] + 0.0157 * rng.standard_normal((n, 3))
v64 = run(p, "rbf", 0.1, 1e-2, 5, 16, 32)
v32 = run(p.astype(np.float32).astype(np.float64), "rbf", 0.1, 1e-2, 5, 16, 32)
print("c4", v64, v32, abs(v32-v64)/abs(v64))
