"""Test-only numpy mirror of librld's row-sharded dataflow (rld_api.cu
build_preconditioner() / run_estimate() / gather_rows()).

Every rank holds rows [row0, row1) of K and of every n-vector block, exactly
as ``paper_2405_03474_b200.parallel.shard_bounds`` and prepare() split them.
The only exchanges are the ones the device path makes through NCCL:

* ``gather``  -- the all-gather of an m x L padded row block + relayout into
  the m x n rows layout (gather_rows: sketch Q per power iteration, the
  Lanczos direction block x_j per step);
* ``allreduce`` -- sums of Gram matrices (CholQR), B = Q K Q^T, the k x k
  inner Gram, sum log base, the fused dot products and the U^T X partials.

Eigensolves, the inner Cholesky, Thomas solves and the Hutchinson mean run
replicated.  The CPU test runs this under ``gloo`` at world sizes 1/2/3 and
checks that the sharded estimate equals the world-1 one and the oracle, which
validates the decomposition the CUDA path implements (the device kernels
themselves are checked by the ``-m gpu`` parity tests).
"""

from __future__ import annotations

import numpy as np

from oracle.rstar_oracle import BREAKDOWN_RTOL, DIAG_FLOOR, KEEP_RTOL, PARTIAL_FRACTIONS, thomas


class Comm:
    """world == 1: identity collectives; otherwise torch.distributed (gloo)."""

    def __init__(self, world: int, rank: int):
        self.world, self.rank = world, rank

    def allreduce(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        if self.world == 1:
            return a
        import torch
        import torch.distributed as dist

        t = torch.from_numpy(a.copy())
        dist.all_reduce(t)
        return t.numpy()

    def gather(self, local, n):
        """local: m x rows -> m x n (gather_rows: pad to L, all-gather [G][m][L], relayout)."""
        m, rows = local.shape
        if self.world == 1:
            return local.copy()
        import torch
        import torch.distributed as dist

        L = -(-n // self.world)
        snd = np.zeros((m, L))
        snd[:, :rows] = local
        parts = [torch.zeros(m * L, dtype=torch.float64) for _ in range(self.world)]
        dist.all_gather(parts, torch.from_numpy(snd.reshape(-1)))
        rcv = np.stack([p.numpy().reshape(m, L) for p in parts])          # [G][m][L]
        full = np.empty((m, n))
        for j in range(n):                                                 # relayout_kernel
            g, jj = divmod(j, L)
            full[:, j] = rcv[g, :, jj]
        return full


def cholqr(Zl, comm, passes):
    for _ in range(passes):
        G = comm.allreduce(Zl @ Zl.T)
        R = np.linalg.cholesky(G).T                                        # G = R^T R
        Zl = np.linalg.solve(R.T, Zl)                                      # rows: Z <- R^-T Z
    return Zl


def sharded_rstar(K, row0, row1, comm, order, V, omega, k, q, t):
    """r* estimate with K[row0:row1, :] on this rank.  V: s x n probes, omega: w x n."""
    n = K.shape[0]
    Kl = K[row0:row1, :]
    diag_l = np.diag(K)[row0:row1]
    # ---- preconditioner (build_preconditioner)
    Y = np.array(omega, dtype=np.float64)
    for it in range(q):
        Zl = Y @ Kl.T                                                      # w x nl (K symmetric)
        Zl = cholqr(Zl, comm, 2 if it + 1 == q else 1)
        Y = comm.gather(Zl, n)
    Zl = Y @ Kl.T
    Ql = Y[:, row0:row1]
    B = comm.allreduce(Ql @ Zl.T)
    theta, Ub = np.linalg.eigh(B)
    top = np.argsort(theta)[::-1][:k]
    A = (Ql.T @ Ub[:, top]) * np.sqrt(np.maximum(theta[top], 0.0))       # nl x k
    base = np.maximum(diag_l - np.sum(A * A, axis=1), DIAG_FLOOR)
    sb = np.sqrt(base)
    logdet_base = comm.allreduce(np.array([np.sum(np.log(base))]))[0]
    At = A / sb[:, None]
    C = comm.allreduce(At.T @ At)
    L = np.linalg.cholesky(np.eye(k) + C)
    logdet_P = logdet_base + 2.0 * np.sum(np.log(np.diag(L)))
    lam, W = np.linalg.eigh(C)
    keep = lam > KEEP_RTOL * max(lam[-1], 1.0)
    U = At @ (W[:, keep] / np.sqrt(lam[keep]))                             # nl x kept
    lam = lam[keep]
    hfac = 1.0 / (1.0 + lam) - 1.0
    gfac = 1.0 / np.sqrt(1.0 + lam) - 1.0
    cfac = np.sqrt(1.0 + lam) - 1.0

    # ---- two-sequence preconditioned Lanczos (run_estimate), s columns in lock step
    Vl = np.asarray(V, dtype=np.float64)[:, row0:row1].T                   # nl x s
    s = Vl.shape[1]
    norms = np.sqrt(comm.allreduce(np.sum(Vl * Vl, axis=0)))
    q0 = Vl / norms
    T = comm.allreduce(U.T @ q0)
    x = (q0 + U @ (gfac[:, None] * T)) / sb[:, None]                       # N^-T q0
    p = (q0 + U @ (cfac[:, None] * T)) * sb[:, None]                       # N q0
    pp = np.zeros_like(p)
    alpha = np.zeros((s, t))
    beta = np.zeros((s, t))
    beta_ref = np.full(s, np.nan)
    live = np.ones(s, dtype=bool)
    size = np.full(s, t)
    for j in range(t):
        xfull = comm.gather(x.T, n)                                        # s x n
        KX = Kl @ xfull.T                                                  # nl x s
        a = comm.allreduce(np.sum(x * KX, axis=0))
        alpha[:, j] = np.where(live, a, alpha[:, j])
        if j == t - 1:
            break
        bprev = beta[:, j - 1] if j else np.zeros(s)
        u = KX - alpha[:, j] * p - bprev * pp
        wv = u / sb[:, None]
        T = comm.allreduce(U.T @ wv)
        z = (wv + U @ (hfac[:, None] * T)) / sb[:, None]                   # P^-1 u
        b = np.sqrt(np.maximum(comm.allreduce(np.sum(u * z, axis=0)), 0.0))
        beta_ref = np.where(np.isnan(beta_ref), b, beta_ref)
        broke = live & (b <= BREAKDOWN_RTOL * np.maximum(beta_ref, np.abs(alpha[:, j])))
        size[broke] = j + 1
        live &= ~broke
        beta[:, j] = np.where(live, b, 0.0)
        safe = np.where(live, b, 1.0)
        pp, p = p, np.where(live, u / safe, 0.0)
        x = np.where(live, z / safe, 0.0)

    # ---- multishift Thomas + Hutchinson (thomas_hutchinson), replicated
    off, poles, residues = PARTIAL_FRACTIONS[order]
    per = np.empty(s)
    for c in range(s):
        m = size[c]
        rhs = np.zeros(m)
        rhs[0] = norms[c]
        acc = off * norms[c] ** 2
        for a_j, c_j in zip(poles, residues):
            acc += c_j * norms[c] * thomas(alpha[c, :m], beta[c, : m - 1], -a_j, rhs)[0]
        per[c] = acc
    trace = float(np.mean(per))
    return logdet_P + trace, logdet_P, trace, per
