"""CPU oracle for the r* rational log-determinant path.

TEST INFRASTRUCTURE ONLY. This module is the checker, never the product:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import it.  The product
package ``paper_2405_03474_b200`` never imports anything under ``oracle/`` and
fails loudly when its CUDA library is missing.

What it is: a float64 numpy restatement of the reference package ``ratlogdet``
(``/root/reference/pkg/src/ratlogdet``), written from its algorithm, not copied.
Each function cites the reference file:line it follows.  Differences in
*structure* (not in arithmetic semantics):

* Lanczos runs all probes in lock-step on an n x s block (the reference loops
  probe by probe, ``estimators.py:86-92``); every column still gets its own
  two-pass full reorthogonalisation and its own lucky-breakdown truncation, so
  each column's recurrence is the reference's.  ``per_probe=True`` restores the
  reference's loop order exactly (used for CPU-baseline timing).
* The kernel matrix may be supplied matrix-free (row blocks generated from the
  points with the reference's r^2 = |x|^2 + |y|^2 - 2 x.y formula), which lets
  the oracle run past the n ~ 30k where a dense float64 K stops fitting in RAM.

Pinning: ``tests/test_oracle.py`` checks this module against golden
vectors produced by the unmodified reference (``tests/golden/make_golden.py``)
to <= 1e-10 relative on well-posed configurations, and bit-for-bit on the RNG
streams.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

# ----------------------------------------------------------------------------
# constants

# Table 1 of arXiv 2405.03474: r_k(z) = b + sum_j c_j / (z - a_j); poles ascending.
# Reference: src/rational.py:70-96.
PARTIAL_FRACTIONS = {
    1: (2.0, (-1.0,), (-4.0,)),
    3: (14.0 / 3.0,
        (-13.92820323027551, -1.0, -0.0717967697244908),
        (-49.52250037431294, -20.0 / 9.0, -0.2552774034648563)),
    5: (86.0 / 15.0,
        (-39.863458189061411, -3.8518399963191827, -1.0,
         -0.25961618368249978, -0.025085630936916615),
        (-140.08241129102026, -6.1858406006156228, -92.0 / 75.0,
         -0.41692913805732562, -0.088152303639431204)),
}

OVERSAMPLE = 10          # src/precond.py:165
DIAG_FLOOR = 1e-12       # src/precond.py:37
KEEP_RTOL = 1e-14        # src/precond.py:97
BREAKDOWN_RTOL = 1e-12   # src/lanczos.py:20
CGS_RTOL = 1e-12         # src/linalg.py:177
PIVOT_FLOOR = 1e-300     # src/linalg.py:140-148
SQRT5 = np.sqrt(5.0)     # src/kernels.py:14


class OracleRankDeficient(Exception):
    pass


class OracleSingularShift(Exception):
    pass


class OracleNotPD(Exception):
    pass


# ----------------------------------------------------------------------------
# random streams (src/linalg.py:64-91, src/probes.py:25-44)

def stream(seed: int, path=()) -> np.random.Generator:
    """Philox keyed by SeedSequence(seed, spawn_key=path) -- src/linalg.py:72-76."""
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(int(seed), spawn_key=tuple(path))))


def probes(kind: str, s: int, n: int, seed: int) -> np.ndarray:
    """s x n probe rows from stream (seed, (2,)) -- src/estimators.py:64, src/probes.py:31-34."""
    g = stream(seed, (2,))
    if kind == "rademacher":
        return 2.0 * g.integers(0, 2, size=(s, n)).astype(np.float64) - 1.0   # src/linalg.py:84-85
    if kind == "gaussian":
        return g.standard_normal((s, n))                                     # src/linalg.py:81-82
    if kind == "normal-orthogonal":                                          # src/probes.py:15-22, 36-44
        blocks, left, i = [], s, 0
        while left > 0:
            sb = min(left, n)
            gb = stream(seed, (2, i))
            Q = cgs2_rows(gb.standard_normal((sb, n)))
            blocks.append(Q * np.sqrt(gb.chisquare(n, sb))[:, None])          # Rng.chi, src/linalg.py:87-88
            left -= sb
            i += 1
        return np.vstack(blocks)
    raise ValueError(f"unknown probe kind {kind!r}")


def sketch(seed: int, attempt: int, w: int, n: int) -> np.ndarray:
    """Gaussian test rows, stream (seed, (1, attempt)) -- src/estimators.py:63, src/precond.py:183."""
    return stream(seed, (1, attempt)).standard_normal((w, n))


# ----------------------------------------------------------------------------
# kernel matrices (src/kernels.py:40-73)

def kernel_of_r(family: str, amplitude: float, ell: float, r):
    a2 = amplitude * amplitude
    if family == "rbf":
        return a2 * np.exp(-(r * r) / (2.0 * ell * ell))
    u = SQRT5 * r / ell
    return a2 * (1.0 + u + u * u / 3.0) * np.exp(-u)


def covariance_block(family, amplitude, ell, jitter, X, rows=None):
    """Rows ``rows`` (a slice) of K = k(x_i, x_j) + jitter*I via the reference's
    r^2 trick (src/kernels.py:65-72).  The full-matrix call symmetrises r^2 like
    the reference; a row block uses the same formula for both orientations."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    sq = np.einsum("ij,ij->i", X, X)
    if rows is None:
        r2 = sq[:, None] + sq[None, :] - 2.0 * (X @ X.T)
        r2 = 0.5 * (r2 + r2.T)
        np.fill_diagonal(r2, 0.0)
        np.maximum(r2, 0.0, out=r2)
        K = kernel_of_r(family, amplitude, ell, np.sqrt(r2))
        K[np.diag_indices(n)] = amplitude * amplitude + jitter
        return K
    lo, hi = rows.start, rows.stop
    Xr = X[lo:hi]
    r2 = sq[lo:hi, None] + sq[None, :] - 2.0 * (Xr @ X.T)
    r2t = sq[None, lo:hi].T + sq[None, :] - 2.0 * (Xr @ X.T)
    r2 = 0.5 * (r2 + r2t)
    np.maximum(r2, 0.0, out=r2)
    idx = np.arange(lo, hi)
    r2[idx - lo, idx] = 0.0
    K = kernel_of_r(family, amplitude, ell, np.sqrt(r2))
    K[idx - lo, idx] = amplitude * amplitude + jitter
    return K


class DenseOperator:
    """K held densely (the reference's only mode)."""

    def __init__(self, K):
        self.K = np.asarray(K, dtype=np.float64)
        self.n = self.K.shape[0]

    def diag(self):
        return np.diag(self.K).copy()

    def __call__(self, V):
        return self.K @ V


class PointsOperator:
    """Matrix-free K @ V from the points, row block by row block."""

    def __init__(self, family, amplitude, ell, jitter, X, block=2048):
        self.args = (family, amplitude, ell, jitter)
        self.X = np.asarray(X, dtype=np.float64)
        self.n = self.X.shape[0]
        self.block = block

    def diag(self):
        fam, a, ell, jit = self.args
        return np.full(self.n, a * a + jit)

    def __call__(self, V):
        V = np.asarray(V, dtype=np.float64)
        out = np.empty((self.n,) + V.shape[1:])
        for lo in range(0, self.n, self.block):
            hi = min(lo + self.block, self.n)
            out[lo:hi] = covariance_block(*self.args, self.X, slice(lo, hi)) @ V
        return out


# ----------------------------------------------------------------------------
# dense primitives (src/linalg.py:110-180)

def cholesky_logdet(K) -> float:
    """2 sum log diag chol(K) -- src/linalg.py:110-122."""
    try:
        L = np.linalg.cholesky(np.asarray(K, dtype=np.float64))
    except np.linalg.LinAlgError as exc:
        raise OracleNotPD(str(exc)) from exc
    return float(2.0 * np.sum(np.log(np.diag(L))))


def thomas(diag, off, shift, rhs):
    """(T + shift I) x = rhs without pivoting -- src/linalg.py:125-156."""
    t = len(diag)
    d = np.asarray(diag, dtype=np.float64) + shift
    e = np.asarray(off, dtype=np.float64)
    c = np.zeros(max(t - 1, 0))
    y = np.zeros(t)
    piv = d[0]
    if abs(piv) < PIVOT_FLOOR:
        raise OracleSingularShift("zero pivot at row 0")
    y[0] = rhs[0] / piv
    if t > 1:
        c[0] = e[0] / piv
    for i in range(1, t):
        piv = d[i] - e[i - 1] * c[i - 1]
        if abs(piv) < PIVOT_FLOOR:
            raise OracleSingularShift(f"zero pivot at row {i}")
        y[i] = (rhs[i] - e[i - 1] * y[i - 1]) / piv
        if i < t - 1:
            c[i] = e[i] / piv
    x = np.zeros(t)
    x[t - 1] = y[t - 1]
    for i in range(t - 2, -1, -1):
        x[i] = y[i] - c[i] * x[i + 1]
    return x


def cgs2_rows(V):
    """Row orthonormalisation, classical Gram-Schmidt applied twice per row,
    RankDeficient below 1e-12 of the row's norm -- src/linalg.py:159-180."""
    V = np.asarray(V, dtype=np.float64)
    m, n = V.shape
    Q = np.empty((m, n))
    for i in range(m):
        w = V[i].copy()
        nrm0 = np.linalg.norm(w)
        if i:
            for _ in range(2):
                w -= Q[:i].T @ (Q[:i] @ w)
        nrm = np.linalg.norm(w)
        if nrm < CGS_RTOL * max(nrm0, 1e-300):
            raise OracleRankDeficient(f"row {i}")
        Q[i] = w / nrm
    return Q


# ----------------------------------------------------------------------------
# preconditioner (src/precond.py:58-118, 168-198, 231-267)

@dataclass
class OraclePreconditioner:
    base: np.ndarray
    A: np.ndarray
    log_det: float
    sqrt_base: np.ndarray
    U: np.ndarray
    lam: np.ndarray
    theta: np.ndarray
    attempts: int

    def solve_sqrt_t(self, X):
        """N^-T X -- src/precond.py:110-115."""
        g = 1.0 / np.sqrt(1.0 + self.lam) - 1.0
        if self.U.shape[1]:
            X = X + self.U @ (g.reshape(-1, *([1] * (X.ndim - 1))) * (self.U.T @ X))
        return X / self.sqrt_base.reshape(-1, *([1] * (X.ndim - 1)))

    def solve_sqrt(self, Z):
        """N^-1 Z -- src/precond.py:102-108."""
        W = Z / self.sqrt_base.reshape(-1, *([1] * (Z.ndim - 1)))
        if not self.U.shape[1]:
            return W
        g = 1.0 / np.sqrt(1.0 + self.lam) - 1.0
        return W + self.U @ (g.reshape(-1, *([1] * (W.ndim - 1))) * (self.U.T @ W))


def range_svd(op, n, k, q, seed, omega=None):
    """Randomised subspace iteration -- src/precond.py:168-198.

    ``omega`` optionally injects the test rows per attempt (list or callable).
    Returns (theta descending (k,), rows (k, n), attempts used)."""
    if not 1 <= k <= n:
        raise ValueError(f"rank must be in 1..{n}, got {k}")
    w = min(k + OVERSAMPLE, n)
    for attempt in range(2):
        try:
            if omega is None:
                Y = sketch(seed, attempt, w, n)
            elif callable(omega):
                Y = omega(attempt)
            else:
                Y = np.asarray(omega[attempt], dtype=np.float64)
            Q = None
            for _ in range(q):
                Y = op(Y.T).T           # rows times symmetric K
                Q = cgs2_rows(Y)
                Y = Q
            B = Q @ op(Q.T)
            theta, Ub = np.linalg.eigh(B)
            top = np.argsort(theta)[::-1][:k]
            return theta[top], (Q.T @ Ub[:, top]).T, attempt + 1
        except OracleRankDeficient:
            if attempt == 1:
                raise
    raise AssertionError("unreachable")


def _finish_preconditioner(A, base, theta=None, attempts=1) -> OraclePreconditioner:
    """Determinant lemma and factored square root of P = diag(base) + A A^T -- src/precond.py:69-100."""
    inner = np.eye(A.shape[1]) + A.T @ (A / base[:, None])
    try:
        L = np.linalg.cholesky(inner)
    except np.linalg.LinAlgError as exc:
        raise OracleNotPD(str(exc)) from exc
    log_det = float(np.sum(np.log(base)) + 2.0 * np.sum(np.log(np.diag(L))))
    sqrt_base = np.sqrt(base)
    At = A / sqrt_base[:, None]
    lam, W = np.linalg.eigh(At.T @ At)
    keep = lam > KEEP_RTOL * max(lam[-1] if lam.size else 0.0, 1.0)
    U = At @ (W[:, keep] / np.sqrt(lam[keep]))
    return OraclePreconditioner(base, A, log_det, sqrt_base, U, lam[keep],
                                np.zeros(0) if theta is None else theta, attempts)


def other_preconditioner(kind, K, k, q, seed, scale) -> OraclePreconditioner:
    """The non-default kinds of build_preconditioner for a dense K -- src/precond.py:201-267:
    diagonal, rank-one (power iteration from stream (seed, (1,))), partial-cholesky(-scaled)
    (greedy largest-diagonal pivots), trunc-svd(-scaled) (dense eigh), rand-svd-scaled."""
    K = np.asarray(K, dtype=np.float64)
    n = K.shape[0]
    if kind not in ("identity", "diagonal", "rank-one") and k > n:
        raise ValueError(f"rank {k} exceeds dimension {n}")                 # precond.py:241-242
    d0 = np.diag(K).copy()

    def floored(A):                                                         # precond.py:231-233
        return np.maximum(d0 - np.sum(A * A, axis=1), DIAG_FLOOR)

    if kind == "diagonal":
        return _finish_preconditioner(np.zeros((n, 0)), d0)
    if kind == "rank-one":                                                  # precond.py:201-213, 249-251
        g = stream(seed, (1,))
        v = g.standard_normal(n)
        v /= np.linalg.norm(v)
        lam = 0.0
        for _ in range(max(100, q * max(k, 1))):
            w = K @ v
            new_lam = float(v @ w)
            v = w / np.linalg.norm(w)
            if lam != 0.0 and abs(new_lam - lam) <= 1e-10 * abs(new_lam):
                lam = new_lam
                break
            lam = new_lam
        A = np.sqrt(max(lam, DIAG_FLOOR)) * v[:, None]
        return _finish_preconditioner(A, floored(A))
    if kind in ("partial-cholesky", "partial-cholesky-scaled"):             # precond.py:215-228
        d = d0.copy()
        C = np.zeros((n, k))
        for j in range(k):
            p = int(np.argmax(d))
            if d[p] <= 0.0:
                C = C[:, :j]
                break
            col = K[:, p] - C[:, :j] @ C[p, :j]
            C[:, j] = col / np.sqrt(d[p])
            d -= C[:, j] ** 2
        base = floored(C) if kind == "partial-cholesky" else np.full(n, scale)
        return _finish_preconditioner(C, base)
    if kind in ("trunc-svd", "trunc-svd-scaled"):                           # precond.py:260-263
        theta, vecs = np.linalg.eigh(K)
        top = np.argsort(theta)[::-1][:k]
        A = vecs[:, top] * np.sqrt(np.maximum(theta[top], 0.0))
    elif kind == "rand-svd-scaled":
        theta, rows, _ = range_svd(DenseOperator(K), n, k, q, seed)
        A = rows.T * np.sqrt(np.maximum(theta, 0.0))
    else:
        raise ValueError(f"unknown preconditioner kind {kind!r}")
    base = np.full(n, scale) if kind.endswith("-scaled") else floored(A)
    return _finish_preconditioner(A, base)


def rand_svd_preconditioner(op, diagK, n, k, q, seed, omega=None) -> OraclePreconditioner:
    """rand-svd branch of build_preconditioner -- src/precond.py:236-267."""
    if k > n:
        raise ValueError(f"rank {k} exceeds dimension {n}")
    theta, rows, attempts = range_svd(op, n, k, q, seed, omega)
    A = rows.T * np.sqrt(np.maximum(theta, 0.0))
    base = np.maximum(diagK - np.sum(A * A, axis=1), DIAG_FLOOR)      # precond.py:231-233
    # determinant lemma with the inner Cholesky -- precond.py:69-80
    inner = np.eye(A.shape[1]) + A.T @ (A / base[:, None])
    try:
        L = np.linalg.cholesky(inner)
    except np.linalg.LinAlgError as exc:
        raise OracleNotPD(str(exc)) from exc
    log_det = float(np.sum(np.log(base)) + 2.0 * np.sum(np.log(np.diag(L))))
    # factored square root -- precond.py:90-100
    sqrt_base = np.sqrt(base)
    At = A / sqrt_base[:, None]
    lam, W = np.linalg.eigh(At.T @ At)
    keep = lam > KEEP_RTOL * max(lam[-1] if lam.size else 0.0, 1.0)
    U = At @ (W[:, keep] / np.sqrt(lam[keep]))
    return OraclePreconditioner(base, A, log_det, sqrt_base, U, lam[keep], theta, attempts)


# ----------------------------------------------------------------------------
# Lanczos (src/lanczos.py:34-84), lock-step over probe columns

def lanczos_block(op, V, t):
    """t Lanczos steps for every column of V (n x s), each column with its own
    two-pass full reorthogonalisation and breakdown test (src/lanczos.py:34-74).

    Returns (Q (t, n, s), alphas (s, t), betas (s, t-1), sizes (s,), norms (s,))."""
    V = np.asarray(V, dtype=np.float64)
    n, s = V.shape
    if t < 1:
        raise ValueError("t must be >= 1")
    if t > n:
        raise ValueError(f"t={t} exceeds operator dimension n={n}")
    norms = np.linalg.norm(V, axis=0)
    if np.any(norms == 0.0):
        raise ValueError("starting vector must be nonzero")
    Q = np.zeros((t, n, s))
    alphas = np.zeros((s, t))
    betas = np.zeros((s, max(t - 1, 0)))
    sizes = np.full(s, t)
    live = np.ones(s, dtype=bool)
    beta_ref = np.full(s, np.nan)
    Q[0] = V / norms
    for j in range(t):
        W = np.array(op(Q[j]), dtype=np.float64)
        alphas[:, j] = np.where(live, np.einsum("nc,nc->c", Q[j], W), alphas[:, j])
        for _ in range(2):
            coef = np.einsum("jnc,nc->jc", Q[: j + 1], W)
            W -= np.einsum("jnc,jc->nc", Q[: j + 1], coef)
        if j == t - 1:
            break
        beta = np.linalg.norm(W, axis=0)
        beta_ref = np.where(np.isnan(beta_ref), beta, beta_ref)
        broke = live & (beta <= BREAKDOWN_RTOL * np.maximum(beta_ref, np.abs(alphas[:, j])))
        sizes[broke] = j + 1
        live &= ~broke
        betas[:, j] = np.where(live, beta, 0.0)
        safe = np.where(live, beta, 1.0)
        Q[j + 1] = np.where(live[None, :], W / safe, 0.0)
    return Q, alphas, betas, sizes, norms


# ----------------------------------------------------------------------------
# the estimator (src/estimators.py:58-96)

@dataclass
class OracleEstimate:
    value: float
    logdet_P: float
    trace_term: float
    per_probe_values: np.ndarray
    wall_time: float
    attempts: int = 1


def identity_preconditioner(n) -> OraclePreconditioner:
    """P = I (src/precond.py:245-246)."""
    z = np.zeros((n, 0))
    return OraclePreconditioner(np.ones(n), z, 0.0, np.ones(n), z, np.zeros(0), np.zeros(0), 0)


def rstar(op, n, order, s, t, probe_kind, k, q, seed, V=None, omega=None, per_probe=False,
          diagK=None, precond="rand-svd", scale=1e-6) -> OracleEstimate:
    """log det P + mean_i z_i^T r_k(N^-1 K N^-T) z_i -- src/estimators.py:77-96.

    ``op`` maps an n x m block to K @ block.  ``V`` optionally injects the s x n
    probe rows; ``omega`` the sketch rows."""
    start = time.perf_counter()
    b, poles, residues = PARTIAL_FRACTIONS[order]
    t = min(t, n)                                                       # estimators.py:62
    if precond == "identity":
        P = identity_preconditioner(n)
    elif precond == "rand-svd":
        P = rand_svd_preconditioner(op, op.diag() if diagK is None else diagK, n, k, q, seed, omega)
    else:   # dense K only (the other kinds of src/precond.py:236-267)
        P = other_preconditioner(precond, op.K, k, q, seed, scale)
    Z = probes(probe_kind, s, n, seed) if V is None else np.asarray(V, dtype=np.float64)

    def aop(X):
        return P.solve_sqrt(op(P.solve_sqrt_t(X)))                      # estimators.py:71-72

    shifts = [-a for a in poles]
    per = np.empty(s)
    groups = [slice(i, i + 1) for i in range(s)] if per_probe else [slice(0, s)]
    for g in groups:
        Zg = Z[g].T                                                     # n x m
        Q, al, be, sizes, norms = lanczos_block(aop, Zg, t)
        for c in range(Zg.shape[1]):
            m = sizes[c]
            rhs = np.zeros(m)
            rhs[0] = norms[c]
            v = Zg[:, c]
            acc = b * float(v @ v)
            Qc = Q[:m, :, c]
            for cj, sig in zip(residues, shifts):
                wv = thomas(al[c, :m], be[c, : m - 1], sig, rhs)
                acc += cj * float(v @ (Qc.T @ wv))
            per[g.start + c] = acc
    trace = float(np.mean(per))
    return OracleEstimate(P.log_det + trace, P.log_det, trace, per,
                          time.perf_counter() - start, P.attempts)


def rstar_dense(K, order=3, s=35, t=20, probe_kind="rademacher", k=25, q=5, seed=0, **kw):
    op = DenseOperator(K)
    return rstar(op, op.n, order, s, t, probe_kind, k, q, seed, **kw)


def rstar_points(family, amplitude, ell, jitter, X, order=3, s=35, t=20, probe_kind="rademacher",
                 k=25, q=5, seed=0, block=2048, **kw):
    op = PointsOperator(family, amplitude, ell, jitter, X, block=block)
    return rstar(op, op.n, order, s, t, probe_kind, k, q, seed, **kw)


# ----------------------------------------------------------------------------
# stochastic Lanczos quadrature (src/estimators.py:99-122) -- SURVEY.md §8(f) row 1

SLQ_EIG_FLOOR = 1e-300   # src/estimators.py:29


def slq(op, n, s, t, probe_kind, seed, V=None, per_probe=False) -> OracleEstimate:
    """mean_i |z_i|^2 sum_j Y[0,j]^2 log(max(theta_j, floor)) over the Ritz pairs of
    each probe's t-step Lanczos on K itself (no preconditioner, src/estimators.py:106),
    with the reference's two-pass full reorthogonalisation (lanczos_block)."""
    start = time.perf_counter()
    t = min(t, n)                                                       # estimators.py:62
    Z = probes(probe_kind, s, n, seed) if V is None else np.asarray(V, dtype=np.float64)
    per = np.empty(s)
    clamped = 0
    groups = [slice(i, i + 1) for i in range(s)] if per_probe else [slice(0, s)]
    for g in groups:
        Zg = Z[g].T
        _, al, be, sizes, norms = lanczos_block(op, Zg, t)
        for c in range(Zg.shape[1]):
            m = sizes[c]
            T = np.diag(al[c, :m]) + np.diag(be[c, : m - 1], 1) + np.diag(be[c, : m - 1], -1)
            theta, Y = np.linalg.eigh(T)                                  # estimators.py:111
            clamped += int(np.count_nonzero(theta <= 0.0))
            theta = np.maximum(theta, SLQ_EIG_FLOOR)
            per[g.start + c] = norms[c] ** 2 * float((Y[0, :] ** 2) @ np.log(theta))
    trace = float(np.mean(per))
    est = OracleEstimate(trace, 0.0, trace, per, time.perf_counter() - start)
    est.clamped_eigs = clamped
    return est


def slq_dense(K, s=35, t=20, probe_kind="rademacher", seed=0, **kw):
    op = DenseOperator(K)
    return slq(op, op.n, s, t, probe_kind, seed, **kw)


def eval_partial(order, z):
    """b + sum_j c_j/(z - a_j) -- src/rational.py:151-160."""
    b, poles, residues = PARTIAL_FRACTIONS[order]
    z = np.asarray(z, dtype=np.float64)
    out = np.full_like(z, b)
    for a, c in zip(poles, residues):
        out = out + c / (z - a)
    return out
