"""Golden vectors for the stand-alone preconditioner seam (rld_precond_build / rld_precond_apply)
from the UNMODIFIED reference ``build_preconditioner`` (src/precond.py:236-267) and its
``solve_sqrt`` / ``solve_sqrt_t`` (src/precond.py:102-115), run in this container only.

Usage:  OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_preconditioner_apply.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

import ratlogdet  # noqa: E402  (the unmodified reference)
from ratlogdet import linalg as rlinalg  # noqa: E402
from ratlogdet import precond as rprecond  # noqa: E402

from paper_2405_03474_b200.workloads import baseline  # noqa: E402  (point sets only)


def main():
    out = []
    for idx, n, kind, rank in [(1, 768, "rand-svd", 48), (1, 768, "rank-one", 1), (2, 1024, "rand-svd", 64),
                               (3, 1024, "trunc-svd-scaled", 32), (1, 768, "diagonal", 0)]:
        wl = baseline(idx, n=n)
        spec = ratlogdet.KernelSpec(wl.spec.family, wl.spec.amplitude, wl.spec.length_scale, wl.spec.jitter)
        M = ratlogdet.build_covariance(spec, wl.points)
        cfg = ratlogdet.PreconditionerConfig(kind, rank, 5, 5e-3)
        P = rprecond.build_preconditioner(M, cfg, rlinalg.Rng(0).child(1))
        g = np.random.default_rng(idx + n)
        Z = g.standard_normal((n, 3))
        rec = dict(name=f"{kind}_{wl.name}_n{n}", config_index=idx, n=n, kind=kind, rank=rank, num_iters=5,
                   scale=5e-3, seed=0, rng_path=[1], log_det=float(P.log_det), z_seed=idx + n,
                   solve_sqrt=[P.solve_sqrt(z).tolist() for z in Z.T],
                   solve_sqrt_t=[P.solve_sqrt_t(z).tolist() for z in Z.T])
        print(rec["name"], rec["log_det"], flush=True)
        out.append(rec)
    (HERE / "golden_preconditioner_apply.json").write_text(json.dumps(out))


if __name__ == "__main__":
    main()
