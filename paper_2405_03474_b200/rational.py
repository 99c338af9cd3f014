"""Partial-fraction constants of the odd-order rational approximations to
log z (Table 1 of arXiv 2405.03474).

r_k(z) = b + sum_j c_j / (z - a_j), poles a_j ascending (most negative first),
r(1) = 0 and r(z) = -r(1/z).  Reference: ``src/rational.py:70-96`` (table),
``src/rational.py:116-119`` (lookup), ``src/rational.py:151-160`` (evaluation).
The shifted solves of the estimator use sigma_j = -a_j > 0.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["RationalPartialFraction", "partial_fraction", "eval_partial"]


@dataclass(frozen=True)
class RationalPartialFraction:
    order: int
    offset: float
    poles: tuple[float, ...]
    residues: tuple[float, ...]


_TABLE = {
    1: RationalPartialFraction(1, 2.0, (-1.0,), (-4.0,)),
    3: RationalPartialFraction(
        3, 14.0 / 3.0,
        (-13.92820323027551, -1.0, -0.0717967697244908),
        (-49.52250037431294, -20.0 / 9.0, -0.2552774034648563)),
    5: RationalPartialFraction(
        5, 86.0 / 15.0,
        (-39.863458189061411, -3.8518399963191827, -1.0, -0.25961618368249978, -0.025085630936916615),
        (-140.08241129102026, -6.1858406006156228, -92.0 / 75.0, -0.41692913805732562,
         -0.088152303639431204)),
}


def partial_fraction(order: int) -> RationalPartialFraction:
    if order not in _TABLE:
        raise ValueError(f"partial fractions exist for odd orders 1, 3, 5; got {order}")
    return _TABLE[order]


def eval_partial(pf: RationalPartialFraction, z):
    z = np.asarray(z, dtype=np.float64)
    out = np.full_like(z, pf.offset, dtype=np.float64)
    for a, c in zip(pf.poles, pf.residues):
        diff = z - a
        if np.any(diff == 0.0):
            raise ZeroDivisionError(f"evaluation at pole {a}")
        out = out + c / diff
    return float(out) if out.ndim == 0 else out
