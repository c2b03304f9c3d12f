"""Error measures of the GPU parity tests (test infrastructure).

``err(a, b)`` = max(rel-l2, max-abs / 10), where rel-l2 = ||a - b||_2 / ||b||_2 (reading
R2) and max-abs = max_j |a_j - b_j| / max_j |b_j|.  Compared against the rel-l2 bar of
the north_star (1e-10 fp64, 1e-4 fp32, 10 eps vs the NUDFT) it also fails when a few
elements -- one bad bin in a million outputs -- are wrong by more than 10x the bar
relative to the largest reference value, which the rel-l2 alone averages away.
"""
import numpy as np

import oracle


def err(a, b) -> float:
    return max(oracle.rel_l2(a, b), oracle.max_abs(a, b) / 10.0)


def both(a, b):
    """(rel-l2, max-abs) for reports."""
    return oracle.rel_l2(a, b), oracle.max_abs(a, b)
