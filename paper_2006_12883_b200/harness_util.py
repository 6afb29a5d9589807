"""Convergence-rate fit used by the order study (API of paradiff/harness_util.py:8-40)."""

from __future__ import annotations

import math

import numpy as np


def fit_slope(nt_values, errors, floor: float = 1e-14, rate_window: float = 0.15) -> float:
    """Observed order: slope of log(error) against log(1/Nt) over the asymptotic tail.

    The usable prefix ends at the first error at or below ``floor`` (round-off
    plateau) or at the first error that fails to decrease.  High-order schemes
    converge faster than their asymptotic rate on coarse grids, so of that prefix
    only the longest tail whose consecutive two-point rates stay within
    ``rate_window`` (relative, plus 0.05 absolute) of the finest pair's rate enters
    the least-squares line.  Fewer than two usable points give NaN.
    """
    nts = [float(v) for v in nt_values]
    errs = [float(v) for v in errors]
    usable = 0
    while usable < len(nts) and errs[usable] > floor and (usable == 0
                                                         or errs[usable] < errs[usable - 1]):
        usable += 1
    if usable < 2:
        return math.nan
    lx = -np.log(nts[:usable])
    ly = np.log(errs[:usable])
    rates = np.diff(ly) / np.diff(lx)
    finest = rates[-1]
    allowed = rate_window * abs(finest) + 0.05
    first = len(rates) - 1
    while first > 0 and abs(rates[first - 1] - finest) <= allowed:
        first -= 1
    return float(np.polyfit(lx[first:], ly[first:], 1)[0])
