"""CPU oracle for the sorted-order plane sums (TEST INFRASTRUCTURE ONLY).

Restates the reference's ``_plane_sum`` (lfbp/arrays.py:211-221): the
n_x*n_y values of every (s, t) slice of a depth plane, sorted ascending and
summed in float64 by numpy (pairwise summation) -- behind
``sum_forward_plane`` / ``sum_backward_plane`` (arrays.py:224-239).
``pairwise_sum`` spells out numpy's summation order (umath loops_utils
``pairwise_sum``: blocks of <= 128 with eight accumulators, halving splits
rounded down to multiples of 8) -- the order the K3 kernel reproduces.
Pinned against values produced by the reference (tests/golden).
"""
from __future__ import annotations

import numpy as np


def plane_sums_oracle(data: np.ndarray) -> np.ndarray:
    """(n_s, n_t, n_z) float64: sorted-order sums of each slice, every plane."""
    data = np.asarray(data)
    n_s, n_t, n_x, n_y, n_z = data.shape
    out = np.empty((n_s, n_t, n_z), dtype=np.float64, order="F")
    for z in range(n_z):
        flat = data[..., z].reshape(n_s, n_t, -1)
        out[..., z] = np.sort(flat, axis=-1).sum(axis=-1, dtype=np.float64)
    return out


def pairwise_sum(values) -> float:
    """numpy's float64 pairwise summation order, in plain Python."""
    a = [float(v) for v in values]

    def rec(lo, n):
        if n < 8:
            res = 0.0
            for i in range(lo, lo + n):
                res += a[i]
            return res
        if n <= 128:
            r = a[lo:lo + 8]
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] += a[lo + i + j]
                i += 8
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                res += a[lo + i]
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return rec(lo, n2) + rec(lo + n2, n - n2)

    return 0.0 + rec(0, len(a))
