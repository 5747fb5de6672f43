"""CPU oracle for the H' consumer (TEST INFRASTRUCTURE ONLY).

Restates the reference's projector (lfbp/projector.py) in numpy:

* ``forward_project``      -- projector.py:55-81 (voxel patterns stamped onto
  the image; the window arithmetic of ``_windows``, projector.py:35-47)
* ``backproject``          -- projector.py:103-126 (pixel patterns from H')
* ``backproject_adjoint``  -- projector.py:84-100 (gather per voxel through H)
* ``safe_divide``          -- projector.py:135-145
* ``rl_run``               -- projector.py:162-196

Pinned against reference outputs in tests/golden/projector_cases.npz; used by
the GPU tests as the checker on random shapes.  float64 accumulation.
"""
from __future__ import annotations

import numpy as np


def pattern_centre(n: int) -> int:
    return (n + 1) // 2 if n % 2 else n // 2 + 1


def _windows(n_grid: int, n_pat: int, centre: int):
    idx = np.arange(n_grid)
    lo = np.maximum(idx + 1 - centre, 0)
    hi = np.minimum(idx + n_pat - centre + 1, n_grid)
    return lo, hi, lo - idx + centre - 1


def forward_project(H: np.ndarray, g: np.ndarray) -> np.ndarray:
    n_s, n_t, n_x, n_y, n_z = H.shape
    nvx, nvy, _ = g.shape
    s_lo, s_hi, a0 = _windows(nvx, n_s, pattern_centre(n_s))
    t_lo, t_hi, b0 = _windows(nvy, n_t, pattern_centre(n_t))
    out = np.zeros((nvx, nvy))
    for z in range(n_z):
        for x in range(nvx):
            for y in range(nvy):
                w = g[x, y, z]
                if w:
                    out[s_lo[x]:s_hi[x], t_lo[y]:t_hi[y]] += w * H[a0[x]:a0[x] + s_hi[x] - s_lo[x],
                                                                   b0[y]:b0[y] + t_hi[y] - t_lo[y],
                                                                   x % n_x, y % n_y, z]
    return out


def backproject(Hp: np.ndarray, f: np.ndarray) -> np.ndarray:
    n_s, n_t, n_x, n_y, n_z = Hp.shape
    npx, npy = f.shape
    x_lo, x_hi, a0 = _windows(npx, n_s, pattern_centre(n_s))
    y_lo, y_hi, b0 = _windows(npy, n_t, pattern_centre(n_t))
    out = np.zeros((npx, npy, n_z))
    for s in range(npx):
        for t in range(npy):
            w = f[s, t]
            if w:
                out[x_lo[s]:x_hi[s], y_lo[t]:y_hi[t], :] += w * Hp[a0[s]:a0[s] + x_hi[s] - x_lo[s],
                                                                   b0[t]:b0[t] + y_hi[t] - y_lo[t],
                                                                   s % n_x, t % n_y, :]
    return out


def backproject_adjoint(H: np.ndarray, f: np.ndarray) -> np.ndarray:
    n_s, n_t, n_x, n_y, n_z = H.shape
    npx, npy = f.shape
    s_lo, s_hi, a0 = _windows(npx, n_s, pattern_centre(n_s))
    t_lo, t_hi, b0 = _windows(npy, n_t, pattern_centre(n_t))
    out = np.zeros((npx, npy, n_z))
    for z in range(n_z):
        for x in range(npx):
            for y in range(npy):
                pat = H[a0[x]:a0[x] + s_hi[x] - s_lo[x], b0[y]:b0[y] + t_hi[y] - t_lo[y], x % n_x, y % n_y, z]
                out[x, y, z] = np.sum(f[s_lo[x]:s_hi[x], t_lo[y]:t_hi[y]] * pat, dtype=np.float64)
    return out


def safe_divide(num, den, eps):
    out = np.zeros(num.shape)
    peak = float(den.max()) if den.size else 0.0
    if peak <= 0.0:
        return out
    ok = den >= eps * peak
    if eps * peak == 0.0:
        ok &= den > 0.0
    np.divide(num, den, out=out, where=ok)
    return out


def rl_run(H, Hp, f, iterations=20, eps=1e-12):
    npx, npy = f.shape
    norm = backproject(Hp, np.ones((npx, npy)))
    g = np.ones((npx, npy, H.shape[4]))
    hist = []
    for _ in range(iterations):
        ratio = safe_divide(f, forward_project(H, g), eps)
        g = g * safe_divide(backproject(Hp, ratio), norm, eps)
        hist.append(float(np.mean((f - forward_project(H, g)) ** 2)))
    return g, hist, norm
