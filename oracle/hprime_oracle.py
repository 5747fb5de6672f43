"""CPU oracle for the H -> H' rearrangement (TEST INFRASTRUCTURE ONLY).

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_2003_09133_b200``) never imports anything under ``oracle/`` and
fails loudly when its CUDA library is missing.

It restates, in numpy, the reference algorithm of
``/root/reference/pkg/src/lfbp/transform.py`` (the pure-Python ``lfbp``
package of arXiv 2003.09133):

* per-axis helpers ``slice_index`` / ``wrap_phase`` / ``target_cell`` /
  ``mirror_index``                                  (transform.py:40-70)
* the per-axis ``(n_pix, n_cell)`` phase table built by walking the
  extended slice window                              (transform.py:73-96)
* the valid mirrored source rows                     (transform.py:99-103)
* the dropped-element count for even pattern sizes   (transform.py:106-110)
* the forward gather into a zero-filled F-ordered output
                                                     (transform.py:113-135)
* the inverse scatter, refused for even sizes        (transform.py:138-155)

Parity pinning: ``tests/golden/`` holds vectors and per-plane SHA-256
digests produced by running the real reference (script
``tests/golden/make_golden.py``); ``tests/test_oracle_golden.py`` checks
this restatement against every one of them, plus the reference's own
known-answer tests (``pkg/tests/test_transform.py``).

A second, independent formulation (``closed_form_hprime``) uses the closed
form derived in SURVEY.md section 0; the tests cross-check the two.

``hprime_oracle(..., threads=k)`` splits the independent depth planes over
``k`` Python threads (numpy's fancy indexing releases the GIL), which is how
``bench.py --impl reference`` runs the reference algorithm on all host
cores.
"""
from __future__ import annotations

import concurrent.futures as _cf
from functools import lru_cache

import numpy as np

__all__ = [
    "slice_index", "wrap_phase", "target_cell", "mirror_index",
    "phase_pair_table", "source_pixels", "dropped_source_count",
    "hprime_oracle", "hprime_oracle_split", "closed_form_hprime", "EvenPixelDimsOracle",
]


class EvenPixelDimsOracle(ValueError):
    """Inverse requested for even n_s or n_t (transform.py:141-144)."""


# --------------------------------------------------------------------------
# per-axis index helpers (1-based, as in the reference contract)

def slice_index(m: int, n_pix: int, n_cell: int) -> int:
    """Window counter re-centred on the core cells (transform.py:40-47)."""
    margin = (n_pix - n_cell) // 2
    return m - margin


def wrap_phase(alpha: int, n_cell: int) -> int:
    """Periodic fold of ``alpha`` into 1..n_cell (transform.py:50-56).

    The reference folds with two explicit branches; the result is the unique
    representative of ``alpha`` modulo ``n_cell`` in 1..n_cell.
    """
    return (alpha - 1) % n_cell + 1


def target_cell(s: int, alpha: int, n_pix: int, n_cell: int) -> int:
    """Pixel phase receiving pattern row ``s`` from slice ``alpha``
    (transform.py:59-65)."""
    return alpha + s - n_cell + (n_cell - 1) // 2 - (n_pix - n_cell) // 2


def mirror_index(s: int, n_pix: int) -> int:
    """180-degree reversal of a pattern coordinate; 0 = dropped (even n)
    (transform.py:68-70)."""
    return (n_pix + (n_pix & 1)) - s


@lru_cache(maxsize=64)
def phase_pair_table(n_pix: int, n_cell: int) -> np.ndarray:
    """1-based source phase for every (pattern row, target phase) pair.

    Follows transform.py:73-96: for pattern row ``s`` the slice window is
    entered at the first counter whose target phase is 1; walking ``n_cell``
    counters from there visits target phases 1..n_cell in order, and the
    folded slice index is the source phase.  Raises ``ValueError`` for an
    even cell or a pattern narrower than the cell (transform.py:83-84).
    """
    if n_cell < 1 or n_cell % 2 == 0 or n_pix < n_cell:
        raise ValueError(f"invalid axis pair n_pix={n_pix}, n_cell={n_cell}")
    margin2 = 2 * ((n_pix - n_cell) // 2)
    half = (n_cell - 1) // 2
    rows = []
    for s in range(1, n_pix + 1):
        m0 = n_cell + margin2 - half + 1 - s     # counter with target phase 1
        row = []
        for k in range(n_cell):
            alpha = slice_index(m0 + k, n_pix, n_cell)
            if target_cell(s, alpha, n_pix, n_cell) != k + 1:   # walk invariant
                raise AssertionError("slice window walk lost its phase")
            row.append(wrap_phase(alpha, n_cell))
        rows.append(row)
    tab = np.asarray(rows, dtype=np.intp).reshape(n_pix, n_cell)
    tab.flags.writeable = False
    return tab


def source_pixels(n_pix: int) -> np.ndarray:
    """0-based mirrored source row for each valid target row
    (transform.py:99-103).  Length n (odd) or n-1 (even)."""
    n_valid = n_pix if n_pix % 2 else n_pix - 1
    return np.array([mirror_index(k, n_pix) - 1 for k in range(1, n_valid + 1)],
                    dtype=np.intp)


def dropped_source_count(shape) -> int:
    """Source elements without a target (transform.py:106-110)."""
    n_s, n_t, n_x, n_y, n_z = (int(v) for v in shape)
    v_s = n_s if n_s % 2 else n_s - 1
    v_t = n_t if n_t % 2 else n_t - 1
    return (n_s * n_t - v_s * v_t) * n_x * n_y * n_z


def _index_sets(shape):
    n_s, n_t, n_x, n_y, _ = shape
    S = source_pixels(n_s)
    T = source_pixels(n_t)
    X = phase_pair_table(n_s, n_x)[S] - 1      # (v_s, n_x), 0-based
    Y = phase_pair_table(n_t, n_y)[T] - 1      # (v_t, n_y), 0-based
    return S, T, X, Y


def _gather_slab(src: np.ndarray, dst: np.ndarray, sets, inverse: bool, y_range=None) -> None:
    S, T, X, Y = sets
    if y_range is not None:                    # output columns y' in [y0, y1) only (forward)
        y0, y1 = y_range
        Y = Y[:, y0:y1]
        dst = dst[..., y0:y1, :]
    sidx = (S[:, None, None, None], T[None, :, None, None],
            X[:, None, :, None], Y[None, :, None, :])
    if inverse:
        # same index set, source and target exchanged (transform.py:150-154)
        dst[sidx] = src
    else:
        dst[:len(S), :len(T)] = src[sidx]      # transform.py:127-130


def hprime_oracle(H: np.ndarray, inverse: bool = False, threads: int = 1) -> np.ndarray:
    """H' (or, with ``inverse``, H from H') of a 5-D F-ordered array.

    ``H`` has shape (n_s, n_t, n_x, n_y, n_z) and dtype float32/float64 (any
    fixed-size dtype is moved bit-exactly).  Returns a new F-ordered array.
    With ``threads > 1`` contiguous z-slabs are processed concurrently; each
    plane is independent, so the result is identical.
    """
    H = np.asarray(H)
    if H.ndim != 5:
        raise ValueError(f"expected a 5-D array, got ndim={H.ndim}")
    shape = tuple(int(v) for v in H.shape)
    n_s, n_t = shape[0], shape[1]
    if inverse and (n_s % 2 == 0 or n_t % 2 == 0):
        raise EvenPixelDimsOracle(f"inverse undefined for even (n_s, n_t)=({n_s}, {n_t})")
    sets = _index_sets(shape)
    out = (np.empty if inverse else np.zeros)(shape, dtype=H.dtype, order="F")
    n_z = shape[4]
    threads = max(1, min(int(threads), n_z))
    if threads == 1:
        _gather_slab(H, out, sets, inverse)
        return out
    bounds = [(n_z * k) // threads for k in range(threads + 1)]
    with _cf.ThreadPoolExecutor(threads) as pool:
        futs = [pool.submit(_gather_slab, H[..., a:b], out[..., a:b], sets, inverse)
                for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
        for f in futs:
            f.result()
    return out


def hprime_oracle_split(H: np.ndarray, threads: int) -> np.ndarray:
    """Forward H' with the work split over ``threads`` host threads by depth
    plane AND output column y' (each H'[..., y', z] is an independent gather),
    so a sample of fewer planes than threads still uses every thread.  Same
    result as ``hprime_oracle(H)``."""
    H = np.asarray(H)
    shape = tuple(int(v) for v in H.shape)
    sets = _index_sets(shape)
    out = np.zeros(shape, dtype=H.dtype, order="F")
    n_y, n_z = shape[3], shape[4]
    per_z = max(1, min(n_y, -(-int(threads) // n_z)))
    tasks = [(z, (n_y * k) // per_z, (n_y * (k + 1)) // per_z) for z in range(n_z) for k in range(per_z)]
    with _cf.ThreadPoolExecutor(max(1, int(threads))) as pool:
        futs = [pool.submit(_gather_slab, H[..., z:z + 1], out[..., z:z + 1], sets, False, (y0, y1))
                for z, y0, y1 in tasks if y1 > y0]
        for f in futs:
            f.result()
    return out


def closed_form_hprime(H: np.ndarray) -> np.ndarray:
    """Independent formulation via the closed form of SURVEY.md section 0:

    H'[i, j, x', y', z] = H[2c_s - i, 2c_t - j, (x' + i - c_s) mod n_x,
                            (y' + j - c_t) mod n_y, z],
    c = floor((n - 1) / 2); rows i = n_s - 1 (even n_s) / j = n_t - 1 (even
    n_t) are zero.  Used only to cross-check ``hprime_oracle``.
    """
    H = np.asarray(H)
    n_s, n_t, n_x, n_y, _ = H.shape
    c_s, c_t = (n_s - 1) // 2, (n_t - 1) // 2
    v_s, v_t = 2 * c_s + 1, 2 * c_t + 1
    i = np.arange(v_s)
    j = np.arange(v_t)
    xs = (np.arange(n_x)[None, :] + i[:, None] - c_s) % n_x          # (v_s, n_x)
    ys = (np.arange(n_y)[None, :] + j[:, None] - c_t) % n_y          # (v_t, n_y)
    out = np.zeros(H.shape, dtype=H.dtype, order="F")
    out[:v_s, :v_t] = H[(2 * c_s - i)[:, None, None, None],
                        (2 * c_t - j)[None, :, None, None],
                        xs[:, None, :, None], ys[None, :, None, :]]
    return out
