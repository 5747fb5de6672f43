"""Seeded synthetic H arrays (input generation, not the hot path).

Two generators:

* ``baseline_psf`` -- the BASELINE.json value laws (U[0,1) times a Gaussian
  envelope, or U[0,1) inside a disc) about the lenslet-shifted pattern
  centre.  The laws are not in the reference, so the conventions are fixed
  here:

  - plane ``z`` (0-based) draws from ``np.random.default_rng([seed, z])``:
    one ``random(n_s*n_t*n_x*n_y)`` call read in F order (s fastest), so
    planes and z-shards can be produced independently and in parallel;
  - 1-based centre for phase (x, y): ``(pc(n_s) + (n_x+1)/2 - x,
    pc(n_t) + (n_y+1)/2 - y)`` with ``pc`` = the reference's
    ``pattern_centre`` (projector.py:26-32);
  - Gaussian envelope ``exp(-d_s^2/(2w^2)) * exp(-d_t^2/(2w^2))`` (separable,
    the factors evaluated by ``_exp_neg`` from +, *, / only, so every host
    produces identical bits), value ``(U * e_s) * e_t`` in float64, then
    cast; disc: ``U`` if ``d_s^2 + d_t^2 <= R^2`` else exactly 0.0.

* ``baseline_psf_device`` -- the same planes generated on the GPU (K6,
  ``lfbp_synth_planes_device``), bit-identical: the host passes each plane's
  PCG64 starting state and the per-axis factor tables, the device jumps
  every lane to its draw and applies the same correctly rounded IEEE
  operations.  C5's 71 GB take well under a second instead of minutes of
  host time and no host memory.

* ``random_psf_like_reference`` -- restates the reference's sparse test
  generator ``random_psf`` (synth.py:181-195: C-order ``rng.random(shape)``
  mask ``< density``, values ``1 - rng.random(shape)``), so the reference's
  own test inputs can be rebuilt on the GPU box where the reference is not
  installed.
"""
from __future__ import annotations

import concurrent.futures as _cf
import os

import numpy as np

from .configs import Workload


def pattern_centre(n: int) -> int:
    """Zero-offset pattern coordinate, 1-based (reference projector.py:26-32)."""
    return (n + 1) // 2 if n % 2 else n // 2 + 1


def _exp_neg(x: np.ndarray) -> np.ndarray:
    """exp(x) for x <= 0 using only IEEE +, *, / (bit-reproducible on any
    host, unlike libm / SIMD exp).  Scale by 2^-12, 24-term Horner series,
    square 12 times; below -745 the result is 0."""
    x = np.asarray(x, dtype=np.float64)
    y = x * (1.0 / 4096.0)
    p = np.ones_like(y)
    for k in range(24, 0, -1):
        p = 1.0 + (y / float(k)) * p
    for _ in range(12):
        p = p * p
    return np.where(x < -745.0, 0.0, p)


def _plane_factors(w: Workload, z: int):
    """Per-axis envelope tables for plane z: es (n_s, n_x), et (n_t, n_y)
    as float64, or the integer offsets for the disc law."""
    n_s, n_t, n_x, n_y, _ = w.shape
    s = np.arange(1, n_s + 1, dtype=np.int64)[:, None]
    t = np.arange(1, n_t + 1, dtype=np.int64)[:, None]
    xs = np.arange(1, n_x + 1, dtype=np.int64)[None, :]
    ys = np.arange(1, n_y + 1, dtype=np.int64)[None, :]
    ds = s - (pattern_centre(n_s) + (n_x + 1) // 2 - xs)       # (n_s, n_x)
    dt = t - (pattern_centre(n_t) + (n_y + 1) // 2 - ys)       # (n_t, n_y)
    if w.law == "disc":
        return ds, dt
    width = w.width(z)
    inv = 1.0 / (2.0 * width * width)
    # exp over the distinct integer offsets, then gathered (fast and exact)
    lo = int(min(ds.min(), dt.min()))
    hi = int(max(ds.max(), dt.max()))
    d = np.arange(lo, hi + 1, dtype=np.float64)
    table = _exp_neg(-(d * d) * inv)
    return table[ds - lo], table[dt - lo]


def baseline_plane(w: Workload, z: int) -> np.ndarray:
    """One depth plane (n_s, n_t, n_x, n_y), F-ordered, dtype of ``w``."""
    n_s, n_t, n_x, n_y, _ = w.shape
    rng = np.random.default_rng([w.seed, z])
    u = rng.random(n_s * n_t * n_x * n_y).reshape((n_s, n_t, n_x, n_y), order="F")
    a, b = _plane_factors(w, z)
    if w.law == "disc":
        r = w.width(z)
        r2 = (a * a)[:, None, :, None] + (b * b)[None, :, None, :]
        vals = np.where(r2 <= r * r, u, 0.0)
    else:
        vals = u * a[:, None, :, None]
        vals *= b[None, :, None, :]
    return np.asfortranarray(vals.astype(w.dtype, copy=False))


def baseline_psf(w: Workload, z_begin: int = 0, z_end: int | None = None,
                 out: np.ndarray | None = None, threads: int | None = None) -> np.ndarray:
    """Planes [z_begin, z_end) of workload ``w`` as one F-ordered array.

    ``out`` (optional) must be an F-contiguous array of the slab's shape and
    dtype, e.g. a pinned-memory view; planes are generated in parallel.
    """
    n_s, n_t, n_x, n_y, n_z = w.shape
    z_end = n_z if z_end is None else z_end
    if not 0 <= z_begin <= z_end <= n_z:
        raise ValueError(f"bad plane range [{z_begin}, {z_end}) for n_z={n_z}")
    shape = (n_s, n_t, n_x, n_y, z_end - z_begin)
    if out is None:
        out = np.empty(shape, dtype=w.dtype, order="F")
    elif out.shape != shape or out.dtype != np.dtype(w.dtype) or not out.flags.f_contiguous:
        raise ValueError("out has the wrong shape, dtype or layout")

    def one(z):
        out[..., z - z_begin] = baseline_plane(w, z)

    threads = threads or min(16, os.cpu_count() or 1)
    if threads <= 1 or z_end - z_begin <= 1:
        for z in range(z_begin, z_end):
            one(z)
    else:
        with _cf.ThreadPoolExecutor(threads) as pool:
            list(pool.map(one, range(z_begin, z_end)))
    return out


def random_psf_like_reference(shape, density: float = 0.05, seed: int = 0,
                              dtype=np.float64) -> np.ndarray:
    """Restatement of the reference's ``random_psf`` draw order
    (synth.py:181-195); returns the F-ordered data array."""
    if not 0.0 < density <= 1.0:
        raise ValueError(f"density must be in (0, 1], got {density}")
    rng = np.random.default_rng(seed)
    shape = tuple(int(v) for v in shape)
    mask = rng.random(shape) < density
    values = 1.0 - rng.random(shape)
    data = np.where(mask, values, 0.0).astype(dtype, copy=False)
    return np.asfortranarray(data)


def _pcg_states(w: Workload, z_begin: int, z_end: int) -> np.ndarray:
    """(n_planes, 4) uint64: the PCG64 state (lo, hi) and increment (lo, hi)
    of ``default_rng([seed, z])`` before its first draw, per plane."""
    m = (1 << 64) - 1
    rows = []
    for z in range(z_begin, z_end):
        st = np.random.default_rng([w.seed, z]).bit_generator.state["state"]
        s, inc = int(st["state"]), int(st["inc"])
        rows.append([s & m, s >> 64, inc & m, inc >> 64])
    return np.asarray(rows, dtype=np.uint64).reshape(-1, 4)


def _device_tables(w: Workload, z_begin: int, z_end: int):
    """Per-plane factor tables for K6: tab_s (n_planes, n_x, n_s) and tab_t
    (n_planes, n_y, n_t) in the kernel's s-fastest order, float64, and the
    disc law's r^2 per plane (None for the product law)."""
    ts, tt, r2 = [], [], []
    for z in range(z_begin, z_end):
        a, b = _plane_factors(w, z)
        if w.law == "disc":
            a = (a * a).astype(np.float64)
            b = (b * b).astype(np.float64)
            r = w.width(z)
            r2.append(r * r)
        ts.append(np.asarray(a, dtype=np.float64).T)
        tt.append(np.asarray(b, dtype=np.float64).T)
    return np.stack(ts), np.stack(tt), (np.asarray(r2, dtype=np.float64) if w.law == "disc" else None)


def baseline_psf_device(w: Workload, z_begin: int = 0, z_end: int | None = None, out=None, device=None,
                        stream=None):
    """Planes [z_begin, z_end) of workload ``w`` generated on the GPU,
    bit-identical to ``baseline_psf``: a CUDA tensor of shape
    (n_s, n_t, n_x, n_y, z_end - z_begin) with Fortran strides (``out``, if
    given, must be such a tensor).  Asynchronous on ``stream``."""
    import ctypes

    import torch

    from . import _native
    from .transform import f_order_empty
    n_s, n_t, n_x, n_y, n_z = w.shape
    z_end = n_z if z_end is None else z_end
    if not 0 <= z_begin <= z_end <= n_z:
        raise ValueError(f"bad plane range [{z_begin}, {z_end}) for n_z={n_z}")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    tdt = torch.float32 if w.itemsize == 4 else torch.float64
    shape = (n_s, n_t, n_x, n_y, z_end - z_begin)
    if out is None:
        out = f_order_empty(shape, tdt, dev)
    elif tuple(out.shape) != shape or out.dtype != tdt or not out.permute(4, 3, 2, 1, 0).is_contiguous():
        raise ValueError("out has the wrong shape, dtype or layout")
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    code = _native.F32 if w.itemsize == 4 else _native.F64
    # at most 1024 planes' tables per launch keeps the tables small
    for a in range(z_begin, z_end, 1024):
        b = min(z_end, a + 1024)
        ts, tt, r2 = _device_tables(w, a, b)
        dst = out.permute(4, 3, 2, 1, 0)[a - z_begin]
        with torch.cuda.stream(stream):   # tables uploaded on the kernel's stream
            states = torch.from_numpy(_pcg_states(w, a, b).view(np.int64)).to(dev)
            ts_d = torch.from_numpy(np.ascontiguousarray(ts)).to(dev)
            tt_d = torch.from_numpy(np.ascontiguousarray(tt)).to(dev)
            r2_d = torch.from_numpy(r2).to(dev) if r2 is not None else None
            rc = _native.lib().lfbp_synth_planes_device(
                ctypes.c_void_p(dst.data_ptr()), code, _native.dims_array(w.shape), b - a,
                ctypes.c_void_p(states.data_ptr()), ctypes.c_void_p(ts_d.data_ptr()), ctypes.c_void_p(tt_d.data_ptr()),
                ctypes.c_void_p(r2_d.data_ptr() if r2_d is not None else 0), ctypes.c_void_p(stream.cuda_stream))
        _native.check(rc)
        # keep the tables alive until the kernel has read them
        stream.synchronize()
    return out
