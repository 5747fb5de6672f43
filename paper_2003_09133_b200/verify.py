"""Verification harness for the device path (reference: bench.py:88's
bitwise ``np.array_equal`` and ``lfbp verify``, cli.py:129-150).

* ``compare_device(a, b)`` -- K2 kernel: number of differing bytes and the
  first differing byte offset of two device buffers.
* ``first_mismatch_index(shape, byte_offset, itemsize)`` -- 0-based
  (s, t, x, y, z) of a byte offset in the F-ordered array, the way
  ``lfbp verify`` reports the first differing element (cli.py:145-150).
* ``plane_digests(t)`` -- per-plane SHA-256 of a device array (planes are
  copied to the host one at a time), comparable with the reference-produced
  golden digests under ``tests/golden/``.
* ``involution_check(h)`` -- applies the kernel twice on the device and
  compares with the input (odd n_s, n_t: the map is an involution,
  reference test_transform.py:157-162).
* ``negative_control(h, hp)`` -- flips one bit of a copy of ``hp`` and
  asserts the comparator catches it.
"""
from __future__ import annotations

import ctypes
import hashlib

from . import _native
from .errors import VerificationFailure


def compare_device(a, b, stream=None) -> tuple[int, int]:
    import torch
    if a.numel() * a.element_size() != b.numel() * b.element_size():
        raise ValueError("buffers differ in size")
    nbytes = a.numel() * a.element_size()
    n_diff = ctypes.c_int64(0)
    first = ctypes.c_int64(-1)
    if stream is None:
        stream = torch.cuda.current_stream(a.device)
    with torch.cuda.device(a.device):
        rc = _native.lib().lfbp_compare_device(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
                                               nbytes, ctypes.byref(n_diff), ctypes.byref(first),
                                               ctypes.c_void_p(stream.cuda_stream))
    _native.check(rc)
    return int(n_diff.value), int(first.value)


def first_mismatch_index(shape, byte_offset: int, itemsize: int) -> tuple[int, ...]:
    e = byte_offset // itemsize
    idx = []
    for n in shape:
        idx.append(e % n)
        e //= n
    return tuple(idx)


def plane_digests(t, shape, threads: int = 8) -> list[str]:
    """SHA-256 of each z-plane's bytes of a device tensor in F layout.

    Planes are copied to pinned host buffers in batches and hashed by a
    thread pool (hashlib releases the GIL)."""
    import concurrent.futures as cf

    import torch
    n_s, n_t, n_x, n_y, n_z = shape
    flat = t.reshape(-1) if t.is_contiguous() else t.permute(4, 3, 2, 1, 0).reshape(-1)
    per = n_s * n_t * n_x * n_y
    batch = max(1, min(n_z, threads))
    bufs = [torch.empty(per, dtype=t.dtype, pin_memory=True) for _ in range(batch)]
    out = [None] * n_z

    def digest(k, z):
        out[z] = hashlib.sha256(memoryview(bufs[k].numpy()).cast("B")).hexdigest()

    with cf.ThreadPoolExecutor(batch) as pool:
        for z0 in range(0, n_z, batch):
            zs = list(range(z0, min(n_z, z0 + batch)))
            for k, z in enumerate(zs):
                bufs[k].copy_(flat[z * per:(z + 1) * per])
            list(pool.map(lambda kz: digest(*kz), enumerate(zs)))
    return out


def involution_check(h, scratch=None) -> tuple[int, int]:
    """(n_diff, first) of rearrange(rearrange(h)) vs h, all on the device."""
    from .transform import hprime_device
    hp = hprime_device(h)
    back = hprime_device(hp, out=scratch)
    return compare_device(back, h)


def negative_control(hp) -> None:
    """A one-bit flip in a copy of ``hp`` must be detected by the comparator."""
    import torch
    bad = hp.clone()
    raw = bad.view(torch.uint8) if bad.is_contiguous() else bad.permute(4, 3, 2, 1, 0).view(torch.uint8)
    flat = raw.reshape(-1)
    pos = flat.numel() // 2 + 3
    flat[pos] ^= 0x10
    n_diff, first = compare_device(hp, bad)
    if n_diff != 1 or first != pos:
        raise VerificationFailure(f"negative control not caught: n_diff={n_diff} first={first} pos={pos}")


def plane_sums_device(t, shape, z_range=None, stream=None):
    """Sorted-order float64 sums of every (s, t) pattern slice (K3 kernel):
    bit-identical to the reference's sum_forward_plane / sum_backward_plane
    (arrays.py:211-239) for every plane.  Returns a CUDA float64 tensor of
    shape (n_s, n_t, n_planes) in F layout."""
    import torch

    from .transform import _code_of
    n_s, n_t, n_x, n_y, n_z = shape
    z0, z1 = (0, n_z) if z_range is None else z_range
    out = torch.empty((z1 - z0, n_t, n_s), dtype=torch.float64, device=t.device).permute(2, 1, 0)
    if stream is None:
        stream = torch.cuda.current_stream(t.device)
    with torch.cuda.device(t.device):
        rc = _native.lib().lfbp_plane_sums_device(ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                                  _native.dims_array(shape), _code_of(t), int(z0), int(z1),
                                                  ctypes.c_void_p(stream.cuda_stream))
    _native.check(rc)
    return out


def rotation_check(h, hp, shape) -> int:
    """Acceptance criterion 3 of the reference (test_acceptance.py:85-99) on
    the device: sum_backward_plane(H') == rotate180(sum_forward_plane(H)) bit
    for bit, every plane.  Returns the number of mismatching (s, t, z)."""
    import torch
    fwd = plane_sums_device(h, shape)
    bwd = plane_sums_device(hp, shape)
    rot = torch.flip(fwd, dims=(0, 1))
    return int((bwd.contiguous().view(torch.int64) != rot.contiguous().view(torch.int64)).sum().item())
