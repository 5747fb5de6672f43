"""Per-depth-slab launcher: z-planes sharded over the GPUs of one box.

Depth planes are independent (reference PAPER.md:162, SPEC.md:218/225,
test_transform.py:141-154) and z is the slowest axis of the F-ordered array,
so a contiguous plane range [z0, z1) is the byte range [z0*P, z1*P) of both
H and H' (P = n_s*n_t*n_x*n_y*itemsize).  Each rank owns one slab; there is
no collective on the data path.  ``torch.distributed`` is used only for the
plumbing around it (barriers and the max-over-ranks timing in bench.py).

``shard_planes`` matches the C-ABI ``lfbp_shard_planes``: shard k of G gets
[floor(k*n_z/G), floor((k+1)*n_z/G)).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native


def shard_planes(n_z: int, n_shards: int, shard: int) -> tuple[int, int]:
    if n_shards < 1 or not 0 <= shard < n_shards or n_z < 0:
        raise ValueError(f"bad shard request n_z={n_z} n_shards={n_shards} shard={shard}")
    return (n_z * shard) // n_shards, (n_z * (shard + 1)) // n_shards


def slab_bytes(shape, itemsize: int, z0: int, z1: int) -> tuple[int, int]:
    """Byte range of planes [z0, z1) in the F-ordered array."""
    n_s, n_t, n_x, n_y, _ = shape
    p = n_s * n_t * n_x * n_y * itemsize
    return z0 * p, z1 * p


def imbalance(n_z: int, n_shards: int) -> float:
    """max/mean planes per shard."""
    sizes = [b - a for a, b in (shard_planes(n_z, n_shards, k) for k in range(n_shards))]
    return max(sizes) / (n_z / n_shards) if n_z else 1.0


def rearrange_multi_host(src: np.ndarray, dst: np.ndarray, devices, inverse: bool = False) -> None:
    """Single-process multi-GPU host-to-host H': one thread per device, each
    streaming its own z-slab (C-ABI ``lfbp_hprime_multi``)."""
    code = {np.dtype(np.float32): _native.F32, np.dtype(np.float64): _native.F64}[np.dtype(src.dtype)]
    if src.shape != dst.shape or src.dtype != dst.dtype:
        raise ValueError("src and dst must match")
    if not (src.flags.f_contiguous and dst.flags.f_contiguous):
        raise ValueError("arrays must be F-contiguous")
    if np.shares_memory(src, dst):
        raise ValueError("src and dst overlap (the rearrangement is not in place; transform.py:113-135 returns a new array)")
    devs = (ctypes.c_int * len(devices))(*devices)
    rc = _native.lib().lfbp_hprime_multi(src.ctypes.data_as(ctypes.c_void_p), dst.ctypes.data_as(ctypes.c_void_p),
                                         _native.dims_array(src.shape), code, int(inverse), len(devices), devs,
                                         _native.HOST_REGISTER)
    _native.check(rc)


def rank_slab(shape, world_size: int, rank: int) -> tuple[tuple[int, ...], int, int]:
    """Shape of this rank's slab and its global plane range."""
    z0, z1 = shard_planes(shape[4], world_size, rank)
    return (shape[0], shape[1], shape[2], shape[3], z1 - z0), z0, z1


def open_shared_host(path: str, shape, dtype, create: bool = False) -> np.ndarray:
    """F-ordered host array backed by a shared file (e.g. under /dev/shm):
    every rank maps the same H' and writes its own slab at byte offset
    z0 * plane_bytes -- the final gather of the z-shards needs no network
    collective."""
    mode = "w+" if create else "r+"
    return np.memmap(path, dtype=dtype, mode=mode, shape=tuple(shape), order="F")


def write_slab(shared: np.ndarray, z0: int, slab: np.ndarray) -> None:
    """Copy this rank's planes into the shared host array."""
    z1 = z0 + slab.shape[4]
    shared[..., z0:z1] = slab


def device_slab_to_shared(shared: np.ndarray, z0: int, t) -> None:
    """D2H of a device slab (F layout CUDA tensor) straight into the shared
    host array at its plane offset."""
    import torch
    n = int(np.prod(t.shape))
    flat_host = torch.from_numpy(shared.reshape(-1, order="F")[z0 * (n // t.shape[4]):][:n].view(np.uint8))
    flat_dev = t.permute(4, 3, 2, 1, 0).reshape(-1).view(torch.uint8)
    flat_host.copy_(flat_dev)
