"""LF5 container streaming.

The reference's LF5 format (lfbp/fileio.py:3-14): a 32-byte little-endian
header -- magic ``b"LF5D"``, u32 version 1, u8 element code (1 = float32,
2 = float64), three zero bytes, five u32 dims -- then the F-ordered payload.
The reference reads the whole file into memory (fileio.py:70) and writes
with ``tofile`` (fileio.py:46-60).  Here:

* ``read_header`` / ``save`` / ``load`` -- host-side format I/O, byte-
  identical to the reference's ``read_lf5`` / ``save`` / ``load_psf``
  (the same FormatError / IoError / DimsError / InvalidDims checks);
* ``transform_file(in, out, inverse=False)`` -- the ``lfbp transform`` CLI
  (cli.py:115-126) file to file through the GPU, plane chunks pread into
  pinned buffers and pwritten at their offsets (C-ABI
  ``lfbp_lf5_transform_file``), never holding the array in host memory;
* ``load_device`` / ``store_device`` -- a z-slab of a file straight into /
  out of HBM (per-rank shard loads for the multi-GPU path).
"""
from __future__ import annotations

import ctypes
import logging
import os
import struct

import numpy as np

from . import _native
from .arrays import Dims5, PsfArray
from .errors import DimsError, FormatError, InvalidDims, IoError

log = logging.getLogger(__name__)

MAGIC = b"LF5D"
VERSION = 1
HEADER = struct.Struct("<4sIB3s5I")
_CODES = {1: np.dtype("<f4"), 2: np.dtype("<f8")}
_CODE_OF = {np.dtype("<f4"): 1, np.dtype("<f8"): 2}


def _path(p) -> bytes:
    return os.fsencode(os.fspath(p))


def read_header(path) -> tuple[tuple[int, ...], np.dtype]:
    """(dims, dtype) of an LF5 file, validated like read_lf5 (fileio.py:63-92)."""
    dims = _native.dims_array((0, 0, 0, 0, 0))
    code = ctypes.c_int(0)
    _native.check(_native.lib().lfbp_lf5_read_header(_path(path), dims, ctypes.byref(code)))
    return tuple(int(v) for v in dims), _CODES[code.value]


def header_bytes(shape, dtype) -> bytes:
    code = _CODE_OF.get(np.dtype(dtype).newbyteorder("<"))
    if code is None:
        raise FormatError(f"unsupported element dtype {dtype}")
    return HEADER.pack(MAGIC, VERSION, code, b"\x00\x00\x00", *[int(v) for v in shape])


def save(array, path) -> None:
    """Write a PsfArray / BackprojArray (or any F-ordered 5-D float array) as
    LF5, byte-identical to the reference's ``save`` (fileio.py:46-60)."""
    data = np.asarray(array) if isinstance(array, np.ndarray) or not hasattr(array, "dims") else array.data
    if data.ndim != 5:
        raise FormatError(f"save expects a 5-D array, got ndim={data.ndim}")
    head = header_bytes(data.shape, data.dtype)
    payload = np.asarray(data, dtype=data.dtype.newbyteorder("<")).ravel(order="F")
    try:
        with open(path, "wb") as fh:
            fh.write(head)
            payload.tofile(fh)
    except OSError as exc:
        raise IoError(f"cannot write {path}: {exc}") from exc


def load(path, cls=PsfArray, allow_invalid_dims: bool = False):
    """Read a whole LF5 file as ``cls`` (PsfArray / BackprojArray) with the
    reference's checks (fileio.py:95-118)."""
    shape, dtype = read_header(path)
    data = np.fromfile(path, dtype=dtype, offset=HEADER.size).reshape(shape, order="F")
    try:
        dims = Dims5(*shape)
    except InvalidDims as exc:
        if not allow_invalid_dims:
            raise DimsError(f"{path}: {exc}") from exc
        return cls._wrap(Dims5.unchecked(*shape), data)
    data.flags.writeable = False
    return cls(dims, data)


def transform_file(in_path, out_path, inverse: bool = False, device: int = 0) -> tuple[int, ...]:
    """H' of an LF5 file into another LF5 file on the GPU (file -> pinned
    chunks -> HBM -> pinned chunks -> file).  Returns the dims.  Errors and
    the even-dims warning follow ``lfbp transform`` (cli.py:115-126)."""
    _native.check(_native.lib().lfbp_lf5_transform_file(_path(in_path), _path(out_path), int(inverse),
                                                         int(device), 0))
    shape, _ = read_header(out_path)
    n_s, n_t = shape[:2]
    if not inverse and (n_s % 2 == 0 or n_t % 2 == 0):
        v_s, v_t = n_s - (1 - n_s % 2), n_t - (1 - n_t % 2)
        dropped = (n_s * n_t - v_s * v_t) * shape[2] * shape[3] * shape[4]
        log.warning("even pixel dims %s: %d source elements have no target and were dropped", (n_s, n_t), dropped)
    return shape


def load_device(path, z_range=None, device=None, stream=None):
    """Planes [z0, z1) of an LF5 file as a CUDA tensor (F layout)."""
    import torch

    from .transform import f_order_empty
    shape, dtype = read_header(path)
    z0, z1 = (0, shape[4]) if z_range is None else (int(z_range[0]), int(z_range[1]))
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    t = f_order_empty((*shape[:4], z1 - z0), torch.float32 if dtype.itemsize == 4 else torch.float64, dev)
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        rc = _native.lib().lfbp_lf5_load_device(_path(path), ctypes.c_void_p(t.data_ptr()), z0, z1,
                                                ctypes.c_void_p(stream.cuda_stream))
    _native.check(rc)
    return t


def store_device(path, t, z0: int = 0, create_shape=None, stream=None) -> None:
    """Write a CUDA tensor's planes into an LF5 file at plane offset z0;
    ``create_shape`` creates the file (header + sized payload) first."""
    import torch
    if create_shape is not None:
        code = 1 if t.element_size() == 4 else 2
        _native.check(_native.lib().lfbp_lf5_create(_path(path), _native.dims_array(create_shape), code))
    n_planes = t.shape[4] if t.dim() == 5 else 1
    if stream is None:
        stream = torch.cuda.current_stream(t.device)
    with torch.cuda.device(t.device):
        rc = _native.lib().lfbp_lf5_store_device(_path(path), ctypes.c_void_p(t.data_ptr()), int(z0),
                                                 int(z0) + int(n_planes), ctypes.c_void_p(stream.cuda_stream))
    _native.check(rc)
