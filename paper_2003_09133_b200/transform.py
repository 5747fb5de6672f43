"""The H -> H' hot path: drop-in replacements and the device API.

Drop-ins (same names, argument meaning, result type and errors as the
reference ``lfbp/transform.py``):

* ``compute_backprojection(psf) -> BackprojArray``        (transform.py:113-135)
* ``compute_psf_from_backprojection(bp) -> PsfArray``      (transform.py:138-155)
* ``dropped_source_count(dims)``                           (transform.py:106-110)

They validate, stream the array through one GPU with the C-ABI
``lfbp_hprime_host`` (chunked H2D / K1 kernel / D2H on three streams) and
return a fresh, read-only, Fortran-ordered array.  Even ``n_s``/``n_t``
log the reference's WARNING containing "dropped" (transform.py:131-134); the
inverse of even dims raises ``EvenPixelDims``.  When the argument is an
instance of the reference's own classes (``lfbp.PsfArray``), the result is
built with the reference's ``_wrap`` and errors use the reference's
exception classes, so the functions can be patched into ``lfbp`` directly
(INTEGRATION.md).

Device API (torch tensors already in HBM, no host copies):

* ``hprime_device(src, out=None, inverse=False, z_range=None, stream=None)``
  -- ``src`` is a CUDA tensor holding the 5-D F-ordered array: either shape
  (n_s, n_t, n_x, n_y, n_z) with Fortran strides, or the C-contiguous
  (n_z, n_y, n_x, n_t, n_s) view of the same memory.
"""
from __future__ import annotations

import ctypes
import importlib
import logging
import os

import numpy as np

from . import _native
from .arrays import BackprojArray, PsfArray
from .errors import EvenPixelDims, InvalidDims, NativeError

log = logging.getLogger(__name__)

_DTYPE_CODE = {np.dtype(np.float32): _native.F32, np.dtype(np.float64): _native.F64}


def _family(obj):
    """(PsfArray, BackprojArray, InvalidDims, EvenPixelDims) of the package
    the argument comes from: the reference's when it is an ``lfbp`` object,
    ours otherwise."""
    mod = type(obj).__module__ or ""
    root = mod.split(".")[0]
    if root and root != __name__.split(".")[0]:
        try:
            arrays = importlib.import_module(root + ".arrays")
            errors = importlib.import_module(root + ".errors")
            return (arrays.PsfArray, arrays.BackprojArray, errors.InvalidDims, errors.EvenPixelDims)
        except (ImportError, AttributeError):
            pass
    return (PsfArray, BackprojArray, InvalidDims, EvenPixelDims)


def dropped_source_count(dims) -> int:
    """Source elements with no target (0 for odd n_s, n_t)."""
    n = _native.lib().lfbp_dropped_source_count(_native.dims_array(dims.shape))
    if n < 0:
        raise InvalidDims(f"invalid dims {tuple(dims.shape)}")
    return int(n)


def _host_flags() -> int:
    """How pageable host arrays reach the GPU (LFBP_HOST_MODE): "stage"
    (default: pinned staging chunks filled by a memcpy thread pool, overlapped
    with the DMA), "register" (pin in place for the call) or "driver"."""
    mode = os.environ.get("LFBP_HOST_MODE", "stage")
    return {"stage": _native.HOST_STAGE, "register": _native.HOST_REGISTER, "driver": 0}.get(mode, _native.HOST_STAGE)


def _out_pinned(nbytes: int) -> bool:
    """Where the drop-in's fresh result array lives (LFBP_OUT_MODE): "pinned"
    (default: a page-locked block from the library's cached host allocator,
    so the D2H lands directly) or "pageable" (plain numpy; the D2H is staged
    through the pipeline's pinned chunks).  Results above LFBP_PIN_MAX_MB
    (default 4096) are pageable: page-locking costs about 0.5 s/GB and a
    71 GB block (C5) would take most of a 200 GB host out of the pageable
    pool."""
    if os.environ.get("LFBP_OUT_MODE", "pinned") != "pinned":
        return False
    return nbytes <= int(os.environ.get("LFBP_PIN_MAX_MB", "4096")) << 20


def _result_array(shape, dtype) -> np.ndarray:
    """The drop-in's fresh F-ordered result: pinned when small enough, and
    pageable when page-locked memory is refused (the reference's plain
    ``np.zeros`` never fails for lack of pinnable memory, so neither may
    this)."""
    nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
    if _out_pinned(nbytes):
        try:
            return _pinned_empty(shape, dtype)
        except NativeError as e:
            log.debug("pinned result of %d bytes refused (%s); using pageable memory", nbytes, e)
    return np.empty(shape, dtype=dtype, order="F")


class _PinnedBlock:
    """Owner of one ``lfbp_host_alloc`` block, exposed to numpy through the
    array interface: the ndarray keeps it alive, and the block goes back to
    the library's cache when the last array on it is gone."""

    ptr = None

    def __init__(self, nbytes: int):
        ptr = ctypes.c_void_p()
        _native.check(_native.lib().lfbp_host_alloc(nbytes, ctypes.byref(ptr)))
        self.ptr = ptr.value
        self.nbytes = nbytes
        self.__array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (self.ptr, False), "version": 3}

    def __del__(self):
        lib = _native._lib
        if lib is not None and self.ptr:
            lib.lfbp_host_free(ctypes.c_void_p(self.ptr))
            self.ptr = None


def _pinned_empty(shape, dtype) -> np.ndarray:
    """F-ordered host array in page-locked memory (no torch involved)."""
    n = int(np.prod(shape)) * np.dtype(dtype).itemsize
    raw = np.asarray(_PinnedBlock(max(n, 1)))
    return raw[:n].view(dtype).reshape(shape, order="F")


def _rearrange_host(data: np.ndarray, dims, inverse: bool, errs, device: int = 0) -> np.ndarray:
    invalid, even = errs
    shape = tuple(int(v) for v in dims.shape)
    code = _DTYPE_CODE.get(np.dtype(data.dtype))
    if code is None:
        raise invalid(f"dtype {data.dtype} is not float32/float64")
    if tuple(data.shape) != shape:
        raise invalid(f"array shape {data.shape} does not match {shape}")
    src = data if data.flags.f_contiguous else np.asfortranarray(data)
    dvec = _native.dims_array(shape)
    rc = _native.lib().lfbp_check_dims(dvec)
    _native.check(rc, invalid, even)
    if inverse and (shape[0] % 2 == 0 or shape[1] % 2 == 0):
        raise even(f"inverse undefined for even pixel dims (n_s, n_t)=({shape[0]}, {shape[1]}): "
                   "the forward mapping drops elements")
    out = _result_array(shape, src.dtype)
    rc = _native.lib().lfbp_hprime_host(src.ctypes.data_as(ctypes.c_void_p), out.ctypes.data_as(ctypes.c_void_p),
                                        dvec, code, int(inverse), int(device), _host_flags())
    _native.check(rc, invalid, even)
    return out


def compute_backprojection(psf, device: int = 0):
    """Rearrange a PSF array into its backprojection array on the GPU.

    Bit-exact drop-in for ``lfbp.compute_backprojection``
    (reference transform.py:113-135).
    """
    psf_cls, bp_cls, invalid, even = _family(psf)
    dims = psf.dims
    out = _rearrange_host(psf.data, dims, False, (invalid, even), device)
    dropped = dropped_source_count(dims)
    if dropped:
        # the reference's logger name when called on reference objects
        logger = log if psf_cls is PsfArray else logging.getLogger(psf_cls.__module__.split(".")[0] + ".transform")
        logger.warning("even pixel dims %s: %d source elements have no target and were dropped",
                       (dims.n_s, dims.n_t), dropped)
    return bp_cls._wrap(dims, out)


def compute_psf_from_backprojection(bp, device: int = 0):
    """Invert the rearrangement on the GPU; exact for odd pixel dims,
    ``EvenPixelDims`` otherwise (reference transform.py:138-155)."""
    psf_cls, bp_cls, invalid, even = _family(bp)
    dims = bp.dims
    if dims.n_s % 2 == 0 or dims.n_t % 2 == 0:
        raise even(f"inverse undefined for even pixel dims (n_s, n_t)=({dims.n_s}, {dims.n_t}): "
                   "the forward mapping drops elements")
    out = _rearrange_host(bp.data, dims, True, (invalid, even), device)
    return psf_cls._wrap(dims, out)


# --------------------------------------------------------------------------
# device API

def _f_strides(shape):
    n_s, n_t, n_x, n_y, _ = shape
    return (1, n_s, n_s * n_t, n_s * n_t * n_x, n_s * n_t * n_x * n_y)


def _dims_of_tensor(t):
    """(n_s, n_t, n_x, n_y, n_z) of a CUDA tensor holding an F-ordered 5-D array."""
    if t.dim() != 5:
        raise InvalidDims(f"expected a 5-D tensor, got {t.dim()}-D")
    shape = tuple(t.shape)
    st = t.stride()
    if st == _f_strides(shape) or t.permute(4, 3, 2, 1, 0).is_contiguous():
        return shape                                     # (n_s, ..., n_z), F strides
    if t.is_contiguous():
        return tuple(reversed(shape))                    # (n_z, ..., n_s) C view
    raise ValueError("tensor must be Fortran-ordered (n_s..n_z) or C-contiguous (n_z..n_s)")


def _code_of(t) -> int:
    size = t.element_size()
    if size == 4:
        return _native.F32
    if size == 8:
        return _native.F64
    raise ValueError(f"element size {size} not supported (4 or 8 bytes)")


_DIMS_CACHE: dict = {}


def _dims_arg(shape):
    """ctypes int64[5] of `shape`, cached (the device API is called per
    launch; building the array is a measurable part of a small call)."""
    d = _DIMS_CACHE.get(shape)
    if d is None:
        if len(_DIMS_CACHE) > 256:
            _DIMS_CACHE.clear()
        d = _DIMS_CACHE[shape] = _native.dims_array(shape)
    return d


def hprime_device(src, out=None, inverse: bool = False, z_range=None, stream=None):
    """H' of a device-resident array (K1 kernel, asynchronous on ``stream``,
    default: torch's current stream).  Returns ``out`` (allocated like
    ``src`` when None).  ``z_range=(z0, z1)`` restricts the planes written."""
    import torch
    if not src.is_cuda:
        raise ValueError("hprime_device needs a CUDA tensor (there is no CPU path)")
    shape = _dims_of_tensor(src)
    if out is None:
        out = torch.empty_like(src)
    if out.shape != src.shape or out.stride() != src.stride() or out.dtype != src.dtype:
        raise ValueError("out must match src in shape, strides and dtype")
    dev = src.device
    if out.device != dev:
        raise ValueError("src and out must be on the same device")
    z0, z1 = (0, shape[4]) if z_range is None else (int(z_range[0]), int(z_range[1]))
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    lib = _native.lib()
    args = (ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(out.data_ptr()), _dims_arg(shape), _code_of(src),
            int(inverse), z0, z1, ctypes.c_void_p(handle))
    if dev.index == torch.cuda.current_device():
        rc = lib.lfbp_hprime_device(*args)
    else:
        with torch.cuda.device(dev):
            rc = lib.lfbp_hprime_device(*args)
    _native.check(rc)
    return out


def f_order_empty(shape, dtype, device="cuda"):
    """Uninitialised CUDA tensor with the reference's F layout."""
    import torch
    n_s, n_t, n_x, n_y, n_z = shape
    strides = (1, n_s, n_s * n_t, n_s * n_t * n_x, n_s * n_t * n_x * n_y)
    return torch.empty_strided(tuple(shape), strides, dtype=dtype, device=device)


def plan(shape, dtype=np.float32) -> dict:
    """The kernel's launch plan for ``shape`` (current device, or B200
    defaults without a GPU)."""
    import json
    buf = ctypes.create_string_buffer(1024)
    code = _DTYPE_CODE[np.dtype(dtype)]
    _native.check(_native.lib().lfbp_plan_json(_native.dims_array(shape), code, buf, len(buf)))
    return json.loads(buf.value.decode())


def plan_candidates(size_class: int = 1) -> list:
    """The autotuner's candidate plans, as (stages, stage_kb, consumer_warps,
    lanes_per_row, order_flags, grid_sms) tuples: size class 1 for launches
    moving >= 256 MB, 0 for 8-256 MB (``lfbp_plan_candidates``; no GPU
    needed)."""
    lib = _native.lib()
    n = lib.lfbp_plan_candidates(int(size_class), None, 0)
    if n < 0:
        _native.check(-n)
    buf = (ctypes.c_int32 * (6 * n))()
    lib.lfbp_plan_candidates(int(size_class), buf, n)
    return [tuple(buf[6 * c:6 * c + 6]) for c in range(n)]


def tune(shape, dtype=np.float32, device: int = 0, z_count: int = 0) -> dict:
    """Tune the kernel plan for ``shape`` ahead of time on library-owned
    scratch buffers (``lfbp_tune``): for launches of ``z_count`` planes
    (0: all) and for the host pipeline's chunks.  Afterwards
    ``hprime_device`` never synchronises.  Returns the tuned plan."""
    code = _DTYPE_CODE[np.dtype(dtype)]
    _native.check(_native.lib().lfbp_tune(_native.dims_array(shape), code, int(device), int(z_count)))
    return plan(shape, dtype)
