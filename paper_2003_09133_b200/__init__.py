"""B200-native H -> H' rearrangement (arXiv 2003.09133), drop-in for the
reference ``lfbp`` hot path.

Public API mirrors ``lfbp/__init__.py:21-23`` for the path:
``compute_backprojection``, ``compute_psf_from_backprojection``,
``dropped_source_count``, the ``Dims5`` / ``PsfArray`` / ``BackprojArray``
types and the ``InvalidDims`` / ``EvenPixelDims`` errors; plus the device
API ``hprime_device`` and the z-slab launcher in ``shard``.
"""
from .arrays import BackprojArray, Dims5, PsfArray
from .errors import (DimMismatch, DimsError, EvenPixelDims, FormatError, InvalidDims, IoError, LfbpError,
                     NativeError, NonFiniteInput, VerificationFailure)
from .transform import (compute_backprojection, compute_psf_from_backprojection, dropped_source_count,
                        f_order_empty, hprime_device, plan, plan_candidates, tune)

__version__ = "0.1.0"

__all__ = [
    "BackprojArray", "Dims5", "PsfArray", "DimMismatch", "DimsError", "EvenPixelDims", "FormatError",
    "InvalidDims", "IoError", "LfbpError", "NativeError", "NonFiniteInput",
    "VerificationFailure", "compute_backprojection", "compute_psf_from_backprojection",
    "dropped_source_count", "f_order_empty", "hprime_device", "plan", "plan_candidates", "tune",
]
