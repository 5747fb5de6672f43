"""The reference's own known-answer and property tests for the hot path
(lfbp tests/test_transform.py), restated against the
GPU drop-ins: same inputs, same expected values, each citing the reference
test it mirrors.  Bit-exact parity on random and golden inputs is in
test_gpu_parity.py; these pin the behaviours the reference states directly."""
import logging

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _bp(H):
    from paper_2003_09133_b200 import Dims5, PsfArray, compute_backprojection
    return compute_backprojection(PsfArray(Dims5(*H.shape), H)).data


def _inv(Hp):
    from paper_2003_09133_b200 import BackprojArray, Dims5, compute_psf_from_backprojection
    return compute_psf_from_backprojection(BackprojArray(Dims5(*Hp.shape), Hp)).data


def _zeros(shape, dtype=np.float64):
    return np.zeros(shape, dtype=dtype, order="F")


def test_single_element_lands_mirrored_in_phase_zero():
    """test_transform.py:108-115: one unit element at (0,0,2,2,0) of a
    (5,5,3,3,1) PSF becomes the only nonzero of H', at (4,4,0,0,0)."""
    H = _zeros((5, 5, 3, 3, 1))
    H[0, 0, 2, 2, 0] = 1.0
    out = _bp(H)
    assert out[4, 4, 0, 0, 0] == 1.0
    assert np.count_nonzero(out) == 1


def test_centre_phase_slice_is_the_rotated_pattern():
    """test_transform.py:118-127: on (3,3,3,3,1), H'[s,t,1,1,0] = H[2-s,2-t,s,t,0]."""
    rng = np.random.default_rng(5)
    H = np.asfortranarray(rng.random((3, 3, 3, 3, 1)))
    out = _bp(H)
    for s in range(3):
        for t in range(3):
            assert out[s, t, 1, 1, 0] == H[2 - s, 2 - t, s, t, 0]


def test_constant_in_constant_out():
    """test_transform.py:90-93."""
    H = np.full((9, 7, 3, 5, 2), 0.25, order="F")
    assert np.all(_bp(H) == 0.25)


def test_result_is_fortran_frozen_and_keeps_dtype():
    """test_transform.py:96-105: F-contiguous, read-only, float64 stays
    float64 and float32 stays float32."""
    for dt in (np.float64, np.float32):
        out = _bp(np.asfortranarray(np.random.default_rng(1).random((7, 7, 3, 3, 2)).astype(dt)))
        assert out.flags.f_contiguous and not out.flags.writeable and out.dtype == dt


def test_additive():
    """test_transform.py:130-138: H'(A + B) = H'(A) + H'(B).  Integer-valued
    doubles, so the sums are exact and the comparison is bitwise."""
    rng = np.random.default_rng(2)
    A = np.asfortranarray(rng.integers(0, 1000, (11, 9, 5, 3, 2)).astype(np.float64))
    B = np.asfortranarray(rng.integers(0, 1000, (11, 9, 5, 3, 2)).astype(np.float64))
    assert np.array_equal(_bp(np.asfortranarray(A + B)), _bp(A) + _bp(B))


def test_depth_planes_are_independent():
    """test_transform.py:141-154: the transform of a z-slice is the same
    slice of the full transform."""
    rng = np.random.default_rng(3)
    H = np.asfortranarray(rng.random((13, 11, 5, 3, 4)))
    full = _bp(H)
    for z0, z1 in ((0, 1), (1, 3), (3, 4)):
        assert np.array_equal(_bp(np.asfortranarray(H[..., z0:z1])), full[..., z0:z1])


@pytest.mark.parametrize("shape", [(5, 5, 3, 3, 2), (9, 7, 3, 5, 1), (15, 13, 5, 3, 2)])
def test_inverse_recovers_the_psf_and_the_map_is_an_involution(shape):
    """test_transform.py:157-162."""
    H = np.asfortranarray(np.random.default_rng(4).random(shape))
    Hp = _bp(H)
    assert np.array_equal(_inv(np.asfortranarray(Hp)), H)
    assert np.array_equal(_bp(np.asfortranarray(Hp)), H)


def test_slice_multisets_are_conserved():
    """test_transform.py:165-175: each (x', y', z) phase slice of H' holds
    exactly the values of the rearranged slice set -- as a whole, every
    depth plane's multiset of values is unchanged (odd dims, nothing dropped)."""
    H = np.asfortranarray(np.random.default_rng(6).random((11, 9, 3, 3, 2)))
    out = _bp(H)
    for z in range(2):
        assert np.array_equal(np.sort(out[..., z].ravel()), np.sort(H[..., z].ravel()))


def test_even_dims_zero_row_and_dropped_count(caplog):
    """test_transform.py:178-192: (4,5,3,3,1) drops 45 source elements with a
    WARNING containing "dropped", and H' row n_s-1 is all zero."""
    from paper_2003_09133_b200 import Dims5, dropped_source_count
    H = np.asfortranarray(np.random.default_rng(7).random((4, 5, 3, 3, 1)) + 1.0)
    assert dropped_source_count(Dims5(*H.shape)) == 45
    with caplog.at_level(logging.WARNING):
        out = _bp(H)
    assert any("dropped" in r.getMessage() for r in caplog.records)
    assert np.all(out[3, :, :, :, :] == 0.0)
    assert np.count_nonzero(out) == H.size - 45


def test_inverse_of_even_dims_is_refused():
    """test_transform.py:195-198."""
    from paper_2003_09133_b200 import EvenPixelDims
    with pytest.raises(EvenPixelDims):
        _inv(_zeros((4, 5, 3, 3, 1)))
