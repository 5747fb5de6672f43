"""Pin the CPU oracle (oracle/hprime_oracle.py) to the real reference.

Golden data in tests/golden/ was produced by running the reference ``lfbp``
(script tests/golden/make_golden.py).  These tests run on CPU only.
"""
import hashlib

import numpy as np
import pytest

from conftest import load_digests
from oracle.hprime_oracle import (EvenPixelDimsOracle, closed_form_hprime, dropped_source_count,
                                  hprime_oracle, mirror_index, phase_pair_table, slice_index,
                                  target_cell, wrap_phase)
from paper_2003_09133_b200.configs import WORKLOADS
from paper_2003_09133_b200.synth import baseline_plane


def test_oracle_matches_every_small_golden_case(golden_small):
    cases, arrays = golden_small
    assert len(cases) >= 20
    for c in cases:
        H = arrays[c["name"] + "__H"]
        want = arrays[c["name"] + "__Hp"]
        got = hprime_oracle(H)
        assert got.dtype == want.dtype and got.flags.f_contiguous
        assert got.tobytes(order="F") == want.tobytes(order="F"), c["name"]
        assert dropped_source_count(H.shape) == c["dropped"], c["name"]
        if c["inverse"]:
            inv = hprime_oracle(H, inverse=True)
            assert inv.tobytes(order="F") == arrays[c["name"] + "__Hinv"].tobytes(order="F"), c["name"]


def test_closed_form_agrees_with_table_walk(golden_small):
    cases, arrays = golden_small
    for c in cases:
        H = arrays[c["name"] + "__H"]
        assert closed_form_hprime(H).tobytes(order="F") == arrays[c["name"] + "__Hp"].tobytes(order="F")


def test_threaded_oracle_equals_single_thread(golden_small):
    cases, arrays = golden_small
    H = arrays["rand_21_21_11_11_3__H"]
    assert hprime_oracle(H, threads=3).tobytes() == hprime_oracle(H).tobytes()


def test_oracle_inverse_refused_for_even():
    with pytest.raises(EvenPixelDimsOracle):
        hprime_oracle(np.zeros((4, 5, 3, 3, 1), order="F"), inverse=True)


# reference known-answer tests restated (pkg/tests/test_transform.py:17-76)
@pytest.mark.parametrize("m,n_pix,n_cell,want", [(1, 5, 3, 0), (7, 9, 3, 4), (2, 3, 3, 2), (5, 6, 3, 4)])
def test_slice_index(m, n_pix, n_cell, want):
    assert slice_index(m, n_pix, n_cell) == want


@pytest.mark.parametrize("alpha,n_cell,want", [(1, 3, 1), (3, 3, 3), (0, 3, 3), (-5, 3, 1), (4, 3, 1),
                                               (7, 3, 1), (5, 1, 1), (-2, 1, 1)])
def test_wrap_phase(alpha, n_cell, want):
    assert wrap_phase(alpha, n_cell) == want


@pytest.mark.parametrize("s,alpha,n_pix,n_cell,want", [(2, 2, 3, 3, 2), (1, 1, 3, 3, 0), (3, 2, 5, 3, 2)])
def test_target_cell(s, alpha, n_pix, n_cell, want):
    assert target_cell(s, alpha, n_pix, n_cell) == want


@pytest.mark.parametrize("s,n_pix,want", [(1, 3, 3), (2, 3, 2), (3, 3, 1), (5, 5, 1), (1, 4, 3), (4, 4, 0)])
def test_mirror_index(s, n_pix, want):
    assert mirror_index(s, n_pix) == want


def test_phase_pair_table_frozen_values():
    assert phase_pair_table(3, 3).tolist() == [[2, 3, 1], [1, 2, 3], [3, 1, 2]]
    assert phase_pair_table(5, 3).tolist() == [[3, 1, 2], [2, 3, 1], [1, 2, 3], [3, 1, 2], [2, 3, 1]]


def test_phase_pair_table_rows_are_cyclic_and_rejects_bad_axes():
    for n_pix, n_cell in [(9, 3), (15, 5), (13, 13), (6, 3), (91, 15)]:
        for row in phase_pair_table(n_pix, n_cell):
            assert sorted(row) == list(range(1, n_cell + 1))
            assert all((b - a) % n_cell == 1 for a, b in zip(row, row[1:]))
    with pytest.raises(ValueError):
        phase_pair_table(4, 4)
    with pytest.raises(ValueError):
        phase_pair_table(3, 5)


def test_single_element_and_centre_slice():
    d = (5, 5, 3, 3, 1)
    H = np.zeros(d, order="F")
    H[0, 0, 2, 2, 0] = 0.625
    Hp = hprime_oracle(H)
    assert Hp[4, 4, 0, 0, 0] == 0.625 and np.count_nonzero(Hp) == 1
    H = np.asfortranarray(np.random.default_rng(9).random((3, 3, 3, 3, 1)))
    Hp = hprime_oracle(H)
    for s in range(3):
        for t in range(3):
            assert Hp[s, t, 1, 1, 0] == H[2 - s, 2 - t, s, t, 0]


def test_generator_is_pinned_and_oracle_matches_reference_digests_c1():
    d = load_digests("C1")
    assert d is not None, "tests/golden/digests_C1.json missing"
    w = WORKLOADS["C1"]
    for z in range(w.shape[4]):
        plane = baseline_plane(w, z)
        assert hashlib.sha256(plane.tobytes(order="F")).hexdigest() == d["input_plane_sha256"][z]
        got = hprime_oracle(plane[..., None])
        assert hashlib.sha256(got.tobytes(order="F")).hexdigest() == d["hprime_plane_sha256"][z]


@pytest.mark.parametrize("cfg", ["C2", "C3", "C4", "C5"])
def test_generator_pinned_first_plane(cfg):
    """Input digests of the big configs reproduce here (plane 0 and last)."""
    d = load_digests(cfg)
    if d is None:
        pytest.skip(f"digests_{cfg}.json not generated")
    w = WORKLOADS[cfg]
    for z in (0, w.shape[4] - 1):
        plane = baseline_plane(w, z)
        assert hashlib.sha256(plane.tobytes(order="F")).hexdigest() == d["input_plane_sha256"][z]


def test_oracle_matches_reference_digest_c2_planes():
    d = load_digests("C2")
    if d is None:
        pytest.skip("digests_C2.json not generated")
    w = WORKLOADS["C2"]
    for z in (0, 25, 50):
        plane = baseline_plane(w, z)
        got = hprime_oracle(plane[..., None])
        assert hashlib.sha256(got.tobytes(order="F")).hexdigest() == d["hprime_plane_sha256"][z]


def test_plane_sums_oracle_matches_reference(golden_small):
    """Sorted-order plane sums (arrays.py:211-239) reproduce the reference's
    sum_forward_plane / sum_backward_plane bit for bit, and the spelled-out
    pairwise order (the K3 kernel's) equals numpy's."""
    from oracle.plane_sums import pairwise_sum, plane_sums_oracle
    cases, arrays = golden_small
    n = 0
    for c in cases:
        key = c["name"] + "__fwdsum"
        if key not in arrays:
            continue
        n += 1
        H, Hp = arrays[c["name"] + "__H"], arrays[c["name"] + "__Hp"]
        assert plane_sums_oracle(H).tobytes() == np.asfortranarray(arrays[key]).tobytes(), c["name"]
        assert plane_sums_oracle(Hp).tobytes() == np.asfortranarray(arrays[c["name"] + "__bwdsum"]).tobytes()
        s, t = H.shape[0] // 2, H.shape[1] // 3
        want = arrays[key][s, t, 0]
        assert pairwise_sum(np.sort(H[s, t, :, :, 0], axis=None)) == want
    assert n >= 20


def test_pairwise_order_long_slices():
    from oracle.plane_sums import pairwise_sum
    rng = np.random.default_rng(3)
    for k in (1, 7, 8, 9, 127, 128, 129, 255, 441, 1000, 5225):
        v = np.sort(rng.random(k).astype(np.float32) * rng.random(k).astype(np.float32) ** 7)
        want = v.reshape(1, 1, k).sum(axis=-1, dtype=np.float64)[0, 0]
        assert pairwise_sum(v) == want, k


def _acceptance_cases():
    import json
    import os

    from conftest import GOLDEN
    with open(os.path.join(GOLDEN, "acceptance_suite.json")) as f:
        return json.load(f)["cases"]


def test_oracle_matches_reference_acceptance_suite():
    """The reference's 50-array acceptance matrix (test_acceptance.py:21-27,
    criterion 1): our redraw of lfbp.random_psf is bit-identical to the
    reference's input and the oracle reproduces the reference's H' for every
    array (digests produced by the reference, tests/golden/make_golden.py)."""
    from paper_2003_09133_b200.synth import random_psf_like_reference
    cases = _acceptance_cases()
    assert len(cases) == 50
    for c in cases:
        H = random_psf_like_reference(tuple(c["shape"]), density=c["density"], seed=c["seed"])
        assert hashlib.sha256(H.tobytes(order="F")).hexdigest() == c["input_sha256"]
        Hp = hprime_oracle(H)
        assert hashlib.sha256(np.asfortranarray(Hp).tobytes(order="F")).hexdigest() == c["hprime_sha256"], c["seed"]
