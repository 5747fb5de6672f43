"""K3 (device sorted-order plane sums) against the reference (GPU; -m gpu).

sum_forward_plane / sum_backward_plane (reference arrays.py:211-239) are
bitwise functions of the value multiset; the device kernel must reproduce
them bit for bit, and the reference's acceptance criterion 3 (180-degree
rotation of the summed planes, test_acceptance.py:85-99) must hold on the
device at full BASELINE size.
"""
import numpy as np
import pytest

from oracle.plane_sums import plane_sums_oracle

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def to_device(H):
    torch = _torch()
    flat = torch.from_numpy(np.array(H.reshape(-1, order="F")))
    return flat.cuda().view(H.shape[::-1]).permute(4, 3, 2, 1, 0)


def host(t):
    return t.permute(2, 1, 0).contiguous().cpu().numpy().transpose(2, 1, 0)


def test_plane_sums_match_reference_golden(golden_small):
    _torch()
    from paper_2003_09133_b200.verify import plane_sums_device
    cases, arrays = golden_small
    n = 0
    for c in cases:
        if c["name"] + "__fwdsum" not in arrays:
            continue
        n += 1
        for which, key in (("__H", "__fwdsum"), ("__Hp", "__bwdsum")):
            A = arrays[c["name"] + which]
            got = host(plane_sums_device(to_device(A), A.shape))
            want = arrays[c["name"] + key]
            assert got.tobytes() == np.asfortranarray(want).astype(np.float64).tobytes(order="F") or \
                np.array_equal(got.view(np.int64), want.view(np.int64)), c["name"] + which
    assert n >= 20


@pytest.mark.parametrize("shape,dtype", [((95, 55, 95, 55, 1), np.float32), ((17, 13, 11, 13, 3), np.float64),
                                         ((9, 7, 31, 17, 2), np.float32), ((3, 3, 1, 1, 4), np.float32),
                                         ((4, 6, 2, 2, 2), np.float64)])
def test_plane_sums_match_oracle_random(shape, dtype):
    _torch()
    from paper_2003_09133_b200.synth import random_psf_like_reference
    from paper_2003_09133_b200.verify import plane_sums_device
    H = random_psf_like_reference(shape, density=0.7, seed=11, dtype=dtype)
    got = host(plane_sums_device(to_device(H), shape))
    assert np.array_equal(got.view(np.int64), plane_sums_oracle(H).view(np.int64))


def test_plane_sums_special_bits_nan_aware(golden_small):
    _torch()
    from paper_2003_09133_b200.verify import plane_sums_device
    cases, arrays = golden_small
    for c in cases:
        if not c["kind"].startswith("bits"):
            continue
        A = arrays[c["name"] + "__H"]
        got = host(plane_sums_device(to_device(A), A.shape))
        want = plane_sums_oracle(A)
        assert np.array_equal(got, want, equal_nan=True), c["name"]


@pytest.mark.parametrize("cfg", ["C2", "C4", "C3"])
def test_rotation_criterion_full_size_on_device(cfg):
    """Criterion 3 at full size: bwd sums of H' == rotated fwd sums of H, all planes."""
    torch = _torch()
    from paper_2003_09133_b200 import f_order_empty, hprime_device
    from paper_2003_09133_b200.configs import WORKLOADS
    from paper_2003_09133_b200.synth import baseline_psf
    from paper_2003_09133_b200.verify import plane_sums_device, rotation_check
    w = WORKLOADS[cfg]
    src = f_order_empty(w.shape, torch.float32 if w.itemsize == 4 else torch.float64)
    flat = src.permute(4, 3, 2, 1, 0).reshape(-1)
    step = 8
    for z0 in range(0, w.shape[4], step):
        z1 = min(w.shape[4], z0 + step)
        flat[z0 * w.plane_elems:z1 * w.plane_elems].copy_(torch.from_numpy(baseline_psf(w, z0, z1).reshape(-1, order="F")))
    hp = hprime_device(src)
    assert rotation_check(src, hp, w.shape) == 0
    # and plane 0's device sums equal the CPU oracle's
    got = host(plane_sums_device(src, w.shape, z_range=(0, 1)))
    want = plane_sums_oracle(baseline_psf(w, 0, 1))
    assert np.array_equal(got.view(np.int64), want.view(np.int64))
