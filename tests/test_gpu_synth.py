"""K6 on the device (-m gpu): the synthesised BASELINE inputs equal the host
generator bit for bit, and at full size carry the input digests the golden
run recorded from the reference session (tests/golden/digests_C*.json)."""
import numpy as np
import pytest

from conftest import load_digests

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("cfg,z0,z1", [("C1", 0, 9), ("C2", 24, 27), ("C3", 0, 1), ("C4", 18, 22), ("C4", 40, 41),
                                       ("C5", 50, 51), ("C5", 0, 1)])
def test_device_planes_equal_host_planes(cfg, z0, z1):
    torch = _torch()
    from paper_2003_09133_b200.configs import WORKLOADS
    from paper_2003_09133_b200.synth import baseline_psf, baseline_psf_device
    w = WORKLOADS[cfg]
    dev = baseline_psf_device(w, z0, z1)
    torch.cuda.synchronize()
    got = dev.permute(4, 3, 2, 1, 0).contiguous().cpu().numpy().reshape(-1)
    want = baseline_psf(w, z0, z1).reshape(-1, order="F")
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("cfg", ["C1", "C2", "C4"])
def test_full_size_input_digests(cfg):
    torch = _torch()
    from paper_2003_09133_b200.configs import WORKLOADS
    from paper_2003_09133_b200.synth import baseline_psf_device
    from paper_2003_09133_b200.verify import plane_digests
    d = load_digests(cfg)
    if d is None:
        pytest.skip(f"digests_{cfg}.json not generated")
    w = WORKLOADS[cfg]
    src = baseline_psf_device(w)
    torch.cuda.synchronize()
    assert plane_digests(src, w.shape) == d["input_plane_sha256"]
