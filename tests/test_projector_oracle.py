"""The projector oracle (oracle/projector_oracle.py) against the reference's
own outputs (tests/golden/projector_cases.npz, produced by lfbp).  CPU only."""
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import projector_oracle as po


@pytest.fixture(scope="module")
def proj():
    return dict(np.load(os.path.join(GOLDEN, "projector_cases.npz")))


def close(a, b, rtol=1e-12):
    denom = np.maximum(np.abs(b), 1e-300)
    return np.max(np.abs(a - b) / denom) < rtol if a.size else True


@pytest.mark.parametrize("name", ["sym", "even", "asym", "f32"])
def test_projections_match_reference(proj, name):
    from oracle.hprime_oracle import hprime_oracle
    H, g, f = proj[name + "__H"], proj[name + "__g"], proj[name + "__f"]
    Hp = hprime_oracle(H)
    assert close(po.forward_project(H, g), proj[name + "__fwd"])
    assert close(po.backproject(Hp, f), proj[name + "__bp"])
    assert close(po.backproject_adjoint(H, f), proj[name + "__adj"])
    assert close(po.backproject(Hp, np.ones(f.shape)), proj[name + "__norm"])


def test_rl_matches_reference(proj):
    from oracle.hprime_oracle import hprime_oracle
    H = proj["rl6__H"]
    g, hist, _ = po.rl_run(H, hprime_oracle(H), proj["rl6__f"], iterations=6)
    assert close(g, proj["rl6__est"], 1e-10)
    assert np.allclose(hist, proj["rl6__mse"], rtol=1e-9, atol=0)


def test_safe_divide_kat():
    out = po.safe_divide(np.ones(4), np.asarray([2.0, 1e-30, 0.0, 4.0]), 1e-12)
    assert out.tolist() == [0.5, 0.0, 0.0, 0.25]
