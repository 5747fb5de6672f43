"""The H' consumer on the GPU (f2; -m gpu): projections and Richardson-Lucy
against the reference's outputs (tests/golden/projector_cases.npz) to the
reference's own tolerance (relative 1e-12 between its two backprojection
forms, test_projector.py:67-82), plus the reference's projector tests and
acceptance criteria 5-6 restated."""
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import projector_oracle as po

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def proj():
    return dict(np.load(os.path.join(GOLDEN, "projector_cases.npz")))


def rel(a, b):
    denom = np.maximum(np.abs(b), 1e-300)
    return float(np.max(np.abs(a - b) / denom)) if a.size else 0.0


def _arrays(H):
    from paper_2003_09133_b200 import Dims5, PsfArray, compute_backprojection
    psf = PsfArray._wrap(Dims5.unchecked(*H.shape), H)
    return psf, compute_backprojection(psf)


@pytest.mark.parametrize("name", ["sym", "even", "asym", "f32"])
def test_projections_match_reference(proj, name):
    _torch()
    from paper_2003_09133_b200.arrays import Image, Volume
    from paper_2003_09133_b200.projector import backproject, backproject_adjoint, forward_project, normalizer
    H, g, f = proj[name + "__H"], proj[name + "__g"], proj[name + "__f"]
    psf, bp = _arrays(H)
    fwd = forward_project(psf, Volume(g)).data
    assert fwd.dtype == np.float64 and rel(fwd, proj[name + "__fwd"]) < 1e-12
    assert rel(backproject(bp, Image(f)).data, proj[name + "__bp"]) < 1e-12
    assert rel(backproject_adjoint(psf, Image(f)).data, proj[name + "__adj"]) < 1e-12
    assert rel(normalizer(bp, f.shape).data, proj[name + "__norm"]) < 1e-12


def test_reference_projector_kats():
    """test_projector.py:19-58 restated: zero volume, one voxel stamps its
    pattern exactly, border clipping, cell-shift equivariance."""
    _torch()
    from paper_2003_09133_b200 import Dims5, PsfArray
    from paper_2003_09133_b200.arrays import Volume
    from paper_2003_09133_b200.projector import forward_project, pattern_centre
    from paper_2003_09133_b200.synth import random_psf_like_reference as rpsf
    psf = PsfArray._wrap(Dims5(9, 9, 3, 3, 2), rpsf((9, 9, 3, 3, 2), seed=0))
    img = forward_project(psf, Volume(np.zeros((15, 15, 2))))
    assert img.shape == (15, 15) and not img.data.any()
    H = rpsf((5, 5, 3, 3, 2), density=1.0, seed=8)
    g = np.zeros((15, 15, 2)); g[7, 6, 1] = 2.0
    img = forward_project(PsfArray._wrap(Dims5(5, 5, 3, 3, 2), H), Volume(g))
    want = np.zeros((15, 15)); c = pattern_centre(5)
    want[7 - (c - 1):7 + c, 6 - (c - 1):6 + c] = 2.0 * H[:, :, 7 % 3, 6 % 3, 1]
    assert np.array_equal(img.data, want)
    ones = PsfArray._wrap(Dims5(5, 5, 3, 3, 1), np.ones((5, 5, 3, 3, 1), order="F"))
    g = np.zeros((7, 7, 1)); g[0, 0, 0] = 1.0
    img = forward_project(ones, Volume(g))
    assert img.data.sum() == 9.0 and np.count_nonzero(img.data) == 9
    H = rpsf((9, 9, 3, 3, 1), density=0.8, seed=4)
    psf = PsfArray._wrap(Dims5(9, 9, 3, 3, 1), H)
    g1 = np.zeros((31, 31, 1)); g1[10, 12, 0] = 1.0
    g2 = np.zeros((31, 31, 1)); g2[13, 12, 0] = 1.0
    f1 = forward_project(psf, Volume(g1)).data
    f2 = forward_project(psf, Volume(g2)).data
    assert np.array_equal(f1[6:15, :], f2[9:18, :])


def test_criterion_5_adjointness_on_gpu():
    """<Hg, f> = <g, H'f> within 1e-10 and the H' path equals the literal
    adjoint within 1e-12, 20 instances (test_acceptance.py:128-152)."""
    _torch()
    from paper_2003_09133_b200 import Dims5, PsfArray, compute_backprojection
    from paper_2003_09133_b200.arrays import Image, Volume
    from paper_2003_09133_b200.projector import backproject, backproject_adjoint, forward_project
    from paper_2003_09133_b200.synth import random_psf_like_reference as rpsf
    worst_rel = worst_pair = 0.0
    for i in range(20):
        psf = PsfArray._wrap(Dims5(9, 9, 3, 3, 3), rpsf((9, 9, 3, 3, 3), density=0.3, seed=2000 + i))
        bp = compute_backprojection(psf)
        rng = np.random.default_rng(3000 + i)
        g = Volume(rng.random((31, 31, 3)))
        f = Image(rng.random((31, 31)))
        lhs = float(np.vdot(forward_project(psf, g).data, f.data))
        via = backproject(bp, f).data
        rhs = float(np.vdot(g.data, via))
        worst_rel = max(worst_rel, abs(lhs - rhs) / abs(lhs))
        worst_pair = max(worst_pair, rel(via, backproject_adjoint(psf, f).data))
    assert worst_rel < 1e-10 and worst_pair < 1e-12


def test_rl_matches_reference(proj):
    _torch()
    from paper_2003_09133_b200.arrays import Image
    from paper_2003_09133_b200.projector import rl_run
    psf, bp = _arrays(proj["rl6__H"])
    st = rl_run(psf, bp, Image(proj["rl6__f"]), iterations=6)
    assert st.iterations == 6 and len(st.mse_history) == 6
    assert rel(st.estimate.data, proj["rl6__est"]) < 1e-9
    assert np.allclose(st.mse_history, proj["rl6__mse"], rtol=1e-9, atol=0)
    assert (st.estimate.data >= 0).all() and st.mse_history[-1] < st.mse_history[0]


def test_criterion_6_rl_recovers_two_point_scene(proj):
    """test_acceptance.py:155-180 on the GPU: top-2 voxels exact, MSE never
    increases, and the estimate tracks the reference's."""
    _torch()
    from paper_2003_09133_b200.arrays import Image
    from paper_2003_09133_b200.projector import rl_run
    psf, bp = _arrays(proj["rl20__H"])
    st = rl_run(psf, bp, Image(proj["rl20__f"]), iterations=20)
    est = st.estimate.data
    order = np.argsort(est.ravel())[::-1]
    top = {tuple(int(i) for i in np.unravel_index(k, est.shape)) for k in order[:2]}
    assert top == {(9, 11, 0), (21, 19, 2)}
    assert sum(b > a for a, b in zip(st.mse_history, st.mse_history[1:])) == 0
    assert st.dead_voxels == int(proj["rl20__dead"])
    assert np.allclose(st.mse_history, proj["rl20__mse"], rtol=1e-6, atol=1e-18)


def test_rl_zero_image_and_argument_checks():
    _torch()
    from paper_2003_09133_b200 import Dims5, DimMismatch, NonFiniteInput, PsfArray, compute_backprojection
    from paper_2003_09133_b200.arrays import Image
    from paper_2003_09133_b200.projector import rl_run
    from paper_2003_09133_b200.synth import random_psf_like_reference as rpsf
    psf = PsfArray._wrap(Dims5(5, 5, 3, 3, 1), rpsf((5, 5, 3, 3, 1), density=0.9, seed=5))
    bp = compute_backprojection(psf)
    st = rl_run(psf, bp, Image(np.zeros((9, 9))), iterations=3)
    assert not st.estimate.data.any() and st.mse_history == [0.0, 0.0, 0.0]
    with pytest.raises(ValueError):
        rl_run(psf, bp, Image(np.zeros((9, 9))), iterations=0)
    other = compute_backprojection(PsfArray._wrap(Dims5(7, 7, 3, 3, 1), rpsf((7, 7, 3, 3, 1), seed=1)))
    with pytest.raises(DimMismatch):
        rl_run(psf, other, Image(np.zeros((9, 9))), iterations=1)
    with pytest.raises(NonFiniteInput):
        rl_run(psf, bp, Image._wrap(np.full((9, 9), np.inf)), iterations=1)


@pytest.mark.parametrize("shape,img", [((15, 13, 5, 3, 2), (40, 33)), ((55, 55, 11, 11, 2), (121, 99)),
                                       ((8, 12, 7, 3, 2), (20, 17))])
def test_random_shapes_match_oracle(shape, img):
    _torch()
    from paper_2003_09133_b200 import Dims5, PsfArray, compute_backprojection
    from paper_2003_09133_b200.arrays import Image, Volume
    from paper_2003_09133_b200.projector import backproject, backproject_adjoint, forward_project
    from paper_2003_09133_b200.synth import random_psf_like_reference as rpsf
    H = rpsf(shape, density=0.5, seed=3, dtype=np.float32)
    psf = PsfArray._wrap(Dims5(*shape), H)
    bp = compute_backprojection(psf)
    rng = np.random.default_rng(4)
    g = rng.random((*img, shape[4]))
    f = rng.random(img)
    assert rel(forward_project(psf, Volume(g)).data, po.forward_project(H, g)) < 1e-12
    assert rel(backproject(bp, Image(f)).data, po.backproject(bp.data, f)) < 1e-12
    assert rel(backproject_adjoint(psf, Image(f)).data, po.backproject_adjoint(H, f)) < 1e-12


def test_forward_projection_is_deterministic():
    """rl_loop reuses the residual projection as the next iteration's
    projection; that is exact only if a projection repeats bit for bit."""
    torch = _torch()
    from paper_2003_09133_b200.projector import _to_device_f, forward_project_device
    from paper_2003_09133_b200.transform import hprime_device
    rng = np.random.default_rng(3)
    H = np.asfortranarray(rng.random((15, 13, 5, 3, 4)))
    g = np.asfortranarray(rng.random((40, 33, 4)))
    Hd, gd = _to_device_f(H, "cuda:0"), _to_device_f(g, "cuda:0")
    Hp = hprime_device(Hd)
    for kw in ({"Hp": Hp}, {}):
        a = forward_project_device(Hd, gd, **kw).clone()
        b = forward_project_device(Hd, gd, **kw)
        torch.cuda.synchronize()
        assert torch.equal(a, b)


def test_rl_kernels_match_reference_safe_divide():
    """lfbp_max_device / lfbp_safe_divide_peak_device / lfbp_rl_update_device
    against _safe_divide (projector.py:135-145), including zero and tiny
    denominators and an all-zero denominator (peak 0)."""
    torch = _torch()
    from paper_2003_09133_b200.projector import DeviceSlabOps
    rng = np.random.default_rng(4)
    num = rng.random(1000) * 3
    for den in (rng.random(1000), np.zeros(1000)):
        den = den.copy()
        den[::7] = 0.0
        den[::11] = 1e-15
        nd, dd = torch.from_numpy(num).cuda(), torch.from_numpy(den).cuda()
        peak = torch.zeros(1, dtype=torch.float64, device="cuda")
        DeviceSlabOps.max(dd, peak)
        assert float(peak.item()) == max(float(den.max()), 0.0)
        out = DeviceSlabOps.divide(nd, dd, 1e-12, peak, torch.empty_like(nd))
        want = po.safe_divide(num, den, 1e-12)
        assert out.cpu().numpy().tobytes() == want.tobytes()
        g0 = rng.random(1000)
        g = torch.from_numpy(g0.copy()).cuda()
        DeviceSlabOps.update(g, nd, dd, 1e-12, peak)
        assert g.cpu().numpy().tobytes() == (g0 * want).tobytes()


def test_rl_sharded_world_one_equals_rl_run(proj):
    """rl_run_sharded through a 1-rank NCCL group (its plane-range slicing
    and setup) gives the single-GPU rl_run result bit for bit."""
    torch = _torch()
    import socket

    import torch.distributed as dist

    from paper_2003_09133_b200.arrays import Image
    from paper_2003_09133_b200.projector import rl_run, rl_run_sharded
    psf, bp = _arrays(proj["rl6__H"])
    img = Image(proj["rl6__f"])
    want = rl_run(psf, bp, img, iterations=6)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        torch.cuda.set_device(0)
        sh = rl_run_sharded(psf, bp, img, iterations=6)
    finally:
        dist.destroy_process_group()
    assert (sh.z0, sh.z1) == (0, psf.dims.n_z)
    assert sh.state.estimate.data.tobytes() == want.estimate.data.tobytes()
    assert sh.state.mse_history == want.mse_history and sh.state.dead_voxels == want.dead_voxels


@pytest.mark.parametrize("shape,img", [((15, 13, 5, 3, 2), (40, 33)), ((8, 12, 7, 3, 2), (20, 17)),
                                       ((20, 18, 5, 7, 3), (33, 41)), ((33, 31, 11, 3, 2), (70, 23)),
                                       # tap classes of N = 17, 21, 31 taps (ceil(n_s / n_x)): the
                                       # multi-block register window + remainder path that the C3/C4
                                       # (N = 21, RL = 7) and C5 (N = 31, RL = 10) geometries take
                                       ((51, 51, 3, 3, 2), (40, 37)), ((85, 83, 5, 5, 2), (47, 44)),
                                       ((63, 63, 3, 3, 2), (45, 41)), ((62, 60, 3, 3, 2), (44, 39)),
                                       ((93, 93, 3, 3, 2), (50, 47)), ((93, 91, 3, 3, 1), (101, 37))])
def test_both_polyphase_forms_match_oracle(shape, img):
    """Every device form against the oracle, odd and even sizes: the H form
    of the forward projection and the H'-stamp backprojection run as
    polyphase convolutions (input-phase patterns), the H' forward and the
    adjoint as polyphase correlations (output-phase patterns)."""
    torch = _torch()
    from oracle.hprime_oracle import hprime_oracle
    from paper_2003_09133_b200.projector import (_to_device_f, _to_host_f, backproject_device,
                                                 forward_project_device)
    from paper_2003_09133_b200.synth import random_psf_like_reference as rpsf
    H = np.asfortranarray(rpsf(shape, density=0.7, seed=11, dtype=np.float64))
    Hp = np.asfortranarray(hprime_oracle(H))
    rng = np.random.default_rng(5)
    g = np.asfortranarray(rng.random((*img, shape[4])))
    f = np.asfortranarray(rng.random(img))
    Hd, Hpd = _to_device_f(H, "cuda:0"), _to_device_f(Hp, "cuda:0")
    gd, fd = _to_device_f(g, "cuda:0"), _to_device_f(f, "cuda:0")
    want_fwd = po.forward_project(H, g)
    assert rel(_to_host_f(forward_project_device(Hd, gd)), want_fwd) < 1e-12           # H form (convolution)
    if shape[0] % 2 and shape[1] % 2:
        assert rel(_to_host_f(forward_project_device(None, gd, Hp=Hpd)), want_fwd) < 1e-12   # H' form
    assert rel(_to_host_f(backproject_device(Hpd, fd, use_hprime=True)), po.backproject(Hp, f)) < 1e-12
    assert rel(_to_host_f(backproject_device(Hd, fd, use_hprime=False)), po.backproject_adjoint(H, f)) < 1e-12
    torch.cuda.synchronize()


def test_rl_even_sizes_match_oracle():
    """RL with even n_s, n_t (H forward and H'-stamp backward, both polyphase
    convolutions on the device) against the oracle's RL."""
    _torch()
    from paper_2003_09133_b200 import Dims5, PsfArray, compute_backprojection
    from paper_2003_09133_b200.arrays import Image
    from paper_2003_09133_b200.projector import rl_run
    from paper_2003_09133_b200.synth import random_psf_like_reference as rpsf
    shape = (12, 10, 5, 3, 3)
    H = rpsf(shape, density=0.8, seed=9, dtype=np.float64)
    psf = PsfArray._wrap(Dims5(*shape), H)
    bp = compute_backprojection(psf)
    f = np.random.default_rng(2).random((25, 19)) + 0.05
    st = rl_run(psf, bp, Image(f), iterations=4)
    g_ref, hist_ref, norm_ref = po.rl_run(H, bp.data, f, iterations=4)
    assert rel(st.normalizer.data, norm_ref) < 1e-12
    assert rel(st.estimate.data, g_ref) < 1e-10
    assert np.allclose(st.mse_history, hist_ref, rtol=1e-10, atol=0)


@pytest.mark.parametrize("shape,img", [((15, 13, 5, 3, 4), (40, 33)), ((21, 19, 7, 5, 2), (64, 71)),
                                       ((12, 10, 3, 5, 3), (29, 30))])
def test_tma_staged_windows_equal_cooperative_fill_bitwise(monkeypatch, shape, img):
    """poly_tma_kernel (TMA-staged windows, zero fill outside the padded
    sub-images, odd window origins) runs the same sums in the same order as
    poly_tile_kernel, so every projection form agrees bit for bit."""
    torch = _torch()
    from paper_2003_09133_b200.projector import _to_device_f, backproject_device, forward_project_device
    from paper_2003_09133_b200.transform import hprime_device
    rng = np.random.default_rng(sum(shape))
    H = np.asfortranarray(rng.random(shape))
    g = np.asfortranarray(rng.random((*img, shape[4])))
    f = np.asfortranarray(rng.random(img))
    Hd, gd, fd = _to_device_f(H, "cuda:0"), _to_device_f(g, "cuda:0"), _to_device_f(f, "cuda:0")
    odd = shape[0] % 2 == 1 and shape[1] % 2 == 1
    Hp = hprime_device(Hd) if odd else None

    def run():
        outs = [forward_project_device(Hd, gd).clone(), backproject_device(Hd, fd, use_hprime=False).clone()]
        if odd:
            outs += [forward_project_device(Hd, gd, Hp=Hp).clone(), backproject_device(Hp, fd).clone()]
        torch.cuda.synchronize()
        return outs
    monkeypatch.setenv("LFBP_PROJ_TMA", "1")
    tma = run()
    monkeypatch.setenv("LFBP_PROJ_TMA", "0")
    coop = run()
    for a, b in zip(tma, coop):
        assert torch.equal(a, b)
