"""The C-ABI library loads and exports every declared symbol; host-only
entry points behave like the reference (no GPU needed, no compute calls)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2003_09133_b200 import Dims5, InvalidDims, _native, plan
from paper_2003_09133_b200.configs import WORKLOADS
from paper_2003_09133_b200.shard import imbalance, shard_planes


def _declared():
    names = set()
    inc = os.path.join(ROOT, "include")
    for fn in os.listdir(inc):
        if fn.endswith(".h"):
            text = open(os.path.join(inc, fn)).read()
            names |= set(re.findall(r"^\s*(?:const\s+)?[\w\*]+\s+\*?(lfbp_\w+)\s*\(", text, re.M))
    return names


def test_library_exports_every_header_symbol():
    lib = _native.lib()
    declared = _declared()
    assert len(declared) >= 11
    for name in declared:
        assert hasattr(lib, name), name
    assert set(_native.EXPORTS) == declared


def test_version_and_no_error_initially():
    assert b"sm_100a" in _native.lib().lfbp_version()


@pytest.mark.parametrize("shape,ok", [
    ((9, 7, 3, 7, 2), True), ((5, 5, 3, 3, 1), True), ((4, 5, 3, 3, 1), True), ((1, 1, 1, 1, 1), True),
    ((9, 9, 4, 3, 1), False), ((9, 9, 3, 2, 1), False), ((2, 9, 3, 3, 1), False), ((9, 2, 3, 3, 1), False),
    ((0, 9, 3, 3, 1), False), ((9, 9, 3, 3, 0), False), ((3, 3, 5, 3, 1), False),
])
def test_check_dims_matches_dims5(shape, ok):
    rc = _native.lib().lfbp_check_dims(_native.dims_array(shape))
    assert (rc == _native.OK) == ok
    if ok:
        Dims5(*shape)
    else:
        assert rc == _native.ERR_INVALID_DIMS
        with pytest.raises(InvalidDims):
            Dims5(*shape)


def test_dropped_source_count():
    f = _native.lib().lfbp_dropped_source_count
    assert f(_native.dims_array((4, 5, 3, 3, 1))) == 45
    assert f(_native.dims_array((9, 9, 3, 3, 3))) == 0
    assert f(_native.dims_array((6, 6, 3, 5, 2))) == (36 - 25) * 15 * 2
    assert f(_native.dims_array((4, 4, 4, 3, 1))) == -1


def test_shard_planes_c_and_python_agree():
    for n_z in (1, 9, 51, 64, 41, 101):
        for g in (1, 2, 4, 8):
            cover = []
            for k in range(g):
                a, b = ctypes.c_int64(), ctypes.c_int64()
                assert _native.lib().lfbp_shard_planes(n_z, g, k, ctypes.byref(a), ctypes.byref(b)) == 0
                assert (a.value, b.value) == shard_planes(n_z, g, k)
                cover.extend(range(a.value, b.value))
            assert cover == list(range(n_z))
    assert imbalance(64, 8) == 1.0
    assert abs(imbalance(51, 8) - 7 / (51 / 8)) < 1e-12


@pytest.mark.parametrize("cfg", list(WORKLOADS))
def test_plans_for_every_config_fit_b200(cfg):
    w = WORKLOADS[cfg]
    p = plan(w.shape, w.dtype)
    assert p["smem_bytes"] <= 232448
    assert p["stages"] >= 2 and p["grid"] >= 148
    assert p["n_units"] < 2 ** 31
    # pitch is congruent to the x-stride mod 16 (linear smem addressing over x)
    n_s, n_t = w.shape[:2]
    assert p["row_pitch"] % 16 == (n_s * n_t * w.itemsize) % 16
    # one staged unit holds J full rows per x (or an i-chunk) plus alignment slack
    run = (p["J"] * n_s if p["n_chunks"] == 1 else p["C"]) * w.itemsize
    assert p["row_pitch"] >= run + 32
    assert p["stage_bytes"] >= w.shape[2] * p["row_pitch"] + 32


def test_plan_chunks_huge_slabs():
    p = plan((4001, 9, 2001, 3, 1), np.float64)
    assert p["n_chunks"] > 1 and p["J"] == 1


def test_compute_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    buf = np.zeros(64, dtype=np.float32)
    ptr = buf.ctypes.data_as(ctypes.c_void_p)
    rc = _native.lib().lfbp_hprime_device(ptr, ptr, _native.dims_array((3, 3, 1, 1, 1)), 1, 0, 0, 1, None)
    assert rc != _native.OK
    out = np.zeros(64, dtype=np.float32)
    rc = _native.lib().lfbp_hprime_host(ptr, out.ctypes.data_as(ctypes.c_void_p),
                                        _native.dims_array((3, 3, 1, 1, 1)), 1, 0, 0, 0)
    assert rc == _native.ERR_CUDA
    assert _native.last_error()


def test_argument_errors():
    lib = _native.lib()
    d = _native.dims_array((5, 5, 3, 3, 1))
    assert lib.lfbp_hprime_device(None, None, d, 1, 0, 0, 1, None) == _native.ERR_ARGUMENT
    assert lib.lfbp_hprime_device(None, None, d, 3, 0, 0, 1, None) == _native.ERR_ARGUMENT
    assert lib.lfbp_hprime_device(None, None, _native.dims_array((4, 5, 3, 3, 1)), 1, 1, 0, 1, None) \
        == _native.ERR_EVEN_PIXEL_DIMS
    assert lib.lfbp_hprime_host(None, None, _native.dims_array((5, 5, 2, 3, 1)), 1, 0, 0, 0) \
        == _native.ERR_INVALID_DIMS


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    """No CPU fallback: without libhprime.so every compute call raises."""
    from paper_2003_09133_b200 import Dims5, NativeError, PsfArray, compute_backprojection
    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setattr(_native, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(NativeError):
        compute_backprojection(PsfArray(Dims5(3, 3, 3, 3, 1), np.ones((3, 3, 3, 3, 1))))


def test_dropin_mirrors_reference_errors_and_types():
    from paper_2003_09133_b200 import BackprojArray, Dims5, EvenPixelDims, InvalidDims, PsfArray
    from paper_2003_09133_b200 import compute_psf_from_backprojection
    with pytest.raises(InvalidDims):
        Dims5(True, 3, 3, 3, 1)
    with pytest.raises(InvalidDims):
        PsfArray(Dims5(3, 3, 3, 3, 1), -np.ones((3, 3, 3, 3, 1)))
    with pytest.raises(InvalidDims):
        PsfArray(Dims5(3, 3, 3, 3, 1), np.full((3, 3, 3, 3, 1), np.nan))
    psf = PsfArray(Dims5(3, 3, 3, 3, 1), np.ones((3, 3, 3, 3, 1), dtype=np.int32))
    assert psf.dtype == np.float64 and not psf.data.flags.writeable and psf.data.flags.f_contiguous
    with pytest.raises(AttributeError):
        psf.dims = None
    # the even-dims inverse is refused before any device work
    with pytest.raises(EvenPixelDims):
        compute_psf_from_backprojection(BackprojArray._wrap(Dims5(4, 5, 3, 3, 1), np.ones((4, 5, 3, 3, 1), order="F")))


def test_multi_host_rejects_overlapping_buffers():
    from paper_2003_09133_b200.shard import rearrange_multi_host
    H = np.zeros((5, 5, 3, 3, 2), dtype=np.float32, order="F")
    with pytest.raises(ValueError, match="overlap"):
        rearrange_multi_host(H, H, [0])


def _build_c_example(tmp_path):
    """examples/hprime_host.c against include/lfbp_hprime.h as plain C99."""
    import subprocess
    from conftest import ROOT
    exe = str(tmp_path / "hprime_host")
    libdir = os.path.join(ROOT, "paper_2003_09133_b200")
    r = subprocess.run(["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "examples", "hprime_host.c"), "-L", libdir, "-lhprime",
                        f"-Wl,-rpath,{libdir}", "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_header_is_plain_c_and_the_abi_runs_from_c(tmp_path):
    import subprocess
    r = subprocess.run([_build_c_example(tmp_path), "--abi"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "abi ok" in r.stdout


@pytest.mark.parametrize("threads", [1, 3, 12, 16])
@pytest.mark.parametrize("nbytes", [34_692_100, (4 << 20) + 4, (64 << 20) + 1, 12 * 64 * 100_003 + 4])
def test_host_copy_covers_every_byte(threads, nbytes):
    """The staging memcpy pool splits [0, n) over its workers: every byte is
    copied whatever n mod workers is.  34,692,100 B is one (155,155,19,19) f32
    plane -- with 12 workers the former split (floor(n/parts) rounded to 64)
    left its last 4 bytes uncopied."""
    src = np.frombuffer(np.random.default_rng(nbytes % 1000).bytes(nbytes), dtype=np.uint8)
    dst = np.zeros(nbytes, dtype=np.uint8)
    rc = _native.lib().lfbp_host_copy(dst.ctypes.data_as(ctypes.c_void_p), src.ctypes.data_as(ctypes.c_void_p),
                                      nbytes, threads)
    assert rc == _native.OK
    assert np.array_equal(dst, src)


def test_plan_candidates_are_exported():
    from paper_2003_09133_b200 import plan_candidates
    large, small = plan_candidates(1), plan_candidates(0)
    assert len(large) >= 8 and len(small) >= 4
    assert all(len(k) == 6 and k[0] >= 1 and k[1] >= 1 and k[2] >= 1 for k in large + small)
    assert len(set(large)) == len(large)
    assert _native.lib().lfbp_plan_candidates(7, None, 0) < 0


@pytest.mark.parametrize("cfg", ["C2", "C3", "C4", "C5"])
def test_round2_plan_flags(monkeypatch, cfg):
    """Planner side of the round-2 kernel options (no GPU): the task consumer
    stages runs at a 16-byte row pitch; z-chunked and dynamic-ticket plans
    keep their flags (also with several producer warps); the tuner's
    candidate list holds each of them."""
    from paper_2003_09133_b200 import plan, plan_candidates
    from paper_2003_09133_b200.configs import WORKLOADS
    w = WORKLOADS[cfg]
    base = plan(w.shape, w.dtype)
    assert base["row_pitch"] % 16 == (w.shape[0] * w.shape[1] * w.itemsize) % 16
    monkeypatch.setenv("LFBP_KFLAGS", "32")
    p = plan(w.shape, w.dtype)
    assert p["flags"] == 32 and p["row_pitch"] % 16 == 0
    assert p["row_pitch"] >= p["J"] * w.shape[0] * w.itemsize + 32
    assert p["stage_bytes"] >= 64 + 16 + w.shape[2] * p["row_pitch"]
    for f in (64, 128, 200):
        monkeypatch.setenv("LFBP_KFLAGS", str(f))
        assert plan(w.shape, w.dtype)["flags"] == f
    monkeypatch.setenv("LFBP_KFLAGS", "128")
    wide = plan((181, 181, 95, 55, 1))     # three producer warps share each ticket
    assert wide["flags"] == 128 and wide["producers"] == 3
    flags = {k[4] for k in plan_candidates(1)}
    assert {32 | 128, 8 | 64, 8 | 128} <= flags
