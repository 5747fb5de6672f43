"""LF5 container host side (no GPU): byte-identical to files the reference
wrote (tests/golden), the reference's header checks (pkg/tests/test_fileio.py
restated), and the C-ABI header parser."""
import hashlib
import struct

import numpy as np
import pytest

from paper_2003_09133_b200 import BackprojArray, Dims5, DimsError, FormatError, InvalidDims, IoError, PsfArray
from paper_2003_09133_b200 import lf5


def sha(path):
    return hashlib.sha256(open(path, "rb").read()).hexdigest()


def test_save_is_byte_identical_to_reference_files(golden_small, golden_lf5, tmp_path):
    cases, arrays = golden_small
    for name, want in golden_lf5.items():
        H = arrays[name + "__H"]
        p = tmp_path / f"{name}.lf5"
        lf5.save(PsfArray(Dims5(*H.shape), H), p)
        assert sha(p) == want["in_sha256"], name
        Hp = arrays[name + "__Hp"]
        q = tmp_path / f"{name}.out.lf5"
        lf5.save(BackprojArray._wrap(Dims5(*Hp.shape), Hp), q)
        assert sha(q) == want["out_sha256"], name


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_roundtrip_and_header(tmp_path, dtype):
    d = Dims5(9, 7, 3, 5, 2)
    H = np.asfortranarray(np.random.default_rng(1).random(d.shape).astype(dtype))
    p = tmp_path / "h.lf5"
    lf5.save(PsfArray(d, H), p)
    blob = p.read_bytes()
    code = 1 if dtype == np.float32 else 2
    assert blob[:32] == b"LF5D" + struct.pack("<I", 1) + bytes([code]) + b"\x00" * 3 + struct.pack("<5I", *d.shape)
    shape, dt = lf5.read_header(p)
    assert shape == d.shape and dt == np.dtype(dtype)
    back = lf5.load(p)
    assert back.data.tobytes(order="F") == H.tobytes(order="F") and not back.data.flags.writeable


@pytest.mark.parametrize("mangle", [
    lambda b: b[:16], lambda b: b"XXXX" + b[4:], lambda b: b[:4] + struct.pack("<I", 9) + b[8:],
    lambda b: b[:8] + b"\x07" + b[9:], lambda b: b[:9] + b"\x00\x01\x00" + b[12:],
    lambda b: b + b"\x00" * 8, lambda b: b[:-8],
])
def test_corrupted_headers_rejected(tmp_path, mangle):
    d = Dims5(3, 3, 3, 3, 1)
    p = tmp_path / "h.lf5"
    lf5.save(PsfArray(d, np.random.default_rng(1).random(d.shape)), p)
    bad = tmp_path / "bad.lf5"
    bad.write_bytes(mangle(p.read_bytes()))
    with pytest.raises(FormatError):
        lf5.read_header(bad)


def test_missing_file_and_dims_contract(tmp_path):
    with pytest.raises(IoError):
        lf5.read_header(tmp_path / "nope.lf5")
    p = tmp_path / "bad.lf5"
    p.write_bytes(b"LF5D" + struct.pack("<I", 1) + b"\x01" + b"\x00" * 3 + struct.pack("<5I", 4, 4, 4, 4, 1)
                  + b"\x00" * (256 * 4))
    with pytest.raises(DimsError):
        lf5.load(p)
    assert lf5.load(p, allow_invalid_dims=True).dims.shape == (4, 4, 4, 4, 1)


def test_negative_values_rejected_on_load(tmp_path):
    d = Dims5(3, 3, 3, 3, 1)
    p = tmp_path / "neg.lf5"
    lf5.save(np.asfortranarray(-np.ones(d.shape)), p)
    with pytest.raises(InvalidDims):
        lf5.load(p)


def test_create_sizes_the_file(tmp_path):
    from paper_2003_09133_b200 import _native
    p = tmp_path / "c.lf5"
    _native.check(_native.lib().lfbp_lf5_create(bytes(p), _native.dims_array((5, 5, 3, 3, 4)), 1))
    assert p.stat().st_size == 32 + 5 * 5 * 3 * 3 * 4 * 4
    assert lf5.read_header(p) == ((5, 5, 3, 3, 4), np.dtype("<f4"))


def test_cli_plan_and_errors(tmp_path, capsys):
    from paper_2003_09133_b200.__main__ import main
    assert main(["plan", "195,195,15,15,51"]) == 0
    assert '"J"' in capsys.readouterr().out
    assert main(["transform", str(tmp_path / "missing.lf5"), str(tmp_path / "o.lf5")]) == 2
    assert "IoError" in capsys.readouterr().err


def test_failed_in_place_transform_leaves_the_input_intact(tmp_path):
    """transform_file(f, f) writes to a temporary next to f and renames it
    only on success: when the transform fails (here: no GPU, or any device
    error) the input file is neither truncated nor deleted, and no temporary
    is left behind."""
    import os

    import torch
    d = Dims5(9, 7, 3, 5, 2)
    H = np.asfortranarray(np.random.default_rng(3).random(d.shape).astype(np.float32))
    p = tmp_path / "h.lf5"
    lf5.save(PsfArray(d, H), p)
    before = sha(p)
    if torch.cuda.is_available():
        pytest.skip("exercises the failure path; the GPU test covers the successful in-place transform")
    with pytest.raises(Exception):
        lf5.transform_file(p, p)
    assert sha(p) == before
    assert sorted(os.listdir(tmp_path)) == ["h.lf5"]
