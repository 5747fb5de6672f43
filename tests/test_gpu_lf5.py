"""LF5 file -> GPU -> LF5 file (GPU; -m gpu): byte-identical to the files the
reference's `lfbp transform` path writes (tests/golden), at full C2 size
against the reference's H' digest, plus z-slab device loads / stores."""
import hashlib

import numpy as np
import pytest

from conftest import load_digests
from oracle.hprime_oracle import hprime_oracle

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def sha(path):
    return hashlib.sha256(open(path, "rb").read()).hexdigest()


def test_transform_file_matches_reference_files(golden_small, golden_lf5, tmp_path, caplog):
    _torch()
    import logging

    from paper_2003_09133_b200 import Dims5, PsfArray, lf5
    cases, arrays = golden_small
    for name, want in golden_lf5.items():
        H = arrays[name + "__H"]
        fin, fout = tmp_path / f"{name}.lf5", tmp_path / f"{name}.out.lf5"
        lf5.save(PsfArray(Dims5(*H.shape), H), fin)
        assert sha(fin) == want["in_sha256"]
        with caplog.at_level(logging.WARNING):
            caplog.clear()
            lf5.transform_file(fin, fout)
        assert sha(fout) == want["out_sha256"], name
        assert ("dropped" in caplog.text) == (H.shape[0] % 2 == 0 or H.shape[1] % 2 == 0)
        if H.shape[0] % 2 and H.shape[1] % 2:   # inverse restores the input file
            back = tmp_path / f"{name}.back.lf5"
            lf5.transform_file(fout, back, inverse=True)
            assert sha(back) == want["in_sha256"]


def test_transform_file_in_place(golden_small, golden_lf5, tmp_path):
    """`transform f f` works like the reference CLI (it loads the whole file
    before saving): the result replaces the input only once it is complete,
    and no temporary is left behind.  A failing in-place call (negative
    values) leaves the input byte for byte."""
    _torch()
    import os

    from paper_2003_09133_b200 import Dims5, InvalidDims, PsfArray, lf5
    cases, arrays = golden_small
    for name, want in list(golden_lf5.items())[:4]:
        H = arrays[name + "__H"]
        f = tmp_path / f"{name}.lf5"
        lf5.save(PsfArray(Dims5(*H.shape), H), f)
        lf5.transform_file(f, f)
        assert sha(f) == want["out_sha256"], name
    assert all(not n.startswith(".") and "lfbp-tmp" not in n for n in os.listdir(tmp_path))
    neg = np.asfortranarray(-np.ones((5, 5, 3, 3, 2), dtype=np.float32))
    g = tmp_path / "neg.lf5"
    lf5.save(neg, g)
    before = sha(g)
    with pytest.raises(InvalidDims):
        lf5.transform_file(g, g)
    assert sha(g) == before
    assert not any("lfbp-tmp" in n for n in os.listdir(tmp_path))


def test_transform_file_errors(tmp_path):
    _torch()
    from paper_2003_09133_b200 import EvenPixelDims, InvalidDims, lf5
    neg = np.asfortranarray(-np.ones((5, 5, 3, 3, 2), dtype=np.float32))
    fin, fout = tmp_path / "neg.lf5", tmp_path / "neg.out.lf5"
    lf5.save(neg, fin)
    with pytest.raises(InvalidDims):
        lf5.transform_file(fin, fout)
    assert not fout.exists()
    even = np.asfortranarray(np.ones((4, 5, 3, 3, 1)))
    lf5.save(even, tmp_path / "even.lf5")
    with pytest.raises(EvenPixelDims):
        lf5.transform_file(tmp_path / "even.lf5", tmp_path / "even.out.lf5", inverse=True)


def test_transform_file_c2_full_size(tmp_path, monkeypatch):
    torch = _torch()
    from paper_2003_09133_b200 import lf5
    from paper_2003_09133_b200.configs import WORKLOADS
    from paper_2003_09133_b200.synth import baseline_psf
    d = load_digests("C2")
    w = WORKLOADS["C2"]
    H = baseline_psf(w)
    fin, fout = tmp_path / "c2.lf5", tmp_path / "c2.out.lf5"
    lf5.save(H, fin)
    del H
    monkeypatch.setenv("LFBP_CHUNK_MB", "128")
    lf5.transform_file(fin, fout)
    h = hashlib.sha256()
    with open(fout, "rb") as f:
        assert f.read(32) == lf5.header_bytes(w.shape, np.float32)
        while True:
            b = f.read(64 << 20)
            if not b:
                break
            h.update(b)
    assert h.hexdigest() == d["hprime_sha256"]


def test_load_and_store_device_slabs(tmp_path):
    torch = _torch()
    from paper_2003_09133_b200 import hprime_device, lf5
    from paper_2003_09133_b200.synth import random_psf_like_reference
    shape = (33, 31, 7, 5, 9)
    H = random_psf_like_reference(shape, density=1.0, seed=2, dtype=np.float32)
    fin = tmp_path / "in.lf5"
    lf5.save(H, fin)
    full = lf5.load_device(fin)
    torch.cuda.synchronize()
    assert full.permute(4, 3, 2, 1, 0).contiguous().cpu().numpy().tobytes() == H.tobytes(order="F")
    # two z-slabs, transformed separately, stored into one output file
    fout = tmp_path / "out.lf5"
    for k, (z0, z1) in enumerate([(0, 4), (4, 9)]):
        slab = lf5.load_device(fin, z_range=(z0, z1))
        lf5.store_device(fout, hprime_device(slab), z0=z0, create_shape=shape if k == 0 else None)
    torch.cuda.synchronize()
    got = np.fromfile(fout, dtype=np.float32, offset=32)
    assert got.tobytes() == hprime_oracle(H).tobytes(order="F")


def test_cli_transform_and_verify(tmp_path, capsys):
    _torch()
    from paper_2003_09133_b200 import lf5
    from paper_2003_09133_b200.__main__ import main
    from paper_2003_09133_b200.synth import random_psf_like_reference
    H = random_psf_like_reference((21, 19, 7, 5, 3), density=0.8, seed=1, dtype=np.float32)
    fin, fout = tmp_path / "in.lf5", tmp_path / "out.lf5"
    lf5.save(H, fin)
    assert main(["transform", str(fin), str(fout)]) == 0
    assert main(["verify", str(fin), "--against", str(fout)]) == 0
    assert "PASS" in capsys.readouterr().out
    bad = np.fromfile(fout, dtype=np.uint8)
    bad[32 + 4 * 100] ^= 1                      # element 100 (0-based, F order)
    bad.tofile(fout)
    assert main(["verify", str(fin), "--against", str(fout)]) == 1
    out = capsys.readouterr().out
    assert "FAIL" in out and "(s,t,x,y,z)=(17, 5, 1, 1, 1)" in out
