"""The reference's own hot-path test files, UNMODIFIED, run against the GPU
drop-in through the unmodified reference package (baseline/_ref, installed
by tools/install_reference.sh): tests/lfbp_dropin_plugin.py rebinds
``lfbp.compute_backprojection`` / ``compute_psf_from_backprojection`` (and
the copies ``lfbp.transform``, ``lfbp.bench``, ``lfbp.cli`` imported) to the
drop-ins before the reference's test modules load -- INTEGRATION.md's swap,
executed.  Files: test_transform.py, test_oracle.py, test_acceptance.py
(with LFBP_ACCEPT_FULL=1: the full-scale (181,181,95,55,1) case), and the
callers' tests test_bench.py, test_cli.py."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

REF = os.path.join(ROOT, "baseline", "_ref")
FILES = ["test_transform.py", "test_oracle.py", "test_acceptance.py", "test_bench.py", "test_cli.py"]
# need matplotlib, which this image lacks; they fail the same way without the drop-in
NEEDS_MATPLOTLIB = ["test_bench.py::test_render_figure", "test_cli.py::test_bench_subcommand"]


def _have_reference():
    return os.path.isdir(os.path.join(REF, "lfbp")) and os.path.isdir(os.path.join(REF, "tests"))


def _run(tmp_path, extra_env=None, files=FILES):
    report = tmp_path / "dropin.json"
    ini = tmp_path / "pytest.ini"
    ini.write_text("[pytest]\n")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tests")])
    env["LFBP_DROPIN_REPORT"] = str(report)
    env.update(extra_env or {})
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "lfbp_dropin_plugin", "-p", "no:cacheprovider",
           "-c", str(ini), "--rootdir", REF]
    cmd += [os.path.join(REF, "tests", f) for f in files]
    cmd += ["-k", " and ".join(f"not {d.split('::')[1]}" for d in NEEDS_MATPLOTLIB)]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=str(tmp_path), timeout=1800)
    rep = json.loads(report.read_text()) if report.exists() else None
    return r, rep


def test_plugin_binds_the_dropins_into_the_reference():
    """CPU: the swap itself (no compute)."""
    if not _have_reference():
        pytest.skip("reference not installed (tools/install_reference.sh)")
    code = ("import sys; sys.path[:0] = [%r, %r, %r]\n"
            "import lfbp_dropin_plugin as p, lfbp, lfbp.cli, lfbp.bench, lfbp.transform\n"
            "from paper_2003_09133_b200 import transform as g\n"
            "bound = p.bind()\n"
            "assert lfbp.compute_backprojection is g.compute_backprojection\n"
            "assert lfbp.transform.compute_psf_from_backprojection is g.compute_psf_from_backprojection\n"
            "assert lfbp.cli.compute_backprojection is g.compute_backprojection\n"
            "assert lfbp.bench.compute_backprojection is g.compute_backprojection\n"
            "print(len(bound))\n") % (REF, ROOT, os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert int(r.stdout.strip()) == 7


@pytest.mark.gpu
def test_reference_hot_path_tests_pass_on_the_gpu_dropin(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not _have_reference():
        pytest.skip("reference not installed (tools/install_reference.sh)")
    r, rep = _run(tmp_path, {"LFBP_ACCEPT_FULL": "1"})
    tail = (r.stdout[-3000:] + r.stderr[-2000:])
    assert r.returncode == 0, tail
    assert rep is not None and rep["exitstatus"] == 0, tail
    assert "lfbp.compute_backprojection" in rep["bound"] and "lfbp.cli.compute_backprojection" in rep["bound"]
    assert rep["launches"] > 100, rep          # the kernels ran: one launch per drop-in call at least
    summary = [l for l in r.stdout.splitlines() if l.strip()][-1]
    assert " passed" in summary and "failed" not in summary and "skipped" not in summary, tail
