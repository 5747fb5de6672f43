"""bench.py contract on CPU: the reference arm prints one JSON line with the
driver's keys (the GPU arm is exercised on the GPU box)."""
import json
import os
import subprocess
import sys

from conftest import ROOT


import pytest

REF_INSTALLED = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "lfbp"))


@pytest.mark.parametrize("arm", ["port", "reference"])
def test_reference_arm_json_line(arm):
    """The reference arm: the oracle's numpy restatement on every host thread
    (default, kind "port"), or with --ref-mode unmodified the unmodified lfbp
    from baseline/_ref, one process per plane (kind "reference", checked
    against the reference's digests)."""
    if arm == "reference" and not REF_INSTALLED:
        pytest.skip("baseline/_ref not installed (tools/install_reference.sh)")
    extra = ["--ref-mode", "unmodified"] if arm == "reference" else []
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                        "--steps", "2", "--warmup", "1", "--cpu-planes", "2", *extra],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == arm and d["cpu_baseline"]["cores"] >= 1
    if arm == "reference":
        assert d["cpu_baseline"]["matches_reference_digests"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["dtype"] == "f32"


def test_reference_arm_under_torchrun_prints_once():
    """N > 1 launch as the driver does it: rank 0 alone runs and prints the
    reference arm's line, the other rank exits 0 without output."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--config", "C1",
                        "--steps", "1", "--warmup", "1", "--cpu-planes", "2"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
