"""bench.py on the GPU (-m gpu): the headline line's keys, and the z-split
multi-rank path -- two ranks on one device over gloo (functional check of
the shard plumbing; the ranks share no data and never wait on each other's
kernels) -- with every rank's planes verified against the reference's
per-plane digests."""
import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _line(stdout):
    lines = [l for l in stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, stdout
    return json.loads(lines[0])


def test_bench_line_on_c2():
    _gpu()
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "C2", "--steps", "5",
                        "--warmup", "3", "--no-cpu", "--e2e-steps", "1"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks",
                "shards"):
        assert key in d, key
    assert d["verified_vs_reference_digests"] is True
    assert d["e2e"]["matches_reference_digests"] is True
    assert d["gpu_launches"] == 5 and d["roofline"]["bound"] == "hbm"
    assert d["config"]["workload"].startswith("C2 ")


def test_bench_z_split_two_ranks_verifies_every_slab():
    _gpu()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, LFBP_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--config", "C2", "--steps", "3", "--warmup", "3", "--no-cpu",
                        "--e2e-steps", "1"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["shards"]["planes_per_rank"] == [25, 26]
    assert [s["planes"] for s in d["shards"]["per_rank"]] == [[0, 25], [25, 51]]
    assert all(s["verified"] is True for s in d["shards"]["per_rank"])
    assert d["verified_vs_reference_digests"] is True
    assert d["e2e"]["matches_reference_digests"] is True
    assert "shared host H'" in d["e2e"].get("host_output", "")   # one host H' gathered from both slabs
