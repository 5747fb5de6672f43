"""The N > 1 z-slab path on CPU: world_size 2 over gloo.

Each rank takes its contiguous plane range of C1 (shard_planes), generates
only those planes, rearranges them (the CPU oracle stands in for the GPU
kernel here) and writes its slab into one shared host array at its own
plane offset -- no collective moves H' data.  Rank 0 then checks the
assembled array against the reference's per-plane digests, and the
max-over-ranks timing reduction bench.py uses.
"""
import hashlib
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, path, result_path):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist

    from oracle.hprime_oracle import hprime_oracle
    from paper_2003_09133_b200.configs import WORKLOADS
    from paper_2003_09133_b200.shard import open_shared_host, rank_slab, write_slab
    from paper_2003_09133_b200.synth import baseline_psf

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = WORKLOADS["C1"]
    slab_shape, z0, z1 = rank_slab(w.shape, world, rank)
    H = baseline_psf(w, z0, z1)
    assert H.shape == slab_shape
    Hp = hprime_oracle(H)                      # stand-in for the per-rank kernel
    if rank == 0:
        open_shared_host(path, w.shape, w.dtype, create=True).flush()
    dist.barrier()
    shared = open_shared_host(path, w.shape, w.dtype)
    write_slab(shared, z0, Hp)
    shared.flush()
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)   # bench.py's max-over-ranks time
    dist.barrier()
    if rank == 0:
        full = open_shared_host(path, w.shape, w.dtype)
        digests = [hashlib.sha256(np.asarray(full[..., z]).tobytes(order="F")).hexdigest()
                   for z in range(w.shape[4])]
        with open(result_path, "w") as f:
            f.write(repr((digests, float(t.item()))))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_z_slabs_over_gloo_assemble_the_reference_result(tmp_path, world):
    from conftest import load_digests
    d = load_digests("C1")
    path = str(tmp_path / "hprime.f32")
    result = str(tmp_path / "result.txt")
    mp.spawn(_worker, args=(world, _free_port(), path, result), nprocs=world, join=True)
    digests, tmax = eval(open(result).read())
    assert digests == d["hprime_plane_sha256"]
    assert tmax == float(world)
