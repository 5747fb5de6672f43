"""The z-sharded Richardson-Lucy loop (projector.rl_loop / rl_run_sharded)
on CPU: world_size 2 over gloo, and world_size 1.

The loop's orchestration -- partial forward projections summed with one
all-reduce per iteration, the normalizer peak reduced with MAX, the
dead-voxel count with SUM, the residual projection reused as the next
iteration's projection, the fused update -- is checked with the CPU oracle
standing in for the device kernels (the product path's DeviceSlabOps only
calls the C-ABI).  Reference: projector.py:162-196, tolerance 1e-12 as in
the reference's own projector tests.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

SHAPE = (9, 9, 3, 3, 5)
IMG = (13, 12)
ITERS = 4


class OracleOps:
    """Same methods as projector.DeviceSlabOps, computed by the oracle on
    CPU tensors (F layout)."""

    def __init__(self, H, Hp):
        self.H, self.Hp = H, Hp

    def forward(self, g, out):
        from oracle.projector_oracle import forward_project
        out.copy_(torch.from_numpy(forward_project(self.H, g.numpy())))
        return out

    def back(self, img, out):
        from oracle.projector_oracle import backproject
        out.copy_(torch.from_numpy(backproject(self.Hp, img.numpy())))
        return out

    @staticmethod
    def max(x, peak):
        peak.fill_(max(float(x.max()), 0.0) if x.numel() else 0.0)
        return peak

    @staticmethod
    def _divide(num, den, eps, pk):
        out = np.zeros(num.shape)
        if pk <= 0.0:
            return out
        ok = den >= eps * pk
        if eps * pk == 0.0:
            ok &= den > 0.0
        np.divide(num, den, out=out, where=ok)
        return out

    def divide(self, num, den, eps, peak, out):
        out.copy_(torch.from_numpy(self._divide(num.numpy(), den.numpy(), eps, float(peak.item()))))
        return out

    def update(self, g, back, norm, eps, peak):
        g.mul_(torch.from_numpy(self._divide(back.numpy(), norm.numpy(), eps, float(peak.item()))))
        return g


def _case():
    from oracle.hprime_oracle import hprime_oracle
    rng = np.random.default_rng(7)
    H = np.asfortranarray(rng.random(SHAPE))
    H[..., 2] *= 0.0                                    # an all-zero plane: dead voxels
    f = rng.random(IMG) + 0.1
    return H, np.asfortranarray(hprime_oracle(H)), f


def _f_tensor(a):
    from paper_2003_09133_b200.projector import _f_empty
    t = _f_empty(a.shape, "cpu")
    t.copy_(torch.from_numpy(np.ascontiguousarray(a)))
    return t


def test_rl_loop_single_rank_matches_oracle():
    from oracle.projector_oracle import rl_run
    from paper_2003_09133_b200.projector import rl_loop
    H, Hp, f = _case()
    g_ref, hist_ref, norm_ref = rl_run(H, Hp, f, iterations=ITERS)
    g, norm, hist, dead = rl_loop(OracleOps(H, Hp), _f_tensor(f), SHAPE[4], ITERS, 1e-12)
    np.testing.assert_allclose(norm.numpy(), norm_ref, rtol=1e-12, atol=0)
    np.testing.assert_allclose(g.numpy(), g_ref, rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(hist, hist_ref, rtol=1e-12)
    assert dead == int(np.count_nonzero(norm_ref < 1e-12 * norm_ref.max()))
    assert dead >= IMG[0] * IMG[1]                      # the zero plane


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2003_09133_b200.projector import rl_loop
    from paper_2003_09133_b200.shard import shard_planes
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    H, Hp, f = _case()
    z0, z1 = shard_planes(SHAPE[4], world, rank)
    ops = OracleOps(np.asfortranarray(H[..., z0:z1]), np.asfortranarray(Hp[..., z0:z1]))
    g, norm, hist, dead = rl_loop(ops, _f_tensor(f), z1 - z0, ITERS, 1e-12, sharded=True)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), g=g.numpy(), norm=norm.numpy(), hist=np.array(hist),
             dead=dead, z0=z0, z1=z1)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_rl_sharded_two_ranks_gloo(tmp_path):
    from oracle.projector_oracle import rl_run
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    H, Hp, f = _case()
    g_ref, hist_ref, norm_ref = rl_run(H, Hp, f, iterations=ITERS)
    dead_ref = int(np.count_nonzero(norm_ref < 1e-12 * norm_ref.max()))
    covered = 0
    for r in range(2):
        d = np.load(tmp_path / f"rank{r}.npz")
        z0, z1 = int(d["z0"]), int(d["z1"])
        covered += z1 - z0
        np.testing.assert_allclose(d["norm"], norm_ref[..., z0:z1], rtol=1e-12, atol=0)
        np.testing.assert_allclose(d["g"], g_ref[..., z0:z1], rtol=1e-12, atol=1e-300)
        np.testing.assert_allclose(d["hist"], hist_ref, rtol=1e-12)   # global residual on every rank
        assert int(d["dead"]) == dead_ref                               # global count on every rank
    assert covered == SHAPE[4]
