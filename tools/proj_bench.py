"""Projector / Richardson-Lucy timing on the GPU box.
    python tools/proj_bench.py [--psf C1] [--image 256] [--iters 5]
Reports per-call time of forward / H'-backprojection and one RL iteration,
the FP64 GFLOP/s (2 flops per multiply-add over the full windows) and the
measured cuBLAS DGEMM rate as the FP64 denominator."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--psf", default="C1")
    ap.add_argument("--image", type=int, default=256)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--quick", action="store_true", help="forward (H') and H'-backprojection only")
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_2003_09133_b200 import f_order_empty, hprime_device
    from paper_2003_09133_b200.configs import WORKLOADS
    from paper_2003_09133_b200.projector import backproject_device, forward_project_device, safe_divide_device
    from paper_2003_09133_b200.synth import baseline_psf
    w = WORKLOADS[a.psf]
    n_s, n_t, n_x, n_y, n_z = w.shape
    H = f_order_empty(w.shape, torch.float32 if w.itemsize == 4 else torch.float64)
    H.permute(4, 3, 2, 1, 0).reshape(-1).copy_(torch.from_numpy(baseline_psf(w).reshape(-1, order="F")))
    Hp = hprime_device(H)
    N = a.image
    g = torch.rand((n_z, N, N), dtype=torch.float64, device="cuda").permute(2, 1, 0)
    f = torch.rand((N, N), dtype=torch.float64, device="cuda").t()

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    macs = float(N) * N * n_s * n_t * n_z
    t_fwd_h = timed(lambda: forward_project_device(H, g))
    t_fwd = timed(lambda: forward_project_device(H, g, Hp=Hp))
    t_bp = timed(lambda: backproject_device(Hp, f))
    if a.quick:
        print(json.dumps({"psf": w.name, "image": N, "rl": os.environ.get("LFBP_PROJ_RL", ""),
                          "tk": os.environ.get("LFBP_PROJ_TK", ""), "forward_ms": round(t_fwd, 3),
                          "backproject_ms": round(t_bp, 3),
                          "forward_fp64_tflops": round(2 * float(N) * N * n_s * n_t * n_z / (t_fwd * 1e-3) / 1e12, 3),
                          "backproject_fp64_tflops": round(2 * float(N) * N * n_s * n_t * n_z / (t_bp * 1e-3) / 1e12, 3)}))
        return
    t_adj = timed(lambda: backproject_device(H, f, use_hprime=False))
    norm = backproject_device(Hp, torch.ones((N, N), dtype=torch.float64, device="cuda").t().contiguous().t())
    scratch = torch.empty(1, dtype=torch.float64, device="cuda")

    def rl_iter():  # the pre-change loop body: fwd, divide, back, divide, mul, fwd
        reproj = forward_project_device(H, g, Hp=Hp)
        ratio = safe_divide_device(f, reproj, 1e-12, scratch=scratch)
        back = backproject_device(H, ratio, use_hprime=False)
        g.mul_(safe_divide_device(back, norm, 1e-12, scratch=scratch))
        forward_project_device(H, g, Hp=Hp)
    t_rl_old = timed(rl_iter, a.iters)

    from paper_2003_09133_b200.projector import DeviceSlabOps
    ops = DeviceSlabOps(H, Hp, n_s % 2 == 1 and n_t % 2 == 1)
    peak = torch.zeros(1, dtype=torch.float64, device="cuda")
    rpeak = torch.zeros(1, dtype=torch.float64, device="cuda")
    ops.max(norm, peak)
    reproj = torch.empty_like(f)
    ratio = torch.empty_like(f)
    bwd = torch.empty_like(g)
    ops.forward(g, reproj)

    def rl_body():  # projector.rl_loop's iteration body, call for call
        ops.max(reproj, rpeak)
        ops.divide(f, reproj, 1e-12, rpeak, ratio)
        ops.back(ratio, bwd)
        ops.update(g, bwd, norm, 1e-12, peak)
        ops.forward(g, reproj)
        return ((f - reproj) ** 2).mean()
    t_rl = timed(rl_body, a.iters)
    x = torch.rand(8192, 8192, dtype=torch.float64, device="cuda")
    t_mm = timed(lambda: x @ x, 3)
    dgemm_tf = 2 * 8192 ** 3 / (t_mm * 1e-3) / 1e12
    res = {"psf": f"{w.name} {w.shape} {np.dtype(w.dtype).name}", "image": [N, N],
           "forward_ms": round(t_fwd, 3), "forward_H_form_ms": round(t_fwd_h, 3), "backproject_ms": round(t_bp, 3), "adjoint_ms": round(t_adj, 3),
           "rl_iteration_ms": round(t_rl, 3), "rl_iteration_two_forward_ms": round(t_rl_old, 3),
           "forward_fp64_tflops": round(2 * macs / (t_fwd * 1e-3) / 1e12, 3),
           "backproject_fp64_tflops": round(2 * macs / (t_bp * 1e-3) / 1e12, 3),
           "adjoint_fp64_tflops": round(2 * macs / (t_adj * 1e-3) / 1e12, 3),
           "dgemm_tflops_measured": round(dgemm_tf, 2)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
