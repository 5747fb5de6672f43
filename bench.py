#!/usr/bin/env python
"""Benchmark of the H -> H' rearrangement (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One step = one pass of the K1 kernel over one whole workload (C2 by default,
BASELINE.json configs[1]: H float32 (195,195,15,15,51), 1.75 GB in + out),
inputs resident in HBM.  Under torchrun (N > 1) every rank owns one C2-shaped
depth stack (z-slab) of its own -- weak scaling, no collective on the data
path; the NCCL process group only carries the barriers and the max-over-ranks
time.  ``--config C3 --strong`` instead shards one C3 array's planes over the
ranks.

Printed by rank 0, one JSON line:
  value        algorithmic GB/s (bytes read + written, 2*N*itemsize per step)
               over all ranks / max-over-ranks device time (CUDA events)
  roofline     dominant kernel (K1) achieved GB/s vs MEASURED_PEAKS.json
  e2e          same metric through the C-ABI host path (pinned host buffers,
               H2D + kernel + D2H every step, wall clock around the
               synchronous call)
  cpu_baseline the reference algorithm (oracle/hprime_oracle.py, the numpy
               restatement of lfbp.compute_backprojection) on a bounded
               sample, all host threads over depth planes
``--impl reference`` prints the same metric for that CPU arm alone.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "H' build GB/s (bytes read+written)"
L2_BYTES = 126 << 20
FALLBACK_HBM_GBS = 6650.0   # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy_ r+w)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.dev = device_index
        self.period = period_s
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._th = None
        self.ok = False

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.dev)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            names = {
                "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
                "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
                "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
            }

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for n, bit in names.items():
                            if r & bit and n != "gpu_idle":
                                self.reasons.add(n)
                    except Exception:
                        pass
                    time.sleep(self.period)

            self._th = threading.Thread(target=run, daemon=True)
            self._th.start()
            self.ok = True
        except Exception:
            self.ok = False
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._th:
            self._th.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples), "source": "nvml"}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml"}


def _dtype_tag(dtype) -> str:
    """The element type the path moves: "f32" / "f64" (copied as 4 / 8-byte words)."""
    return {4: "f32", 8: "f64"}[np.dtype(dtype).itemsize]


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_sample(w, planes: int, threads: int, reps: int):
    """Time the reference algorithm (numpy restatement) on `planes` planes of
    workload `w` with `threads` host threads; returns (seconds, bytes r+w)."""
    from oracle.hprime_oracle import hprime_oracle
    from paper_2003_09133_b200.synth import baseline_psf
    H = baseline_psf(w, 0, planes)
    hprime_oracle(H[..., :1], threads=1)   # warm the index tables
    times = []
    for _ in range(reps):
        t = time.perf_counter()
        hprime_oracle(H, threads=threads)
        times.append(time.perf_counter() - t)
    return statistics.median(times), 2 * H.nbytes


def run_reference(args, w):
    rank, world, _ = _dist()
    if world > 1 and rank != 0:
        return 0
    planes = min(w.shape[4], max(args.cpu_planes, os.cpu_count() or 1))
    threads = min(os.cpu_count() or 1, planes)
    from oracle.hprime_oracle import hprime_oracle
    from paper_2003_09133_b200.synth import baseline_psf
    H = baseline_psf(w, 0, planes)
    for _ in range(args.warmup):
        hprime_oracle(H, threads=threads)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        hprime_oracle(H, threads=threads)
        times.append(time.perf_counter() - t)
    total = sum(times)
    gbs = 2 * H.nbytes * args.steps / total / 1e9
    sample = f"{planes} of {w.shape[4]} planes of {w.name} {w.shape} per step (planes are independent)"
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * total / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": _dtype_tag(w.dtype), "data": "synthetic (seeded BASELINE law)",
        "config": {"workload": f"{w.name} {w.shape} {np.dtype(w.dtype).name} seed {w.seed}",
                   "sample_planes": planes},
        "helems_per_s": round(H.size * args.steps / total, 1),
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": sample,
                         "what": "oracle/hprime_oracle.py: numpy restatement of lfbp.compute_backprojection "
                                 "(transform.py:113-135), depth planes split over host threads"},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _max_over_ranks(x: float, world: int, device) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _verify_against_golden(out, w, shape):
    from paper_2003_09133_b200.verify import plane_digests
    path = os.path.join(ROOT, "tests", "golden", f"digests_{w.name}.json")
    if not os.path.exists(path) or tuple(shape) != tuple(w.shape):
        return None
    with open(path) as f:
        want = json.load(f)["hprime_plane_sha256"]
    return plane_digests(out, shape) == want


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--strong", action="store_true", help="shard one array's planes over ranks")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-planes", type=int, default=8)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (the driver already does this)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", "--master-port=29517", os.path.abspath(__file__), *sys.argv[1:]]
        os.execvp(cmd[0], cmd)
    from paper_2003_09133_b200.configs import WORKLOADS
    w = WORKLOADS[args.config]
    if args.impl == "reference":
        return run_reference(args, w)

    import torch
    import torch.distributed as dist

    from paper_2003_09133_b200 import _native, f_order_empty, hprime_device, plan
    from paper_2003_09133_b200.shard import shard_planes
    from paper_2003_09133_b200.synth import baseline_psf

    rank, world, local = _dist()
    # one process per GPU; LFBP_BENCH_BACKEND=gloo (+ device = local % count)
    # only exercises the multi-rank plumbing on a box with fewer GPUs
    backend = os.environ.get("LFBP_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    # this rank's slab
    if args.strong:
        z0, z1 = shard_planes(w.shape[4], world, rank)
    else:
        z0, z1 = 0, w.shape[4]
    shape = (*w.shape[:4], z1 - z0)
    tdt = torch.float32 if w.itemsize == 4 else torch.float64
    host_in = torch.empty(w.plane_elems * (z1 - z0), dtype=tdt, pin_memory=True)
    hin = host_in.numpy().reshape(shape, order="F")
    baseline_psf(w, z0, z1, out=hin)
    src = f_order_empty(shape, tdt, dev)
    src.permute(4, 3, 2, 1, 0).reshape(-1).copy_(host_in)
    out = f_order_empty(shape, tdt, dev)
    n_elems = w.plane_elems * (z1 - z0)
    step_bytes = 2 * n_elems * w.itemsize
    stream = torch.cuda.current_stream(dev)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier(device_ids=[local]) if backend == "nccl" else dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        hprime_device(src, out=out, stream=stream)
    barrier()

    # inputs smaller than 2x L2 (C1): flush L2 between steps by writing a
    # 512 MB buffer outside the per-step events, and time the steps only
    flush = None
    if step_bytes < 2 * L2_BYTES:
        flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    l0 = _native.launch_count()
    with ClockSampler(local) as clk:
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for k in range(args.steps):
            if flush is not None:
                flush.fill_(k & 0xff)
            starts[k].record(stream)
            hprime_device(src, out=out, stream=stream)
            ends[k].record(stream)
        t1.record(stream)
        barrier()
    launches = _native.launch_count() - l0
    kern_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    elapsed_ms = sum(kern_ms) if flush is not None else t0.elapsed_time(t1)
    max_ms = _max_over_ranks(elapsed_ms, world, dev if backend == "nccl" else "cpu")

    verified = None
    if not args.no_verify and rank == 0:
        verified = _verify_against_golden(out, w, shape)

    # end-to-end through the C-ABI host path, pinned host buffers
    e2e = None
    if not args.no_e2e:
        import ctypes
        host_out = torch.empty_like(host_in, pin_memory=True)
        code = _native.F32 if w.itemsize == 4 else _native.F64
        dvec = _native.dims_array(shape)

        def host_call():
            rc = _native.lib().lfbp_hprime_host(ctypes.c_void_p(host_in.data_ptr()),
                                                ctypes.c_void_p(host_out.data_ptr()), dvec, code, 0, local, 0)
            _native.check(rc)

        host_call()
        barrier()
        t = time.perf_counter()
        for _ in range(args.e2e_steps):
            host_call()
        barrier()
        e2e_s = time.perf_counter() - t
        e2e_s = _max_over_ranks(e2e_s, world, dev if backend == "nccl" else "cpu")
        ok = hashlib.sha256(host_out.numpy().tobytes()).hexdigest() == hashlib.sha256(
            out.permute(4, 3, 2, 1, 0).contiguous().view(-1).cpu().numpy().tobytes()).hexdigest()
        e2e = {"value": round(world * step_bytes * args.e2e_steps / e2e_s / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": n_elems * w.itemsize, "d2h_bytes_per_step": n_elems * w.itemsize,
               "steps": args.e2e_steps, "ms_per_step": round(1e3 * e2e_s / args.e2e_steps, 3),
               "path": "lfbp_hprime_host (C-ABI): pinned host H -> chunked H2D/K1/D2H on 3 streams -> pinned host H'",
               "matches_device_result": ok, "timing": "wall clock around the synchronous call, max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        planes = min(w.shape[4], max(args.cpu_planes, os.cpu_count() or 1))
        threads = min(os.cpu_count() or 1, planes)
        secs, nbytes = cpu_sample(w, planes, threads, reps=3)
        cpu = {"value": round(nbytes / secs / 1e9, 4), "unit": "GB/s", "cores": threads, "kind": "port",
               "sample": f"{planes} of {w.shape[4]} planes of {w.name}, median of 3, depth planes over {threads} threads",
               "what": "oracle/hprime_oracle.py (numpy restatement of lfbp.compute_backprojection)"}

    if rank == 0:
        peak, peak_src = _peaks()
        avg_kern_ms = statistics.mean(kern_ms)
        achieved = step_bytes / (avg_kern_ms * 1e-3) / 1e9
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_full_summary.json")
        if os.path.exists(prof):
            try:
                with open(prof) as f:
                    pj = json.load(f)
                if pj.get("workload") == w.name and pj.get("shape") == list(shape):
                    traffic = pj.get("dram_bytes_per_launch")
            except (OSError, ValueError):
                pass
        value = world * step_bytes * args.steps / (max_ms * 1e-3) / 1e9
        p = plan(shape, w.dtype)
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(max_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
            "dtype": _dtype_tag(w.dtype), "data": "synthetic (seeded BASELINE.json law, see synth.py)",
            "config": {"workload": f"{w.name} {w.shape} {np.dtype(w.dtype).name} seed {w.seed}",
                       "per_rank_shape": list(shape),
                       "parallelism": f"z-slab x{world}, no collective on the data path",
                       "l2": (f"inputs larger than L2 ({n_elems * w.itemsize / 1e9:.2f} GB per array vs 0.126 GB)"
                              if flush is None else
                              "L2 flushed between steps (512 MB write outside the per-step events); "
                              "value = bytes / sum of per-step kernel times"),
                       "kernel_plan": p},
            "helems_per_s": round(world * n_elems * args.steps / (max_ms * 1e-3), 1),
            "frac_of_8tbs_nominal": round(value / world / 8000.0, 4),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                         "kernel": "hp::hprime_kernel (K1)", "kernel_ms_avg": round(avg_kern_ms, 4),
                         "kernel_ms_min": round(min(kern_ms), 4),
                         "algorithmic_bytes_per_launch": step_bytes},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "first_timed_launch": l0,
            "clocks": clk.summary(),
            "verified_vs_reference_digests": verified,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local]) if backend == "nccl" else dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
