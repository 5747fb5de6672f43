#!/usr/bin/env python
"""Benchmark of the H -> H' rearrangement (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--weak]
                    [--impl ours|reference]

Workload: C5 by default -- BASELINE.json configs[4], H float32
(631,631,21,21,101), 70.9 GB in + 70.9 GB out resident on one GPU, the
largest single-GPU configuration.  One step = one pass of the K1 kernel over
this rank's planes, inputs resident in HBM (generated on the device by K6,
bit-identical to the host generator).

Multi-GPU (torchrun, one process per GPU): the north_star z-split -- the
config's n_z planes are split into contiguous slabs, one per rank
(``shard_planes``), and every rank runs K1 on its slab; no collective on the
data path (NCCL only carries barriers and the max-over-ranks time).  Total
work is fixed, so ``scaling`` is "strong"; the N=1 line is the single-GPU
headline.  ``--weak`` instead gives every rank a full replica.

Rank 0 prints one JSON line:
  value        algorithmic GB/s (bytes read + written, 2*N*itemsize per step)
               summed over ranks / max-over-ranks device time (CUDA events)
  roofline     dominant kernel (K1) achieved GB/s vs MEASURED_PEAKS.json
  e2e          same metric through the C-ABI host path lfbp_hprime_host on
               each rank's whole slab: pinned host H -> chunked H2D / K1 /
               D2H -> pinned host H' every step, wall clock around the
               synchronous call, max over ranks
  shards       per-rank planes, kernel ms and digest verification
  cpu_baseline the UNMODIFIED reference lfbp.compute_backprojection
               (baseline/_ref, single-threaded numpy as shipped) on one plane
               of the same config (chunked: planes are independent);
               cpu_baseline_port: the oracle's numpy restatement on all host
               threads
``--impl reference`` prints the same metric for the CPU arm alone: the
oracle's numpy restatement of the reference on every host thread, on a
bounded plane sample of the same config (``--ref-mode unmodified``: the
unmodified reference from baseline/_ref, one process per plane).
"""
from __future__ import annotations

import argparse
import ctypes
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
REF_DIR = os.path.join(ROOT, "baseline", "_ref")  # the reference install (side measurements only)


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
        med = statistics.median(self.samples) if self.ok and self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "source": "nvml"}


def _dtype_tag(dtype) -> str:
    """The element type the path moves: "f32" / "f64" (copied as 4 / 8-byte words)."""
    return {4: "f32", 8: "f64"}[np.dtype(dtype).itemsize]


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _workload_tag(w) -> str:
    return f"{w.name} {w.shape} {np.dtype(w.dtype).name} seed {w.seed}"


def _golden_plane_digests(w):
    path = os.path.join(ROOT, "tests", "golden", f"digests_{w.name}.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f)["hprime_plane_sha256"]


# ---------------------------------------------------------------- CPU legs

def _threads() -> int:
    return max(1, os.cpu_count() or 1)


def cpu_reference_one_plane(w, z: int):
    """The unmodified reference (baseline/_ref lfbp, single-threaded numpy as
    shipped) on plane z of the workload; returns the cpu_baseline object or
    None when the reference is not installed."""
    if not os.path.isdir(os.path.join(REF_DIR, "lfbp")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import lfbp  # noqa: E402  (the reference package, unmodified)

    from paper_2003_09133_b200.synth import baseline_psf
    H = baseline_psf(w, z, z + 1)
    psf = lfbp.PsfArray._wrap(lfbp.Dims5(*H.shape), H)
    t = time.perf_counter()
    bp = lfbp.compute_backprojection(psf)
    secs = time.perf_counter() - t
    want = _golden_plane_digests(w)
    ok = None if want is None else hashlib.sha256(bp.data.tobytes(order="F")).hexdigest() == want[z]
    return {"value": round(2 * H.nbytes / secs / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "reference",
            "sample": f"plane {z} of {w.shape[4]} of {w.name} (chunked: planes are independent, "
                      f"reference test_transform.py:141-154), one run",
            "seconds": round(secs, 3),
            "what": "lfbp.compute_backprojection from baseline/_ref (the unmodified reference, "
                    "single-threaded numpy as shipped: reference bench.py:99-105)",
            "host_threads_available": _threads(), "matches_reference_digest": ok}


def cpu_port_sample(w, planes: int, threads: int, reps: int = 1):
    """The oracle's numpy restatement on `planes` planes with `threads` host
    threads (split over planes and output columns); (seconds, bytes r+w)."""
    from oracle.hprime_oracle import hprime_oracle_split
    from paper_2003_09133_b200.synth import baseline_psf
    z0 = max(0, w.shape[4] // 2 - planes // 2)
    H = baseline_psf(w, z0, z0 + planes)
    hprime_oracle_split(H[..., :1], threads)   # warm the index tables
    times = []
    for _ in range(reps):
        t = time.perf_counter()
        hprime_oracle_split(H, threads)
        times.append(time.perf_counter() - t)
    return statistics.median(times), 2 * H.nbytes, z0


def _port_planes(w, requested: int) -> int:
    """Planes per CPU sample: ~1.5 GB of H (C5: 2 planes, C2: 16)."""
    if requested > 0:
        return min(w.shape[4], requested)
    return max(1, min(w.shape[4], (3 << 29) // (w.plane_elems * w.itemsize)))


def _ref_plane_worker(wname, z, steps, warmup, bar, q):
    """One process of the reference arm: the unmodified lfbp (baseline/_ref)
    transforms plane z of the workload `warmup` + `steps` times; the timed
    steps start together (barrier) and report (t_start, t_end, digest)."""
    try:
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        import lfbp  # noqa: E402  (the reference package, unmodified)

        from paper_2003_09133_b200.configs import WORKLOADS
        from paper_2003_09133_b200.synth import baseline_psf
        w = WORKLOADS[wname]
        H = baseline_psf(w, z, z + 1, threads=1)
        psf = lfbp.PsfArray._wrap(lfbp.Dims5(*H.shape), H)
        for _ in range(warmup):
            lfbp.compute_backprojection(psf)
        spans, digest = [], None
        for _ in range(steps):
            bar.wait()
            t0 = time.time()
            bp = lfbp.compute_backprojection(psf)
            spans.append((t0, time.time()))
            digest = hashlib.sha256(bp.data.tobytes(order="F")).hexdigest()
            del bp
        q.put((z, spans, digest, H.nbytes, None))
    except BaseException as e:  # report, never hang the barrier of the others
        bar.abort()
        q.put((z, None, None, 0, f"{type(e).__name__}: {e}"))


def run_reference_processes(args, w, procs: int):
    """The unmodified reference on `procs` planes at once, one process per
    plane (planes are independent, reference test_transform.py:141-154);
    step time = last end - first start over the processes."""
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    nz = w.shape[4]
    zs = [(nz // 2 - procs // 2 + k) % nz for k in range(procs)]
    bar = ctx.Barrier(procs)
    q = ctx.Queue()
    warm = min(args.warmup, 1)
    ps = [ctx.Process(target=_ref_plane_worker, args=(w.name, z, args.steps, warm, bar, q)) for z in zs]
    for pr in ps:
        pr.start()
    res = []
    import queue
    while len(res) < len(ps):
        try:
            res.append(q.get(timeout=10))
        except queue.Empty:
            dead = [pr for pr in ps if pr.exitcode not in (None, 0)]
            if dead:   # a worker died without reporting (e.g. the OOM killer)
                for pr in ps:
                    pr.kill()
                raise RuntimeError(f"reference worker exited with code {dead[0].exitcode}")
    for pr in ps:
        pr.join()
    errs = [r[4] for r in res if r[4]]
    if errs:
        raise RuntimeError(errs[0])
    step_s = [max(r[1][k][1] for r in res) - min(r[1][k][0] for r in res) for k in range(args.steps)]
    want = _golden_plane_digests(w)
    ok = None if want is None else all(r[2] == want[r[0]] for r in res)
    nbytes = sum(2 * r[3] for r in res)
    return step_s, nbytes, sorted(zs), ok, warm


def run_reference(args, w):
    """--impl reference: the reference algorithm on the box's host cores, a
    bounded plane sample of the same workload per step.  Default (this
    tier's reference arm): the oracle's numpy restatement of
    lfbp.compute_backprojection on every host thread -- the reference is
    Python, so there is no compiled oracle/_ref.  --ref-mode unmodified runs
    the UNMODIFIED lfbp from baseline/_ref instead (single-threaded numpy as
    shipped, one process per plane on every host thread), a side
    measurement."""
    rank, world, _ = _dist()
    if world > 1 and rank != 0:
        return 0
    threads = _threads()
    sample = None
    if args.ref_mode == "unmodified":
        if not os.path.isdir(os.path.join(REF_DIR, "lfbp")):
            raise SystemExit("--ref-mode unmodified needs baseline/_ref (tools/install_reference.sh)")
        procs = max(1, min(threads, w.shape[4], args.cpu_planes or threads))
        # bound host memory: ~3 x plane bytes per process (reference peak RSS)
        try:
            avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
            procs = max(1, min(procs, int(0.6 * avail // (4 * w.plane_elems * w.itemsize))))
        except (ValueError, OSError):
            pass
        times, nbytes, zs, ok, warm = run_reference_processes(args, w, procs)
        kind, cores = "reference", procs
        what = ("lfbp.compute_backprojection from baseline/_ref (the unmodified reference, single-threaded "
                "numpy as shipped), one process per plane")
        sample = (f"{procs} planes {zs[0]}..{zs[-1]} of {w.shape[4]} of {w.name} per step, one per process "
                  f"(chunked: planes are independent, reference test_transform.py:141-154); warm-up {warm}")
        extra = {"matches_reference_digests": ok}
    else:
        from oracle.hprime_oracle import hprime_oracle_split
        from paper_2003_09133_b200.synth import baseline_psf
        planes = _port_planes(w, args.cpu_planes)
        z0 = max(0, w.shape[4] // 2 - planes // 2)
        H = baseline_psf(w, z0, z0 + planes)
        for _ in range(args.warmup):
            hprime_oracle_split(H, threads)
        times = []
        for _ in range(args.steps):
            t = time.perf_counter()
            hprime_oracle_split(H, threads)
            times.append(time.perf_counter() - t)
        nbytes = 2 * H.nbytes
        kind, cores = "port", threads
        what = ("oracle/hprime_oracle.py: numpy restatement of lfbp.compute_backprojection "
                "(transform.py:113-135), planes and output columns split over host threads")
        sample = (f"planes [{z0}, {z0 + planes}) of {w.shape[4]} of {w.name} per step (chunked: planes are "
                  f"independent, reference test_transform.py:141-154)")
        extra = {}
    total = sum(times)
    gbs = nbytes * args.steps / total / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * total / args.steps, 3),
        "higher_is_better": True, "scaling": "strong" if not args.weak else "weak", "vs_baseline": None,
        "dtype": _dtype_tag(w.dtype), "data": "synthetic (seeded BASELINE.json law, see synth.py)",
        "config": {"workload": _workload_tag(w)},
        "helems_per_s": round(nbytes / (2 * w.itemsize) * args.steps / total, 1),
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": cores, "kind": kind, "sample": sample,
                         "what": what, "host_threads_available": threads, **extra},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU arm

def _max_over_ranks(x: float, world: int, device) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _gather_objects(obj, world: int):
    if world == 1:
        return [obj]
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, obj)
    return out


class HostBuffer:
    """One host array of `nbytes` for the e2e leg: page-locked from the
    library allocator (lfbp_host_alloc: huge pages, registered) when the host
    can pin it, else pageable (then the host path stages it)."""

    def __init__(self, nbytes: int, pinned: bool):
        from paper_2003_09133_b200.errors import NativeError
        from paper_2003_09133_b200.transform import _PinnedBlock
        self.pinned = False
        if pinned:
            try:
                self.arr = np.asarray(_PinnedBlock(nbytes))[:nbytes]
                self.pinned = True
            except NativeError:
                pass
        if not self.pinned:
            self.arr = np.empty(nbytes, dtype=np.uint8)
            self.arr[::4096] = 0   # fault the pages in outside the timed region

    def free(self):
        from paper_2003_09133_b200 import _native
        self.arr = None            # the block goes back to the library (released below)
        _native.lib().lfbp_host_cache_release()


class SharedHostOut:
    """The z-split's one host H' for the e2e leg: a file under /dev/shm that
    every rank maps (``shard.open_shared_host``); this rank writes its slab
    [z0, z1) in place, page-locked with cudaHostRegister outside the timed
    region.  ``ok`` is False (private buffers are used) when /dev/shm cannot
    hold the array."""

    def __init__(self, w, z0, z1, plane_bytes, rank, world, barrier):
        import torch
        self.path = f"/dev/shm/lfbp_bench_{os.environ.get('MASTER_PORT', '0')}_{w.name}.hp"
        self.rank, self.barrier, self.registered, self.arr, self._mm = rank, barrier, False, None, None
        free = 0
        try:
            st = os.statvfs("/dev/shm")
            free = st.f_bavail * st.f_frsize
        except OSError:
            pass
        self.ok = all(_gather_objects(free > 1.05 * w.nbytes + (2 << 30), world))
        if not self.ok:
            return
        if rank == 0:
            with open(self.path, "wb") as f:
                f.truncate(w.nbytes)
        barrier()
        from paper_2003_09133_b200.shard import open_shared_host
        self._mm = open_shared_host(self.path, (w.nbytes,), np.uint8)
        self.arr = self._mm[z0 * plane_bytes:z1 * plane_bytes]
        if self.arr.size:
            self.arr[::4096] = 0                       # fault the tmpfs pages in, outside the timed region
            rc = torch.cuda.cudart().cudaHostRegister(self.arr.ctypes.data, self.arr.size, 0)
            self.registered = int(rc) == 0

    def free(self):
        import torch
        if self.registered:
            torch.cuda.cudart().cudaHostUnregister(self.arr.ctypes.data)
            self.registered = False
        self.arr = self._mm = None
        if self.ok:
            self.barrier()
            if self.rank == 0:
                try:
                    os.unlink(self.path)
                except OSError:
                    pass


def _host_plane_digests(buf: np.ndarray, plane_bytes: int, n_planes: int) -> list[str]:
    import concurrent.futures as cf

    def one(z):
        return hashlib.sha256(memoryview(buf[z * plane_bytes:(z + 1) * plane_bytes])).hexdigest()

    with cf.ThreadPoolExecutor(min(16, _threads())) as pool:
        return list(pool.map(one, range(n_planes)))


def _all_verified(shard_info):
    """True when every rank with planes matched the reference digests, False
    if one did not, None when verification was skipped."""
    vals = [s["verified"] for s in shard_info if s["planes"][1] > s["planes"][0]]
    if not vals or any(v is None for v in vals):
        return None
    return all(vals)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--weak", action="store_true", help="every rank a full replica instead of the z-split")
    ap.add_argument("--strong", action="store_true", help="(default) z-split of one array over the ranks")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-mode", default="port", choices=["port", "unmodified"],
                    help="reference arm: the oracle port on every host thread (default), or the unmodified "
                         "lfbp from baseline/_ref, one process per plane")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-planes", type=int, default=0, help="planes per CPU sample (0: about 1.5 GB)")
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
    from paper_2003_09133_b200.shard import imbalance, shard_planes
    from paper_2003_09133_b200.synth import baseline_psf_device
    from paper_2003_09133_b200.verify import plane_digests

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
    red_dev = dev if backend == "nccl" else "cpu"

    # this rank's slab
    if args.weak:
        z0, z1 = 0, w.shape[4]
    else:
        z0, z1 = shard_planes(w.shape[4], world, rank)
    nz = z1 - z0
    shape = (*w.shape[:4], nz)
    tdt = torch.float32 if w.itemsize == 4 else torch.float64
    n_elems = w.plane_elems * nz
    plane_bytes = w.plane_elems * w.itemsize
    step_bytes = 2 * n_elems * w.itemsize
    src = f_order_empty(shape, tdt, dev)
    out = f_order_empty(shape, tdt, dev)
    stream = torch.cuda.current_stream(dev)
    t_setup = time.perf_counter()
    if nz:
        baseline_psf_device(w, z0, z1, out=src)
    torch.cuda.synchronize(dev)
    setup_s = time.perf_counter() - t_setup

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier(device_ids=[local]) if backend == "nccl" else dist.barrier()
        torch.cuda.synchronize(dev)

    def step():
        if nz:
            hprime_device(src, out=out, stream=stream)

    # the first call autotunes the plan on these buffers (lfbp_hprime_device)
    for _ in range(args.warmup):
        step()
    barrier()

    # inputs smaller than 2x L2 (C1): flush L2 between steps by writing a
    # 512 MB buffer outside the per-step events, and time the steps only
    flush = None
    if step_bytes < 2 * L2_BYTES and nz:
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
            step()
            ends[k].record(stream)
        t1.record(stream)
        barrier()
    launches = _native.launch_count() - l0
    kern_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    elapsed_ms = sum(kern_ms) if flush is not None else t0.elapsed_time(t1)
    max_ms = _max_over_ranks(elapsed_ms, world, red_dev)

    # every rank checks its planes against the reference's per-plane digests
    verified = None
    if not args.no_verify and nz:
        want = _golden_plane_digests(w)
        if want is not None:
            verified = plane_digests(out, shape, threads=min(16, _threads())) == want[z0:z1]
        torch._C._host_emptyCache()   # the digest staging buffers, before the e2e leg pins its own

    # end to end through the C-ABI host path on this rank's whole slab; under
    # the z-split every rank writes its slab straight into ONE shared host H'
    # (a /dev/shm file mapped by every rank, shard.open_shared_host) -- the
    # final gather of the z-shards, no collective
    e2e = None
    shared = None
    if not args.no_e2e and world > 1 and not args.weak and os.environ.get("LFBP_BENCH_SHARED_OUT", "1") != "0":
        shared = SharedHostOut(w, z0, z1, plane_bytes, rank, world, barrier)
    if not args.no_e2e and nz:
        nbytes = n_elems * w.itemsize
        hin = HostBuffer(nbytes, pinned=True)
        hout = shared if shared is not None and shared.ok else HostBuffer(nbytes, pinned=hin.pinned)
        torch.from_numpy(hin.arr).copy_(src.permute(4, 3, 2, 1, 0).reshape(-1).view(torch.uint8))
        code = _native.F32 if w.itemsize == 4 else _native.F64
        dvec = _native.dims_array(shape)
        lib = _native.lib()

        def host_call():
            rc = lib.lfbp_hprime_host(ctypes.c_void_p(hin.arr.ctypes.data), ctypes.c_void_p(hout.arr.ctypes.data),
                                      dvec, code, 0, local, _native.HOST_STAGE)
            _native.check(rc)

        host_call()
        barrier()
        t = time.perf_counter()
        for _ in range(args.e2e_steps):
            host_call()
        barrier()
        e2e_s = _max_over_ranks(time.perf_counter() - t, world, red_dev)
        want = _golden_plane_digests(w)
        ok = (None if want is None else
              _host_plane_digests(hout.arr, plane_bytes, nz) == want[z0:z1])
        e2e_total = step_bytes if args.weak else 2 * w.nbytes
        e2e = {"value": round((world if args.weak else 1) * e2e_total * args.e2e_steps / e2e_s / 1e9, 3),
               "unit": "GB/s", "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
               "bytes_per_step_note": "per rank (this rank's slab)",
               "steps": args.e2e_steps, "ms_per_step": round(1e3 * e2e_s / args.e2e_steps, 3),
               "path": "lfbp_hprime_host (C-ABI) on the rank's whole slab: host H -> chunked H2D/K1/D2H on "
                       "3 streams -> host H'",
               "host_buffers": "pinned (lfbp_host_alloc)" if hin.pinned else
                               "pageable, staged through pinned chunks (LFBP_HOST_STAGE)",
               "matches_reference_digests": ok, "timing": "wall clock around the synchronous call, max over ranks"}
        if hout is shared:
            e2e["host_output"] = (f"one shared host H' ({shared.path}, mapped by every rank; each rank's slab "
                                  f"page-locked in place: {shared.registered}); digests read back from it")
        hin.free()
        hout.free()
    elif shared is not None:
        shared.free()

    shard_info = _gather_objects({"rank": rank, "planes": [z0, z1], "kernel_ms_avg": round(statistics.mean(kern_ms), 4)
                                  if kern_ms and nz else 0.0, "verified": verified,
                                  "e2e_verified": e2e["matches_reference_digests"] if e2e else None}, world)
    if e2e is not None:
        e2e["matches_reference_digests"] = _all_verified(
            [{"planes": s["planes"], "verified": s["e2e_verified"]} for s in shard_info])

    cpu = cpu_port = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_reference_one_plane(w, w.shape[4] // 2)
        except Exception as e:   # the reference leg must not sink the bench line
            cpu = {"error": f"{type(e).__name__}: {e}"}
        planes = _port_planes(w, args.cpu_planes)
        threads = _threads()
        secs, nbytes, zs = cpu_port_sample(w, planes, threads)
        cpu_port = {"value": round(nbytes / secs / 1e9, 4), "unit": "GB/s", "cores": threads, "kind": "port",
                    "sample": f"planes [{zs}, {zs + planes}) of {w.name}, planes and output columns over {threads} "
                              f"threads (chunked)",
                    "what": "oracle/hprime_oracle.py (numpy restatement of lfbp.compute_backprojection)"}
        if cpu is None or "error" in cpu:
            cpu, cpu_port = cpu_port, cpu

    if rank == 0:
        peak, peak_src = _peaks()
        avg_kern_ms = statistics.mean(kern_ms)
        achieved = step_bytes / (avg_kern_ms * 1e-3) / 1e9
        traffic = traffic_src = None
        prof = os.path.join(ROOT, "profiles", "ncu_full_summary.json")
        if os.path.exists(prof):
            try:
                with open(prof) as f:
                    pj = json.load(f)
                # a capture of the same plane geometry (a z-slab of the workload
                # for C5, whose 142 GB ncu would have to save and restore per
                # replay pass) scales by planes: K1's traffic is per plane
                ps = pj.get("shape")
                if pj.get("workload") == w.name and ps and list(ps[:4]) == list(shape[:4]) and ps[4] > 0:
                    traffic = round(pj["dram_bytes_per_launch"] * shape[4] / ps[4])
                    traffic_src = f"{pj.get('source')} ({ps[4]}-plane capture, scaled to {shape[4]} planes)" \
                        if ps[4] != shape[4] else pj.get("source")
            except (OSError, ValueError):
                pass
        total_bytes = (world if args.weak else 1) * (step_bytes if args.weak else 2 * w.nbytes)
        value = total_bytes * args.steps / (max_ms * 1e-3) / 1e9
        p = plan(shape, w.dtype)
        sizes = [s["planes"][1] - s["planes"][0] for s in shard_info]
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(max_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
            "dtype": _dtype_tag(w.dtype), "data": "synthetic (seeded BASELINE.json law, generated on the device "
                                                  "by K6, bit-identical to synth.py)",
            "config": {"workload": _workload_tag(w),
                       "per_rank_shape": list(shape),
                       "parallelism": (f"z-slab x{world} (contiguous plane ranges), no collective on the data path"
                                       if not args.weak else f"replica x{world}, no collective on the data path"),
                       "l2": (f"inputs larger than L2 ({n_elems * w.itemsize / 1e9:.2f} GB per array vs 0.126 GB)"
                              if flush is None else
                              "L2 flushed between steps (512 MB write outside the per-step events); "
                              "value = bytes / sum of per-step kernel times"),
                       "kernel_plan": p},
            "helems_per_s": round(total_bytes / (2 * w.itemsize) * args.steps / (max_ms * 1e-3), 1),
            "frac_of_8tbs_nominal": round(value / world / 8000.0, 4),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": peak_src,
                         "kernel": "hp::hprime_kernel (K1)", "kernel_ms_avg": round(avg_kern_ms, 4),
                         "kernel_ms_min": round(min(kern_ms), 4),
                         "algorithmic_bytes_per_launch": step_bytes},
            "shards": {"planes_per_rank": sizes, "imbalance_max_over_mean": round(imbalance(w.shape[4], world), 4)
                       if not args.weak else 1.0, "per_rank": shard_info},
            "cpu_baseline": cpu, "cpu_baseline_port": cpu_port, "e2e": e2e, "gpu_launches": launches,
            "first_timed_launch": l0, "clocks": clk.summary(),
            "verified_vs_reference_digests": _all_verified(shard_info),
            "setup_s": round(setup_s, 2),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local]) if backend == "nccl" else dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
