"""Does K1's efficiency depend on the per-plane working set?  (TLB-reach probe)

Same unit geometry, different plane sizes: vary n_y (and n_z to keep the
total near --gb GB) at fixed (n_s, n_t, n_x), fixed plan, autotune off.
Concurrent units all lie in one z-plane, so the pages touched at once are
~2 x plane bytes / 2 MB.  Prints one JSON line per shape.

    python tools/tlb_probe.py --base 399,399,19 --ny 2,4,6,8,10,13,16,19 --plan 4,48,12,16
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class Nvml:
    """Median SM clock / power and the throttle reasons seen while active."""

    def __init__(self):
        import pynvml
        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(0)

    def __enter__(self):
        import threading
        self.clk, self.pw, self.rs = [], [], 0
        self.stop = threading.Event()

        def run():
            while not self.stop.is_set():
                self.clk.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.pw.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000)
                self.rs |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                time.sleep(0.01)
        self.th = threading.Thread(target=run, daemon=True)
        self.th.start()
        return self

    def __exit__(self, *exc):
        self.stop.set()
        self.th.join()

    def summary(self):
        import statistics
        return {"sm_mhz": statistics.median(self.clk) if self.clk else None,
                "watts": round(statistics.median(self.pw), 1) if self.pw else None,
                "reasons": hex(self.rs & ~1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--base", default="399,399,19")
    ap.add_argument("--ny", default="2,4,6,8,10,13,16,19")
    ap.add_argument("--plan", default="4,48,12,16")
    ap.add_argument("--gb", type=float, default=8.0)
    ap.add_argument("--f64", action="store_true")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--secs", type=float, default=0.0, help="time each leg for about this long instead of --reps")
    ap.add_argument("--kflags", type=int, default=0)
    a = ap.parse_args()
    import torch

    from paper_2003_09133_b200 import f_order_empty, hprime_device
    os.environ["LFBP_AUTOTUNE"] = "0"
    os.environ["LFBP_KFLAGS"] = str(a.kflags)
    for k, v in zip(("LFBP_STAGES", "LFBP_STAGE_KB", "LFBP_CONSUMER_WARPS", "LFBP_SUBWARP"), a.plan.split(",")):
        os.environ[k] = v
    n_s, n_t, n_x = (int(v) for v in a.base.split(","))
    tdt = torch.float64 if a.f64 else torch.float32
    e = 8 if a.f64 else 4
    for ny in (int(v) for v in a.ny.split(",")):
        plane = n_s * n_t * n_x * ny * e
        nz = max(1, int(a.gb * 1e9 / 2 / plane))
        shape = (n_s, n_t, n_x, ny, nz)
        src = f_order_empty(shape, tdt)
        src.permute(4, 3, 2, 1, 0).reshape(-1).uniform_()
        out = f_order_empty(shape, tdt)
        for _ in range(3):
            hprime_device(src, out=out)
        reps = a.reps
        if a.secs:
            torch.cuda.synchronize()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record()
            hprime_device(src, out=out)
            t1.record()
            torch.cuda.synchronize()
            reps = max(3, int(a.secs * 1e3 / t0.elapsed_time(t1)))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with Nvml() as nk:
            e0.record()
            for _ in range(reps):
                hprime_device(src, out=out)
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        # plain copy of the same bytes for comparison
        fs, fo = src.permute(4, 3, 2, 1, 0).reshape(-1), out.permute(4, 3, 2, 1, 0).reshape(-1)
        for _ in range(3):
            fo.copy_(fs)
        torch.cuda.synchronize()
        with Nvml() as nc:
            e0.record()
            for _ in range(reps):
                fo.copy_(fs)
            e1.record()
            torch.cuda.synchronize()
        cms = e0.elapsed_time(e1) / reps
        nbytes = 2 * src.numel() * e
        print(json.dumps({"shape": shape, "plane_mb": round(plane / 1e6, 1), "pages_2mb_rw": round(2 * plane / 2**21),
                          "plan": a.plan, "reps": reps, "kflags": a.kflags, "ms": round(ms, 4), "GBps": round(nbytes / ms / 1e6, 1),
                          "copy_GBps": round(nbytes / cms / 1e6, 1),
                          "k1_nvml": nk.summary(), "copy_nvml": nc.summary()}), flush=True)
        del src, out, fs, fo
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
