"""Alternate two K1 plans window by window in one process, with NVML state
(SM / memory clock, GPU and memory temperature, power, throttle reasons)
sampled at each window boundary: separates plan effects from drifting
device state.

    python tools/alternate.py --config C2 --plans "4,48,8,8;2,96,8,8" --cycles 12 --reps 40
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--plans", default="4,48,8,8;2,96,8,8")
    ap.add_argument("--cycles", type=int, default=12)
    ap.add_argument("--reps", type=int, default=40)
    a = ap.parse_args()
    import pynvml
    import torch

    from paper_2003_09133_b200 import f_order_empty, hprime_device
    from paper_2003_09133_b200.configs import WORKLOADS
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())

    def state():
        d = {"sm": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
             "mem": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
             "gpu_c": pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU),
             "w": round(pynvml.nvmlDeviceGetPowerUsage(h) / 1000),
             "rs": hex(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h) & ~1)}
        try:
            d["mem_c"] = pynvml.nvmlDeviceGetFieldValues(h, [pynvml.NVML_FI_DEV_MEMORY_TEMP])[0].value.uiVal
        except Exception:
            pass
        return d

    w = WORKLOADS[a.config]
    tdt = torch.float32 if w.itemsize == 4 else torch.float64
    src = f_order_empty(w.shape, tdt)
    src.permute(4, 3, 2, 1, 0).reshape(-1).uniform_()
    out = f_order_empty(w.shape, tdt)
    keys = ("LFBP_STAGES", "LFBP_STAGE_KB", "LFBP_CONSUMER_WARPS", "LFBP_SUBWARP", "LFBP_KFLAGS")
    plans = a.plans.split(";")
    for c in range(a.cycles):
        for pl in plans:
            for k, v in zip(keys, pl.split(",") + [""] * len(keys)):
                os.environ[k] = v
            hprime_device(src, out=out)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.reps):
                hprime_device(src, out=out)
            e1.record()
            torch.cuda.synchronize()
            st = state()
            print(json.dumps({"cycle": c, "plan": pl, "GBps": round(2 * w.nbytes * a.reps / e0.elapsed_time(e1) / 1e6, 1),
                              **st}), flush=True)


if __name__ == "__main__":
    main()
