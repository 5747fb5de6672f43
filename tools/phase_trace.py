"""Per-launch K1 times over several bursts separated by idle gaps, with an
NVML sampler (SM / memory clock, power, temperature, throttle reasons):
separates one-time warm-up effects from power / thermal state.
    python tools/phase_trace.py 631,631,21,21,101 --bursts 3 --launches 60 --gap 5"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("shape")
    ap.add_argument("--bursts", type=int, default=3)
    ap.add_argument("--launches", type=int, default=60)
    ap.add_argument("--gap", type=float, default=5.0)
    ap.add_argument("--f64", action="store_true")
    ap.add_argument("--tag", default="")
    ap.add_argument("--op", default="k1")
    a = ap.parse_args()
    import pynvml
    import torch

    from paper_2003_09133_b200 import f_order_empty, hprime_device
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    shape = tuple(int(v) for v in a.shape.split(","))
    dt = torch.float64 if (a.f64 or os.environ.get("LFBP_PT_F64")) else torch.float32
    src = f_order_empty(shape, dt)
    src.permute(4, 3, 2, 1, 0).reshape(-1).uniform_()
    out = f_order_empty(shape, dt)
    nbytes = src.numel() * src.element_size()
    fs, fo = src.permute(4, 3, 2, 1, 0).reshape(-1), out.permute(4, 3, 2, 1, 0).reshape(-1)

    def op():
        if a.op == "k1":
            hprime_device(src, out=out)
        else:
            fo.copy_(fs)

    op()
    torch.cuda.synchronize()
    samples = []
    stop = threading.Event()
    t0 = time.perf_counter()

    def sampler():
        while not stop.is_set():
            try:
                samples.append([round(time.perf_counter() - t0, 3),
                                pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                                round(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0, 1),
                                pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU),
                                hex(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))])
            except Exception:
                pass
            time.sleep(0.02)

    th = threading.Thread(target=sampler, daemon=True)
    th.start()
    bursts = []
    for b in range(a.bursts):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.launches)]
        tb = time.perf_counter() - t0
        for e0, e1 in ev:
            e0.record()
            op()
            e1.record()
        torch.cuda.synchronize()
        gbs = [round(2 * nbytes / e0.elapsed_time(e1) / 1e6, 1) for e0, e1 in ev]
        bursts.append({"t_start": round(tb, 3), "GBps": gbs})
        time.sleep(a.gap)
    stop.set()
    th.join()
    print(json.dumps({"tag": a.tag, "op": a.op, "shape": shape, "bursts": bursts, "nvml": samples}), flush=True)


if __name__ == "__main__":
    main()
