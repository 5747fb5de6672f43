"""Device-to-device copy bandwidth (torch copy_, read + write bytes) at the
BASELINE array sizes, burst (first iterations) and sustained (~1 s of
back-to-back copies) -- the denominator K1 competes with at each size."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2003_09133_b200.configs import WORKLOADS
    for name in ("C2", "C3", "C4", "C5"):
        w = WORKLOADS[name]
        n = w.nbytes // 4
        a = torch.empty(n, dtype=torch.float32, device="cuda")
        b = torch.empty(n, dtype=torch.float32, device="cuda")
        a.fill_(1.0)
        b.copy_(a)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        burst = 2 * w.nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9
        reps = max(3, int(1.0 / max(e0.elapsed_time(e1) * 1e-3, 1e-6)))
        e0.record()
        for _ in range(reps):
            b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        sus = 2 * w.nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
        print(json.dumps({"config": name, "bytes_rw": 2 * w.nbytes, "copy_burst_GBps": round(burst, 1),
                          "copy_sustained_GBps": round(sus, 1), "reps": reps}), flush=True)
        del a, b
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
