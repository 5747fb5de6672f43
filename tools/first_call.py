"""What a user sees on the first call in a fresh process: wall time of the
drop-in ``compute_backprojection`` on a pageable C2 array, first call (CUDA
context, library load, pinned output and workspace allocation) and the
calls after it.

    python tools/first_call.py [--config C2] [--calls 3]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--calls", type=int, default=3)
    ap.add_argument("--breakdown", action="store_true",
                    help="time torch import, CUDA context and a pinned allocation of |H| before the calls")
    a = ap.parse_args()
    pre = {}
    if a.breakdown:
        t = time.perf_counter()
        import torch
        pre["torch_import_s"] = round(time.perf_counter() - t, 3)
        t = time.perf_counter()
        torch.empty(1, device="cuda")
        torch.cuda.synchronize()
        pre["cuda_context_s"] = round(time.perf_counter() - t, 3)
    t0 = time.perf_counter()
    from paper_2003_09133_b200 import Dims5, PsfArray, compute_backprojection
    from paper_2003_09133_b200.configs import WORKLOADS
    from paper_2003_09133_b200.synth import baseline_psf
    t_import = time.perf_counter() - t0
    w = WORKLOADS[a.config]
    H = baseline_psf(w)
    if a.breakdown:
        t = time.perf_counter()
        buf = torch.empty(w.nbytes, dtype=torch.uint8, pin_memory=True)
        pre["pinned_alloc_s"] = round(time.perf_counter() - t, 3)
        del buf
    psf = PsfArray._wrap(Dims5(*w.shape), H)
    times = []
    for _ in range(a.calls):
        t = time.perf_counter()
        bp = compute_backprojection(psf)
        times.append(time.perf_counter() - t)
        del bp
    print(json.dumps({"config": a.config, "import_s": round(t_import, 3),
                      "call_s": [round(v, 4) for v in times], "bytes_rw": 2 * w.nbytes, **pre}), flush=True)


if __name__ == "__main__":
    main()
