"""Host cost per call of the device API on a tiny array (the GPU work is
negligible, so back-to-back calls measure the CPU side): the Python
``hprime_device`` wrapper, the bare ctypes call with prebuilt arguments, and
torch's ``copy_`` of the same bytes for scale.

    python tools/call_overhead.py [--calls 20000]
"""
import argparse
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=20000)
    ap.add_argument("--shape", default="5,5,3,3,1")
    a = ap.parse_args()
    import torch

    from paper_2003_09133_b200 import _native, f_order_empty, hprime_device
    shape = tuple(int(v) for v in a.shape.split(","))
    src = f_order_empty(shape, torch.float32)
    src.permute(4, 3, 2, 1, 0).reshape(-1).uniform_()
    out = f_order_empty(shape, torch.float32)
    lib = _native.lib()
    dvec = _native.dims_array(shape)
    sp, dp = ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(out.data_ptr())
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    fs, fo = src.permute(4, 3, 2, 1, 0).reshape(-1), out.permute(4, 3, 2, 1, 0).reshape(-1)
    arms = {
        "hprime_device (python wrapper)": lambda: hprime_device(src, out=out),
        "lfbp_hprime_device (bare ctypes)": lambda: lib.lfbp_hprime_device(sp, dp, dvec, 1, 0, 0, shape[4], stream),
        "torch copy_ (same bytes)": lambda: fo.copy_(fs),
    }
    res = {}
    for name, fn in arms.items():
        for _ in range(200):
            fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(a.calls):
            fn()
        host = time.perf_counter() - t
        torch.cuda.synchronize()
        res[name] = round(host / a.calls * 1e6, 2)
    print(json.dumps({"shape": shape, "us_per_call_host": res}), flush=True)


if __name__ == "__main__":
    main()
