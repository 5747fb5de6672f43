"""Per-chunk timeline of the pinned host pipeline (LFBP_TRACE=1 prints one
line per chunk to stderr: h2d start/end, kernel end, d2h start/end in ms).

    python tools/e2e_trace.py [--config C2] 2> trace.txt
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    a = ap.parse_args()
    import torch

    from paper_2003_09133_b200 import _native
    from paper_2003_09133_b200.configs import WORKLOADS
    w = WORKLOADS[a.config]
    tdt = torch.float32 if w.itemsize == 4 else torch.float64
    pin_in = torch.rand(w.n_elems, dtype=tdt).pin_memory()
    pin_out = torch.empty(w.n_elems, dtype=tdt, pin_memory=True)
    code = _native.F32 if w.itemsize == 4 else _native.F64
    dvec = _native.dims_array(w.shape)

    def call():
        _native.check(_native.lib().lfbp_hprime_host(ctypes.c_void_p(pin_in.data_ptr()),
                                                     ctypes.c_void_p(pin_out.data_ptr()), dvec, code, 0, 0, 0))
    call()
    call()
    os.environ["LFBP_TRACE"] = "1"
    call()


if __name__ == "__main__":
    main()
