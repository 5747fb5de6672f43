"""Host-path probe on the GPU box: drop-in / C-ABI host-to-host timings.

    python tools/e2e_probe.py [--config C2]

Times (wall clock, synchronous calls): the pinned-buffer C-ABI path at
several chunk sizes, the drop-in ``compute_backprojection`` on a pageable
numpy array with and without per-call host registration, and checks every
result against the device path's bytes.
"""
from __future__ import annotations

import argparse
import ctypes
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--dropin-only", action="store_true", help="skip the PCIe and C-ABI legs")
    ap.add_argument("--modes", default="stage,register,driver")
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_2003_09133_b200 import Dims5, PsfArray, _native, compute_backprojection
    from paper_2003_09133_b200.configs import WORKLOADS
    from paper_2003_09133_b200.synth import baseline_psf
    w = WORKLOADS[a.config]
    tdt = torch.float32 if w.itemsize == 4 else torch.float64
    pin_in = torch.empty(w.n_elems, dtype=tdt, pin_memory=True)
    pin_out = torch.empty(w.n_elems, dtype=tdt, pin_memory=True)
    H = pin_in.numpy().reshape(w.shape, order="F")
    baseline_psf(w, out=H)
    code = _native.F32 if w.itemsize == 4 else _native.F64
    dvec = _native.dims_array(w.shape)
    step_bytes = 2 * w.nbytes

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            t = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t)
        return min(ts), sorted(ts)[len(ts) // 2]

    # PCIe ceilings: H2D alone, D2H alone, both at once (separate streams)
    dev_a = torch.empty(w.n_elems, dtype=tdt, device="cuda")
    dev_b = torch.empty(w.n_elems, dtype=tdt, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def h2d():
        with torch.cuda.stream(s1):
            dev_a.copy_(pin_in, non_blocking=True)
        s1.synchronize()

    def d2h():
        with torch.cuda.stream(s2):
            pin_out.copy_(dev_b, non_blocking=True)
        s2.synchronize()

    def both():
        with torch.cuda.stream(s1):
            dev_a.copy_(pin_in, non_blocking=True)
        with torch.cuda.stream(s2):
            pin_out.copy_(dev_b, non_blocking=True)
        s1.synchronize()
        s2.synchronize()
    legs = () if a.dropin_only else (("h2d", h2d, w.nbytes), ("d2h", d2h, w.nbytes), ("h2d+d2h", both, 2 * w.nbytes))
    for name, fn, nb in legs:
        best, med = timed(fn)
        print(json.dumps({"path": "pcie " + name, "best_ms": round(best * 1e3, 2), "GBps": round(nb / best / 1e9, 2)}),
              flush=True)
    del dev_a, dev_b
    ref = None
    chunk_env = os.environ.get("LFBP_CHUNK_MB")
    for mb in ((70,) if a.dropin_only else (34, 70)):
        os.environ["LFBP_CHUNK_MB"] = str(mb)

        def call():
            _native.check(_native.lib().lfbp_hprime_host(ctypes.c_void_p(pin_in.data_ptr()),
                                                         ctypes.c_void_p(pin_out.data_ptr()), dvec, code, 0, 0, 0))
        best, med = timed(call)
        dig = hashlib.sha256(pin_out.numpy().tobytes()).hexdigest()
        ref = ref or dig
        print(json.dumps({"path": "c-abi pinned", "chunk_mb": mb, "best_ms": round(best * 1e3, 2),
                          "med_ms": round(med * 1e3, 2), "GBps_rw": round(step_bytes / best / 1e9, 2),
                          "same": dig == ref}), flush=True)
    os.environ.pop("LFBP_CHUNK_MB", None)
    if chunk_env:
        os.environ["LFBP_CHUNK_MB"] = chunk_env
    pageable = np.array(H, order="F")
    pageable.flags.writeable = False
    psf = PsfArray._wrap(Dims5(*w.shape), pageable)
    for reg in a.modes.split(","):
        os.environ["LFBP_HOST_MODE"] = reg
        out = {}

        def dropin():
            out["bp"] = compute_backprojection(psf)
        best, med = timed(dropin)
        dig = hashlib.sha256(out["bp"].data.tobytes(order="F")).hexdigest()
        print(json.dumps({"path": "drop-in pageable input", "host_mode": reg,
                          "copy_threads": os.environ.get("LFBP_COPY_THREADS", "default"),
                          "chunk_mb": os.environ.get("LFBP_CHUNK_MB", "64"), "best_ms": round(best * 1e3, 2),
                          "med_ms": round(med * 1e3, 2), "GBps_rw": round(step_bytes / best / 1e9, 2),
                          "same": dig == ref}), flush=True)


if __name__ == "__main__":
    main()
