"""The drop-in compute_backprojection on a host C5 array (70.9 GB numpy in,
70.9 GB numpy out): wall time of the first call in the process and of a
second call, and the per-plane digests of the result against the
reference's.  python tools/c5_dropin.py [--config C5]"""
import argparse
import concurrent.futures as cf
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    a = ap.parse_args()
    import numpy as np

    from paper_2003_09133_b200 import Dims5, PsfArray, compute_backprojection
    from paper_2003_09133_b200.configs import WORKLOADS
    from paper_2003_09133_b200.synth import baseline_psf
    w = WORKLOADS[a.config]
    t = time.perf_counter()
    H = baseline_psf(w, threads=min(16, os.cpu_count() or 1))
    gen_s = time.perf_counter() - t
    psf = PsfArray._wrap(Dims5(*w.shape), H)
    times = []
    bp = None
    for _ in range(2):
        bp = None
        t = time.perf_counter()
        bp = compute_backprojection(psf)
        times.append(round(time.perf_counter() - t, 3))
    data = bp.data.reshape(-1, order="F")
    pe = w.plane_elems

    def dig(z):
        return hashlib.sha256(memoryview(data[z * pe:(z + 1) * pe]).cast("B")).hexdigest()

    with cf.ThreadPoolExecutor(16) as pool:
        got = list(pool.map(dig, range(w.shape[4])))
    with open(os.path.join(ROOT, "tests", "golden", f"digests_{w.name}.json")) as f:
        want = json.load(f)["hprime_plane_sha256"]
    print(json.dumps({"config": w.name, "shape": w.shape, "bytes_each_way": H.nbytes, "host_generate_s": round(gen_s, 1),
                      "call_s": times, "GBps_rw": [round(2 * H.nbytes / s / 1e9, 2) for s in times],
                      "result_pinned": bool(getattr(bp.data, "base", None) is not None and
                                            type(bp.data.base).__name__ != "ndarray"),
                      "matches_reference_digests": got == want, "read_only": not bp.data.flags.writeable,
                      "f_contiguous": bp.data.flags.f_contiguous}), flush=True)


if __name__ == "__main__":
    main()
