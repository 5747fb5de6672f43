"""Does K1's rate depend on where H and H' sit in memory?  The same plans
on views of one larger allocation at different byte offsets of H' (and H).

    python tools/placement.py --config C2 --plans "4,48,8,8;2,96,8,8" --offsets 0,16,4096,65536,1048576
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
    ap.add_argument("--offsets", default="0,16,4096,65536,1048576,2097152,3145728")
    ap.add_argument("--which", default="dst", choices=["dst", "src"])
    ap.add_argument("--reps", type=int, default=60)
    a = ap.parse_args()
    import torch

    from paper_2003_09133_b200 import hprime_device
    from paper_2003_09133_b200.configs import WORKLOADS
    w = WORKLOADS[a.config]
    tdt = torch.float32 if w.itemsize == 4 else torch.float64
    n = w.nbytes // w.itemsize
    offs = [int(v) for v in a.offsets.split(",")]
    slack = (max(offs) + 4096) // w.itemsize
    big_src = torch.empty(n + slack, dtype=tdt, device="cuda").uniform_()
    big_dst = torch.empty(n + slack, dtype=tdt, device="cuda")
    keys = ("LFBP_STAGES", "LFBP_STAGE_KB", "LFBP_CONSUMER_WARPS", "LFBP_SUBWARP", "LFBP_KFLAGS")

    def view(t, off):
        return t[off // w.itemsize: off // w.itemsize + n].view(w.shape[::-1]).permute(4, 3, 2, 1, 0)

    for off in offs:
        src = view(big_src, off if a.which == "src" else 0)
        out = view(big_dst, off if a.which == "dst" else 0)
        res = {}
        for pl in a.plans.split(";"):
            for k, v in zip(keys, pl.split(",") + [""] * len(keys)):
                os.environ[k] = v
            for _ in range(3):
                hprime_device(src, out=out)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.reps):
                hprime_device(src, out=out)
            e1.record()
            torch.cuda.synchronize()
            res[pl] = round(2 * w.nbytes * a.reps / e0.elapsed_time(e1) / 1e6, 1)
        print(json.dumps({"config": a.config, "which": a.which, "offset": off,
                          "src_ptr_mod_2mb": src.data_ptr() % (1 << 21), "dst_ptr_mod_2mb": out.data_ptr() % (1 << 21),
                          "GBps": res}), flush=True)


if __name__ == "__main__":
    main()
