"""K1 on a 16-plane C5 slab placed at different spots of two full-size C5
allocations (and in small allocations of its own): does the accessed
footprint or the placement decide the rate?  Short bursts at full clock."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2003_09133_b200 import hprime_device
    full = (631, 631, 21, 21, 101)
    slab = (631, 631, 21, 21, 16)
    P = 631 * 631 * 21 * 21
    small_src = torch.empty(P * 16, dtype=torch.float32, device="cuda")
    small_out = torch.empty(P * 16, dtype=torch.float32, device="cuda")
    big_src = torch.empty(P * 101, dtype=torch.float32, device="cuda")
    big_out = torch.empty(P * 101, dtype=torch.float32, device="cuda")
    big_src.uniform_()
    small_src.uniform_()

    def view(flat, z0, nz):
        return flat[z0 * P:(z0 + nz) * P].view(nz, 21, 21, 631, 631).permute(4, 3, 2, 1, 0)

    cases = {
        "small_small": (view(small_src, 0, 16), view(small_out, 0, 16)),
        "big_start": (view(big_src, 0, 16), view(big_out, 0, 16)),
        "big_end": (view(big_src, 84, 16), view(big_out, 84, 16)),
        "big_mid": (view(big_src, 40, 16), view(big_out, 40, 16)),
        "src_big_out_small": (view(big_src, 40, 16), view(small_out, 0, 16)),
        "full": (view(big_src, 0, 101), view(big_out, 0, 101)),
    }
    for _ in range(2):
        for name, (s, o) in cases.items():
            nbytes = s.numel() * 4
            for _ in range(2):
                hprime_device(s, out=o)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10 if name != "full" else 4
            e0.record()
            for _ in range(reps):
                hprime_device(s, out=o)
            e1.record()
            torch.cuda.synchronize()
            print(json.dumps({"case": name, "GBps": round(2 * nbytes * reps / e0.elapsed_time(e1) / 1e6, 1)}), flush=True)
            time.sleep(3)


if __name__ == "__main__":
    main()
