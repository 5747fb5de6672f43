"""Bit-exactness of every unit order (LFBP_KFLAGS / LFBP_TILE_Y variants)
against the default plan on one shape: the orders permute the work units,
so every variant must write the same H'.
    python tools/order_check.py 631,631,21,21,4"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2003_09133_b200 import f_order_empty, hprime_device
    from paper_2003_09133_b200.verify import compare_device
    shape = tuple(int(v) for v in sys.argv[1].split(","))
    src = f_order_empty(shape, torch.float32)
    src.permute(4, 3, 2, 1, 0).reshape(-1).uniform_()
    ref = hprime_device(src)
    res = []
    for flags, ty in [("8", "1"), ("8", "2"), ("8", "3"), ("8", "4"), ("8", "7"), ("8", str(shape[3])), ("4", ""),
                      ("0", "3"), ("16", ""), ("24", "1"), ("64", ""), ("72", "1"), ("80", "")]:
        os.environ["LFBP_KFLAGS"], os.environ["LFBP_TILE_Y"] = flags, ty
        out = hprime_device(src)
        n, _ = compare_device(out, ref)
        res.append({"flags": flags, "tile_y": ty, "n_diff": n})
    print(json.dumps({"shape": shape, "checks": res}))


if __name__ == "__main__":
    main()
