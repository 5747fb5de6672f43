"""PCIe probe: single large copies vs plane-sized chunked copies, one or two
streams per direction, alone and with both directions at once (pinned host).

    python tools/pcie_probe.py [--mb 1745] [--chunk-mb 34]
"""
import argparse
import json
import time


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=1745)
    ap.add_argument("--chunk-mb", type=int, default=34)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch
    n = a.mb * 1000 * 1000 // 4
    cn = a.chunk_mb * 1000 * 1000 // 4
    hin = torch.empty(n, dtype=torch.float32, pin_memory=True)
    hout = torch.empty(n, dtype=torch.float32, pin_memory=True)
    din = torch.empty(n, dtype=torch.float32, device="cuda")
    dout = torch.empty(n, dtype=torch.float32, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(4)]

    def run(h2d, d2h, chunked, nstreams):
        def go():
            if chunked:
                for i, o in enumerate(range(0, n, cn)):
                    e = min(n, o + cn)
                    if h2d:
                        with torch.cuda.stream(streams[i % nstreams]):
                            din[o:e].copy_(hin[o:e], non_blocking=True)
                    if d2h:
                        with torch.cuda.stream(streams[2 + i % nstreams]):
                            hout[o:e].copy_(dout[o:e], non_blocking=True)
            else:
                if h2d:
                    with torch.cuda.stream(streams[0]):
                        din.copy_(hin, non_blocking=True)
                if d2h:
                    with torch.cuda.stream(streams[2]):
                        hout.copy_(dout, non_blocking=True)
            torch.cuda.synchronize()
        go()
        ts = []
        for _ in range(a.reps):
            t = time.perf_counter()
            go()
            ts.append(time.perf_counter() - t)
        t = min(ts)
        nb = n * 4 * (int(h2d) + int(d2h))
        return {"h2d": h2d, "d2h": d2h, "chunked": chunked, "streams_per_dir": nstreams, "ms": round(t * 1e3, 2),
                "GBps": round(nb / t / 1e9, 2)}
    for h2d, d2h in ((True, False), (False, True), (True, True)):
        print(json.dumps(run(h2d, d2h, False, 1)), flush=True)
        for ns in (1, 2):
            print(json.dumps(run(h2d, d2h, True, ns)), flush=True)


if __name__ == "__main__":
    main()
