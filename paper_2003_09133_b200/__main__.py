"""Command line for the H' path: ``python -m paper_2003_09133_b200 ...``.

Mirrors the reference CLI's hot-path subcommands (lfbp/cli.py) on the GPU:

* ``transform IN OUT [--inverse] [--device N]`` -- cli.py:115-126, file to
  file through the GPU (LF5 streaming, never loading the array on the host);
* ``verify IN [--against OUT] [--device N]`` -- cli.py:129-150.  The
  reference checks its rearrangement against a brute-force oracle; here the
  device result is checked by the device invariants (involution and the
  rotation criterion of the sorted-order plane sums) and, with ``--against``,
  byte for byte against a stored H' file, reporting the first differing
  1-based (s,t,x,y,z) like the reference;
* ``plan SHAPE [--f64]`` -- the kernel's launch plan for a shape.

Exit codes follow the reference (cli.py:402-407): 0 ok, 1 mismatch / OS
error, 2 library error.
"""
from __future__ import annotations

import argparse
import json
import logging
import sys
import time


def _cmd_transform(args) -> int:
    from .lf5 import transform_file
    t0 = time.perf_counter()
    shape = transform_file(args.input, args.output, inverse=args.inverse, device=args.device)
    print(f"{'x'.join(map(str, shape))} rearranged on cuda:{args.device} in "
          f"{time.perf_counter() - t0:.3f} s -> {args.output}", file=sys.stderr)
    return 0


def _cmd_verify(args) -> int:
    import numpy as np
    import torch

    from . import hprime_device
    from .lf5 import load_device, read_header
    from .verify import compare_device, first_mismatch_index, involution_check, rotation_check
    shape, dtype = read_header(args.input)
    label = "x".join(map(str, shape))
    with torch.cuda.device(args.device):
        h = load_device(args.input, device=args.device)
        hp = hprime_device(h)
        if args.against:
            other_shape, _ = read_header(args.against)
            if other_shape != shape:
                from .errors import InvalidDims
                raise InvalidDims(f"{args.against} dims {other_shape} do not match {args.input} dims {shape}")
            stored = load_device(args.against, device=args.device)
            n_diff, first = compare_device(hp, stored)
            if n_diff:
                coord = tuple(i + 1 for i in first_mismatch_index(shape, first, np.dtype(dtype).itemsize))
                print(f"FAIL {label}: {n_diff} bytes differ, first at (s,t,x,y,z)={coord}")
                return 1
        checks = []
        if shape[0] % 2 and shape[1] % 2:
            n_diff, _ = involution_check(h)
            checks.append(("involution", n_diff == 0))
            checks.append(("rotation of plane sums", rotation_check(h, hp, shape) == 0))
    bad = [name for name, ok in checks if not ok]
    if bad:
        print(f"FAIL {label}: {', '.join(bad)}")
        return 1
    what = "stored backprojection matches the GPU rearrangement bitwise" if args.against else \
        "GPU rearrangement passes the device invariants"
    print(f"PASS {label}: {what} ({', '.join(n for n, _ in checks) or 'even dims: byte compare only'})")
    return 0


def _cmd_plan(args) -> int:
    import numpy as np

    from .transform import plan
    shape = tuple(int(v) for v in args.shape.split(","))
    print(json.dumps(plan(shape, np.float64 if args.f64 else np.float32)))
    return 0


def main(argv=None) -> int:
    from .errors import LfbpError
    ap = argparse.ArgumentParser(prog="python -m paper_2003_09133_b200")
    ap.add_argument("-v", "--verbose", action="store_true")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("transform", help="H' (or H with --inverse) of an LF5 file, on the GPU")
    p.add_argument("input")
    p.add_argument("output")
    p.add_argument("--inverse", action="store_true")
    p.add_argument("--device", type=int, default=0)
    p.set_defaults(func=_cmd_transform)
    p = sub.add_parser("verify", help="check the GPU rearrangement of an LF5 file")
    p.add_argument("input")
    p.add_argument("--against")
    p.add_argument("--device", type=int, default=0)
    p.set_defaults(func=_cmd_verify)
    p = sub.add_parser("plan", help="launch plan for n_s,n_t,n_x,n_y,n_z")
    p.add_argument("shape")
    p.add_argument("--f64", action="store_true")
    p.set_defaults(func=_cmd_plan)
    try:
        args = ap.parse_args(argv)
        logging.basicConfig(stream=sys.stderr, format="%(levelname)s: %(message)s",
                            level=logging.INFO if args.verbose else logging.WARNING)
        return args.func(args)
    except LfbpError as exc:
        print(f"{type(exc).__name__}: {exc}", file=sys.stderr)
        return 2
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
