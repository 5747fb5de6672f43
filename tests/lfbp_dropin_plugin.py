"""pytest plugin (``-p lfbp_dropin_plugin``): run the reference's OWN test
files with the GPU drop-ins bound into the unmodified ``lfbp`` package --
the two-line swap of INTEGRATION.md section 1, applied before the test
modules import ``lfbp``.

Every module of the reference that holds the hot-path names gets the GPU
versions: ``lfbp`` (``__init__.py:21-23``), ``lfbp.transform``
(``transform.py:113-155``), and the callers that imported the names at
load time, ``lfbp.bench`` (``bench.py:25``) and ``lfbp.cli``
(``cli.py:28``).  With ``LFBP_DROPIN_REPORT=<path>`` the plugin writes, at
session end, how many kernels the library launched and which functions
were bound, so the outer test can prove the GPU path ran.
"""
from __future__ import annotations

import json
import os

BOUND = ("compute_backprojection", "compute_psf_from_backprojection")


def bind():
    import importlib

    import lfbp

    from paper_2003_09133_b200 import transform as gpu
    mods = [lfbp] + [importlib.import_module(f"lfbp.{m}") for m in ("transform", "bench", "cli")]
    done = []
    for mod in mods:
        for name in BOUND:
            if hasattr(mod, name):
                setattr(mod, name, getattr(gpu, name))
                done.append(f"{mod.__name__}.{name}")
    return done


def pytest_configure(config):
    config._lfbp_dropin_bound = bind()


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("LFBP_DROPIN_REPORT")
    if not path:
        return
    from paper_2003_09133_b200 import _native
    with open(path, "w") as f:
        json.dump({"bound": getattr(session.config, "_lfbp_dropin_bound", []),
                   "launches": int(_native.launch_count()), "exitstatus": int(exitstatus)}, f)
