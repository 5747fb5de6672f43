"""Generate the golden fixtures by running the REAL reference (``lfbp``).

Run in the dev container, where the read-only reference is mounted:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--configs C1,C2,C3,C4] [--small] [--acceptance]

Outputs (committed):

* ``tests/golden/small_cases.npz`` -- full input / H' / inverse arrays for the
  reference's own test shapes (pkg/tests/test_transform.py, test_oracle.py,
  test_acceptance.py) plus bit-pattern edge cases, each produced by
  ``lfbp.compute_backprojection`` / ``lfbp.compute_psf_from_backprojection``.
* ``tests/golden/acceptance_suite.json`` -- SHA-256 of the input and of the
  reference's H' for each of the 50 arrays of the reference's acceptance
  suite (test_acceptance.py:21-27).
* ``tests/golden/digests_<C>.json`` -- per-plane SHA-256 of the BASELINE
  workload input (our seeded generator) and of the reference's H' for it.
  Planes are transformed in slabs of ``--slab`` planes; z-planes are
  independent (reference test_transform.py:141-154), so slab results equal
  the whole-array result plane for plane.

The GPU box has no ``/root/reference``: tests there read only these files.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.environ.get("LFBP_REFERENCE_SRC", "/root/reference/pkg/src"))

import lfbp  # noqa: E402  (the reference)
from lfbp import Dims5  # noqa: E402

from paper_2003_09133_b200.configs import WORKLOADS  # noqa: E402
from paper_2003_09133_b200.synth import baseline_psf  # noqa: E402

# (name, shape, kind, density, seed, dtype)
SMALL_CASES = [
    ("ones_9_7_3_7_2", (9, 7, 3, 7, 2), "ones", None, None, np.float64),
    ("single_5_5_3_3_1", (5, 5, 3, 3, 1), "single", None, None, np.float64),
    ("centre_3_3_3_3_1", (3, 3, 3, 3, 1), "rng9", None, 9, np.float64),
    ("rand_5_5_3_3_2", (5, 5, 3, 3, 2), "random", 0.05, 0, np.float64),
    ("rand_5_5_3_3_1_f32", (5, 5, 3, 3, 1), "random", 0.05, 3, np.float32),
    ("rand_9_7_3_5_2_a", (9, 7, 3, 5, 2), "random", 0.4, 1, np.float64),
    ("rand_9_9_3_3_3", (9, 9, 3, 3, 3), "random", 0.3, 24, np.float64),
    ("rand_15_13_5_3_2", (15, 13, 5, 3, 2), "random", 0.3, 35, np.float64),
    ("rand_21_21_11_11_1", (21, 21, 11, 11, 1), "random", 0.3, 65, np.float64),
    ("rand_9_7_3_7_2", (9, 7, 3, 7, 2), "random", 0.5, 21, np.float64),
    ("rand_19_11_9_5_2", (19, 11, 9, 5, 2), "random", 0.1, 1040, np.float64),
    ("rand_7_9_5_3_2", (7, 9, 5, 3, 2), "random", 0.3, 26, np.float64),
    ("rand_21_21_11_11_3", (21, 21, 11, 11, 3), "random", 0.1, 1044, np.float32),
    ("even_4_5_3_3_1", (4, 5, 3, 3, 1), "uniform5", None, 5, np.float64),
    ("even_6_6_3_5_1", (6, 6, 3, 5, 1), "random", 0.3, 19, np.float64),
    ("even_4_6_3_5_1", (4, 6, 3, 5, 1), "random", 0.5, 19, np.float32),
    ("even_10_5_5_5_2", (10, 5, 5, 5, 2), "random", 0.5, 7, np.float32),
    ("even_8_12_7_3_2", (8, 12, 7, 3, 2), "random", 0.5, 8, np.float64),
    ("unit_1_1_1_1_1", (1, 1, 1, 1, 1), "random", 1.0, 1, np.float64),
    ("cell1_3_3_1_1_2", (3, 3, 1, 1, 2), "random", 1.0, 2, np.float32),
    ("tall_13_3_3_3_2", (13, 3, 3, 3, 2), "random", 0.7, 3, np.float32),
    ("cell_eq_7_7_7_7_1", (7, 7, 7, 7, 1), "random", 0.7, 4, np.float64),
    ("bits_17_11_5_3_3_f32", (17, 11, 5, 3, 3), "bits32", None, 11, np.float32),
    ("bits_13_9_3_5_2_f64", (13, 9, 3, 5, 2), "bits64", None, 12, np.float64),
    ("bits_even_6_4_3_3_2_f32", (6, 4, 3, 3, 2), "bits32", None, 13, np.float32),
    ("rand_89_89_11_11_1_f32", (89, 89, 11, 11, 1), "random", 0.1, 1046, np.float32),
]


def _input(shape, kind, density, seed, dtype):
    if kind == "ones":
        return np.ones(shape, dtype=dtype, order="F")
    if kind == "single":
        a = np.zeros(shape, dtype=dtype, order="F")
        a[0, 0, 2, 2, 0] = 0.625
        return a
    if kind == "rng9":
        return np.asfortranarray(np.random.default_rng(seed).random(shape).astype(dtype))
    if kind == "uniform5":
        return np.asfortranarray((1.0 - np.random.default_rng(seed).random(shape)).astype(dtype))
    if kind == "random":
        return lfbp.random_psf(Dims5(*shape), density=density, seed=seed, dtype=dtype).data
    if kind in ("bits32", "bits64"):
        # arbitrary bit patterns: NaN payloads, -0.0, denormals, infinities
        rng = np.random.default_rng(seed)
        it = np.uint32 if kind == "bits32" else np.uint64
        raw = rng.integers(0, np.iinfo(it).max, size=shape, dtype=it, endpoint=True)
        flat = raw.reshape(-1)
        specials = np.array([0x80000000, 0x00000001, 0x7F800000, 0xFF800000,
                             0x7FC00001, 0xFFBADBAD, 0x007FFFFF], dtype=np.uint64)
        if kind == "bits64":
            specials = np.array([0x8000000000000000, 1, 0x7FF0000000000000,
                                 0x7FF8000000000123, 0xFFF4000000000001,
                                 0x000FFFFFFFFFFFFF], dtype=np.uint64)
        flat[:len(specials)] = specials.astype(it)
        return np.asfortranarray(raw.view(dtype))
    raise ValueError(kind)


def make_small(path):
    arrays = {}
    manifest = []
    for name, shape, kind, density, seed, dtype in SMALL_CASES:
        H = _input(shape, kind, density, seed, dtype)
        dims = Dims5(*shape)
        psf = lfbp.PsfArray._wrap(dims, np.asfortranarray(H))
        bp = lfbp.compute_backprojection(psf)
        arrays[name + "__H"] = np.asfortranarray(H)
        arrays[name + "__Hp"] = np.asfortranarray(bp.data)
        if kind not in ("bits32", "bits64"):   # PsfArray values: nonnegative, no NaN
            # the reference's sorted-order plane sums (arrays.py:211-239), every plane
            arrays[name + "__fwdsum"] = np.stack(
                [lfbp.sum_forward_plane(psf, z) for z in range(1, shape[4] + 1)], axis=-1)
            arrays[name + "__bwdsum"] = np.stack(
                [lfbp.sum_backward_plane(bp, z) for z in range(1, shape[4] + 1)], axis=-1)
        odd = shape[0] % 2 == 1 and shape[1] % 2 == 1
        if odd:
            inv = lfbp.compute_psf_from_backprojection(lfbp.BackprojArray._wrap(dims, np.asfortranarray(H)))
            arrays[name + "__Hinv"] = np.asfortranarray(inv.data)
        manifest.append({"name": name, "shape": list(shape), "dtype": np.dtype(dtype).name,
                         "kind": kind, "density": density, "seed": seed, "inverse": odd,
                         "dropped": int(lfbp.dropped_source_count(dims))})
    # LF5 files written by the reference: input and `lfbp transform` output
    import tempfile
    lf5 = {}
    with tempfile.TemporaryDirectory() as td:
        for name in ("rand_19_11_9_5_2", "rand_21_21_11_11_3", "even_10_5_5_5_2", "rand_5_5_3_3_1_f32"):
            H = arrays[name + "__H"]
            dims = Dims5(*H.shape)
            fin, fout = os.path.join(td, "in.lf5"), os.path.join(td, "out.lf5")
            lfbp.save(lfbp.PsfArray(dims, H), fin)
            lfbp.save(lfbp.compute_backprojection(lfbp.load_psf(fin)), fout)
            lf5[name] = {"in_sha256": hashlib.sha256(open(fin, "rb").read()).hexdigest(),
                         "out_sha256": hashlib.sha256(open(fout, "rb").read()).hexdigest()}
    np.savez_compressed(path, **arrays)
    with open(path.replace(".npz", ".json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "lfbp " + lfbp.__version__,
                   "numpy": np.__version__, "cases": manifest, "lf5": lf5}, f, indent=1)
    print(f"wrote {path}: {len(manifest)} cases")


def make_projector(path):
    """Reference projector outputs (projector.py:55-196) for the GPU f2 path."""
    out = {}
    rng = np.random.default_rng(17)
    cases = []
    # (name, psf, volume shape, image shape)
    psf = lfbp.random_psf(Dims5(9, 9, 3, 3, 3), density=0.4, seed=17)
    cases.append(("sym", psf, rng.random((31, 31, 3)), rng.random((31, 31))))
    psf = lfbp.random_psf(Dims5(6, 6, 3, 5, 2), density=0.6, seed=6)
    cases.append(("even", psf, rng.random((17, 19, 2)), rng.random((17, 19))))
    psf = lfbp.random_psf(Dims5(19, 11, 9, 5, 2), density=0.5, seed=19)
    cases.append(("asym", psf, rng.random((23, 29, 2)), rng.random((23, 29))))
    psf = lfbp.random_psf(Dims5(5, 5, 3, 3, 1), density=1.0, seed=3, dtype=np.float32)
    cases.append(("f32", psf, np.ones((9, 9, 1)), np.ones((9, 9))))
    for name, psf, g, f in cases:
        bp = lfbp.compute_backprojection(psf)
        out[name + "__H"] = np.asfortranarray(psf.data)
        out[name + "__g"] = np.asfortranarray(g)
        out[name + "__f"] = np.asfortranarray(f)
        out[name + "__fwd"] = lfbp.forward_project(psf, lfbp.Volume(g)).data
        out[name + "__bp"] = lfbp.backproject(bp, lfbp.Image(f)).data
        out[name + "__adj"] = lfbp.backproject_adjoint(psf, lfbp.Image(f)).data
        out[name + "__norm"] = lfbp.normalizer(bp, f.shape).data
    # RL: reference test_projector.py:140-150 and acceptance criterion 6
    psf = lfbp.random_psf(Dims5(5, 5, 3, 3, 2), density=0.9, seed=15)
    g = np.zeros((11, 11, 2)); g[5, 5, 0] = 1.0; g[2, 8, 1] = 0.5
    img = lfbp.forward_project(psf, lfbp.Volume(g))
    st = lfbp.rl_run(psf, lfbp.compute_backprojection(psf), img, iterations=6)
    out["rl6__H"] = np.asfortranarray(psf.data)
    out["rl6__f"] = img.data
    out["rl6__est"] = st.estimate.data
    out["rl6__mse"] = np.asarray(st.mse_history)
    layout = lfbp.MlaLayout.rect(5.0)
    optics = lfbp.SpotOptics(sigma=0.7, fnumber=4.0, z_step=3.0, sigma_gain=0.3, focal_plane=0)
    psf = lfbp.synth_psf(layout, Dims5(17, 17, 5, 5, 3), optics)
    g = np.zeros((31, 31, 3)); g[9, 11, 0] = 1.0; g[21, 19, 2] = 1.0
    img = lfbp.forward_project(psf, lfbp.Volume(g))
    st = lfbp.rl_run(psf, lfbp.compute_backprojection(psf), img, iterations=20)
    out["rl20__H"] = np.asfortranarray(psf.data)
    out["rl20__f"] = img.data
    out["rl20__est"] = st.estimate.data
    out["rl20__mse"] = np.asarray(st.mse_history)
    out["rl20__dead"] = np.asarray(st.dead_voxels)
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays")


def make_digests(cfg: str, slab: int):
    w = WORKLOADS[cfg]
    n_s, n_t, n_x, n_y, n_z = w.shape
    in_planes, out_planes = [], []
    h_in, h_out = hashlib.sha256(), hashlib.sha256()
    t_ref = 0.0
    for z0 in range(0, n_z, slab):
        z1 = min(n_z, z0 + slab)
        H = baseline_psf(w, z0, z1)
        psf = lfbp.PsfArray._wrap(Dims5(n_s, n_t, n_x, n_y, z1 - z0), H)
        t = time.perf_counter()
        Hp = lfbp.compute_backprojection(psf).data
        t_ref += time.perf_counter() - t
        for k in range(z1 - z0):
            a = H[..., k].tobytes(order="F")
            b = Hp[..., k].tobytes(order="F")
            in_planes.append(hashlib.sha256(a).hexdigest())
            out_planes.append(hashlib.sha256(b).hexdigest())
            h_in.update(a)
            h_out.update(b)
        print(f"  {cfg} planes [{z0},{z1}) done, reference time so far {t_ref:.1f} s", flush=True)
        del H, Hp, psf
    doc = {"config": cfg, "shape": list(w.shape), "dtype": np.dtype(w.dtype).name,
           "seed": w.seed, "law": w.law, "slab_planes": slab,
           "reference_seconds_total": round(t_ref, 3),
           "input_sha256": h_in.hexdigest(), "hprime_sha256": h_out.hexdigest(),
           "input_plane_sha256": in_planes, "hprime_plane_sha256": out_planes,
           "generator": "tests/golden/make_golden.py (lfbp.compute_backprojection on "
                        "paper_2003_09133_b200.synth.baseline_psf input)"}
    path = os.path.join(HERE, f"digests_{cfg}.json")
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    print(f"wrote {path}")


# the reference's randomized acceptance matrix (test_acceptance.py:21-27):
# (dims, number of arrays), seeds 1000, 1001, ... in order, density 0.1
ACCEPTANCE_SUITE = [((9, 9, 3, 3, 3), 20), ((15, 13, 5, 3, 2), 12), ((19, 11, 9, 5, 2), 8),
                    ((21, 21, 11, 11, 3), 6), ((89, 89, 11, 11, 2), 4)]


def make_acceptance(path):
    """Digests of the reference's H' (and of its inverse) for the 50 arrays of
    its acceptance suite, drawn by lfbp.random_psf; the tests redraw them with
    synth.random_psf_like_reference (bit-identical, checked here)."""
    from paper_2003_09133_b200.synth import random_psf_like_reference
    cases = []
    seed = 1000
    for shape, count in ACCEPTANCE_SUITE:
        for _ in range(count):
            psf = lfbp.random_psf(Dims5(*shape), density=0.1, seed=seed)
            mine = random_psf_like_reference(shape, density=0.1, seed=seed)
            assert psf.data.tobytes(order="F") == mine.tobytes(order="F"), "generator restatement drifted"
            bp = lfbp.compute_backprojection(psf)
            inv = lfbp.compute_psf_from_backprojection(bp)
            assert np.array_equal(inv.data, psf.data)
            cases.append({"shape": list(shape), "seed": seed, "density": 0.1,
                          "input_sha256": hashlib.sha256(psf.data.tobytes(order="F")).hexdigest(),
                          "hprime_sha256": hashlib.sha256(bp.data.tobytes(order="F")).hexdigest()})
            seed += 1
    doc = {"source": "lfbp test_acceptance.py:21-27 suite, lfbp.random_psf(density=0.1, seeds 1000..1049), "
                     "lfbp.compute_backprojection", "cases": cases}
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    print(f"wrote {path}: {len(cases)} cases")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--acceptance", action="store_true")
    ap.add_argument("--small", action="store_true")
    ap.add_argument("--configs", default="")
    ap.add_argument("--slab", type=int, default=8)
    a = ap.parse_args()
    if a.small:
        make_small(os.path.join(HERE, "small_cases.npz"))
        make_projector(os.path.join(HERE, "projector_cases.npz"))
    if a.acceptance:
        make_acceptance(os.path.join(HERE, "acceptance_suite.json"))
    for c in [c for c in a.configs.split(",") if c]:
        make_digests(c, a.slab)


if __name__ == "__main__":
    main()
