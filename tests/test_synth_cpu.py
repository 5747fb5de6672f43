"""K6 (device synthesis of the BASELINE inputs) restated on the CPU: the
PCG64 jump-ahead and the value law the kernel implements reproduce numpy's
``default_rng([seed, z]).random`` stream and ``synth.baseline_plane`` bit for
bit (the GPU test compares the kernel itself)."""
import numpy as np
import pytest

from paper_2003_09133_b200.configs import WORKLOADS
from paper_2003_09133_b200.synth import _device_tables, _pcg_states, baseline_plane

MULT = 0x2360ED051FC65DA44385DF649FCCF645
M128 = (1 << 128) - 1


def _jump(k, inc):
    """(A, C) with s_k = A s_0 + C, by squaring (as lcg_jump in synth.cuh)."""
    a, c, A, C = MULT, inc, 1, 0
    while k:
        if k & 1:
            A, C = (a * A) & M128, (a * C + c) & M128
        c = (a * c + c) & M128
        a = (a * a) & M128
        k >>= 1
    return A, C


def _draw(state, inc, e):
    A, C = _jump(e + 1, inc)
    s = (A * state + C) & M128
    hi, lo = s >> 64, s & ((1 << 64) - 1)
    x = hi ^ lo
    rot = s >> 122
    out = ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)
    return (out >> 11) * (1.0 / 9007199254740992.0)


@pytest.mark.parametrize("cfg,z", [("C1", 0), ("C1", 8), ("C4", 20), ("C4", 3), ("C2", 25)])
def test_kernel_algorithm_reproduces_numpy(cfg, z):
    w = WORKLOADS[cfg]
    n_s, n_t, n_x, n_y, _ = w.shape
    P = n_s * n_t * n_x * n_y
    st = _pcg_states(w, z, z + 1)[0]
    state = int(st[0]) | (int(st[1]) << 64)
    inc = int(st[2]) | (int(st[3]) << 64)
    u_all = np.random.default_rng([w.seed, z]).random(P)
    plane = baseline_plane(w, z).reshape(-1, order="F")
    ts, tt, r2 = _device_tables(w, z, z + 1)
    ts, tt = ts[0].reshape(-1), tt[0].reshape(-1)
    rng = np.random.default_rng(123)
    for e in [0, 1, 31, 32, P - 1] + list(rng.integers(0, P, 40)):
        e = int(e)
        u = _draw(state, inc, e)
        assert u == u_all[e]
        s, r = e % n_s, e // n_s
        t, r = r % n_t, r // n_t
        x, y = r % n_x, r // n_x
        a, b = ts[s + n_s * x], tt[t + n_t * y]
        v = (u if a + b <= r2[0] else 0.0) if r2 is not None else (u * a) * b
        assert np.array(v).astype(w.dtype).tobytes() == plane[e:e + 1].tobytes()
