"""The BASELINE.json workloads C1..C5 and their value laws.

Shapes are (n_s, n_t, n_x, n_y, n_z): PSF rows/columns, source phase behind
the lenslet, depth -- the reference's H[s, t, x, y, z] layout
(arrays.py:3-23 of the reference ``lfbp`` package).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    shape: tuple[int, int, int, int, int]
    dtype: type
    seed: int
    law: str              # "gauss" or "disc"
    a: float              # width (gauss sigma) or radius law: a + b*|z - zc|
    b: float
    zc: int

    @property
    def itemsize(self) -> int:
        return np.dtype(self.dtype).itemsize

    @property
    def n_elems(self) -> int:
        n = 1
        for v in self.shape:
            n *= v
        return n

    @property
    def plane_elems(self) -> int:
        n_s, n_t, n_x, n_y, _ = self.shape
        return n_s * n_t * n_x * n_y

    @property
    def nbytes(self) -> int:
        return self.n_elems * self.itemsize

    def width(self, z: int) -> float:
        return self.a + self.b * abs(z - self.zc)

    def with_planes(self, n_z: int) -> "Workload":
        """Same law on a different depth count (used for bounded samples)."""
        n_s, n_t, n_x, n_y, _ = self.shape
        return Workload(self.name, (n_s, n_t, n_x, n_y, n_z), self.dtype, self.seed,
                        self.law, self.a, self.b, self.zc)


WORKLOADS: dict[str, Workload] = {
    "C1": Workload("C1", (55, 55, 11, 11, 9), np.float32, 0, "gauss", 3.0, 2.0, 4),
    "C2": Workload("C2", (195, 195, 15, 15, 51), np.float32, 1, "gauss", 4.0, 1.5, 25),
    "C3": Workload("C3", (399, 399, 19, 19, 64), np.float32, 2, "gauss", 5.0, 2.0, 32),
    "C4": Workload("C4", (273, 273, 13, 13, 41), np.float64, 3, "disc", 4.0, 3.0, 20),
    "C5": Workload("C5", (631, 631, 21, 21, 101), np.float32, 4, "gauss", 6.0, 2.0, 50),
}
