"""Kernel specs and the BASELINE.json workload configs (pure Python, no GPU).

Formulas (BASELINE.json ``configs``), 1-based indices:

* green  (kind 0): K = exp(-i kappa rho) / rho, rho = |x_i - y_j|,
  x_i = (i_1/n, .., i_d/n, 0..), y_j = (j_1/n, .., j_d/n, 0..) + offset.
  Plates (d=2): offset (0, 0, 1).  Cubes (d=3): offset (2, 0, 0).
  kappa = 2 pi n / ppw (ppw = 8 points per wavelength in BASELINE).
* dft    (kind 1): K = exp(-2 pi i x.k), x_p = (i_p - 1)/n, k_p = j_p - 1 - n/2,
  phase reduced exactly as (sum (i_p-1)(j_p-1-n/2)) mod n; optional two-sided
  per-mode bit reversal.
* radon2d (kind 2): K = exp(2 pi i Phi), Phi = x.k + sqrt(c1^2 k1^2 + c2^2 k2^2),
  c1 = (2 + sin 2pi x1 sin 2pi x2)/16, c2 = (2 + cos 2pi x1 cos 2pi x2)/16,
  x_p = (i_p - 1)/n, k_p = j_p - 1 - n/2.
* radon3d (kind 3): K = exp(2 pi i Phi), Phi = x.k + c |k|,
  c = (3 + sin 2pi x1 sin 2pi x2 sin 2pi x3)/100; x.k reduced
  exactly mod 1 as for radon2d.
* nudft   (kind 4): type-2 non-uniform DFT K = exp(2 pi i x^i . y^j),
  y^j_k = (j_k - 1)/n, x^i_k uniform in [0, n-1] from derive_seed(seed, {0x4E,
  flat(i), k}) (SPEC.md kernels: counter-based locations).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

GREEN, DFT, RADON2D, RADON3D, NUDFT = 0, 1, 2, 3, 4


@dataclass(frozen=True)
class KernelSpec:
    kind: int
    d: int
    n: int
    kappa: float = 0.0
    offset: tuple = (0.0, 0.0, 0.0)
    bitrev: bool = False
    seed: int = 0  # NUDFT locations

    def describe(self) -> str:
        name = {GREEN: "green", DFT: "dft", RADON2D: "radon2d", RADON3D: "radon3d", NUDFT: "nudft"}[self.kind]
        return f"{name}(d={self.d}, n={self.n})"


def green_plates(n: int, ppw: float = 8.0) -> KernelSpec:
    return KernelSpec(GREEN, 2, n, 2 * math.pi * n / ppw, (0.0, 0.0, 1.0))


def green_cubes(n: int, ppw: float = 8.0, offset=(2.0, 0.0, 0.0)) -> KernelSpec:
    return KernelSpec(GREEN, 3, n, 2 * math.pi * n / ppw, tuple(offset))


def dft(d: int, n: int, bitrev: bool = True) -> KernelSpec:
    return KernelSpec(DFT, d, n, 0.0, (0.0, 0.0, 0.0), bitrev)


def radon2d(n: int) -> KernelSpec:
    return KernelSpec(RADON2D, 2, n)


def radon3d(n: int) -> KernelSpec:
    return KernelSpec(RADON3D, 3, n)


def nudft(d: int, n: int, seed: int = 1) -> KernelSpec:
    return KernelSpec(NUDFT, d, n, seed=seed)


def level_rule(n: int, cb: int = 8) -> int:
    """Largest even L with n / 2^L >= C_b."""
    L = 0
    while (n >> (L + 2)) >= cb and n % (1 << (L + 2)) == 0:
        L += 2
    return L


@dataclass(frozen=True)
class Config:
    name: str
    spec: KernelSpec
    tol: float
    cb: int = 8
    seed: int = 2411_03029
    input_seed: int = 7
    nv: int = 1
    note: str = ""

    @property
    def L(self) -> int:
        return level_rule(self.spec.n, self.cb)

    @property
    def points(self) -> int:
        return self.spec.n ** self.spec.d


# BASELINE.json "configs", in order.
CONFIGS = [
    Config("green_plates_n64", green_plates(64), 1e-6),
    Config("green_cubes_n64", green_cubes(64), 1e-6),
    Config("green_cubes_n256", green_cubes(256), 1e-4),
    Config("dft6_n16", dft(6, 16), 1e-8, cb=1,
           note="C_b=1 (L=4): C_b=8 gives L=0 (SURVEY F4); two-sided bit reversal (App. A3)"),
    Config("radon2d_n1024", radon2d(1024), 1e-6),
]
BY_NAME = {c.name: c for c in CONFIGS}

# ProxyStrategy (q, row_cap) per config for the north_star accuracy gate --
# 1000 sampled outputs against direct dense sums -- measured on B200
# (profiles/r2_accuracy_sweep.jsonl).  The reference default
# (q = 3, row_cap = 2^17, id.hpp:50-55) is proxy-deficient for these
# operators: with every proxy row (ProxyMode::All) the same butterflies land at
# 0.2-0.7 tol at sizes where All is feasible, so the loss is the
# Cartesian-product row sample, not the composition; the error falls
# monotonically with the row cap.  Measured sampled error / tol:
#   green_plates_n64  (4, 2^17): 0.69          green_cubes_n64 (3, 2^23): 0.65
#   green_cubes_n256  (6, 2^27): 0.97 (1058 s construction, 1248 s before the pipelined panels; (4, 2^25): 1.23, 2^23: 2.0-2.5, 2^21: 6.8)
#   dft6_n16          (3, 2^17): 1e-7 (exact: every ID has rank 1)
#   radon2d_n1024     (12, 2^23): 0.87 (609 s construction; (8, 2^21): 5.3, default 2256-4375)
ACCURACY_STRATEGY = {
    "green_plates_n64": (4, 1 << 17),
    "green_cubes_n64": (3, 1 << 23),
    "green_cubes_n256": (6, 1 << 27),
    "dft6_n16": (3, 1 << 17),
    "radon2d_n1024": (12, 1 << 23),
}
