"""Problem configurations C1..C5 of BASELINE.json, plus small test-only variants.

This module holds NO arithmetic of the method (no time stepping, no rSVD, no
Parareal).  It only names the problems: grid sizes, interval counts, ranks and
seeds.  Both the CPU oracle (`oracle/`) and the CUDA path consume it.

Readings of BASELINE.json that the paper leaves open are the Z-list of
SURVEY.md §8(c); each field cites the one it uses.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

BASE_SEED = 2508088730          # SURVEY §8(d) "Seeds: base seed 2508088730 + config index"


@dataclass(frozen=True)
class Config:
    name: str
    dim: int            # 1 or 2 spatial dimensions
    n: int              # interior points per side (1D: n DOFs; 2D: n*n DOFs)
    T: float            # final time
    N: int              # Parareal intervals
    m: int              # implicit-Euler steps per interval (paper: 100*T/10)
    k: int              # truncation rank R_n
    p: int              # oversampling
    K: int              # Parareal iterations (BJ; Z12 for C2..C4)
    problem: str        # "heat" | "reaction_diffusion"
    u0: str             # initial-value recipe name (generators.py)
    source: str         # source recipe name (generators.py)
    nsrc: int = 1       # number of independent source terms sharing G' (C4: 64)
    seed: int = BASE_SEED

    @property
    def l(self) -> int:
        return self.k + self.p

    @property
    def n_dof(self) -> int:
        return self.n if self.dim == 1 else self.n * self.n

    @property
    def h(self) -> float:
        return 1.0 / (self.n + 1)

    @property
    def dT(self) -> float:
        return self.T / self.N

    @property
    def dt(self) -> float:
        return self.T / (self.N * self.m)

    # Seed offsets, Z4: Omega uses seed, u0 seed+1, sources seed+2.
    @property
    def seed_omega(self) -> int:
        return self.seed

    @property
    def seed_u0(self) -> int:
        return self.seed + 1

    @property
    def seed_src(self) -> int:
        return self.seed + 2

    def build_dof_steps(self) -> int:
        """N * 2l * n_dof * m: forward + adjoint sketch solves."""
        return self.N * 2 * self.l * self.n_dof * self.m

    def parareal_dof_steps(self) -> int:
        """Offsets b_n plus K iterations of N*nsrc fine solves."""
        return (self.K + 1) * self.N * self.nsrc * self.n_dof * self.m


C1 = Config("C1", 1, 127, 1.0, 16, 64, 8, 4, 8, "heat", "x1mx", "c1", seed=BASE_SEED + 0)
C2 = Config("C2", 1, 4095, 1.0, 64, 256, 32, 8, 8, "heat", "sine20", "c2", seed=BASE_SEED + 1)
C3 = Config("C3", 2, 255, 0.5, 64, 128, 64, 10, 8, "heat", "smooth2d", "bump1", seed=BASE_SEED + 2)
C4 = Config("C4", 1, 16383, 2.0, 256, 128, 48, 16, 8, "reaction_diffusion", "x1mx", "c4",
            nsrc=64, seed=BASE_SEED + 3)
C5 = Config("C5", 2, 511, 1.0, 512, 64, 96, 16, 10, "heat", "smooth2d", "bump4", seed=BASE_SEED + 4)

CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5)}

# Test-only variants (SURVEY §4 "Extra test-only variants"): small k so that
# Parareal takes several iterations, and small grids the oracle finishes in
# seconds while still spanning several GPU tiles and a ragged tail.
T1 = replace(C1, name="T1", n=200, N=8, m=12, k=3, p=2, K=6)
T1_K1 = replace(C1, name="T1k1", n=157, N=6, m=10, k=1, p=1, K=6)
T4 = replace(C4, name="T4", n=301, N=8, m=16, k=4, p=4, K=6, nsrc=5)
T2D = replace(C3, name="T2D", n=63, N=6, m=10, k=6, p=3, K=5)
# non-symmetric (convection-diffusion) operators: A != A^T, so F'^* is a true
# transposed solve (rSVD step 3) -- small and at C4's grid
T4N = replace(C4, name="T4N", problem="convection_diffusion", n=301, N=8, m=16, k=4, p=4, K=6, nsrc=5)
C4N = replace(C4, name="C4N", problem="convection_diffusion")
# more sources (12) than source terms (8): the offsets go through the source basis
T4S = replace(T4, name="T4S", nsrc=12)
VARIANTS = {c.name: c for c in (T1, T1_K1, T4, T2D, T4N, C4N, T4S)}


def get(name: str) -> Config:
    if name in CONFIGS:
        return CONFIGS[name]
    return VARIANTS[name]

# C5 geometry on fewer intervals (the 511^2 grid, k = 96, p = 16, the same
# dt = 1/(512*64)): the full-size 2D Parareal the oracle can follow on one GPU
C5G = replace(C5, name="C5G", N=16, T=C5.T * 16 / 512)
VARIANTS[C5G.name] = C5G

# the paper's Experiment 2 (eq. ex2):
# time-dependent conductivity, Neumann conditions, linear finite elements with
# 100 elements (n = 101 nodes), 100 time steps on [0, 1] in N = 10 intervals,
# rank R = 5 with p = 1 oversampling vector; problem data in
# workloads/exp2.py.  E2FD: the finite-difference (M = I, non-symmetric A)
# version; E2L: the same problem at GPU scale (4096 nodes, 64 x 64 steps).
E2 = Config("E2", 1, 101, 1.0, 10, 10, 5, 1, 8, "exp2_fem", "exp2", "exp2", seed=BASE_SEED + 5)
E2FD = replace(E2, name="E2FD", problem="exp2_fd")
E2L = replace(E2, name="E2L", n=4096, N=64, m=64, k=16, p=4)
for _c in (E2, E2FD, E2L):
    VARIANTS[_c.name] = _c
