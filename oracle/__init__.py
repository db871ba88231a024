"""CPU oracle for arXiv 2508.08873 (Parareal with spectral coarse solvers).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import, call, link or execute anything
under oracle/.  The product path (paper_2508_08873_b200) never does; it fails
loudly when its CUDA library is missing.

Plain, slow, obviously correct: fp64 numpy plus one textbook C routine
(oracle/csrc/oracle_thomas.c).  It shares no code with the CUDA path; the only
common import is `workloads` (seeded input generators, no method arithmetic).

Modules and the passages they follow:
  rng.py       Gaussian test vectors, Philox4x64-10 + Box-Muller
  fine.py      backward-Euler fine solver F_n, F_n', F_n'^*, b_n
  linalg.py    Householder QR, one-sided Jacobi SVD
  rsvd.py      randomized SVD steps 1-6, spectral G_n
  parareal.py  Parareal iteration, update norms
  bounds.py    a priori / a posteriori bounds

Parity status: every function is pinned by tests/test_oracle_*.py (see
DESIGN.md "Oracle pins"); none is "parity unpinned".
"""
