"""Gaussian test vectors omega_i of rSVD step 1 -- TEST INFRASTRUCTURE ONLY.

The paper only asks for "some appropriate probability distribution on V"
(P:259-260); BASELINE.json fixes i.i.d. N(0,1).  The sketch Omega_n is far too
large to pass in (C5: 1.5e10 values), so the CUDA path and this oracle each
implement the same counter-based generator (reading R-RNG):

  Philox4x64-10 (Salmon et al., SC'11), key = (seed, 0),
  counter = (i // 4, c, q, s)   for row i, column c (0..l-1), interval q (0-based),
                                stream s (0: Omega; 2: the independent adjoint sketch);
  the four 64-bit outputs x0..x3 give rows 4*(i//4) + 0..3 by Box-Muller:
      u1 = ((x0 >> 11) + 1) * 2^-53  in (0, 1],   u2 = (x1 >> 11) * 2^-53,
      z0 = sqrt(-2 ln u1) cos(2 pi u2),  z1 = sqrt(-2 ln u1) sin(2 pi u2),
  and likewise (x2, x3) -> z2, z3.
2D problems number the interior DOFs row = ix * n + iy.

Pinned in tests/test_oracle_rng.py against numpy.random.Philox (an
independent implementation of the same bijection) and against N(0,1)
moments.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
PHILOX_M0 = 0xD2E7470EE14C6C93
PHILOX_M1 = 0xCA5A826395121157
PHILOX_W0 = 0x9E3779B97F4A7C15
PHILOX_W1 = 0xBB67AE8584CAA73B


def _mulhilo64(a: int, b: np.ndarray):
    """(hi, lo) of the 128-bit product a*b for a scalar a and uint64 array b."""
    b = b.astype(np.uint64)
    mask = np.uint64(0xFFFFFFFF)
    a_lo, a_hi = np.uint64(a & 0xFFFFFFFF), np.uint64(a >> 32)
    b_lo, b_hi = b & mask, b >> np.uint64(32)
    with np.errstate(over="ignore"):
        ll = a_lo * b_lo
        lh = a_lo * b_hi
        hl = a_hi * b_lo
        hh = a_hi * b_hi
        mid = (ll >> np.uint64(32)) + (lh & mask) + (hl & mask)
        lo = (ll & mask) | ((mid & mask) << np.uint64(32))
        hi = hh + (lh >> np.uint64(32)) + (hl >> np.uint64(32)) + (mid >> np.uint64(32))
    return hi, lo


def philox4x64_10(c0, c1, c2, c3, k0: int, k1: int):
    """Philox4x64 with 10 rounds on arrays of counters; returns 4 uint64 arrays."""
    c = [np.asarray(x, dtype=np.uint64) for x in (c0, c1, c2, c3)]
    c = np.broadcast_arrays(*c)
    c = [x.copy() for x in c]
    k0, k1 = k0 & 0xFFFFFFFFFFFFFFFF, k1 & 0xFFFFFFFFFFFFFFFF
    for r in range(10):
        if r > 0:
            k0 = (k0 + PHILOX_W0) & 0xFFFFFFFFFFFFFFFF
            k1 = (k1 + PHILOX_W1) & 0xFFFFFFFFFFFFFFFF
        hi0, lo0 = _mulhilo64(PHILOX_M0, c[0])
        hi1, lo1 = _mulhilo64(PHILOX_M1, c[2])
        c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
    return c


def _box_muller(xa, xb):
    u1 = ((xa >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53
    u2 = (xb >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    r = np.sqrt(-2.0 * np.log(u1))
    th = 2.0 * np.pi * u2
    return r * np.cos(th), r * np.sin(th)


def gaussian_sketch(seed: int, interval: int, nrows: int, ncols: int, stream: int = 0) -> np.ndarray:
    """Omega_q (nrows x ncols), i.i.d. N(0,1), for 0-based interval q.  The
    fourth counter word selects an independent stream (0: the sketch Omega of
    step 1; 2: the independent adjoint sketch Psi)."""
    nb = (nrows + 3) // 4
    blk = np.arange(nb, dtype=np.uint64)[:, None]
    col = np.arange(ncols, dtype=np.uint64)[None, :]
    x0, x1, x2, x3 = philox4x64_10(blk, col, np.uint64(interval), np.uint64(stream), seed, 0)
    z0, z1 = _box_muller(x0, x1)
    z2, z3 = _box_muller(x2, x3)
    out = np.stack([z0, z1, z2, z3], axis=1).reshape(nb * 4, ncols)
    return np.ascontiguousarray(out[:nrows])
