"""Pins for oracle/rng.py (Gaussian test vectors; reading R-RNG)."""
import numpy as np
import pytest

from oracle.rng import gaussian_sketch, philox4x64_10


@pytest.mark.parametrize("key,ctr", [((0, 0), (0, 0, 0, 0)),
                                     ((5, 7), (3, 9, 11, 13)),
                                     ((2508088730, 0), (17, 40, 63, 0)),
                                     ((2**64 - 1, 2**64 - 1), (2**64 - 2, 2**64 - 1, 2**64 - 1, 2**64 - 1))])
def test_philox_matches_numpy_bitgenerator(key, ctr):
    # numpy's Philox (4x64-10) increments the counter before each block, so a
    # state counter of ctr-1 yields the block for ctr.
    big = sum(c << (64 * i) for i, c in enumerate(ctr))
    big = (big - 1) % 2**256
    prev = [(big >> (64 * i)) & (2**64 - 1) for i in range(4)]
    bg = np.random.Philox(key=np.array(key, dtype=np.uint64),
                          counter=np.array(prev, dtype=np.uint64))
    ref = bg.random_raw(4)
    got = philox4x64_10(*[np.uint64(c) for c in ctr], *key)
    assert [int(x) for x in got] == [int(x) for x in ref]


def test_philox_known_answer_zero():
    # Random123 known-answer vector for philox4x64_10 with zero counter and key.
    got = [int(x) for x in philox4x64_10(0, 0, 0, 0, 0, 0)]
    assert got == [0x16554D9ECA36314C, 0xDB20FE9D672D0FDC, 0xD7E772CEE186176B, 0x7E68B68AEC7BA23B]


def test_sketch_layout_and_determinism():
    a = gaussian_sketch(123, 4, 37, 6)
    b = gaussian_sketch(123, 4, 41, 6)
    assert a.shape == (37, 6)
    np.testing.assert_array_equal(a, b[:37])            # rows independent of nrows
    assert not np.array_equal(a, gaussian_sketch(123, 5, 37, 6))   # interval changes stream
    assert not np.array_equal(a, gaussian_sketch(124, 4, 37, 6))   # seed changes stream
    # column c of interval q does not depend on how many columns were asked for
    np.testing.assert_array_equal(gaussian_sketch(9, 1, 20, 3), gaussian_sketch(9, 1, 20, 8)[:, :3])


def test_sketch_is_standard_normal():
    z = gaussian_sketch(2508088730, 0, 40000, 25).ravel()
    assert abs(z.mean()) < 5e-3
    assert abs(z.var() - 1.0) < 1e-2
    assert abs(np.mean(z ** 3)) < 2e-2
    assert abs(np.mean(z ** 4) - 3.0) < 5e-2
    # independence of the pair (cos, sin) outputs
    zz = gaussian_sketch(7, 0, 40000, 1)[:, 0]
    assert abs(np.corrcoef(zz[0::2], zz[1::2])[0, 1]) < 2e-2
