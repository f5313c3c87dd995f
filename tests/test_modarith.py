# SPDX-License-Identifier: Apache-2.0
"""Integer identities the device helpers (csrc/hg_device.cuh) rely on, checked with exact
Python integers for every BASELINE prime: the product Barrett of `mulmod` (one IMAD.HI on the
top k+1 bits) and the Shoup bound of `mul_shoup_lazy`."""
import random

import pytest

from paper_1908_04172_b200 import workloads as W

PRIMES = sorted(set(W.N8192["chain"] + [W.N8192["special"]] + [q for q in W.N16384["chain"][1:]]))
M32 = (1 << 32) - 1


def mulmod_dev(a, b, q):
    k = q.bit_length()
    bsh, bmu = k - 1, (1 << (k + 31)) // q
    assert bmu < (1 << 32)
    x = a * b
    xs = (x >> bsh) & M32
    assert xs == x >> bsh  # fits 32 bits
    qhat = (xs * bmu) >> 32
    r = (x - qhat * q) & M32
    assert x - qhat * q == r and 0 <= r < 3 * q  # remainder + at most 2q, no wrap
    r = min(r, (r - 2 * q) & M32)
    r = min(r, (r - q) & M32)
    return r


@pytest.mark.parametrize("q", PRIMES)
def test_mulmod_barrett32(q):
    assert q < (1 << 30)
    rng = random.Random(q)
    edge = [0, 1, 2, q - 2, q - 1, q // 2, (1 << (q.bit_length() - 1)), (1 << q.bit_length()) - 1]
    cases = [(a, b) for a in edge for b in edge] + [(rng.randrange(1 << q.bit_length()),
                                                     rng.randrange(1 << q.bit_length())) for _ in range(20000)]
    for a, b in cases:
        assert mulmod_dev(a, b, q) == (a * b) % q, (a, b)


@pytest.mark.parametrize("q", PRIMES)
def test_shoup_lazy_range(q):
    rng = random.Random(q + 1)
    for _ in range(5000):
        w = rng.randrange(q)
        wsh = (w << 32) // q
        for x in (0, M32, rng.randrange(1 << 32), 4 * q - 1):
            qhat = (x * wsh) >> 32
            r = (x * w - qhat * q) & M32
            assert r == x * w - qhat * q and r < 2 * q and r % q == (x * w) % q
