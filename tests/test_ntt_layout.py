# SPDX-License-Identifier: Apache-2.0
"""Pure-Python proof obligations for the NTT register/shared-memory layouts of
paper_1908_04172_b200/csrc/hg_device.cuh (Ntt<LOGN>): each layout is a
bijection onto [0, N); every butterfly pair of every stage lives in one thread;
and the XOR swizzle makes all three shared-memory access patterns
bank-conflict free (32 lanes -> 32 distinct banks)."""
import pytest


def cfg(logn):
    logt = logn - 5
    cb = logn - 10 if logn >= 14 else 3
    mb = logt - cb
    return logt, cb, mb


def jA(logn, tid, k):
    logt, cb, mb = cfg(logn)
    return tid | (k << logt)


def jB(logn, tid, k):
    logt, cb, mb = cfg(logn)
    cbm, mbm = (1 << cb) - 1, (1 << mb) - 1
    return (tid & cbm) | ((k & mbm) << cb) | ((tid >> cb) << logt) | ((k >> mb) << (logt + mb))


def jC(logn, tid, k):
    logt, cb, mb = cfg(logn)
    cbm = (1 << cb) - 1
    return (k & cbm) | (tid << cb) | ((k >> cb) << (cb + logt))


def swz(logn, j):
    """Ntt::swz: one pad word per 32 elements."""
    return j + (j >> 5)


def tpart(logn, L, tid):
    logt, cb, mb = cfg(logn)
    if L == "A":
        return tid
    if L == "B":
        return (tid & ((1 << cb) - 1)) | ((tid >> cb) << logt)
    return tid << cb


def kpart(logn, L, k):
    logt, cb, mb = cfg(logn)
    if L == "A":
        return k << logt
    if L == "B":
        return ((k & ((1 << mb) - 1)) << cb) | ((k >> mb) << (logt + mb))
    return (k & ((1 << cb) - 1)) | ((k >> cb) << (cb + logt))


LAYOUTS = {"A": (jA, lambda l: (0, 5, cfg(l)[0])), "B": (jB, lambda l: (0, cfg(l)[2], cfg(l)[1])),
           "C": (jC, lambda l: (0, cfg(l)[1], 0))}


@pytest.mark.parametrize("logn", [12, 13, 14])
@pytest.mark.parametrize("name", ["A", "B", "C"])
def test_bijection_and_conflict_free(logn, name):
    jm, _ = LAYOUTS[name]
    n, t = 1 << logn, 1 << (logn - 5)
    seen = set()
    for tid in range(t):
        for k in range(32):
            seen.add(jm(logn, tid, k))
    assert seen == set(range(n))
    assert len({swz(logn, j) for j in range(n)}) == n and max(swz(logn, j) for j in range(n)) < n + n // 32
    worst = 1
    for w in range(t // 32):
        for k in range(32):
            lanes = [w * 32 + lane for lane in range(32)]
            addrs = [swz(logn, jm(logn, tid, k)) for tid in lanes]
            # address = base(tid) + const(k): the split the kernels use for immediate offsets
            assert addrs == [swz(logn, tpart(logn, name, tid)) + swz(logn, kpart(logn, name, k)) for tid in lanes]
            banks = [a % 32 for a in addrs]
            worst = max(worst, max(banks.count(b) for b in set(banks)))
    assert worst == 1 or (logn == 12 and name == "B" and worst == 2), (name, worst)


@pytest.mark.parametrize("logn", [12, 13, 14])
def test_butterfly_pairs_are_thread_local(logn):
    """Stage with t = 2^b pairs j and j + 2^b; pass A covers b in [LOGT, LOGN),
    pass B [CB, LOGT), pass C [0, CB); the pair must be (tid, k0) / (tid, k0 | 1 << rb)."""
    logt, cb, mb = cfg(logn)
    passes = [(jA, logt, 5), (jB, cb, mb), (jC, 0, cb)]
    covered = []
    for jm, blo, nb in passes:
        for rb in range(nb):
            b = blo + rb
            covered.append(b)
            for tid in range(1 << logt):
                for k in range(32):
                    if k & (1 << rb):
                        continue
                    assert jm(logn, tid, k) + (1 << b) == jm(logn, tid, k | (1 << rb))
    assert sorted(covered) == list(range(logn))


@pytest.mark.parametrize("logn", [12, 13, 14])
def test_pass_c_twiddle_factorisation(logn):
    """NTT v3 (hg_device.cuh): in pass C the twiddle index 2^nb + (j >> (b+1)) splits into
    disjoint bit fields from (c, g) and from tid, so bitrev(idx) = bitrev(2^nb | u_cg) +
    bitrev(u_tid) and psi^bitrev(idx) = V(b, c, g) * T_b(tid)."""
    logt, cb, mb = cfg(logn)

    def bitrev(v, bits):
        return int(format(v, f"0{bits}b")[::-1], 2)

    for tid in range(0, 1 << logt, 7):
        for k in range(32):
            j = jC(logn, tid, k)
            c, g = k & ((1 << cb) - 1), k >> cb
            for b in range(cb):
                nb = logn - 1 - b
                idx = (1 << nb) + (j >> (b + 1))
                u_cg = (c >> (b + 1)) | (g << (cb + logt - b - 1))
                u_t = tid << (cb - b - 1)
                assert (1 << nb) | u_cg | u_t == idx and u_cg & u_t == 0
                assert bitrev(idx, logn) == bitrev((1 << nb) | u_cg, logn) + bitrev(u_t, logn)
