# SPDX-License-Identifier: Apache-2.0
"""Pins the C restatement oracle (oracle/henet_oracle.c) to the reference:
golden fixtures produced by the unmodified reference (oracle/gen_golden.py) and
the reference tests' own known answers.  CPU only."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import cbind as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint64).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def small():
    g = dict(np.load(os.path.join(GOLD, "small_n64.npz")))
    oc = O.OracleContext(int(g["n"]), [int(q) for q in g["chain"]], int(g["special"]), float(g["scale"]))
    return g, oc


def test_small_roots_and_ntt(small):
    g, oc = small
    L = len(g["chain"])
    assert [oc.ntt_root(i) for i in range(L + 1)] == [int(x) for x in g["roots"]]
    for i in range(L + 1):
        assert np.array_equal(oc.ntt(i, g["ntt_in"][i]), g["ntt_fwd"][i])
        assert np.array_equal(oc.ntt(i, g["ntt_in"][i], inverse=True), g["ntt_inv"][i])
        assert np.array_equal(oc.ntt(i, oc.ntt(i, g["ntt_in"][i]), inverse=True), g["ntt_in"][i])


def test_small_encoders(small):
    g, oc = small
    L = len(g["chain"])
    for i, v in enumerate(g["enc_vals"]):
        for j, s in enumerate(g["enc_scales"]):
            assert np.array_equal(oc.encode_scalar(v, L, s), g["enc_scalar"][i, j]), (v, s)
    assert np.array_equal(oc.encode_vector(g["vec_slots"], L, float(g["scale"])), g["enc_vector"])


def test_small_keys_encrypt_ops(small):
    g, oc = small
    sk, rk = oc.keygen(17)
    assert np.array_equal(sk, g["sk"]) and np.array_equal(rk, g["rk"])
    ct = oc.encrypt_tensor(sk, g["samples"], 23)
    assert np.array_equal(ct, g["ct"])
    dec = oc.decrypt_tensor(sk, ct, float(g["ct_scale"]), 0, g["samples"].shape[0])
    assert np.array_equal(dec, g["decrypt"])
    assert np.array_equal(oc.mul_ct_pt_scalar(ct, g["mul_res"]), g["mul"])
    assert np.array_equal(oc.add_ct_ct(ct[:2], ct[2:4]), g["add"])
    sq = oc.square(ct[:2])
    assert np.array_equal(sq, g["square"])
    rl = oc.relinearize(sq, rk)
    assert np.array_equal(rl, g["relin"])
    L = len(g["chain"])
    assert np.array_equal(oc.rescale(rl, L - 1), g["rescale"])
    assert np.array_equal(oc.rescale(rl, 1), g["rescale2"])


@pytest.fixture(scope="module")
def big():
    with open(os.path.join(GOLD, "baseline_n8192.json")) as f:
        g = json.load(f)
    p = g["params"]
    return g, O.OracleContext(p["n"], p["chain"], p["special"], p["scale"])


def _residues(seed, shape, chain):
    from oracle.gen_golden import residues
    return residues(seed, shape, chain)


def test_baseline_ntt_rescale(big):
    from oracle.gen_golden import splitmix64
    g, oc = big
    p = g["params"]
    chain, special, n = p["chain"], p["special"], p["n"]
    assert [oc.ntt_root(i) for i in range(len(chain) + 1)] == g["roots"]
    for i, q in enumerate(chain + [special]):
        assert h(oc.ntt(i, splitmix64(100 + i, n) % np.uint64(q))) == g["ntt_fwd"][str(i)]
    ct = _residues(200, (3, 2, len(chain), n), chain)
    assert h(oc.rescale(ct, 5)) == g["rescale_6_to_5"]
    assert h(oc.rescale(ct, 2)) == g["rescale_6_to_2"]


def test_baseline_keys_relin_encode(big):
    g, oc = big
    p = g["params"]
    sk, rk = oc.keygen(7)
    assert h(sk) == g["keygen_seed7"]["sk"] and h(rk) == g["keygen_seed7"]["rk"]
    ct5 = _residues(300, (2, 2, 5, p["n"]), p["chain"])
    sq = oc.square(ct5)
    assert h(sq) == g["square_l5"]
    rl = oc.relinearize(sq, rk)
    assert h(rl) == g["relin_l5_seed7key"]
    assert h(oc.rescale(rl, 4)) == g["relin_rescale_l5"]
    slots = np.load(os.path.join(GOLD, "vec_slots_n8192.npy"))
    assert h(oc.encode_vector(slots, 6, p["scale"])) == g["encode_vector_l6"]


def test_baseline_c1_dense_subset(big):
    from paper_1908_04172_b200 import workloads as W
    g, oc = big
    p = g["params"]
    wl = W.dense_layer()
    blob = np.frombuffer(wl.blob, dtype="<f4")
    man = json.loads(wl.manifest)
    wm = man["weights"]
    w = blob[wm["fc_w"]["offset"] // 4: wm["fc_w"]["offset"] // 4 + 845 * 100].reshape(845, 100)
    b = blob[wm["fc_b"]["offset"] // 4: wm["fc_b"]["offset"] // 4 + 100]
    x = _residues(400, (845, 2, 6, p["n"]), p["chain"])
    outs = [0, 57, 99]
    got = oc.dense(x, w, 6, p["scale"], bias=b, rescale=True, outputs=outs)
    for k, j in enumerate(outs):
        assert h(got[k]) == g["c1_dense_outputs"][j], j


def test_reference_kats():
    """proj/tests/test_encoding.cpp:84-91 and proj/tests/test_modmath.cpp:45-89"""
    with open(os.path.join(GOLD, "kat.json")) as f:
        k = json.load(f)
    oc = O.OracleContext(8, [17], 0, 16.0)
    assert list(oc.encode_scalar(1.0, 1, 16.0)) == k["encode_scalar_q17_scale16"]["1.0"] == [16]
    assert list(oc.encode_scalar(-1.0, 1, 16.0)) == k["encode_scalar_q17_scale16"]["-1.0"] == [1]
    assert O.barrett_64(100, 17) == k["barrett_100_mod_17"] == 15
    assert O.barrett_64(100, 7) == 2
    rng = np.random.default_rng(1)
    for q in (17, 97, 7681, 1073692673, 1099511922689):
        for _ in range(2000):
            lo, hi = int(rng.integers(0, 2 ** 63)), int(rng.integers(0, q))
            assert O.barrett_128(lo, hi, q) == ((hi << 64) + lo) % q
            if q < 2 ** 32:
                z = int(rng.integers(0, 2 ** 63))
                assert O.barrett_64(z, q) == z % q


@pytest.mark.parametrize("n,q", [(4, 17), (8, 17), (16, 97), (16, 7681)])
def test_ntt_matches_schoolbook(n, q):
    """proj/tests/test_modmath.cpp:159-185: pointwise NTT product == negacyclic convolution."""
    oc = O.OracleContext(n, [q], 0, 1.0)
    rng = np.random.default_rng(n + q)
    for _ in range(50):
        a = rng.integers(0, q, n, dtype=np.uint64)
        b = rng.integers(0, q, n, dtype=np.uint64)
        A, B = oc.ntt(0, a), oc.ntt(0, b)
        prod = oc.ntt(0, (A.astype(object) * B.astype(object) % q).astype(np.uint64), inverse=True)
        want = [0] * n
        for i in range(n):
            for j in range(n):
                k = i + j
                v = int(a[i]) * int(b[j])
                if k >= n:
                    want[k - n] -= v
                else:
                    want[k] += v
        assert [int(x) for x in prod] == [w % q for w in want]


def test_scalar_encoding_lemma():
    """proj/tests/test_encoding.cpp:93-114: expand(encode_scalar(r)) == encode_vector(const r)
    on the P12 preset (N=4096, three ~2^30 primes)."""
    oc = O.OracleContext(4096, [1073750017, 1073815553, 1073872897], 1099511799809, 2.0 ** 30)
    rng = np.random.default_rng(13)
    for trial in range(6):
        r = (rng.random() - 0.5) * (200.0 if trial % 2 == 0 else 0.9)
        level = 3 if trial % 2 == 0 else 1 + int(rng.integers(0, 3))
        res = oc.encode_scalar(r, level, 2.0 ** 30)
        vec = oc.encode_vector(np.full(2048, r, dtype=np.complex128), level, 2.0 ** 30)
        assert np.array_equal(vec, np.repeat(res[:, None], 4096, axis=1))


@pytest.mark.parametrize("params,k,m", [("N8192", 40, 7), ("N16384", 24, 5)])
def test_dense_lazy_matches_mac_chain(params, k, m):
    """oc_dense_lazy (one 128-bit sum per residue, used for the K = 4096 c5b check) gives the
    residues of mac_output's per-tap mul + add chain (oc_dense), rescale included."""
    from paper_1908_04172_b200 import workloads as W
    p = getattr(W, params)
    oc = O.OracleContext(p["n"], p["chain"], p["special"], p["scale"])
    x = W.random_ciphertexts(p, k, seed=3)
    w = np.random.default_rng(4).normal(0, 0.1, (k, m)).astype(np.float32)
    w[0, 0] = 0.0
    L = len(p["chain"])
    for rescale in (True, False):
        assert np.array_equal(oc.dense_lazy(x, w, L, rescale), oc.dense(x, w, L, p["scale"], rescale=rescale))
