# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE ONLY -- generates the golden fixtures in tests/golden/ by
running the UNMODIFIED reference (oracle/_ref/libhenet_ref.so, the henet headers
under /root/reference compiled by oracle/Makefile).  Run in the build container:

    python oracle/gen_golden.py

Fixtures:
  small_n64.npz              full inputs + reference outputs at N=64 (3 chain
                             primes + special) for every hot-path function
  baseline_n8192.json        sha256 of reference outputs at the BASELINE
                             N=8192 parameters, inputs from splitmix64 (so they
                             are reproducible without numpy's generators)
  kat.json                   the reference tests' own known answers
                             (proj/tests/test_encoding.cpp:84-91,
                             proj/tests/test_modmath.cpp:45-89)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import refbind as R  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")

MASK = (1 << 64) - 1


def splitmix64(seed: int, count: int) -> np.ndarray:
    """Deterministic u64 stream (Steele et al.), vectorised; fixture inputs."""
    idx = np.arange(1, count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + idx * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def residues(seed, shape, chain):
    """u64 array (..., L, N) of residues mod chain[limb] from splitmix64."""
    n = int(np.prod(shape))
    raw = splitmix64(seed, n).reshape(shape)
    L = shape[-2]
    q = np.array(chain[:L], dtype=np.uint64).reshape((1,) * (len(shape) - 2) + (L, 1))
    return raw % q


def is_prime(n):
    if n < 2:
        return False
    for p in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if n % p == 0:
            return n == p
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def primes_below(bits, n, count, skip=()):
    out, q = [], ((1 << bits) // (2 * n)) * (2 * n) + 1
    while len(out) < count:
        q -= 2 * n
        if is_prime(q) and q not in skip:
            out.append(q)
    return out


def h(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint64).tobytes()).hexdigest()


def small():
    n = 64
    chain = [primes_below(30, n, 1)[0]] + primes_below(24, n, 2)
    special = primes_below(30, n, 2)[1]
    scale = float(2 ** 20)
    ref = R.RefContext(n, chain, special, scale)
    L = len(chain)
    out = {"n": n, "chain": np.array(chain, np.uint64), "special": special, "scale": scale}
    out["roots"] = np.array([ref.ntt_root(i) for i in range(L + 1)], np.uint64)
    limbs = residues(1, (L + 1, n), chain + [special]) if False else None
    ntt_in = np.stack([splitmix64(10 + i, n) % np.uint64(q) for i, q in enumerate(chain + [special])])
    out["ntt_in"] = ntt_in
    out["ntt_fwd"] = np.stack([ref.ntt(i, ntt_in[i]) for i in range(L + 1)])
    out["ntt_inv"] = np.stack([ref.ntt(i, ntt_in[i], inverse=True) for i in range(L + 1)])
    vals = np.array([0.0, 1.0, -1.0, 0.5, -0.5, 0.123456789, -3.75, 1e-7, 2.5, -0.0625])
    scales = np.array([scale, 2.0 ** 40, 1234.5678])
    enc = np.zeros((len(vals), len(scales), L), np.uint64)
    for i, v in enumerate(vals):
        for j, s in enumerate(scales):
            enc[i, j] = ref.encode_scalar(v, L, s)
    out["enc_vals"], out["enc_scales"], out["enc_scalar"] = vals, scales, enc
    rng = np.random.default_rng(5)
    slots = rng.uniform(-1, 1, n // 2) + 1j * rng.uniform(-1, 1, n // 2)
    out["vec_slots"] = slots
    out["enc_vector"] = ref.encode_vector(slots, L, scale)
    keys = ref.keygen(17, True)
    out["sk"], out["rk"] = keys.sk_words(), keys.rk_words()
    samples = rng.uniform(0, 1, (n // 2, 5))
    out["samples"] = samples
    ct, sc = ref.encrypt_tensor(keys, samples, 23)
    out["ct"], out["ct_scale"] = ct, sc
    out["decrypt"] = ref.decrypt_tensor(keys, ct, sc, 0, n // 2)
    res = ref.encode_scalar(-0.3, L, scale)
    out["mul_res"] = res
    out["mul"], _ = ref.mul_ct_pt_scalar(ct, sc, res, scale)
    out["add"] = ref.add_ct_ct(ct[:2], ct[2:4], sc)
    sq, sqs = ref.square(ct[:2], sc)
    out["square"] = sq
    out["relin"] = ref.relinearize(keys, sq, sqs)
    out["rescale"], _ = ref.rescale(out["relin"], sqs, L - 1)
    out["rescale2"], _ = ref.rescale(out["relin"], sqs, 1)
    np.savez_compressed(os.path.join(GOLD, "small_n64.npz"), **out)
    print("small_n64.npz written")


def baseline():
    from paper_1908_04172_b200 import workloads as W
    p = W.N8192
    n, chain, special = p["n"], p["chain"], p["special"]
    ref = R.RefContext(n, chain, special, p["scale"])
    L = len(chain)
    g = {"params": p, "input_generator": "splitmix64(seed) % q, see oracle/gen_golden.py"}
    g["roots"] = [ref.ntt_root(i) for i in range(L + 1)]
    g["ntt_fwd"] = {}
    for i, q in enumerate(chain + [special]):
        x = splitmix64(100 + i, n) % np.uint64(q)
        g["ntt_fwd"][str(i)] = h(ref.ntt(i, x))
    ct = residues(200, (3, 2, L, n), chain)
    g["rescale_6_to_5"] = h(ref.rescale(ct, 2.0 ** 48, 5)[0])
    g["rescale_6_to_2"] = h(ref.rescale(ct, 2.0 ** 48, 2)[0])
    keys = ref.keygen(7, True)
    g["keygen_seed7"] = {"sk": h(keys.sk_words()), "rk": h(keys.rk_words())}
    ct5 = residues(300, (2, 2, 5, n), chain)
    sq, sqs = ref.square(ct5, 2.0 ** 24)
    g["square_l5"] = h(sq)
    rl = ref.relinearize(keys, sq, sqs)
    g["relin_l5_seed7key"] = h(rl)
    g["relin_rescale_l5"] = h(ref.rescale(rl, sqs, 4)[0])
    rng = np.random.default_rng(8)
    slots = rng.uniform(-1, 1, n // 2) + 1j * rng.uniform(-1, 1, n // 2)
    np.save(os.path.join(GOLD, "vec_slots_n8192.npy"), slots)
    g["encode_vector_l6"] = h(ref.encode_vector(slots, L, p["scale"]))
    # c1 dense layer, outputs 0..3 (inputs: splitmix residues, weights: workloads.dense_layer())
    wl = W.dense_layer()
    x = residues(400, (845, 2, L, n), chain)
    outw, osc, _ = ref.execute(None, wl.manifest, wl.blob, x, p["scale"], patch=True)
    g["c1_dense_outputs"] = [h(outw[j]) for j in range(outw.shape[0])]
    g["c1_dense_scale"] = osc
    with open(os.path.join(GOLD, "baseline_n8192.json"), "w") as f:
        json.dump(g, f, indent=1)
    print("baseline_n8192.json written")


def kat():
    k = {}
    r17 = R.RefContext(8, [17], 0, 16.0)
    k["encode_scalar_q17_scale16"] = {"1.0": [int(x) for x in r17.encode_scalar(1.0, 1, 16.0)],
                                      "-1.0": [int(x) for x in r17.encode_scalar(-1.0, 1, 16.0)]}
    r7 = R.RefContext(8, [17], 0, 16.0)
    k["barrett_100_mod_17"] = int(r7.barrett(0, np.array([100], np.uint64), b64=True)[0])
    with open(os.path.join(GOLD, "kat.json"), "w") as f:
        json.dump(k, f, indent=1)
    print("kat.json written", k)


def plans():
    """Reference plan_rescaling output for every workload graph (lazy, naive, patched)."""
    from paper_1908_04172_b200 import workloads as W
    p = W.N8192
    ref = R.RefContext(p["n"], p["chain"], p["special"], p["scale"])
    out = {}
    for wl in (W.dense_layer(), W.cryptonets(), W.cryptonets_relu(), W.toy_cryptonets(),
               W.cryptonets_relu(packing=0)):
        out[wl.name] = {"lazy": ref.plan(wl.manifest, wl.blob, 0), "naive": ref.plan(wl.manifest, wl.blob, 1),
                        "patched": ref.plan(wl.manifest, wl.blob, 0, patch=True)}
    with open(os.path.join(GOLD, "plans_n8192.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("plans_n8192.json written")


if __name__ == "__main__":
    os.makedirs(GOLD, exist_ok=True)
    small()
    baseline()
    kat()
    plans()
