# SPDX-License-Identifier: Apache-2.0
"""GPU client side vs the reference's CPU client (oracle/_ref, all host threads) on the c2
batch: encrypt_tensor of 4096 images x 784 pixels, decrypt_tensor of the 10 logits.
Times are host wall clock around the public calls (host arrays in, host arrays out)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import refbind as R
from paper_1908_04172_b200 import henet as H, workloads as Wk

p = Wk.N8192
ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
ref = R.RefContext(p["n"], p["chain"], p["special"], p["scale"])
keys = ref.keygen(3, True)
sk = H.SecretKey(ctx, keys.sk_words())
imgs = Wk.synthetic_images((1, 28, 28), 4096, 1)


def best(fn, n):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        r = fn()
        ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts), r


H.encrypt_tensor(ctx, sk, imgs, 5)
g_ms, ct = best(lambda: H.encrypt_tensor(ctx, sk, imgs, 5), 5)
r_ms, (words, sc) = best(lambda: ref.encrypt_tensor(keys, imgs, 5), 2)
assert np.array_equal(ct.to_words(), words)
logits = H.CipherTensor.from_words(ctx, Wk.random_ciphertexts(p, 10, seed=3, level=2), 2.0 ** 40)
lw = logits.to_words()
gd_ms, _ = best(lambda: H.decrypt_tensor(ctx, sk, logits, 4096), 5)
rd_ms, _ = best(lambda: ref.decrypt_tensor(keys, lw, 2.0 ** 40, 0, 4096), 3)
print(f"encrypt_tensor 4096 x 784 (c2 batch): GPU {g_ms:.1f} ms, reference CPU ({os.cpu_count()} threads) "
      f"{r_ms:.1f} ms, {r_ms / g_ms:.1f}x; bit-exact")
print(f"decrypt_tensor 10 logits x 4096: GPU {gd_ms:.2f} ms, reference CPU (1 thread, its decrypt_tensor is serial) "
      f"{rd_ms:.1f} ms, {rd_ms / gd_ms:.1f}x")
