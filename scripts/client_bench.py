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

# c3: CryptoNets-ReLU under complex packing (8192 images), client-aided ReLU refreshes --
# GPU engine as the provider vs the reference's execute with its LocalProvider (host threads)
wl = Wk.cryptonets_relu()
imgs3 = Wk.synthetic_images(wl.input_shape, wl.batch, 8)
words3, sc3 = ref.encrypt_tensor(keys, imgs3, 9, packing=1)
model = H.PlainModel.load(wl.manifest, wl.blob)
plan = H.RescalePlan.plan(ctx, model)
inp = H.CipherTensor.from_words(ctx, words3, sc3, packing=1, shape=wl.input_shape)
eng = H.RefreshEngine(ctx, sk, 99)
H.execute(ctx, model, plan, inp, None, eng)
g3_ms, out3 = best(lambda: H.execute(ctx, model, plan, inp, None, eng), 3)
r3_ms, (want3, _, _) = best(lambda: ref.execute(keys, wl.manifest, wl.blob, words3, sc3, refresh_seed=99), 1)
assert np.array_equal(out3.to_words(), want3)
print(f"c3 execute with client-aided ReLU refreshes (8192 images): GPU {g3_ms:.1f} ms "
      f"({8192 / g3_ms * 1e3:.0f} img/s), reference CPU ({os.cpu_count()} threads) {r3_ms:.0f} ms "
      f"({8192 / r3_ms * 1e3:.0f} img/s), {r3_ms / g3_ms:.0f}x; bit-exact")
