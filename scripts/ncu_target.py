# SPDX-License-Identifier: Apache-2.0
"""Small ncu target: two executions of the c2 CryptoNets-shaped network (4096
images) through hg_execute, with the same inputs/parameters as bench.py."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1908_04172_b200 import henet as H, workloads as Wk

p = Wk.N8192
wl = Wk.cryptonets()
ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
L = len(p["chain"])
rng = np.random.default_rng(100)
kw = np.empty((L, 2, L + 1, p["n"]), dtype=np.uint64)
for t, q in enumerate(p["chain"] + [p["special"]]):
    kw[:, :, t, :] = rng.integers(0, q, size=(L, 2, p["n"]), dtype=np.uint64)
rk = H.RelinKey(ctx, kw)
model = H.PlainModel.load(wl.manifest, wl.blob)
plan = H.RescalePlan.plan(ctx, model)
inp = H.CipherTensor.from_words(ctx, Wk.random_ciphertexts(p, wl.input_count, seed=7), p["scale"], shape=wl.input_shape)
for _ in range(int(os.environ.get("NCU_STEPS", "2"))):
    out = H.execute(ctx, model, plan, inp, rk)
ctx.synchronize()
print("ok", out.level, out.count)
