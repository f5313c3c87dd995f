# SPDX-License-Identifier: Apache-2.0
"""Per-kernel time of one c3 execution (CryptoNets-ReLU, complex packing, 8192 images) with
both ReLU refreshes on the GPU engine (library profiler, serialised launches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
from paper_1908_04172_b200 import henet as H, workloads as Wk

p = Wk.N8192
ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
wl = Wk.cryptonets_relu()
model = H.PlainModel.load(wl.manifest, wl.blob)
plan = H.RescalePlan.plan(ctx, model)
L = len(p["chain"])
rng = np.random.default_rng(1)
s = rng.integers(-1, 2, p["n"])
w = np.zeros((1, 2, L, p["n"]), dtype=np.uint64)
for i, q in enumerate(p["chain"]):
    w[0, 0, i] = np.where(s < 0, q - 1, s).astype(np.uint64)
t = H.CipherTensor.from_words(ctx, w, 1.0)
H.ntt_forward(ctx, t)
skw = np.zeros((L + 1, p["n"]), dtype=np.uint64)
skw[:L] = t.to_words()[0, 0]
sk = H.SecretKey(ctx, skw)
imgs = Wk.synthetic_images(wl.input_shape, wl.batch, 8)
x = H.encrypt_tensor(ctx, sk, imgs, 9, packing=1, shape=wl.input_shape)
eng = H.RefreshEngine(ctx, sk, 99)
for _ in range(2):
    H.execute(ctx, model, plan, x, None, eng)
ctx.synchronize()
H.prof_enable(True)
H.execute(ctx, model, plan, x, None, eng)
ctx.synchronize()
H.prof_enable(False)
rep = H.prof_report()
tot = sum(v["ms"] for v in rep.values())
for k, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"]):
    print(f"{k:28s} {v['ms']:8.3f} ms  {v['launches']:5d} launches  {v['ms'] / tot:.3f}")
print(f"total kernel ms {tot:.3f}")
