# SPDX-License-Identifier: Apache-2.0
"""Stress of the two-lane schedule: groups of 10 c2 steps alternating over LANES contexts,
timed group by group; prints the distribution (looks for stalls from TMEM / memory-pool
contention between the lanes' kernels)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1908_04172_b200 import henet as H, workloads as Wk

p = Wk.N8192
wl = Wk.cryptonets()
L = len(p["chain"])
rng = np.random.default_rng(100)
kw = np.empty((L, 2, L + 1, p["n"]), dtype=np.uint64)
for t, q in enumerate(p["chain"] + [p["special"]]):
    kw[:, :, t, :] = rng.integers(0, q, size=(L, 2, p["n"]), dtype=np.uint64)
model = H.PlainModel.load(wl.manifest, wl.blob)
words = Wk.random_ciphertexts(p, wl.input_count, seed=7)
nl = int(os.environ.get("LANES", "2"))
lanes = []
for i in range(nl):
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
    lanes.append((ctx, H.RelinKey(ctx, kw), H.RescalePlan.plan(ctx, model),
                  H.CipherTensor.from_words(ctx, words, p["scale"], shape=wl.input_shape)))
groups = int(os.environ.get("GROUPS", "60"))
ms = []
outs = []
for g in range(groups + 2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(10):
        ctx, rk, plan, inp = lanes[i % nl]
        outs.append(H.execute(ctx, model, plan, inp, rk))
        if len(outs) > 2 * nl:
            outs.pop(0)
    torch.cuda.synchronize()
    if g >= 2:
        ms.append((time.perf_counter() - t0) * 100)
ms = np.array(ms)
print(f"lanes {nl}: {groups} groups of 10 steps: ms/step min {ms.min():.3f} median {np.median(ms):.3f} "
      f"p95 {np.percentile(ms, 95):.3f} max {ms.max():.3f}; groups over 1.2x median: {(ms > 1.2 * np.median(ms)).sum()}")
