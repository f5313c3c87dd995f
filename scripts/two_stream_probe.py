# SPDX-License-Identifier: Apache-2.0
"""Throughput of the c2 step with one batch in flight (one context / stream) against two
independent batches in flight (two contexts on the same GPU, steps issued alternately)."""
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

lanes = []
for i in range(int(os.environ.get("LANES", "2"))):
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
    rk = H.RelinKey(ctx, kw)
    plan = H.RescalePlan.plan(ctx, model)
    inp = H.CipherTensor.from_words(ctx, words, p["scale"], shape=wl.input_shape)
    lanes.append((ctx, rk, plan, inp))


def run(n, nl):
    outs = []
    for i in range(n):
        ctx, rk, plan, inp = lanes[i % nl]
        outs.append(H.execute(ctx, model, plan, inp, rk))
        if len(outs) > 2 * nl:
            outs.pop(0)
    return outs


for nl in range(1, len(lanes) + 1):
    run(6, nl)
    torch.cuda.synchronize()
    K = 40
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run(K, nl)
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) * 1e3 / K)
    print(f"lanes {nl}: {best:.3f} ms per step, {4096 / best * 1e3:.0f} images/s")
