# SPDX-License-Identifier: Apache-2.0
"""Lazy vs naive rescaling on the GPU path (the paper's Table 4 comparison): the c1 dense
layer 845 -> 100 (+ bias, terminal rescale) and the c2 CryptoNets-shaped network, each run
under both RescalePlan modes on the same device-resident input; ms per execute (CUDA
events, median of 5) and the executed rescale count."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1908_04172_b200 import henet as H, workloads as Wk

p = Wk.N8192
ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
L = len(p["chain"])
rng = np.random.default_rng(100)
kw = np.empty((L, 2, L + 1, p["n"]), dtype=np.uint64)
for t, q in enumerate(p["chain"] + [p["special"]]):
    kw[:, :, t, :] = rng.integers(0, q, size=(L, 2, p["n"]), dtype=np.uint64)
rk = H.RelinKey(ctx, kw)
for wl in (Wk.dense_layer(), Wk.cryptonets()):
    model = H.PlainModel.load(wl.manifest, wl.blob)
    inp = H.CipherTensor.from_words(ctx, Wk.random_ciphertexts(p, wl.input_count, seed=7), p["scale"],
                                    shape=wl.input_shape)
    res = {}
    for mode, name in ((H.RESCALE_LAZY, "lazy"), (H.RESCALE_NAIVE, "naive")):
        plan = H.RescalePlan.plan(ctx, model, mode)
        if wl.patch_terminal_rescale:  # c1: the terminal Dot rescales
            nodes = {}
            for nid in ("input", "fc", "out"):
                dec, lin, lout, sc = plan.node(nid)
                nodes[nid] = (dec, lin, lout, sc)
            dec, lin, lout, sc = nodes["fc"]
            q = p["chain"][lin - 1]
            s_fc = (p["scale"] * p["scale"]) / q
            nodes["fc"] = (1, lin, lin - 1, s_fc)
            nodes["out"] = (0, lin - 1, lin - 1, s_fc)
            plan = H.RescalePlan.from_nodes(mode, 100 if mode == H.RESCALE_LAZY else 84500, nodes)
        ms = []
        for i in range(6):
            st = H.ExecutionStats()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ctx.synchronize()
            e0.record()
            out = H.execute(ctx, model, plan, inp, rk, None, st)
            ctx.synchronize()
            e1.record()
            e1.synchronize()
            if i:
                ms.append(e0.elapsed_time(e1))
        res[name] = (float(np.median(ms)), st.rescale_ops, out.to_words())
    same_level = res["lazy"][2].shape == res["naive"][2].shape
    print(f"{wl.name}: lazy {res['lazy'][0]:.2f} ms ({res['lazy'][1]} rescales), naive {res['naive'][0]:.2f} ms "
          f"({res['naive'][1]} rescales), naive/lazy {res['naive'][0] / res['lazy'][0]:.1f}x, "
          f"output levels equal: {same_level}")
