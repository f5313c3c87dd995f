# SPDX-License-Identifier: Apache-2.0
"""Where the time of one c4-sized refresh (9600 ciphertexts, N = 16384) goes: host wall clock,
device span (events on the context stream) and the sum of kernel times (library profiler)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_1908_04172_b200 import henet as H, workloads as Wk

p = Wk.N16384
ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
sk = bench.c4_secret_key(H, ctx, p, 5)
eng = H.RefreshEngine(ctx, sk, 77)
eng.set_relu_clip(6.0)
ext = torch.cuda.ExternalStream(ctx.stream())
n = int(os.environ.get("N_CT", "9600"))
acts = np.random.default_rng(6).normal(0, 1, (ctx.slot_count(), n))
x = H.encrypt_tensor(ctx, sk, acts, 7)
ctx.synchronize()
for i in range(4):
    prof = i == 3
    if prof:
        H.prof_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    t0 = time.perf_counter()
    y = eng.apply(1, 1, i, x)
    e1.record(ext)
    ctx.synchronize()
    t1 = time.perf_counter()
    if prof:
        H.prof_enable(False)
        rep = H.prof_report()
        ks = sum(v["ms"] for v in rep.values())
        print(f"kernel sum {ks:.1f} ms: " + ", ".join(f"{k} {v['ms']:.1f}" for k, v in sorted(rep.items(), key=lambda kv: -kv[1]['ms'])))
    print(f"refresh {n}: wall {1e3 * (t1 - t0):.1f} ms, device span {e0.elapsed_time(e1):.1f} ms")
    del y
