# SPDX-License-Identifier: Apache-2.0
"""Per-kernel time of one c4 tile (bench.py --workload c4) with the library profiler."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
from paper_1908_04172_b200 import henet as H, workloads as Wk

p = Wk.N16384
ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
hw = bench.C4_TILE + 2
wl = Wk.mobilenet_block(hw=hw)
model = H.PlainModel.load(wl.manifest, wl.blob)
plan = H.RescalePlan.plan(ctx, model)
sk = bench.c4_secret_key(H, ctx, p, 5)
acts = np.random.default_rng(6).normal(0, 1, (ctx.slot_count(), wl.input_count))
x = H.encrypt_tensor(ctx, sk, acts, 7, shape=wl.input_shape)
eng = H.RefreshEngine(ctx, sk, 77)
eng.set_relu_clip(6.0)
H.execute(ctx, model, plan, x, None, eng)
ctx.synchronize()
H.prof_enable(True)
H.execute(ctx, model, plan, x, None, eng)
ctx.synchronize()
H.prof_enable(False)
rep = H.prof_report()
tot = sum(v["ms"] for v in rep.values())
for k, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"]):
    print(f"{k:28s} {v['ms']:9.2f} ms  {v['launches']:6d} launches  {v['ms'] / tot:.3f}")
print(f"total kernel ms {tot:.1f}")
