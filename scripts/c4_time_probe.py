import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import bench
from paper_1908_04172_b200 import henet as H, workloads as Wk
p = Wk.N16384
ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
sk = bench.c4_secret_key(H, ctx, p, 5)
eng = H.RefreshEngine(ctx, sk, 77); eng.set_relu_clip(6.0)
for n in (960, 9600):
    acts = np.random.default_rng(6).normal(0, 1, (ctx.slot_count(), n))
    t0 = time.perf_counter(); x = H.encrypt_tensor(ctx, sk, acts, 7); ctx.synchronize(); t1 = time.perf_counter()
    print(f"encrypt {n}: {1e3*(t1-t0):.1f} ms (host-side incl. sample transposition)")
    for i in range(2):
        t0 = time.perf_counter(); y = eng.apply(1, 1, 0, x); ctx.synchronize(); t1 = time.perf_counter()
        print(f"refresh {n}: {1e3*(t1-t0):.1f} ms")
hw = 10
wl = Wk.mobilenet_block(hw=hw)
model = H.PlainModel.load(wl.manifest, wl.blob)
plan = H.RescalePlan.plan(ctx, model)
acts = np.random.default_rng(6).normal(0, 1, (ctx.slot_count(), wl.input_count))
x = H.encrypt_tensor(ctx, sk, acts, 7, shape=wl.input_shape)
for keep in (False, True):
    model.keep_encodings(keep)
    for i in range(2):
        t0 = time.perf_counter(); out = H.execute(ctx, model, plan, x, None, eng); ctx.synchronize(); t1 = time.perf_counter()
        print(f"execute keep={keep}: {1e3*(t1-t0):.1f} ms")
