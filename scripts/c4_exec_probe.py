# SPDX-License-Identifier: Apache-2.0
"""c4 tile executes back to back: device span per execute, and (odd iterations) the kernel-time sum."""
import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
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
eng = H.RefreshEngine(ctx, sk, 77); eng.set_relu_clip(6.0)
ext = torch.cuda.ExternalStream(ctx.stream())
out = None
for i in range(int(os.environ.get('ITERS', '8'))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof = i % 2 == 1
    H.prof_enable(prof)
    e0.record(ext); t0 = time.perf_counter()
    out = H.execute(ctx, model, plan, x, None, eng)
    e1.record(ext); e1.synchronize(); t1 = time.perf_counter()
    H.prof_enable(False)
    ks = ""
    if prof:
        rep = H.prof_report()
        ks = f" kernel sum {sum(v['ms'] for v in rep.values()):.1f} ms (" + ", ".join(f"{k} {v['ms']:.0f}" for k, v in sorted(rep.items(), key=lambda kv: -kv[1]['ms'])[:4]) + ")"
    nm = ""
    if os.environ.get("HG_NODE_TIMING"):
        import ctypes
        from paper_1908_04172_b200._lib import lib
        arr = (ctypes.c_double * 11)()
        lib.hg_last_exec_node_ms(ctx.handle, arr)
        nm = " nodes: conv %.0f relu %.0f" % (arr[6], arr[8])
    print(f"execute {i}: device {e0.elapsed_time(e1):.1f} ms wall {1e3*(t1-t0):.1f} ms{ks}{nm}")
