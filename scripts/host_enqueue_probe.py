import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1908_04172_b200 import henet as H, workloads as Wk
p = Wk.N8192; wl = Wk.cryptonets(); L = len(p["chain"])
rng = np.random.default_rng(100)
kw = np.empty((L, 2, L + 1, p["n"]), dtype=np.uint64)
for t, q in enumerate(p["chain"] + [p["special"]]):
    kw[:, :, t, :] = rng.integers(0, q, size=(L, 2, p["n"]), dtype=np.uint64)
model = H.PlainModel.load(wl.manifest, wl.blob)
words = Wk.random_ciphertexts(p, wl.input_count, seed=7)
ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
rk = H.RelinKey(ctx, kw); plan = H.RescalePlan.plan(ctx, model)
inp = H.CipherTensor.from_words(ctx, words, p["scale"], shape=wl.input_shape)
for _ in range(5): out = H.execute(ctx, model, plan, inp, rk)
torch.cuda.synchronize()
# host time of an execute call when the GPU queue is empty vs. device time
hs = []
for _ in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); out = H.execute(ctx, model, plan, inp, rk); t1 = time.perf_counter()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    hs.append(((t1 - t0) * 1e3, (t2 - t0) * 1e3))
hs = np.array(hs)
print("execute() host call ms: median %.3f min %.3f max %.3f; call+sync ms: median %.3f" % (np.median(hs[:,0]), hs[:,0].min(), hs[:,0].max(), np.median(hs[:,1])))
# back-to-back: host time of 50 calls without sync
torch.cuda.synchronize(); t0 = time.perf_counter()
outs=[]
for _ in range(50):
    outs.append(H.execute(ctx, model, plan, inp, rk)); outs=outs[-2:]
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print("50 back-to-back: host enqueue %.3f ms/step, total %.3f ms/step" % ((t1-t0)*20, (t2-t0)*20))
