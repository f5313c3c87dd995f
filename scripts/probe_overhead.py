import sys, time, subprocess, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1908_04172_b200 import henet as H, workloads as Wk
p = Wk.N8192; wl = Wk.cryptonets()
ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
L = 6; rng = np.random.default_rng(1)
kw = np.empty((L, 2, L + 1, p["n"]), dtype=np.uint64)
for t, q in enumerate(p["chain"] + [p["special"]]):
    kw[:, :, t, :] = rng.integers(0, q, size=(L, 2, p["n"]), dtype=np.uint64)
rk = H.RelinKey(ctx, kw)
model = H.PlainModel.load(wl.manifest, wl.blob); plan = H.RescalePlan.plan(ctx, model)
inp = H.CipherTensor.from_words(ctx, Wk.random_ciphertexts(p, 784, 7), p["scale"], shape=wl.input_shape)
for _ in range(3): out = H.execute(ctx, model, plan, inp, rk)
ctx.synchronize()
def timed(n, label):
    t0 = time.perf_counter(); hs=[]
    for _ in range(n):
        a = time.perf_counter(); out = H.execute(ctx, model, plan, inp, rk); hs.append((time.perf_counter()-a)*1e3)
    ctx.synchronize(); t = (time.perf_counter()-t0)*1e3/n
    print(label, "ms/step", round(t,3), "host ms per call", [round(x,2) for x in hs[:5]], flush=True)
timed(10, "plain")
pr = subprocess.Popen(["nvidia-smi","--query-gpu=clocks.sm","--format=csv","-lms","200"], stdout=subprocess.DEVNULL)
timed(10, "with nvidia-smi starting")
time.sleep(2)
timed(10, "with nvidia-smi running")
pr.terminate()
timed(20, "plain again")
H.prof_enable(True); timed(2, "prof"); H.prof_enable(False); print(H.prof_report())
