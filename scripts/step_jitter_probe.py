# SPDX-License-Identifier: Apache-2.0
"""Per-step device times of the c2 step (CUDA events on the context stream after every
execute) over many steps: looks for rare long steps."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
stream = torch.cuda.ExternalStream(ctx.stream())
for _ in range(5): out = H.execute(ctx, model, plan, inp, rk)
torch.cuda.synchronize()
N = int(os.environ.get("STEPS", "600"))
sync_every = int(os.environ.get("SYNC_EVERY", "0"))
evs = [torch.cuda.Event(enable_timing=True) for _ in range(N + 1)]
host = []
evs[0].record(stream)
outs = []
for i in range(N):
    t0 = time.perf_counter()
    outs.append(H.execute(ctx, model, plan, inp, rk)); outs = outs[-2:]
    evs[i + 1].record(stream)
    host.append((time.perf_counter() - t0) * 1e3)
    if sync_every and (i + 1) % sync_every == 0:
        torch.cuda.synchronize()
torch.cuda.synchronize()
d = np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(N)])
host = np.array(host)
med = np.median(d)
bad = np.where(d > 1.3 * med)[0]
print(f"steps {N} sync_every {sync_every}: device ms median {med:.3f} min {d.min():.3f} max {d.max():.3f}; long steps (>1.3x): {len(bad)}")
for i in bad[:12]:
    print(f"  step {i}: device {d[i]:.3f} ms, host call {host[i]:.3f} ms")
