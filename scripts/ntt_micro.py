# SPDX-License-Identifier: Apache-2.0
"""Micro-benchmark of the batched NTT kernels (k_ntt) at N=8192: CUDA-event time per
transform for a batch of 8450 limbs (845 ciphertexts x 2 polys x 5 limbs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1908_04172_b200 import henet as H, workloads as Wk

p = Wk.N8192
ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
x = Wk.random_ciphertexts(p, 845, seed=1, level=5)
t = H.CipherTensor.from_words(ctx, x, 1.0)
s = torch.cuda.ExternalStream(ctx.stream())
reps = int(os.environ.get("REPS", "5"))
for inv in (False, True):
    f = H.ntt_inverse if inv else H.ntt_forward
    f(ctx, t); ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        f(ctx, t)
    e1.record(s); e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    rows = 845 * 2 * 5
    bf = rows * 4096 * 13
    print(f"{'inv' if inv else 'fwd'}: {ms:.3f} ms for {rows} transforms = {ms * 1e3 / rows * 148:.2f} us/transform/SM, "
          f"{bf * 3 / (ms * 1e-3) / 1e12:.2f} Tops (3/butterfly), {rows * 8192 * 8 / (ms * 1e-3) / 1e9:.0f} GB/s")
