# SPDX-License-Identifier: Apache-2.0
"""ncu target: one c5b wide dense layer (4096 -> 4096 at N=16384, + rescale) on device inputs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1908_04172_b200 import henet as H, workloads as Wk
from paper_1908_04172_b200.sharded import OutputShardedDense

K = M = int(os.environ.get("C5B_K", "4096"))
p = Wk.N16384
ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
L = len(p["chain"])
layer = OutputShardedDense(ctx, Wk.wide_dense_weights(k=K, m=M), 0, 1)
x = H.CipherTensor(ctx, K, 2, L, p["scale"], shape=[K])
ctx.synchronize()
xv = x.torch_view(0).view(K, 2, L, p["n"])
for i, q in enumerate(p["chain"]):
    xv[:, :, i, :] = torch.randint(0, q, (K, 2, p["n"]), device="cuda:0", dtype=torch.int64)
torch.cuda.synchronize()
out = layer.forward(x)
ctx.synchronize()
print("ok", out.count, out.level)
