# SPDX-License-Identifier: Apache-2.0
"""ncu / timing target: the c4 block's three linear layers (1x1 expand 16->96, 3x3 depthwise
pad 1, 1x1 project 96->24) on one 10x10 tile of random wide ciphertexts, ReLU6 removed, with
per-node CUDA-event times (HG_NODE_TIMING) printed once the layers have run twice."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_04172_b200 import henet as H, workloads as Wk

p = Wk.N16384
ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
wl = Wk.mobilenet_block(hw=int(os.environ.get("C4_HW", "10")))
j = json.loads(wl.manifest)
j["nodes"] = [n for n in j["nodes"] if n["op"] != "Relu"]
for n in j["nodes"]:
    n["inputs"] = [{"relu6a": "expand", "relu6b": "dw"}.get(i, i) for i in n.get("inputs", [])]
model = H.PlainModel.load(json.dumps(j), wl.blob)
plan = H.RescalePlan.plan(ctx, model)
x = H.CipherTensor.from_words(ctx, Wk.random_ciphertexts(p, wl.input_count, seed=9), p["scale"], shape=wl.input_shape)
for it in range(int(os.environ.get("NCU_STEPS", "2"))):
    st = H.ExecutionStats()
    out = H.execute(ctx, model, plan, x, None, None, stats=st)
    ctx.synchronize()
    print("c4 linear", it, [(k, round(v, 2)) for k, v in st.layer_ms])
