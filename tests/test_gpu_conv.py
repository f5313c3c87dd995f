# SPDX-License-Identifier: Apache-2.0
"""Convolution (k_mac_conv) vs the C restatement of eval_convolution
(henet/graph.hpp:956-993) over geometries beyond the c2 layer: 9, 25, 75 and 200 taps per
window, F = 1, 3, 5, 6, 8 filters, padding on every side, strides 1-3, ragged sizes,
bias on poly 0, and all-(q-1) inputs (largest accumulator sums)."""
import numpy as np
import pytest

from paper_1908_04172_b200 import henet as H
from paper_1908_04172_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    from oracle import cbind as O
    p = W.N8192
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
    oc = O.OracleContext(p["n"], p["chain"], p["special"], p["scale"])
    return {"ctx": ctx, "oc": oc, "p": p}


def _run(ctx, x, shape, w, b, stride, pad, scale):
    F, C, win, _ = w.shape
    m = H.PlainModel()
    m.add_weight("w", list(w.shape), w)
    if b is not None:
        m.add_weight("b", [F], b)
    m.add_node("input", "Input", [], {"shape": list(shape)})
    m.add_node("conv", "Convolution", ["input"], {"stride": stride, "window": win, "filters": F, "pad": list(pad)},
               "w", "b" if b is not None else "")
    m.add_node("out", "Output", ["conv"])
    m.finalize()
    L = x.shape[2]
    plan = H.RescalePlan.from_nodes(0, 0, {"input": (0, L, L, scale), "conv": (0, L, L, scale * scale),
                                           "out": (0, L, L, scale * scale)})
    return H.execute(ctx, m, plan, H.CipherTensor.from_words(ctx, x, scale, shape=list(shape))).to_words()


CASES = [
    # (C, IH, IW, F, win, stride, pad (top, left, bottom, right), level, bias, edge)
    (1, 28, 28, 5, 5, 2, (0, 0, 1, 1), 6, False, False),   # c2 conv1
    (1, 9, 9, 1, 3, 1, (1, 1, 1, 1), 6, True, False),      # F = 1, pad all round
    (3, 8, 8, 8, 5, 1, (2, 2, 2, 2), 6, True, False),      # 75 taps: 3 k steps, N = 32 on every limb
    (8, 6, 7, 3, 5, 3, (0, 2, 1, 0), 6, False, False),     # 200 taps: 7 k steps, stride 3, ragged
    (2, 5, 5, 6, 3, 2, (1, 0, 0, 1), 6, True, True),       # all (q-1) residues
    # 1x1, stride 1, unpadded: the batched tensor-core Dot (positions as columns)
    (16, 5, 6, 24, 1, 1, (0, 0, 0, 0), 6, True, False),    # MobileNetV2 project-like, ragged 5x6
    (40, 3, 4, 130, 1, 1, (0, 0, 0, 0), 6, True, True),    # 2 k steps, 2 M tiles, all (q-1)
    (4, 6, 6, 3, 1, 2, (0, 0, 0, 0), 6, False, False),     # 1x1 stride 2: tap-gather kernel
    # single channel, 5x5, stride 2 (the CryptoNets first-layer family): padding on every side, ragged outputs
    (1, 28, 28, 5, 5, 2, (1, 1, 0, 0), 6, True, True),     # c2 conv1 padded top-left, bias, all (q-1)
    (1, 12, 11, 8, 5, 2, (2, 1, 1, 2), 6, True, False),    # F = 8, 6 x 5 outputs
    (1, 7, 9, 3, 5, 2, (0, 0, 0, 0), 6, False, False),     # 2 x 3 outputs
    (1, 5, 5, 1, 5, 2, (0, 0, 0, 0), 6, True, False),      # one output position, F = 1
    (1, 9, 10, 2, 5, 2, (2, 2, 2, 2), 6, True, True),      # 5 x 5 outputs, padding all round, all (q-1)
    (1, 10, 9, 7, 5, 2, (0, 1, 1, 0), 6, False, False),    # F = 7
]


def test_depthwise_conv_vs_oracle(env):
    """Block-diagonal weights (a depthwise layer as the reference sees it): the
    GPU runs one 1 -> 1 convolution per channel; the result is the full convolution's."""
    p, oc = env["p"], env["oc"]
    C, IH, IW, win = 6, 7, 7, 3
    rng = np.random.default_rng(31)
    w = np.zeros((C, C, win, win), np.float32)
    for c in range(C):
        w[c, c] = rng.normal(0, 0.1, (win, win))
    b = rng.normal(0, 0.01, C).astype(np.float32)
    x = W.random_ciphertexts(p, C * IH * IW, seed=32)
    got = _run(env["ctx"], x, (C, IH, IW), w, b, 1, (1, 1, 1, 1), p["scale"])
    sel = [0, 6, 24, 48, 49, 100, 150, 293, 294 - 1]
    want = oc.conv(x, w, (C, IH, IW), 1, (1, 1, 1, 1), 6, p["scale"], bias=b, rescale=False, outputs=sel)
    for k, e in enumerate(sel):
        assert np.array_equal(got[e], want[k]), e


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"C{c[0]}_{c[1]}x{c[2]}_F{c[3]}_w{c[4]}_s{c[5]}_L{c[7]}")
def test_conv_vs_oracle_geometries(env, case):
    C, IH, IW, F, win, stride, pad, level, bias, edge = case
    p, oc = env["p"], env["oc"]
    rng = np.random.default_rng(C * 1000 + IH * 10 + F)
    w = rng.normal(0, 0.05, (F, C, win, win)).astype(np.float32)
    b = rng.normal(0, 0.01, F).astype(np.float32) if bias else None
    count = C * IH * IW
    if edge:
        q = np.array(p["chain"][:level], dtype=np.uint64)[None, None, :, None]
        x = np.broadcast_to(q - 1, (count, 2, level, p["n"])).copy()
    else:
        x = W.random_ciphertexts(p, count, seed=17 + F, level=level)
    got = _run(env["ctx"], x, (C, IH, IW), w, b, stride, pad, p["scale"])
    OH = (IH + pad[0] + pad[2] - win) // stride + 1
    OW = (IW + pad[1] + pad[3] - win) // stride + 1
    n_out = F * OH * OW
    sel = sorted(set([0, n_out - 1, OW - 1, (OH - 1) * OW, n_out // 2] + list(range(0, n_out, max(1, n_out // 7)))))
    want = oc.conv(x, w, (C, IH, IW), stride, pad, level, p["scale"], bias=b, rescale=False, outputs=sel)
    for k, e in enumerate(sel):
        assert np.array_equal(got[e], want[k]), e
