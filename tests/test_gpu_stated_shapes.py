# SPDX-License-Identifier: Apache-2.0
"""Residue parity at the shapes BASELINE.json states for configs 4 and 5b.

c4: the MobileNetV2 block 16 -> 96 -> 24 (1x1 expand, ReLU6, 3x3 depthwise pad 1, ReLU6,
1x1 project) on a 3x3 tile of real encryptions (every padded corner / edge / interior
window of the depthwise layer), with both client-aided ReLU6 refreshes done
  (a) by the reference's clamp provider through the GPU executor's callback, and
  (b) by the GPU refresh engine,
against the reference.

The reference side is evaluated layer by layer with the unmodified `execute()` and
NonlinearityEngine-equivalent refresh (oracle/ref/ref_capi.cpp `clip_apply`):
  expand + ReLU6a  : one execute of Input -> Convolution(1x1) -> Relu -> Output
                     (the Relu refresh is the executor's layer_seq 0),
  depthwise        : 96 executes of the single-channel 3x3 convolution (SURVEY H8 --
                     the reference has no grouped convolution; the block-diagonal graph the
                     GPU runs differs from it only by taps whose weight is 0.0, whose
                     product mul_ct_pt_scalar(x, encode_scalar(0)) is the all-zero
                     ciphertext, so the sums are identical residue for residue),
  ReLU6b           : the same refresh at layer_seq 1 (graph.hpp:819,850),
  project          : one execute of Input -> Convolution(1x1) -> Output.
The equivalence of the block-diagonal and per-channel forms is itself checked against the
reference's full block-diagonal execute at a small shape in
tests/test_gpu_wide.py::test_c4_block_relu6_provider_bit_exact.

c5b: the wide dense layer at K = 4096 inputs (N = 16384, 40-bit limb 0) with an M = 160
output slice (one full 128-row tensor-core tile plus a ragged 32-row one) through the
patched one-rescale-per-output plan: every output against the C restatement (pinned to the
reference in tests/test_oracle_golden.py), and three outputs (first, the first of the
ragged tile, last) against the reference's own execute.
"""
import json

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

from oracle import refbind as R  # noqa: E402
from paper_1908_04172_b200 import henet as H  # noqa: E402
from paper_1908_04172_b200 import workloads as W  # noqa: E402

REFRESH_SEED = 77


@pytest.fixture(scope="module")
def wenv():
    p = W.N16384
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
    ref = R.RefContext(p["n"], p["chain"], p["special"], p["scale"])
    keys = ref.keygen(43, False)
    sk = H.SecretKey(ctx, keys.sk_words())
    return dict(p=p, ctx=ctx, ref=ref, keys=keys, sk=sk)


def _conv_model(name, cin, hw, filters, window, pad, w, relu=False):
    blob = W.Blob()
    blob.add("w", list(w.shape), w)
    nodes = [W._node("input", "Input", attrs={"shape": [cin, hw, hw]}),
             W._node("conv", "Convolution", ["input"],
                     {"stride": 1, "window": window, "filters": filters, "pad": pad}, "w")]
    last = "conv"
    if relu:
        nodes.append(W._node("relu", "Relu", ["conv"]))
        last = "relu"
    nodes.append(W._node("out", "Output", [last]))
    j = {"name": name, "packing": "real", "preset": "P14", "weights": blob.table, "nodes": nodes}
    return json.dumps(j), blob.bytes()


def _weights(wl):
    j = json.loads(wl.manifest)
    blob = np.frombuffer(wl.blob, dtype="<f4")
    out = {}
    for name, e in j["weights"].items():
        cnt = int(np.prod(e["shape"]))
        out[name] = blob[e["offset"] // 4:e["offset"] // 4 + cnt].reshape(e["shape"])
    return out


def _c4_reference_layerwise(ref, keys, wl, hw, words, sc):
    """The reference's c4 block output for `words`, layer by layer (module docstring)."""
    wt = _weights(wl)
    cin, expand = wt["exp_w"].shape[1], wt["exp_w"].shape[0]
    cout = wt["proj_w"].shape[0]
    pos = hw * hw
    R.set_relu_clip(6.0)
    try:
        man, blob = _conv_model("expand", cin, hw, expand, 1, [0, 0, 0, 0], wt["exp_w"], relu=True)
        a, a_sc, st = ref.execute(keys, man, blob, words, sc, refresh_seed=REFRESH_SEED,
                                  out_capacity=expand * pos * words[0].size)
        assert st["rescale_ops"] == 0 and a.shape[0] == expand * pos
        dw = np.empty_like(a)
        dw_sc = None
        for c in range(expand):
            wc = np.ascontiguousarray(wt["dw_w"][c, c].reshape(1, 1, 3, 3))
            assert not np.any(np.delete(wt["dw_w"][c], c, axis=0)), "depthwise weights must be block diagonal"
            man, blob = _conv_model(f"dw{c}", 1, hw, 1, 3, [1, 1, 1, 1], wc)
            o, o_sc, _ = ref.execute(None, man, blob, a[c * pos:(c + 1) * pos], a_sc)
            dw[c * pos:(c + 1) * pos] = o
            assert dw_sc is None or dw_sc == o_sc
            dw_sc = o_sc
        b = ref.nonlin_apply(keys, 1, 1, 1, REFRESH_SEED, dw, dw_sc, 0)
        b_sc = ref.scale  # fresh encryptions at (L, default scale)
    finally:
        R.set_relu_clip(0.0)
    man, blob = _conv_model("project", expand, hw, cout, 1, [0, 0, 0, 0], wt["proj_w"])
    out, out_sc, _ = ref.execute(None, man, blob, b, b_sc)
    return out, out_sc


@pytest.fixture(scope="module")
def c4_case(wenv):
    ref, keys = wenv["ref"], wenv["keys"]
    hw = 3
    wl = W.mobilenet_block(hw=hw)  # the stated channel shape: 16 -> 96 -> 24
    acts = np.random.default_rng(21).normal(0, 1, (8192, wl.input_count))
    words, sc = ref.encrypt_tensor(keys, acts, 22)
    want, want_sc = _c4_reference_layerwise(ref, keys, wl, hw, words, sc)
    return dict(wl=wl, acts=acts, words=words, sc=sc, want=want, want_sc=want_sc)


def test_c4_stated_shape_reference_provider(wenv, c4_case):
    """c4 16->96->24 block, ReLU6 refreshes by the reference's clamp provider through the
    GPU executor's NonlinearityProvider callback (graph.hpp:1060-1101)."""
    ctx, ref, keys = wenv["ctx"], wenv["ref"], wenv["keys"]
    wl = c4_case["wl"]
    model = H.PlainModel.load(wl.manifest, wl.blob)
    plan = H.RescalePlan.plan(ctx, model)
    assert plan.planned_rescale_ops == 0

    def provider(kind, window, layer_seq, req):
        R.set_relu_clip(6.0)
        try:
            return ref.nonlin_apply(keys, kind, window, layer_seq, REFRESH_SEED, req.to_words(), req.scale,
                                    req.packing)
        finally:
            R.set_relu_clip(0.0)

    stats = H.ExecutionStats()
    x = H.CipherTensor.from_words(ctx, c4_case["words"], c4_case["sc"], shape=wl.input_shape)
    out = H.execute(ctx, model, plan, x, None, provider, stats)
    assert out.scale == c4_case["want_sc"]
    assert np.array_equal(out.to_words(), c4_case["want"])
    assert stats.nonlin_elements == 2 * 96 * 9


def test_c4_stated_shape_gpu_refresh_engine(wenv, c4_case):
    """Same block with the input encrypted and both ReLU6 refreshes done on the GPU
    (hg_encrypt_tensor, hg_refresh_engine_apply with the [0, 6] clamp)."""
    ctx, sk = wenv["ctx"], wenv["sk"]
    wl = c4_case["wl"]
    x = H.encrypt_tensor(ctx, sk, c4_case["acts"], 22, shape=wl.input_shape)
    assert x.scale == c4_case["sc"]
    assert np.array_equal(x.to_words(), c4_case["words"])
    model = H.PlainModel.load(wl.manifest, wl.blob)
    eng = H.RefreshEngine(ctx, sk, REFRESH_SEED)
    eng.set_relu_clip(6.0)
    out = H.execute(ctx, model, H.RescalePlan.plan(ctx, model), x, None, eng)
    assert out.scale == c4_case["want_sc"]
    assert np.array_equal(out.to_words(), c4_case["want"])
    # decrypted: the project layer of a ReLU6-clamped cleartext forward pass
    dec = H.decrypt_tensor(ctx, sk, out, 64)
    wt = _weights(wl)
    a = c4_case["acts"][:64].reshape(64, 16, 3, 3)
    e = np.clip(np.einsum("bchw,fc->bfhw", a, wt["exp_w"][:, :, 0, 0].astype(np.float64)), 0, 6)
    ep = np.pad(e, ((0, 0), (0, 0), (1, 1), (1, 1)))
    d = np.zeros_like(e)
    for ky in range(3):
        for kx in range(3):
            d += ep[:, :, ky:ky + 3, kx:kx + 3] * np.array([wt["dw_w"][c, c, ky, kx] for c in range(96)])[None, :, None, None]
    d = np.clip(d, 0, 6)
    pr = np.einsum("bchw,fc->bfhw", d, wt["proj_w"][:, :, 0, 0].astype(np.float64)).reshape(64, -1)
    assert np.max(np.abs(dec - pr)) < 1e-3


def test_c5b_stated_k4096_bit_exact(wenv):
    """c5b: dense K = 4096 -> M = 160 slice at N = 16384 (40-bit limb 0), patched
    one-rescale-per-output plan, tensor-core contraction (both the u32 30-bit-limb kernel and
    the 5-plane 40-bit kernel at 128 k-steps) and the hybrid rescale."""
    ctx, ref, p = wenv["ctx"], wenv["ref"], wenv["p"]
    from oracle import cbind as O
    K, M = 4096, 160
    wfull = W.wide_dense_weights(5, K, K)
    wslice = np.ascontiguousarray(wfull[:, :M])
    wl = _dense_workload(wslice)
    x = W.random_ciphertexts(p, K, seed=31)
    model = H.PlainModel.load(wl.manifest, wl.blob)
    rp = ref.plan(wl.manifest, wl.blob, patch=True)
    nodes = {n["id"]: (n["decision"], n["level_in"], n["level_out"],
                       np.array([n["scale_out_bits"]], dtype=np.uint64).view(np.float64)[0]) for n in rp["nodes"]}
    plan = H.RescalePlan.from_nodes(0, rp["planned_rescale_ops"], nodes)
    out = H.execute(ctx, model, plan, H.CipherTensor.from_words(ctx, x, p["scale"], shape=[K]))
    got = out.to_words()
    assert got.shape == (M, 2, 7, p["n"])
    # all 160 outputs against the C restatement (128-bit lazy sums, one rescale per output)
    oc = O.OracleContext(p["n"], p["chain"], p["special"], p["scale"])
    want = oc.dense_lazy(x, wslice, 8, rescale=True)
    assert np.array_equal(got, want)
    # three outputs against the reference's own execute (its Dot over the selected columns)
    cols = [0, 128, M - 1]
    wl3 = _dense_workload(np.ascontiguousarray(wslice[:, cols]))
    r3, r3_sc, _ = ref.execute(None, wl3.manifest, wl3.blob, x, p["scale"], patch=True)
    assert r3_sc == out.scale
    assert np.array_equal(got[cols], r3)


def _dense_workload(w):
    k, m = w.shape
    blob = W.Blob()
    blob.add("fc_w", [k, m], w)
    j = {"name": f"dense-{k}-{m}", "packing": "real", "preset": "P14", "weights": blob.table,
         "nodes": [W._node("input", "Input", attrs={"shape": [k]}),
                   W._node("fc", "Dot", ["input"], weight_ref="fc_w"),
                   W._node("out", "Output", ["fc"])]}
    return W.Workload(f"dense_{k}_{m}", json.dumps(j), blob.bytes(), [k], 0, 8192, patch_terminal_rescale=True)
