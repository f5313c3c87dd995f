# SPDX-License-Identifier: Apache-2.0
"""GPU parity against the C restatement oracle (oracle/henet_oracle.c, itself
pinned to the reference by tests/test_oracle_golden.py).  This suite needs only
sources in this repository, so it runs even where oracle/_ref is absent."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import cbind as O  # noqa: E402
from paper_1908_04172_b200 import henet as H  # noqa: E402
from paper_1908_04172_b200 import workloads as W  # noqa: E402


@pytest.fixture(scope="module")
def env():
    p = W.N8192
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
    oc = O.OracleContext(p["n"], p["chain"], p["special"], p["scale"])
    sk, rk_words = oc.keygen(31)
    return dict(p=p, ctx=ctx, oc=oc, sk=sk, rk_words=rk_words, rk=H.RelinKey(ctx, rk_words))


def test_ntt_every_prime(env):
    ctx, oc, p = env["ctx"], env["oc"], env["p"]
    x = W.random_ciphertexts(p, 1, seed=3)
    t = H.CipherTensor.from_words(ctx, x, 1.0)
    H.ntt_inverse(ctx, t)
    got = t.to_words()
    for k in range(2):
        for i in range(6):
            assert np.array_equal(got[0, k, i], oc.ntt(i, x[0, k, i], inverse=True))


@pytest.mark.parametrize("level", [6, 4, 2])
def test_rescale_levels(env, level):
    ctx, oc, p = env["ctx"], env["oc"], env["p"]
    x = W.random_ciphertexts(p, 2, seed=level, level=level)
    got = H.rescale_next(ctx, H.CipherTensor.from_words(ctx, x, 2.0 ** 40)).to_words()
    assert np.array_equal(got, oc.rescale(x, level - 1))


@pytest.mark.parametrize("level", [6, 5, 2])
def test_relin_levels(env, level):
    ctx, oc, p = env["ctx"], env["oc"], env["p"]
    x = W.random_ciphertexts(p, 2, seed=40 + level, level=level)
    t = H.CipherTensor.from_words(ctx, x, p["scale"])
    want = oc.relinearize(oc.square(x), env["rk_words"])
    assert np.array_equal(H.square_relin(ctx, t, env["rk"]).to_words(), want)
    y = W.random_ciphertexts(p, 2, seed=50 + level, level=level)
    ty = H.CipherTensor.from_words(ctx, y, p["scale"])
    prod = H.mul_ct_ct(ctx, t, ty)
    assert np.array_equal(prod.to_words(), oc.mul_ct_ct(x, y))
    assert np.array_equal(H.relinearize(ctx, prod, env["rk"]).to_words(), oc.relinearize(oc.mul_ct_ct(x, y),
                                                                                         env["rk_words"]))


def test_edge_values(env):
    """All-zero and all-(q-1) ciphertexts: extreme residues through every kernel."""
    ctx, oc, p = env["ctx"], env["oc"], env["p"]
    q = np.array(p["chain"], dtype=np.uint64)[None, None, :, None]
    for x in (np.zeros((2, 2, 6, p["n"]), np.uint64), np.broadcast_to(q - 1, (2, 2, 6, p["n"])).copy()):
        t = H.CipherTensor.from_words(ctx, x, p["scale"])
        assert np.array_equal(H.rescale_next(ctx, t).to_words(), oc.rescale(x, 5))
        x5 = x[:, :, :5]
        t5 = H.CipherTensor.from_words(ctx, x5, p["scale"])
        want = oc.rescale(oc.relinearize(oc.square(x5), env["rk_words"]), 4)
        assert np.array_equal(H.square_relin(ctx, t5, env["rk"], rescale=True).to_words(), want)


def test_upload_rejects_out_of_range(env):
    ctx, p = env["ctx"], env["p"]
    x = W.random_ciphertexts(p, 1, seed=9)
    x[0, 1, 3, 17] = p["chain"][3]
    with pytest.raises(H.ValidationError, match="residue out of range"):
        H.CipherTensor.from_words(ctx, x, 1.0)


def test_op_errors_mirror_reference(env):
    ctx, p = env["ctx"], env["p"]
    a = H.CipherTensor.from_words(ctx, W.random_ciphertexts(p, 1, seed=1, level=1), 1.0)
    with pytest.raises(H.ValidationError, match="cannot rescale below level 1"):
        H.rescale_next(ctx, a)
    b = H.CipherTensor.from_words(ctx, W.random_ciphertexts(p, 1, seed=2), 1.0)
    c = H.CipherTensor.from_words(ctx, W.random_ciphertexts(p, 1, seed=3), 2.0)
    with pytest.raises(H.ValidationError, match="scale mismatch"):
        H.add_ct_ct(ctx, b, c)
    with pytest.raises(H.ValidationError, match="relinearize expects a size-3"):
        H.relinearize(ctx, b, env["rk"])
    cx = H.CipherTensor.from_words(ctx, W.random_ciphertexts(p, 1, seed=4), 1.0, packing=H.PACKING_COMPLEX)
    with pytest.raises(H.ValidationError, match="undefined under complex packing"):
        H.square(ctx, cx)


def test_dense_and_conv_layers_vs_oracle(env):
    """Dot (with bias) and Convolution through hg_execute vs the oracle's mac_output."""
    ctx, oc, p = env["ctx"], env["oc"], env["p"]
    wl = W.dense_layer()
    m = H.PlainModel.load(wl.manifest, wl.blob)
    import json
    man = json.loads(wl.manifest)
    blob = np.frombuffer(wl.blob, dtype="<f4")
    wm = man["weights"]
    w = blob[wm["fc_w"]["offset"] // 4:][:845 * 100].reshape(845, 100)
    b = blob[wm["fc_b"]["offset"] // 4:][:100]
    x = W.random_ciphertexts(p, 845, seed=12)
    plan = H.RescalePlan.from_nodes(0, 100, {"input": (0, 6, 6, p["scale"]),
                                             "fc": (1, 6, 5, p["scale"] ** 2 / p["chain"][5]),
                                             "out": (0, 5, 5, p["scale"] ** 2 / p["chain"][5])})
    out = H.execute(ctx, m, plan, H.CipherTensor.from_words(ctx, x, p["scale"], shape=[845])).to_words()
    sel = [0, 41, 99]
    want = oc.dense(x, w, 6, p["scale"], bias=b, rescale=True, outputs=sel)
    for k, j in enumerate(sel):
        assert np.array_equal(out[j], want[k]), j

    wl = W.cryptonets()
    man = json.loads(wl.manifest)
    blob = np.frombuffer(wl.blob, dtype="<f4")
    cw = blob[man["weights"]["conv1_w"]["offset"] // 4:][:125].reshape(5, 1, 5, 5)
    x = W.random_ciphertexts(p, 784, seed=13)
    mm = H.PlainModel()
    mm.add_weight("w", [5, 1, 5, 5], cw)
    mm.add_node("input", "Input", [], {"shape": [1, 28, 28]})
    mm.add_node("conv", "Convolution", ["input"], {"stride": 2, "window": 5, "filters": 5, "pad": [0, 0, 1, 1]}, "w")
    mm.add_node("out", "Output", ["conv"])
    mm.finalize()
    plan = H.RescalePlan.plan_params(p["chain"], p["scale"], mm)  # terminal conv: Skip (no rescale)
    out = H.execute(ctx, mm, plan, H.CipherTensor.from_words(ctx, x, p["scale"], shape=[1, 28, 28])).to_words()
    sel = [0, 12, 168, 169, 500, 844]  # corners (padding) and interior
    want = oc.conv(x, cw, (1, 28, 28), 2, (0, 0, 1, 1), 6, p["scale"], rescale=False, outputs=sel)
    for k, e in enumerate(sel):
        assert np.array_equal(out[e], want[k]), e


def test_toy_network_decrypts(env):
    """End-to-end on real encryptions from the oracle: decrypted logits vs a cleartext forward."""
    ctx, oc, p = env["ctx"], env["oc"], env["p"]
    wl = W.toy_cryptonets()
    imgs = W.synthetic_images(wl.input_shape, wl.batch, 5)
    ct = oc.encrypt_tensor(env["sk"], imgs, 9)
    m = H.PlainModel.load(wl.manifest, wl.blob)
    plan = H.RescalePlan.plan(ctx, m)
    out = H.execute(ctx, m, plan, H.CipherTensor.from_words(ctx, ct, p["scale"], shape=wl.input_shape), env["rk"])
    dec = oc.decrypt_tensor(env["sk"], out.to_words(), out.scale, 0, wl.batch)
    import json
    man = json.loads(wl.manifest)
    blob = np.frombuffer(wl.blob, dtype="<f4").astype(np.float64)
    g = lambda k, s: blob[man["weights"][k]["offset"] // 4:][:int(np.prod(s))].reshape(s)
    cw, w1, w2 = g("conv_w", (2, 1, 3, 3)), g("fc1_w", (18, 4)), g("fc2_w", (4, 2))
    x = imgs.reshape(-1, 1, 8, 8)
    conv = np.zeros((x.shape[0], 2, 3, 3))
    for f in range(2):
        for yy in range(3):
            for xx in range(3):
                conv[:, f, yy, xx] = (x[:, 0, 2 * yy:2 * yy + 3, 2 * xx:2 * xx + 3] * cw[f, 0]).sum((1, 2))
    h1 = (conv ** 2).reshape(-1, 18) @ w1
    want = (h1 ** 2) @ w2
    assert np.abs(dec - want).max() < 1e-3


def test_dense_tensor_core_path_bit_exact(env):
    """tcgen05.mma.kind::i8 byte-plane contraction (default) == IMAD path (HG_DENSE_TC=0) == oracle,
    on the c1 layer (845 -> 100 + bias + rescale) and a K=100 -> M=10 layer (fc2 shape)."""
    import json
    import os
    p, oc = env["p"], env["oc"]
    os.environ["HG_DENSE_TC"] = "0"
    try:
        ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
    finally:
        del os.environ["HG_DENSE_TC"]
    ctx_tc = env["ctx"]
    for wl, K, M, level in ((W.dense_layer(), 845, 100, 6), (W.dense_layer(seed=9, k=100, m=10), 100, 10, 6)):
        m = H.PlainModel.load(wl.manifest, wl.blob)
        x = W.random_ciphertexts(p, K, seed=21 + K)
        sc2 = p["scale"] ** 2 / p["chain"][level - 1]
        nodes = {"input": (0, level, level, p["scale"]), "fc": (1, level, level - 1, sc2),
                 "out": (0, level - 1, level - 1, sc2)}
        outs = []
        for c in (ctx, ctx_tc):
            plan = H.RescalePlan.from_nodes(0, M, nodes)
            outs.append(H.execute(c, m, plan, H.CipherTensor.from_words(c, x, p["scale"], shape=[K])).to_words())
        assert np.array_equal(outs[0], outs[1]), (K, M)
        man = json.loads(wl.manifest)
        blob = np.frombuffer(wl.blob, dtype="<f4")
        wm = man["weights"]
        w = blob[wm["fc_w"]["offset"] // 4:][:K * M].reshape(K, M)
        b = blob[wm["fc_b"]["offset"] // 4:][:M]
        want = oc.dense(x, w, level, p["scale"], bias=b, rescale=True, outputs=[0, M - 1])
        assert np.array_equal(outs[1][0], want[0]) and np.array_equal(outs[1][M - 1], want[1])
