# SPDX-License-Identifier: Apache-2.0
"""Wide (u64) path: BASELINE configs 4 / 5b parameters (N=16384, chain [40, 30 x 7] bits
+ 40-bit special prime, scale 2^30) against the reference (oracle/_ref), bit-exact."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import refbind as R  # noqa: E402
from paper_1908_04172_b200 import henet as H  # noqa: E402
from paper_1908_04172_b200 import workloads as W  # noqa: E402


@pytest.fixture(scope="module")
def env():
    p = W.N16384
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
    ref = R.RefContext(p["n"], p["chain"], p["special"], p["scale"])
    return dict(p=p, ctx=ctx, ref=ref, keys=ref.keygen(3, False))


def test_ntt_every_prime_wide(env):
    ctx, ref, p = env["ctx"], env["ref"], env["p"]
    assert [ctx.ntt_root(i) for i in range(9)] == [ref.ntt_root(i) for i in range(9)]
    x = W.random_ciphertexts(p, 1, seed=1)
    t = H.CipherTensor.from_words(ctx, x, 1.0)
    H.ntt_forward(ctx, t)
    got = t.to_words()
    for k in range(2):
        for i in range(8):
            assert np.array_equal(got[0, k, i], ref.ntt(i, x[0, k, i])), (k, i)
    H.ntt_inverse(ctx, t)
    assert np.array_equal(t.to_words(), x)


def test_rescale_mul_add_wide(env):
    ctx, ref, p = env["ctx"], env["ref"], env["p"]
    x = W.random_ciphertexts(p, 2, seed=2)
    sc = 2.0 ** 60
    t = H.CipherTensor.from_words(ctx, x, sc)
    for target in (7, 2, 1):
        want, wsc = ref.rescale(x, sc, target)
        got = H.rescale(ctx, t, target)
        assert got.scale == wsc and np.array_equal(got.to_words(), want), target
    res = ref.encode_scalar(0.4321, 8, p["scale"])
    want, wsc = ref.mul_ct_pt_scalar(x, sc, res, p["scale"])
    got = H.mul_ct_pt_scalar(ctx, t, res, p["scale"])
    assert got.scale == wsc and np.array_equal(got.to_words(), want)
    y = W.random_ciphertexts(p, 2, seed=3)
    assert np.array_equal(H.add_ct_ct(ctx, t, H.CipherTensor.from_words(ctx, y, sc)).to_words(),
                          ref.add_ct_ct(x, y, sc))


def test_encoders_wide(env):
    ctx, ref, p = env["ctx"], env["ref"], env["p"]
    vals = np.random.default_rng(4).normal(0, 0.1, 64)
    for scale in (p["scale"], 2.0 ** 60):
        got = H.encode_scalars(ctx, vals, 8, scale)
        for v, g in zip(vals, got):
            assert np.array_equal(g, ref.encode_scalar(v, 8, scale))
    rng = np.random.default_rng(5)
    s = rng.uniform(-1, 1, 8192) + 1j * rng.uniform(-1, 1, 8192)
    assert np.array_equal(H.encode_vector(ctx, s, 8, p["scale"]), ref.encode_vector(s, 8, p["scale"]))


def _run_both(env, wl, count_override=None, seed=7, mode=0):
    ctx, ref, p = env["ctx"], env["ref"], env["p"]
    x = W.random_ciphertexts(p, wl.input_count, seed=seed)
    want, want_sc, st = ref.execute(None, wl.manifest, wl.blob, x, p["scale"], mode=mode,
                                    patch=wl.patch_terminal_rescale)
    rp = ref.plan(wl.manifest, wl.blob, mode=mode, patch=wl.patch_terminal_rescale)
    nodes = {n["id"]: (n["decision"], n["level_in"], n["level_out"],
                       np.array([n["scale_out_bits"]], dtype=np.uint64).view(np.float64)[0]) for n in rp["nodes"]}
    plan = H.RescalePlan.from_nodes(mode, rp["planned_rescale_ops"], nodes)
    model = H.PlainModel.load(wl.manifest, wl.blob)
    out = H.execute(ctx, model, plan, H.CipherTensor.from_words(ctx, x, p["scale"], shape=wl.input_shape))
    assert out.scale == want_sc
    assert np.array_equal(out.to_words(), want)


def test_dense_c5b_shape_small_bit_exact(env):
    """c5b topology (dense + one rescale per output, 40-bit limb 0) at K=96, M=40."""
    _run_both(env, W.wide_dense(k=96, m=40))


def test_dense_naive_wide_bit_exact(env):
    """Naive per-term rescaling with the 40-bit limb (hybrid u32 / u64 rescale per term)."""
    _run_both(env, W.wide_dense(k=12, m=5), mode=1)


def test_conv_c4_shape_small_bit_exact(env):
    """c4 linear layers (1x1 expand, 3x3 block-diagonal depthwise with pad 1, 1x1 project) on a
    4x4 tile, without the client-aided ReLU6 (linear chain only: zero rescales, lazy plan)."""
    import json
    wl = W.mobilenet_block(hw=4, cin=4, expand=6, cout=3)
    j = json.loads(wl.manifest)
    j["nodes"] = [n for n in j["nodes"] if n["op"] != "Relu"]
    for n in j["nodes"]:
        n["inputs"] = [{"relu6a": "expand", "relu6b": "dw"}.get(i, i) for i in n.get("inputs", [])]
    wl.manifest = json.dumps(j)
    ctx, ref, p = env["ctx"], env["ref"], env["p"]
    x = W.random_ciphertexts(p, wl.input_count, seed=9)
    want, want_sc, st = ref.execute(None, wl.manifest, wl.blob, x, p["scale"])
    model = H.PlainModel.load(wl.manifest, wl.blob)
    plan = H.RescalePlan.plan(ctx, model)
    assert plan.planned_rescale_ops == st["rescale_ops"]
    out = H.execute(ctx, model, plan, H.CipherTensor.from_words(ctx, x, p["scale"], shape=wl.input_shape))
    assert out.scale == want_sc
    assert np.array_equal(out.to_words(), want)


def test_c4_block_relu6_provider_bit_exact(env):
    """Full c4 block on a 4x4 tile of real encryptions of N(0,1) activations: 1x1 expand,
    ReLU6, 3x3 depthwise (pad 1), ReLU6, 1x1 project.  ReLU6 is client-aided: the Relu nodes
    go through the provider, here the reference's refresh with a [0, 6] clamp,
    called from the GPU executor's callback exactly as the reference executor calls it."""
    ctx, ref, p, keys = env["ctx"], env["ref"], env["p"], env["keys"]
    wl = W.mobilenet_block(hw=4, cin=4, expand=6, cout=3)
    acts = np.random.default_rng(12).normal(0, 1, (ctx.slot_count(), wl.input_count))
    words, sc = ref.encrypt_tensor(keys, acts, 13)
    R.set_relu_clip(6.0)
    try:
        want, want_sc, st = ref.execute(keys, wl.manifest, wl.blob, words, sc, refresh_seed=77)
        model = H.PlainModel.load(wl.manifest, wl.blob)
        plan = H.RescalePlan.plan(ctx, model)
        assert plan.planned_rescale_ops == st["rescale_ops"]

        def provider(kind, window, layer_seq, req):
            return ref.nonlin_apply(keys, kind, window, layer_seq, 77, req.to_words(), req.scale, req.packing)

        stats = H.ExecutionStats()
        out = H.execute(ctx, model, plan, H.CipherTensor.from_words(ctx, words, sc, shape=wl.input_shape), None,
                        provider, stats)
    finally:
        R.set_relu_clip(0.0)
    assert out.scale == want_sc
    assert np.array_equal(out.to_words(), want)
    assert stats.nonlin_elements == 2 * 6 * 4 * 4  # two ReLU6 layers over (6, 4, 4)


def test_wide_relinearize_bit_exact(env):
    """Relinearization with the 40-bit limb 0 and special prime (u64 kernels,
    henet/ckks.hpp:442-499), and square -> relinearize -> rescale, against the reference."""
    ctx, ref, p = env["ctx"], env["ref"], env["p"]
    keys = ref.keygen(5, True)
    rk = H.RelinKey(ctx, keys.rk_words())
    for level in (8, 3):
        x = W.random_ciphertexts(p, 2, seed=11 + level, level=level)
        sq, sq_sc = ref.square(x, p["scale"])
        want = ref.relinearize(keys, sq, sq_sc)
        got = H.relinearize(ctx, H.CipherTensor.from_words(ctx, sq, sq_sc), rk)
        assert np.array_equal(got.to_words(), want), level
        want_r, want_sc = ref.rescale(want, sq_sc, level - 1)
        got_r = H.square_relin(ctx, H.CipherTensor.from_words(ctx, x, p["scale"]), rk, rescale=True)
        assert got_r.scale == want_sc and np.array_equal(got_r.to_words(), want_r), level
