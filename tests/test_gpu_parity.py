# SPDX-License-Identifier: Apache-2.0
"""GPU parity: every hot-path op of libhenet_b200.so against the reference
library itself (oracle/_ref, the unmodified henet headers compiled here) on
identical inputs.  Integer results must be bit-exact."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import refbind as R  # noqa: E402
from paper_1908_04172_b200 import henet as H  # noqa: E402
from paper_1908_04172_b200 import workloads as W  # noqa: E402


@pytest.fixture(scope="module")
def env():
    p = W.N8192
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
    ref = R.RefContext(p["n"], p["chain"], p["special"], p["scale"])
    keys = ref.keygen(11, True)
    rk = H.RelinKey(ctx, keys.rk_words())
    return dict(p=p, ctx=ctx, ref=ref, keys=keys, rk=rk)


def test_ntt_roots_match(env):
    ctx, ref = env["ctx"], env["ref"]
    for i in range(len(env["p"]["chain"]) + 1):
        assert ctx.ntt_root(i) == ref.ntt_root(i)


def test_ntt_forward_inverse_bit_exact(env):
    ctx, ref, p = env["ctx"], env["ref"], env["p"]
    L = len(p["chain"])
    words = W.random_ciphertexts(p, 3, seed=5)
    t = H.CipherTensor.from_words(ctx, words, 1.0)
    H.ntt_forward(ctx, t)
    got = t.to_words()
    for e in range(3):
        for k in range(2):
            for i in range(L):
                assert np.array_equal(got[e, k, i], ref.ntt(i, words[e, k, i])), (e, k, i)
    H.ntt_inverse(ctx, t)
    assert np.array_equal(t.to_words(), words)


def test_rescale_bit_exact(env):
    ctx, ref, p = env["ctx"], env["ref"], env["p"]
    words = W.random_ciphertexts(p, 4, seed=6)
    sc = 2.0 ** 48
    t = H.CipherTensor.from_words(ctx, words, sc)
    for target in (5, 3, 1):
        want, wsc = ref.rescale(words, sc, target)
        out = H.rescale(ctx, t, target)
        assert out.level == target
        assert out.scale == wsc
        assert np.array_equal(out.to_words(), want), target


def test_mul_scalar_and_add_bit_exact(env):
    ctx, ref, p = env["ctx"], env["ref"], env["p"]
    a = W.random_ciphertexts(p, 3, seed=7)
    b = W.random_ciphertexts(p, 3, seed=8)
    res = ref.encode_scalar(-0.123456, 6, p["scale"])
    want, wsc = ref.mul_ct_pt_scalar(a, p["scale"], res, p["scale"])
    ta = H.CipherTensor.from_words(ctx, a, p["scale"])
    tb = H.CipherTensor.from_words(ctx, b, p["scale"])
    got = H.mul_ct_pt_scalar(ctx, ta, res, p["scale"])
    assert got.scale == wsc
    assert np.array_equal(got.to_words(), want)
    assert np.array_equal(H.add_ct_ct(ctx, ta, tb).to_words(), ref.add_ct_ct(a, b, p["scale"]))


def test_square_relin_rescale_bit_exact(env):
    ctx, ref, p, keys, rk = env["ctx"], env["ref"], env["p"], env["keys"], env["rk"]
    for level in (6, 5, 3):
        words = W.random_ciphertexts(p, 3, seed=10 + level, level=level)
        sc = 2.0 ** 24
        sq, sqs = ref.square(words, sc)
        rl = ref.relinearize(keys, sq, sqs)
        t = H.CipherTensor.from_words(ctx, words, sc)
        got = H.square_relin(ctx, t, rk, rescale=False)
        assert got.scale == sqs
        assert np.array_equal(got.to_words(), rl), level
        want_rs, rs_sc = ref.rescale(rl, sqs, level - 1)
        got_rs = H.square_relin(ctx, t, rk, rescale=True)
        assert got_rs.level == level - 1 and got_rs.scale == rs_sc
        assert np.array_equal(got_rs.to_words(), want_rs), level
        # unfused op-by-op path
        t3 = H.square(ctx, t)
        assert np.array_equal(t3.to_words(), sq)
        assert np.array_equal(H.relinearize(ctx, t3, rk).to_words(), rl)


def test_encode_scalars_bit_exact(env):
    ctx, ref, p = env["ctx"], env["ref"], env["p"]
    rng = np.random.default_rng(3)
    vals = np.concatenate([rng.normal(0, 0.05, 200), rng.uniform(-3, 3, 50), [0.0, 1.0, -1.0, 0.5, -0.5, 2.5]])
    for scale in (p["scale"], 2.0 ** 48, 16777216.0 * 1.0000001, 3.3e9):
        for level in (6, 3, 1):
            ok, want = [], []
            bad = None
            for v in vals:
                try:
                    want.append(ref.encode_scalar(v, level, scale))
                    ok.append(v)
                except R.RefError:
                    bad = v
            got = H.encode_scalars(ctx, np.array(ok), level, scale)
            assert np.array_equal(got, np.array(want)), (scale, level)
            if bad is not None:  # the reference rejects it -> so must the GPU path
                with pytest.raises(H.ValidationError):
                    H.encode_scalars(ctx, np.array([bad]), level, scale)


def test_encode_vector_bit_exact(env):
    ctx, ref, p = env["ctx"], env["ref"], env["p"]
    rng = np.random.default_rng(4)
    for n_slots, cplx in ((4096, False), (4096, True), (100, True)):
        s = rng.uniform(-1, 1, n_slots) + (1j * rng.uniform(-1, 1, n_slots) if cplx else 0)
        for level in (6, 2):
            got = H.encode_vector(ctx, s, level, p["scale"])
            want = ref.encode_vector(s, level, p["scale"])
            assert np.array_equal(got, want), (n_slots, cplx, level)


def test_decode_vector_bit_exact(env):
    """decode_slots of plaintexts: encode -> decode round trips and arbitrary residues, equal
    to the reference's doubles bit for bit."""
    ctx, ref, p = env["ctx"], env["ref"], env["p"]
    rng = np.random.default_rng(8)
    for level in (6, 3, 1):
        slots = rng.uniform(-1, 1, 4096) + 1j * rng.uniform(-1, 1, 4096)
        pt = ref.encode_vector(slots, level, p["scale"])
        got = H.decode_vector(ctx, pt, p["scale"])
        assert np.array_equal(got, ref.decode(pt, p["scale"]))
        assert np.abs(got - slots).max() < 1e-3
        raw = W.random_ciphertexts(p, 1, seed=level, level=level)[0, 0]
        assert np.array_equal(H.decode_vector(ctx, raw, 2.0 ** 40), ref.decode(raw, 2.0 ** 40))


def _run_both(env, wl, seed=21, threads=0, check_plan=True, mode=0):
    ctx, ref, keys, rk = env["ctx"], env["ref"], env["keys"], env["rk"]
    imgs = W.synthetic_images(wl.input_shape, wl.batch, seed)
    words, sc = ref.encrypt_tensor(keys, imgs, seed + 1, packing=wl.packing)
    want, want_sc, st = ref.execute(keys, wl.manifest, wl.blob, words, sc, mode=mode,
                                    patch=wl.patch_terminal_rescale, threads=threads, refresh_seed=99)
    model = H.PlainModel.load(wl.manifest, wl.blob)
    rp = ref.plan(wl.manifest, wl.blob, mode=mode, patch=wl.patch_terminal_rescale)
    nodes = {n["id"]: (n["decision"], n["level_in"], n["level_out"],
                       np.array([n["scale_out_bits"]], dtype=np.uint64).view(np.float64)[0]) for n in rp["nodes"]}
    plan = H.RescalePlan.from_nodes(mode, rp["planned_rescale_ops"], nodes)
    if check_plan and not wl.patch_terminal_rescale:
        own = H.RescalePlan.plan(ctx, model, mode)
        assert own.planned_rescale_ops == rp["planned_rescale_ops"]
        for nid, v in nodes.items():
            assert own.node(nid) == v, nid
    inp = H.CipherTensor.from_words(ctx, words, sc, packing=wl.packing, shape=wl.input_shape)

    def provider(kind, window, layer_seq, req):
        return ref.nonlin_apply(keys, kind, window, layer_seq, 99, req.to_words(), req.scale, req.packing)

    stats = H.ExecutionStats()
    out = H.execute(ctx, model, plan, inp, rk, provider, stats)
    assert out.scale == want_sc
    assert stats.rescale_ops == st["rescale_ops"]
    got = out.to_words()
    assert got.shape == want.shape
    assert np.array_equal(got, want)
    return imgs, got, out


def test_execute_toy_bit_exact(env):
    _run_both(env, W.toy_cryptonets())


def test_two_contexts_interleaved_bit_exact(env):
    """Two contexts on one GPU (bench.py's lanes: independent batches in flight on two streams),
    executes issued alternately without synchronising in between: every result equals the
    reference's, so the lanes' kernels share the device (TMEM, auxiliary stream) safely."""
    p, ref, keys = env["p"], env["ref"], env["keys"]
    wl = W.toy_cryptonets()
    model = H.PlainModel.load(wl.manifest, wl.blob)
    lanes, wants = [], []
    for lane in range(2):
        imgs = W.synthetic_images(wl.input_shape, wl.batch, 40 + lane)
        words, sc = ref.encrypt_tensor(keys, imgs, 50 + lane, packing=wl.packing)
        want, want_sc, _ = ref.execute(keys, wl.manifest, wl.blob, words, sc, refresh_seed=99)
        ctx = env["ctx"] if lane == 0 else H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
        rk = env["rk"] if lane == 0 else H.RelinKey(ctx, keys.rk_words())
        plan = H.RescalePlan.plan(ctx, model)
        inp = H.CipherTensor.from_words(ctx, words, sc, packing=wl.packing, shape=wl.input_shape)
        lanes.append((ctx, rk, plan, inp))
        wants.append((want, want_sc))
    outs = []
    for i in range(8):
        ctx, rk, plan, inp = lanes[i % 2]
        outs.append(H.execute(ctx, model, plan, inp, rk))
    for i, out in enumerate(outs):
        want, want_sc = wants[i % 2]
        assert out.scale == want_sc
        assert np.array_equal(out.to_words(), want), i


def test_execute_c1_dense_bit_exact(env):
    _run_both(env, W.dense_layer())


@pytest.mark.slow
def test_execute_c2_cryptonets_bit_exact(env):
    _run_both(env, W.cryptonets())


@pytest.mark.slow
def test_execute_c3_relu_complex_bit_exact(env):
    _run_both(env, W.cryptonets_relu())


# Naive rescaling (henet/graph.hpp:905-933 under RescaleMode::Naive): every ct x pt term is
# rescaled before accumulation and the bias is added at the rescaled level and scale.
def test_execute_toy_naive_bit_exact(env):
    _run_both(env, W.toy_cryptonets(), mode=1)


def test_execute_dense_naive_bias_bit_exact(env):
    _run_both(env, W.dense_layer(seed=5, k=40, m=7), mode=1)


def test_execute_dense_naive_complex_bias_bit_exact(env):
    _run_both(env, W.dense_layer(seed=6, k=24, m=5, batch=8192, packing=1), mode=1)


def test_execute_dense_lazy_complex_bias_bit_exact(env):
    _run_both(env, W.dense_layer(seed=6, k=24, m=5, batch=8192, packing=1))


def test_execute_zero_weights_bit_exact(env):
    """All-zero (and signed-zero) weights: the output is the bias alone
    (proj/tests/test_graph.cpp:247), bit-exact against the reference for both packings."""
    _run_both(env, W.dense_layer(seed=8, k=30, m=6, w_scale=0.0))
    _run_both(env, W.dense_layer(seed=9, k=30, m=6, batch=8192, packing=1, w_scale=0.0))
    _run_both(env, W.dense_layer(seed=10, k=30, m=6, w_scale=0.0), mode=1)


def test_kept_encodings_equal_jit(env):
    """JIT == precompiled (proj/tests/test_graph.cpp:404-439): a model that keeps its weight
    encodings across executes gives bit-identical ciphertexts on every run, and again after the
    cache is dropped."""
    ctx, ref, keys, rk = env["ctx"], env["ref"], env["keys"], env["rk"]
    for wl in (W.toy_cryptonets(), W.dense_layer(seed=7, k=60, m=9)):
        imgs = W.synthetic_images(wl.input_shape, wl.batch, 4)
        words, sc = ref.encrypt_tensor(keys, imgs, 5, packing=wl.packing)
        model = H.PlainModel.load(wl.manifest, wl.blob)
        plan = H.RescalePlan.plan(ctx, model)
        inp = H.CipherTensor.from_words(ctx, words, sc, shape=wl.input_shape)
        jit = H.execute(ctx, model, plan, inp, rk).to_words()
        model.keep_encodings(True)
        for _ in range(3):
            assert np.array_equal(H.execute(ctx, model, plan, inp, rk).to_words(), jit)
        model.keep_encodings(False)
        assert np.array_equal(H.execute(ctx, model, plan, inp, rk).to_words(), jit)
