# SPDX-License-Identifier: Apache-2.0
"""The reference's own parameter presets (make_parameters, henet/params.hpp:74-101) on the
GPU path, bit-exact against the reference (oracle/_ref):

  P11  N = 2^11, one 54-bit prime, no special prime  (client-aided ReLU networks)
  P12  N = 2^12, three ~2^30 primes above 2^30, 41-bit special prime
  P13  N = 2^13, 51-bit anchor + five 41-bit primes, 50-bit special prime
  P14  N = 2^14, 51-bit anchor + seven 41-bit primes, 50-bit special prime

All four run on the u64 kernels (hg_wide.cu): relinearization for any primes < 2^62
(k_relin_*_w, henet/ckks.hpp:442-499), rescale by primes >= 2^32 (centred corrections
beyond i32, henet/ckks.hpp:504-524), and the 128-bit MAC contractions.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import refbind as R  # noqa: E402
from paper_1908_04172_b200 import henet as H  # noqa: E402
from paper_1908_04172_b200 import workloads as W  # noqa: E402

PRESETS = ["P11", "P12", "P13", "P14"]


@pytest.fixture(scope="module", params=PRESETS)
def penv(request):
    p = W.PRESETS[request.param]
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
    ref = R.RefContext(p["n"], p["chain"], p["special"], p["scale"])
    keys = ref.keygen(17, p["special"] != 0)
    return dict(name=request.param, p=p, ctx=ctx, ref=ref, keys=keys)


def _rand(p, count, seed, level=None):
    rng = np.random.default_rng(seed)
    L = level or len(p["chain"])
    out = np.empty((count, 2, L, p["n"]), dtype=np.uint64)
    for i, q in enumerate(p["chain"][:L]):
        out[:, :, i, :] = rng.integers(0, q, size=(count, 2, p["n"]), dtype=np.uint64)
    return out


def test_preset_context_roots(penv):
    ctx, ref, p = penv["ctx"], penv["ref"], penv["p"]
    full = len(p["chain"]) + (1 if p["special"] else 0)
    assert [ctx.ntt_root(i) for i in range(full)] == [ref.ntt_root(i) for i in range(full)]
    x = _rand(p, 1, 1)
    t = H.CipherTensor.from_words(ctx, x, 1.0)
    H.ntt_inverse(ctx, t)
    got = t.to_words()
    for i in range(len(p["chain"])):
        assert np.array_equal(got[0, 0, i], ref.ntt(i, x[0, 0, i], inverse=True)), i


def test_preset_rescale_every_level(penv):
    """Rescale drops the last chain prime (>= 2^32 for P13/P14: 64-bit corrections)."""
    ctx, ref, p = penv["ctx"], penv["ref"], penv["p"]
    L = len(p["chain"])
    if L < 2:
        pytest.skip("one prime: nothing to rescale")
    x = _rand(p, 3, 2)
    sc = p["scale"] ** 2
    t = H.CipherTensor.from_words(ctx, x, sc)
    for target in range(L - 1, 0, -1):
        want, wsc = ref.rescale(x, sc, target)
        got = H.rescale(ctx, t, target)
        assert got.scale == wsc and np.array_equal(got.to_words(), want), target


def test_preset_relinearize_bit_exact(penv):
    """relinearize of a size-3 ciphertext at the top level and one below, and the eval_square
    body square -> relinearize -> rescale (henet/graph.hpp:995-1008)."""
    ctx, ref, p, keys = penv["ctx"], penv["ref"], penv["p"], penv["keys"]
    if not p["special"]:
        with pytest.raises(H.ValidationError):
            H.RelinKey(ctx, np.zeros(1, dtype=np.uint64))
        return
    rk = H.RelinKey(ctx, keys.rk_words())
    L = len(p["chain"])
    for level in sorted({L, max(1, L - 1)}, reverse=True):
        x = _rand(p, 3, 10 + level, level=level)
        sc = p["scale"]
        sq, sq_sc = ref.square(x, sc)
        want = ref.relinearize(keys, sq, sq_sc)
        t3 = H.CipherTensor.from_words(ctx, sq, sq_sc)
        got = H.relinearize(ctx, t3, rk)
        assert got.scale == sq_sc
        assert np.array_equal(got.to_words(), want), level
        if level >= 2:
            want_r, want_sc = ref.rescale(want, sq_sc, level - 1)
            got_r = H.square_relin(ctx, H.CipherTensor.from_words(ctx, x, sc), rk, rescale=True)
            assert got_r.scale == want_sc
            assert np.array_equal(got_r.to_words(), want_r), level


def test_preset_network_bit_exact(penv):
    """A whole network per preset on real encryptions: the CryptoNets-shaped toy (conv ->
    square -> dense -> square -> dense, lazy plan, four rescales) where the chain is deep
    enough (P13, P14), the CryptoNets-ReLU topology with client-aided refreshes (the
    reference's engine, depth 1) at P11 and P12."""
    ctx, ref, p, keys = penv["ctx"], penv["ref"], penv["p"], penv["keys"]
    slots = p["n"] // 2
    if len(p["chain"]) >= 5:
        wl = W.toy_cryptonets(batch=64)
        imgs = W.synthetic_images(wl.input_shape, 64, 3)
        words, sc = ref.encrypt_tensor(keys, imgs, 5)
        want, want_sc, st = ref.execute(keys, wl.manifest, wl.blob, words, sc)
        rk = H.RelinKey(ctx, keys.rk_words())
        model = H.PlainModel.load(wl.manifest, wl.blob)
        plan = H.RescalePlan.plan(ctx, model)
        assert plan.planned_rescale_ops == st["rescale_ops"]
        stats = H.ExecutionStats()
        out = H.execute(ctx, model, plan, H.CipherTensor.from_words(ctx, words, sc, shape=wl.input_shape), rk,
                        None, stats)
        assert stats.relin_ops == st["relin_ops"] and stats.rescale_ops == st["rescale_ops"]
    else:
        wl = W.toy_cryptonets_relu(batch=slots)
        imgs = W.synthetic_images(wl.input_shape, slots, 3)
        words, sc = ref.encrypt_tensor(keys, imgs, 5)
        want, want_sc, st = ref.execute(keys, wl.manifest, wl.blob, words, sc, refresh_seed=31)
        model = H.PlainModel.load(wl.manifest, wl.blob)
        plan = H.RescalePlan.plan(ctx, model)
        assert plan.planned_rescale_ops == 0

        def provider(kind, window, layer_seq, req):
            return ref.nonlin_apply(keys, kind, window, layer_seq, 31, req.to_words(), req.scale, req.packing)

        out = H.execute(ctx, model, plan, H.CipherTensor.from_words(ctx, words, sc, shape=wl.input_shape), None,
                        provider)
    assert out.scale == want_sc
    assert np.array_equal(out.to_words(), want)


def test_preset_gpu_client_round_trip(penv):
    """GPU encrypt_tensor == the reference's, and the GPU refresh engine == the reference's
    NonlinearityEngine, under every preset (u64 client kernels at N = 2^11 .. 2^14)."""
    ctx, ref, p, keys = penv["ctx"], penv["ref"], penv["p"], penv["keys"]
    slots = p["n"] // 2
    sk = H.SecretKey(ctx, keys.sk_words())
    samples = np.random.default_rng(7).uniform(-1, 1, (slots, 3))
    want, wsc = ref.encrypt_tensor(keys, samples, 9)
    got = H.encrypt_tensor(ctx, sk, samples, 9)
    assert got.scale == wsc and np.array_equal(got.to_words(), want)
    eng = H.RefreshEngine(ctx, sk, 13)
    wl = W.toy_cryptonets_relu(batch=slots)
    imgs = W.synthetic_images(wl.input_shape, slots, 4)
    words, sc = ref.encrypt_tensor(keys, imgs, 6)
    want, want_sc, _ = ref.execute(keys, wl.manifest, wl.blob, words, sc, refresh_seed=13)
    model = H.PlainModel.load(wl.manifest, wl.blob)
    out = H.execute(ctx, model, H.RescalePlan.plan(ctx, model),
                    H.CipherTensor.from_words(ctx, words, sc, shape=wl.input_shape), None, eng)
    assert out.scale == want_sc
    assert np.array_equal(out.to_words(), want)
