# SPDX-License-Identifier: Apache-2.0
"""GPU client side against the reference library (oracle/_ref):

* encrypt_tensor (henet/graph.hpp:68-91): ciphertext words bit-exact for real and
  complex packing, both through the counter-mode ChaCha20 sampler and through the serial
  stream walk that handles rejections (HG_ENC_SERIAL=1 forces it for every ciphertext).
* decrypt (henet/ckks.hpp:256-268): plaintext residues c0 + c1 s (+ c2 s^2), exact.
* decrypt_tensor (henet/graph.hpp:93-103): decoded values bit-exact (the decoder's x87
  long double conversion is emulated), on fresh encryptions, on size-3 ciphertexts and on
  a network's output.
* NonlinearityEngine (henet/graph.hpp:699-741) on the GPU (RefreshEngine): refreshed
  ciphertexts bit-exact for ReLU and window max, real and complex packing, and as the
  provider of whole CryptoNets-ReLU executions."""
import os

import numpy as np
import pytest

from oracle import refbind as R
from paper_1908_04172_b200 import henet as H
from paper_1908_04172_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    p = W.N8192
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
    ref = R.RefContext(p["n"], p["chain"], p["special"], p["scale"])
    keys = ref.keygen(31, True)
    sk = H.SecretKey(ctx, keys.sk_words())
    return dict(p=p, ctx=ctx, ref=ref, keys=keys, sk=sk)


@pytest.mark.parametrize("packing,batch,count,serial", [(0, 4096, 12, False), (1, 8192, 7, False),
                                                        (0, 1000, 3, True), (1, 2, 2, True), (0, 1, 1, False)])
def test_encrypt_tensor_bit_exact(env, packing, batch, count, serial):
    ctx, ref, keys, sk = env["ctx"], env["ref"], env["keys"], env["sk"]
    rng = np.random.default_rng(batch + count)
    samples = rng.uniform(-1, 1, (batch, count))
    want, wsc = ref.encrypt_tensor(keys, samples, 1234 + count, packing=packing)
    if serial:
        os.environ["HG_ENC_SERIAL"] = "1"
    try:
        got = H.encrypt_tensor(ctx, sk, samples, 1234 + count, packing)
    finally:
        os.environ.pop("HG_ENC_SERIAL", None)
    assert got.scale == wsc
    assert np.array_equal(got.to_words(), want)


def test_encrypt_rejects_like_reference(env):
    ctx, sk = env["ctx"], env["sk"]
    with pytest.raises(H.ValidationError, match="batch exceeds slot capacity"):
        H.encrypt_tensor(ctx, sk, np.zeros((4097, 1)), 1, 0)
    with pytest.raises(H.ValidationError, match="complex packing needs an even batch"):
        H.encrypt_tensor(ctx, sk, np.zeros((3, 1)), 1, 1)
    with pytest.raises(H.ValidationError, match="exceeds q_level/2|too large"):
        H.encrypt_tensor(ctx, sk, np.full((4, 1), 1e30), 1, 0)
    with pytest.raises(H.ValidationError, match="batch must be non-empty"):
        H.encrypt_tensor(ctx, sk, np.zeros((0, 1)), 1, 0)


def _decrypt_np(p, skw, words):
    """m = c0 + c1 s (+ c2 s^2) mod q_i, the definition (henet/ckks.hpp:256-268)."""
    cnt, polys, level, n = words.shape
    q = np.array(p["chain"][:level], dtype=np.uint64)[:, None]
    s = skw[:level]
    m = (words[:, 0] + (words[:, 1] * s) % q) % q
    if polys == 3:
        m = (m + (words[:, 2] * ((s * s) % q)) % q) % q
    return m


def test_decrypt_residues_exact(env):
    ctx, p, keys, sk = env["ctx"], env["p"], env["keys"], env["sk"]
    skw = keys.sk_words()
    for level, polys in ((6, 2), (3, 2), (5, 3), (1, 2)):
        words = W.random_ciphertexts(p, 5, seed=level * 10 + polys, level=level)
        if polys == 3:
            words = np.concatenate([words, W.random_ciphertexts(p, 5, seed=99, level=level)[:, :1]], axis=1)
        t = H.CipherTensor.from_words(ctx, words, 2.0 ** 30)
        assert np.array_equal(H.decrypt(ctx, sk, t), _decrypt_np(p, skw, words))


@pytest.mark.parametrize("packing,batch", [(0, 4096), (1, 8192), (0, 10)])
def test_decrypt_tensor_fresh_vs_reference(env, packing, batch):
    ctx, ref, keys, sk = env["ctx"], env["ref"], env["keys"], env["sk"]
    samples = np.random.default_rng(batch).uniform(-2, 2, (max(batch, 2), 6))
    words, sc = ref.encrypt_tensor(keys, samples, 77, packing=packing)
    t = H.CipherTensor.from_words(ctx, words, sc, packing=packing)
    got = H.decrypt_tensor(ctx, sk, t, batch)
    want = ref.decrypt_tensor(keys, words, sc, packing, batch)
    assert np.array_equal(got, want)
    assert np.abs(got - samples[:batch]).max() < 1e-3


def test_decrypt_tensor_network_output_and_size3(env):
    ctx, ref, keys, sk, p = env["ctx"], env["ref"], env["keys"], env["sk"], env["p"]
    wl = W.toy_cryptonets()
    imgs = W.synthetic_images(wl.input_shape, wl.batch, 5)
    words, sc = ref.encrypt_tensor(keys, imgs, 9)
    out_w, out_sc, _ = ref.execute(keys, wl.manifest, wl.blob, words, sc)
    t = H.CipherTensor.from_words(ctx, out_w, out_sc)
    got = H.decrypt_tensor(ctx, sk, t, wl.batch)
    want = ref.decrypt_tensor(keys, out_w, out_sc, 0, wl.batch)
    assert np.array_equal(got, want)
    # size-3 (square without relinearisation) at level 6
    sq, sq_sc = ref.square(words[:3], sc)
    t3 = H.CipherTensor.from_words(ctx, sq, sq_sc)
    got3 = H.decrypt_tensor(ctx, sk, t3, wl.batch)
    want3 = ref.decrypt_tensor(keys, sq, sq_sc, 0, wl.batch)
    assert np.array_equal(got3, want3)


def test_encrypt_execute_decrypt_on_gpu(env):
    """The whole client-server-client loop on the GPU vs the reference's plaintext logits."""
    ctx, ref, keys, sk = env["ctx"], env["ref"], env["keys"], env["sk"]
    wl = W.toy_cryptonets()
    imgs = W.synthetic_images(wl.input_shape, wl.batch, 6)
    rk = H.RelinKey(ctx, keys.rk_words())
    x = H.encrypt_tensor(ctx, sk, imgs, 11, shape=wl.input_shape)
    model = H.PlainModel.load(wl.manifest, wl.blob)
    out = H.execute(ctx, model, H.RescalePlan.plan(ctx, model), x, rk)
    got = H.decrypt_tensor(ctx, sk, out, wl.batch)
    words, sc = ref.encrypt_tensor(keys, imgs, 11)
    out_w, out_sc, _ = ref.execute(keys, wl.manifest, wl.blob, words, sc)
    assert np.array_equal(out.to_words(), out_w)
    assert np.array_equal(got, ref.decrypt_tensor(keys, out_w, out_sc, 0, wl.batch))


@pytest.mark.parametrize("kind,window,packing", [(1, 1, 0), (1, 1, 1), (2, 4, 0), (2, 9, 1)])
def test_refresh_engine_bit_exact(env, kind, window, packing):
    ctx, ref, keys, sk, p = env["ctx"], env["ref"], env["keys"], env["sk"], env["p"]
    batch = 4096 if packing == 0 else 8192
    samples = np.random.default_rng(window).uniform(-1, 1, (batch, 3 * window))
    words, sc = ref.encrypt_tensor(keys, samples, 5, packing=packing)
    # a rescaled product, like a layer output: scale != 2^24, level 5
    res = ref.encode_scalar(0.75, 6, p["scale"])
    prod, psc = ref.mul_ct_pt_scalar(words, sc, res, p["scale"], packing)
    low, lsc = ref.rescale(prod, psc, 5, packing)
    eng = H.RefreshEngine(ctx, sk, 1234)
    for layer_seq in (0, 3):
        want = ref.nonlin_apply(keys, kind, window, layer_seq, 1234, low, lsc, packing)
        got = eng.apply(kind, window, layer_seq, H.CipherTensor.from_words(ctx, low, lsc, packing=packing))
        assert np.array_equal(got.to_words(), want)


def test_decrypt_crt_fast_path_and_fallback_bit_exact_u32(env):
    """The decoder's three-limb CRT fast path on the 30/24-bit chain (q_0 q_1 q_2 ~ 2^78) and
    its full-Garner fallback (uniform residues: coefficients near Q / 2) in one tensor."""
    ctx, ref, keys, sk, p = env["ctx"], env["ref"], env["keys"], env["sk"], env["p"]
    samples = np.random.default_rng(23).normal(0, 1, (4096, 3))
    fresh, sc = ref.encrypt_tensor(keys, samples, 24)
    mixed = np.concatenate([fresh, W.random_ciphertexts(p, 3, seed=25)], axis=0)
    t = H.CipherTensor.from_words(ctx, mixed, sc)
    got = H.decrypt_tensor(ctx, sk, t, 4096)
    want = ref.decrypt_tensor(keys, mixed, sc, 0, 4096)
    assert np.array_equal(got, want, equal_nan=True)


@pytest.mark.parametrize("packing", [1, 0])
def test_refresh_engine_as_provider_cryptonets_relu(env, packing):
    """c3 (CryptoNets-ReLU, client-aided refresh) executed with the GPU engine as provider."""
    ctx, ref, keys, sk = env["ctx"], env["ref"], env["keys"], env["sk"]
    wl = W.cryptonets_relu(packing=packing, batch=8192 if packing else 4096)
    imgs = W.synthetic_images(wl.input_shape, wl.batch, 8)
    words, sc = ref.encrypt_tensor(keys, imgs, 9, packing=packing)
    want, want_sc, _ = ref.execute(keys, wl.manifest, wl.blob, words, sc, refresh_seed=99)
    model = H.PlainModel.load(wl.manifest, wl.blob)
    inp = H.CipherTensor.from_words(ctx, words, sc, packing=packing, shape=wl.input_shape)
    out = H.execute(ctx, model, H.RescalePlan.plan(ctx, model), inp, None, H.RefreshEngine(ctx, sk, 99))
    assert out.scale == want_sc
    assert np.array_equal(out.to_words(), want)


def test_c3_packed_vs_unpacked_slot_for_slot(env):
    """BASELINE c3's own check: the CryptoNets-ReLU network on 8192 images under complex
    packing (two images per slot) against the same network on the two 4096-image halves under
    real packing, all on the GPU (encrypt, execute with the GPU refresh engine, decrypt);
    decrypted logits agree slot for slot within the north star's 1e-3, and each run is itself
    bit-exact against the reference elsewhere (test_refresh_engine_as_provider_cryptonets_relu)."""
    ctx, sk = env["ctx"], env["sk"]
    imgs = W.synthetic_images([1, 28, 28], 8192, 17)
    wl_c = W.cryptonets_relu(packing=1, batch=8192)
    wl_r = W.cryptonets_relu(packing=0, batch=4096)
    mc, mr = H.PlainModel.load(wl_c.manifest, wl_c.blob), H.PlainModel.load(wl_r.manifest, wl_r.blob)
    xc = H.encrypt_tensor(ctx, sk, imgs, 18, 1, shape=wl_c.input_shape)
    yc = H.execute(ctx, mc, H.RescalePlan.plan(ctx, mc), xc, None, H.RefreshEngine(ctx, sk, 99))
    packed = H.decrypt_tensor(ctx, sk, yc, 8192)
    halves = []
    for h in range(2):
        xr = H.encrypt_tensor(ctx, sk, imgs[h * 4096:(h + 1) * 4096], 19 + h, 0, shape=wl_r.input_shape)
        yr = H.execute(ctx, mr, H.RescalePlan.plan(ctx, mr), xr, None, H.RefreshEngine(ctx, sk, 100 + h))
        halves.append(H.decrypt_tensor(ctx, sk, yr, 4096))
    unpacked = np.concatenate(halves, axis=0)
    assert packed.shape == unpacked.shape == (8192, 10)
    assert np.isfinite(packed).all()
    assert float(np.abs(packed - unpacked).max()) < 1e-3


# ---- wide contexts (BASELINE c4/c5b parameters: N = 16384, 40-bit limb 0, u64 residues) ----
@pytest.fixture(scope="module")
def wenv():
    p = W.N16384
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
    ref = R.RefContext(p["n"], p["chain"], p["special"], p["scale"])
    keys = ref.keygen(41, False)
    sk = H.SecretKey(ctx, keys.sk_words())
    return dict(p=p, ctx=ctx, ref=ref, keys=keys, sk=sk)


@pytest.mark.parametrize("packing,serial", [(0, False), (1, False), (0, True)])
def test_wide_encrypt_decrypt_bit_exact(wenv, packing, serial):
    ctx, ref, keys, sk, p = wenv["ctx"], wenv["ref"], wenv["keys"], wenv["sk"], wenv["p"]
    batch = 8192 if packing == 0 else 16384
    samples = np.random.default_rng(3).normal(0, 1, (batch, 3))
    want, wsc = ref.encrypt_tensor(keys, samples, 55, packing=packing)
    if serial:
        os.environ["HG_ENC_SERIAL"] = "1"
    try:
        got = H.encrypt_tensor(ctx, sk, samples, 55, packing)
    finally:
        os.environ.pop("HG_ENC_SERIAL", None)
    assert got.scale == wsc
    assert np.array_equal(got.to_words(), want)
    dec = H.decrypt_tensor(ctx, sk, got, batch)
    assert np.array_equal(dec, ref.decrypt_tensor(keys, want, wsc, packing, batch))
    # plaintext residues c0 + c1 s, checked with Python integers on a slice
    m = H.decrypt(ctx, sk, got)
    skw = keys.sk_words()
    for limb in (0, 3, 7):
        q = p["chain"][limb]
        for n in (0, 1, 4095, 16383):
            c0, c1 = int(want[1, 0, limb, n]), int(want[1, 1, limb, n])
            assert int(m[1, limb, n]) == (c0 + c1 * int(skw[limb, n])) % q


def test_wide_decrypt_crt_fast_path_and_fallback_bit_exact(wenv):
    """The decoder's two-limb CRT fast path (q_0 q_1 ~ 2^70) against the reference's full
    reconstruction: fresh encryptions (small coefficients, fast path) and uniform residues
    (coefficients near Q / 2: every one takes the full Garner fallback), in one tensor, and
    the same tensor with the fast path switched off in a subprocess-free way (HG_CRT_FAST is
    read once, so only the mixed tensor is checked here)."""
    ctx, ref, keys, sk, p = wenv["ctx"], wenv["ref"], wenv["keys"], wenv["sk"], wenv["p"]
    samples = np.random.default_rng(21).normal(0, 1, (8192, 3))
    fresh, sc = ref.encrypt_tensor(keys, samples, 56)
    rnd = W.random_ciphertexts(p, 3, seed=57)
    mixed = np.concatenate([fresh, rnd], axis=0)
    t = H.CipherTensor.from_words(ctx, mixed, sc)
    got = H.decrypt_tensor(ctx, sk, t, 8192)
    want = ref.decrypt_tensor(keys, mixed, sc, 0, 8192)
    assert np.array_equal(got, want, equal_nan=True)


def test_wide_c4_block_gpu_relu6_refresh_bit_exact(wenv):
    """BASELINE c4 on a 4x4 tile with both client-aided ReLU6 refreshes on the GPU engine
    (clamp to [0, 6]) vs the reference executor with the harness's clamp provider."""
    ctx, ref, keys, sk = wenv["ctx"], wenv["ref"], wenv["keys"], wenv["sk"]
    wl = W.mobilenet_block(hw=4, cin=4, expand=6, cout=3)
    acts = np.random.default_rng(12).normal(0, 1, (ctx.slot_count(), wl.input_count))
    words, sc = ref.encrypt_tensor(keys, acts, 13)
    R.set_relu_clip(6.0)
    try:
        want, want_sc, _ = ref.execute(keys, wl.manifest, wl.blob, words, sc, refresh_seed=77)
    finally:
        R.set_relu_clip(0.0)
    model = H.PlainModel.load(wl.manifest, wl.blob)
    eng = H.RefreshEngine(ctx, sk, 77)
    eng.set_relu_clip(6.0)
    x = H.encrypt_tensor(ctx, sk, acts, 13, shape=wl.input_shape)
    assert np.array_equal(x.to_words(), words)
    out = H.execute(ctx, model, H.RescalePlan.plan(ctx, model), x, None, eng)
    assert out.scale == want_sc
    assert np.array_equal(out.to_words(), want)
