# SPDX-License-Identifier: Apache-2.0
"""The narrow (u32) kernels are templated over the ring degree (N = 2^12 .. 2^14: CTA of
N/32 threads, pass split, TMEM scratch of 64 * N/4096 columns).  The BASELINE configs
exercise N = 8192; these cases run the other two degrees against the reference:
N = 4096 with the 24/30-bit chain of configs 1-3, and N = 16384 with a chain of 30-bit
primes (all < 2^30, so the u32 path, not the wide one)."""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import refbind as R  # noqa: E402
from paper_1908_04172_b200 import henet as H  # noqa: E402
from paper_1908_04172_b200 import workloads as W  # noqa: E402

PARAMS = {
    4096: dict(n=4096, chain=W.N8192["chain"], special=W.N8192["special"], scale=float(2 ** 24)),
    16384: dict(n=16384, chain=[1073643521, 1073479681, 1073184769, 1073053697, 1072857089, 1072496641],
                special=1071513601, scale=float(2 ** 24)),
}


@pytest.fixture(scope="module", params=sorted(PARAMS))
def env(request):
    p = PARAMS[request.param]
    assert all(q < 2 ** 30 and q % (2 * p["n"]) == 1 for q in p["chain"] + [p["special"]])
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
    ref = R.RefContext(p["n"], p["chain"], p["special"], p["scale"])
    keys = ref.keygen(13, True)
    return dict(p=p, ctx=ctx, ref=ref, keys=keys, rk=H.RelinKey(ctx, keys.rk_words()))


def test_ntt_rescale(env):
    ctx, ref, p = env["ctx"], env["ref"], env["p"]
    L = len(p["chain"])
    words = W.random_ciphertexts(p, 2, seed=1)
    t = H.CipherTensor.from_words(ctx, words, 2.0 ** 48)
    H.ntt_forward(ctx, t)
    got = t.to_words()
    for i in range(L):
        assert np.array_equal(got[1, 0, i], ref.ntt(i, words[1, 0, i])), i
    H.ntt_inverse(ctx, t)
    assert np.array_equal(t.to_words(), words)
    for target in (L - 1, 2):
        want, wsc = ref.rescale(words, 2.0 ** 48, target)
        out = H.rescale(ctx, t, target)
        assert out.scale == wsc and np.array_equal(out.to_words(), want), target


def test_square_relin_rescale(env):
    ctx, ref, p, keys, rk = env["ctx"], env["ref"], env["p"], env["keys"], env["rk"]
    L = len(p["chain"])
    for level in (L, 3):
        words = W.random_ciphertexts(p, 2, seed=20 + level, level=level)
        sq, sqs = ref.square(words, 2.0 ** 24)
        rl = ref.relinearize(keys, sq, sqs)
        t = H.CipherTensor.from_words(ctx, words, 2.0 ** 24)
        assert np.array_equal(H.square_relin(ctx, t, rk, rescale=False).to_words(), rl), level
        want_rs, _ = ref.rescale(rl, sqs, level - 1)
        assert np.array_equal(H.square_relin(ctx, t, rk, rescale=True).to_words(), want_rs), level


def test_toy_network(env):
    """conv -> square -> dense -> square -> dense on real encryptions."""
    ctx, ref, p, keys, rk = env["ctx"], env["ref"], env["p"], env["keys"], env["rk"]
    wl = W.toy_cryptonets(batch=p["n"] // 2)
    j = json.loads(wl.manifest)
    j["preset"] = {4096: "P12", 16384: "P14"}[p["n"]]
    wl.manifest = json.dumps(j)
    imgs = W.synthetic_images(wl.input_shape, wl.batch, 31)
    words, sc = ref.encrypt_tensor(keys, imgs, 32)
    want, want_sc, st = ref.execute(keys, wl.manifest, wl.blob, words, sc)
    model = H.PlainModel.load(wl.manifest, wl.blob)
    plan = H.RescalePlan.plan(ctx, model)
    assert plan.planned_rescale_ops == st["rescale_ops"]
    out = H.execute(ctx, model, plan, H.CipherTensor.from_words(ctx, words, sc, shape=wl.input_shape), rk)
    assert out.scale == want_sc
    assert np.array_equal(out.to_words(), want)
