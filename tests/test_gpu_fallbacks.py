# SPDX-License-Identifier: Apache-2.0
"""The alternate kernel paths stay bit-exact: each environment switch (read once per
process by the library) selects a different kernel for the same operation, so every case
runs in its own subprocess and compares with the reference (oracle/_ref).

  HG_DENSE_TC=0   Dot on the CUDA-core IMAD kernel instead of the int8 tensor cores
  HG_WIDE_TC=0    the 40-bit limb of a wide Dot on the CUDA-core 128-bit MAC kernel
  HG_CONV_FP64=0  convolution MACs all on IMAD.WIDE (no DFMA split)
  HG_AUX_STREAM=0 special-prime key switch on the main stream
  HG_UPLOAD_HOST_NARROW=0  hg_tensor_upload copies u64 words and narrows them on the GPU
  HG_UPLOAD_DIRECT_FRAC=0 / 1  host packing only / everything raw through the GPU narrowing
  HG_UPLOAD_PACK24=0 / HG_UPLOAD_AVX512=0  u32 bus words / the SSE2 packer
  HG_CONV1X1_DOT=0  1x1 convolutions on the tap-gather kernel instead of the batched Dot
  HG_TC_PPC=3     3 positions per CTA in the batched Dot (ragged last chunk)
  HG_DWCONV=0     depthwise (grouped 1 -> 1) wide convolutions on the tap-gather kernel
  HG_DWCONV_SMEM=0  the depthwise kernel without the shared-memory input tile
  HG_NTT_W32=0    wide NTTs all on the 64-bit transform
  HG_FFT_CLUSTER=0  N = 2^14 encode/decode FFTs on one CTA in global memory (no 2-CTA cluster)
  HG_CRT_FAST=0   the decoder's full Garner CRT for every coefficient
  HG_DEC_FUSE=0 / HG_ENC_FUSE=0  decrypt combine / encrypt combine as separate kernels
  HG_ENCODE_FUSE=0  encode's residues as a separate kernel before the plaintext NTT
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from oracle import refbind as R
from paper_1908_04172_b200 import henet as H, workloads as W

def run(p, wl, seed, keys_relin):
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
    ref = R.RefContext(p["n"], p["chain"], p["special"], p["scale"])
    keys = ref.keygen(5, keys_relin)
    if wl.name.startswith("c5b") or wl.name.startswith("c4"):
        x = W.random_ciphertexts(p, wl.input_count, seed=seed)
        sc = p["scale"]
    else:
        imgs = W.synthetic_images(wl.input_shape, wl.batch, seed)
        x, sc = ref.encrypt_tensor(keys, imgs, seed + 1, packing=wl.packing)
    want, want_sc, st = ref.execute(keys if keys_relin else None, wl.manifest, wl.blob, x, sc,
                                    patch=wl.patch_terminal_rescale)
    rp = ref.plan(wl.manifest, wl.blob, patch=wl.patch_terminal_rescale)
    nodes = {n["id"]: (n["decision"], n["level_in"], n["level_out"],
                       np.array([n["scale_out_bits"]], dtype=np.uint64).view(np.float64)[0]) for n in rp["nodes"]}
    plan = H.RescalePlan.from_nodes(0, rp["planned_rescale_ops"], nodes)
    model = H.PlainModel.load(wl.manifest, wl.blob)
    rk = None
    if keys_relin:
        rk = H.RelinKey(ctx, keys.rk_words())
    out = H.execute(ctx, model, plan, H.CipherTensor.from_words(ctx, x, sc, shape=wl.input_shape), rk)
    assert out.scale == want_sc, (out.scale, want_sc)
    assert np.array_equal(out.to_words(), want)

def c4_linear():
    # the c4 block's linear layers (1x1 expand, 3x3 depthwise pad 1, 1x1 project), ReLU6 removed
    import json
    wl = W.mobilenet_block(hw=4, cin=4, expand=6, cout=3)
    j = json.loads(wl.manifest)
    j["nodes"] = [n for n in j["nodes"] if n["op"] != "Relu"]
    for n in j["nodes"]:
        n["inputs"] = [{"relu6a": "expand", "relu6b": "dw"}.get(i, i) for i in n.get("inputs", [])]
    wl.manifest = json.dumps(j)
    return wl

def c4_refresh():
    # the c4 block on a 4x4 tile with both ReLU6 refreshes on the GPU engine (N = 2^14
    # encrypt / decrypt / FFTs) against the reference executor with the clamp provider
    p = W.N16384
    ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
    ref = R.RefContext(p["n"], p["chain"], p["special"], p["scale"])
    keys = ref.keygen(41, False)
    sk = H.SecretKey(ctx, keys.sk_words())
    wl = W.mobilenet_block(hw=4, cin=4, expand=6, cout=3)
    acts = np.random.default_rng(12).normal(0, 1, (ctx.slot_count(), wl.input_count))
    words, sc = ref.encrypt_tensor(keys, acts, 13)
    R.set_relu_clip(6.0)
    want, want_sc, _ = ref.execute(keys, wl.manifest, wl.blob, words, sc, refresh_seed=77)
    model = H.PlainModel.load(wl.manifest, wl.blob)
    eng = H.RefreshEngine(ctx, sk, 77)
    eng.set_relu_clip(6.0)
    x = H.encrypt_tensor(ctx, sk, acts, 13, shape=wl.input_shape)
    assert np.array_equal(x.to_words(), words)
    out = H.execute(ctx, model, H.RescalePlan.plan(ctx, model), x, None, eng)
    assert out.scale == want_sc
    assert np.array_equal(out.to_words(), want)
    assert np.array_equal(H.decrypt_tensor(ctx, sk, out, 8192), ref.decrypt_tensor(keys, want, want_sc, 0, 8192))

which = sys.argv[2]
if which == "c4refresh":
    c4_refresh()
elif which == "toy":
    run(W.N8192, W.toy_cryptonets(), 3, True)
elif which == "c4lin":
    run(W.N16384, c4_linear(), 5, False)
else:
    run(W.N16384, W.wide_dense(k=96, m=40), 4, False)
print("OK")
'''


@pytest.mark.parametrize("env,which", [
    ({"HG_DENSE_TC": "0"}, "toy"),
    ({"HG_CONV_FP64": "0"}, "toy"),
    ({"HG_AUX_STREAM": "0"}, "toy"),
    ({"HG_UPLOAD_HOST_NARROW": "0"}, "toy"),
    ({"HG_UPLOAD_DIRECT_FRAC": "0"}, "toy"),
    ({"HG_UPLOAD_DIRECT_FRAC": "1"}, "toy"),
    ({"HG_UPLOAD_PACK24": "0"}, "toy"),
    ({"HG_UPLOAD_AVX512": "0", "HG_UPLOAD_PACK24": "0"}, "toy"),
    ({"HG_WIDE_TC": "0"}, "wide"),
    ({"HG_DENSE_TC": "0"}, "wide"),
    ({"HG_CONV1X1_DOT": "0"}, "c4lin"),
    ({"HG_WIDE_TC": "0"}, "c4lin"),
    ({"HG_TC_PPC": "3"}, "c4lin"),
    ({"HG_DWCONV": "0"}, "c4lin"),
    ({"HG_DWCONV_SMEM": "0"}, "c4lin"),
    ({"HG_NTT_W32": "0"}, "c4lin"),
    ({"HG_FFT_CLUSTER": "0"}, "c4refresh"),
    ({"HG_CRT_FAST": "0"}, "c4refresh"),
    ({"HG_DEC_FUSE": "0", "HG_ENC_FUSE": "0"}, "c4refresh"),
    ({"HG_ENCODE_FUSE": "0"}, "c4refresh"),
    ({}, "c4refresh"),
    ({}, "c4lin"),
])
def test_alternate_paths_bit_exact(env, which):
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, which], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
