# SPDX-License-Identifier: Apache-2.0
"""hg_tensor_upload of reference-format u64 words (henet/serialize.hpp:61-63 word order):
host threads validate each word against its limb's prime and pack it to u32 in 2 MB
chunks, DMA'd as they are packed.  Round trips must be exact across many chunks and
ragged tails, and an out-of-range word anywhere -- first word, a late chunk, a word
>= 2^32 -- must raise the reference's "residue out of range"."""
import numpy as np
import pytest

from paper_1908_04172_b200 import henet as H
from paper_1908_04172_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    p = W.N8192
    return H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])


@pytest.mark.parametrize("count,level", [(1, 1), (3, 6), (97, 5), (300, 6)])
def test_upload_round_trip(ctx, count, level):
    x = W.random_ciphertexts(W.N8192, count, seed=count + level, level=level)
    t = H.CipherTensor.from_words(ctx, x, 1.0)
    assert np.array_equal(t.to_words(), x)
    # re-upload into the same tensor (staging reuse) with different words
    y = W.random_ciphertexts(W.N8192, count, seed=count + level + 1, level=level)
    t2 = H.CipherTensor.from_words(ctx, y, 1.0)
    assert np.array_equal(t2.to_words(), y)


@pytest.mark.parametrize("where", ["first", "late", "wide"])
def test_upload_rejects_out_of_range_any_chunk(ctx, where):
    p = W.N8192
    x = W.random_ciphertexts(p, 120, seed=4)  # 11.8 M words: 23 chunks
    if where == "first":
        x[0, 0, 0, 0] = p["chain"][0]
    elif where == "late":
        x[119, 1, 5, 8191] = p["chain"][5] + 7
    else:
        x[60, 0, 2, 100] = np.uint64(1) << np.uint64(32)
    with pytest.raises(H.ValidationError, match="residue out of range"):
        H.CipherTensor.from_words(ctx, x, 1.0)


def test_upload_max_residues_round_trip(ctx):
    """All-(q - 1) words: the largest 24-bit residue needs all 3 bus bytes (pack24) and the
    30-bit limb all 4."""
    p = W.N8192
    q = np.array(p["chain"], dtype=np.uint64)[None, None, :, None]
    x = np.broadcast_to(q - np.uint64(1), (40, 2, len(p["chain"]), p["n"])).copy()
    t = H.CipherTensor.from_words(ctx, x, 1.0)
    assert np.array_equal(t.to_words(), x)


def test_upload_reports_bus_bytes(ctx):
    """hg_last_upload_h2d_bytes: the raw share (HG_UPLOAD_DIRECT_FRAC of the ciphertexts, u64)
    plus the packed chunks -- 3 bytes per residue of a prime < 2^24 when the host packs 24-bit
    words (AVX-512 VBMI), else 4."""
    import ctypes
    import os
    p = W.N8192
    count, L, n = 300, 6, p["n"]
    x = W.random_ciphertexts(p, count, seed=9, level=L)
    H.CipherTensor.from_words(ctx, x, 1.0)
    got = ctypes.c_uint64(0)
    H.lib.hg_last_upload_h2d_bytes(ctypes.byref(got))
    f = float(os.environ.get("HG_UPLOAD_DIRECT_FRAC", "0.15"))
    direct = int(count * f)
    per_res_4 = 2 * L * n * 4
    per_res_p = 2 * n * sum(3 if q < (1 << 24) else 4 for q in p["chain"][:L])
    raw = direct * 2 * L * n * 8
    if os.environ.get("HG_UPLOAD_DYNAMIC", "1") != "0":
        # dynamic split: the raw share follows the host's packing speed; every word crosses the bus
        # once, packed (3 or 4 bytes) or raw (8 bytes), raw in whole 2 MB chunks
        lo = count * min(per_res_4, per_res_p)
        assert lo <= got.value <= count * 2 * L * n * 8, got.value
        return
    assert got.value in (raw + (count - direct) * per_res_4, raw + (count - direct) * per_res_p), got.value


def test_upload_static_split_round_trip_and_bus_bytes():
    """HG_UPLOAD_DYNAMIC=0 (read once per process, hence the subprocess): the fixed raw share
    -- multi-chunk round trip, an out-of-range word in the raw share and in the packed part,
    and the bus bytes of the fixed split."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = r'''
import ctypes, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
from paper_1908_04172_b200 import henet as H, workloads as W
p = W.N8192
ctx = H.CkksContext(p["n"], p["chain"], p["special"], p["scale"])
count, L, n = 300, 6, p["n"]
x = W.random_ciphertexts(p, count, seed=9, level=L)
t = H.CipherTensor.from_words(ctx, x, 1.0)
assert np.array_equal(t.to_words(), x)
got = ctypes.c_uint64(0)
H.lib.hg_last_upload_h2d_bytes(ctypes.byref(got))
direct = int(count * 0.15)
per4 = 2 * L * n * 4
perp = 2 * n * sum(3 if q < (1 << 24) else 4 for q in p["chain"][:L])
raw = direct * 2 * L * n * 8
assert got.value in (raw + (count - direct) * per4, raw + (count - direct) * perp), got.value
for e in (3, count - 2):  # packed part, raw share (the last 15% of the ciphertexts)
    y = x.copy()
    y[e, 1, 2, 77] = p["chain"][2]
    try:
        H.CipherTensor.from_words(ctx, y, 1.0)
        raise SystemExit("accepted an out-of-range word")
    except H.ValidationError as ex:
        assert "residue out of range" in str(ex)
print("OK")
'''
    env = {**os.environ, "HG_UPLOAD_DYNAMIC": "0", "HG_UPLOAD_DIRECT_FRAC": "0.15"}
    r = subprocess.run([sys.executable, "-c", script, root], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
