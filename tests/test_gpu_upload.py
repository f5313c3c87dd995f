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
