# SPDX-License-Identifier: Apache-2.0
"""Wire format: put_tensor / get_tensor (henet/protocol.hpp:335-358)
around serialize_ciphertext (henet/serialize.hpp:95-124).  The reference's own serializer
(oracle/_ref) produces the bytes; hg_tensor_deserialize must land them on the device
unchanged, hg_tensor_serialize must reproduce them byte for byte, and malformed messages
must fail with the reference's messages."""
import struct

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
    return dict(p=p, ctx=ctx, ref=ref)


@pytest.mark.parametrize("count,polys,level,packing,dims", [(784, 2, 6, 0, [1, 28, 28]), (10, 2, 2, 1, [10]),
                                                            (3, 3, 5, 0, [3]), (1, 2, 1, 0, [])])
def test_wire_round_trip_bit_exact(env, count, polys, level, packing, dims):
    ctx, ref, p = env["ctx"], env["ref"], env["p"]
    w = W.random_ciphertexts(p, count, seed=count + level, level=level)
    if polys == 3:
        w = np.concatenate([w, W.random_ciphertexts(p, count, seed=5, level=level)[:, :1]], axis=1)
    sc = 2.0 ** 48 / 16760833.0
    data = ref.put_tensor(w, sc, packing, dims)
    t = H.CipherTensor.deserialize(env["ctx"], data)
    assert t.info()[:5] == (count, polys, level, sc, packing)
    assert t.shape == (dims if dims else [])
    assert np.array_equal(t.to_words(), w)
    out = t.serialize()
    assert out == data
    back, bsc = ref.get_tensor(out)
    assert bsc == sc and np.array_equal(back, w)


def _msg(env, **kw):
    p = env["p"]
    w = W.random_ciphertexts(p, 2, seed=1, level=3)
    return bytearray(env["ref"].put_tensor(w, 2.0 ** 24, 0, [2])), w


def test_wire_rejects_like_reference(env):
    ctx, p = env["ctx"], env["p"]
    data, w = _msg(env)
    hdr = 1 + 4 + 4 + 8  # ndims, dims[0], count, first ciphertext length
    cases = []
    bad = bytearray(data); bad[hdr] = ord("X"); cases.append((bad, "bad magic"))
    bad = bytearray(data); bad[hdr + 4] = 2; cases.append((bad, "unsupported wire version"))
    bad = bytearray(data); struct.pack_into("<I", bad, hdr + 5, 4096); cases.append((bad, "degree does not match"))
    bad = bytearray(data); struct.pack_into("<Q", bad, hdr + 20, 17); cases.append((bad, "modulus list does not match"))
    bad = bytearray(data); bad[hdr + 19] = 4; cases.append((bad, "2 or 3 polynomials"))
    bad = bytearray(data); bad[hdr + 10] = 2; cases.append((bad, "unknown packing mode"))
    bad = bytearray(data); struct.pack_into("<d", bad, hdr + 11, -1.0); cases.append((bad, "scale must be positive"))
    bad = bytearray(data); struct.pack_into("<I", bad, 5, 3); cases.append((bad, "element count mismatch"))
    cases.append((bytearray(data[:-5]), "truncated"))
    words_at = hdr + 20 + 8 * 3
    bad = bytearray(data); struct.pack_into("<Q", bad, words_at + 8 * 100, p["chain"][0]); cases.append((bad, "out of range"))
    for b, msg in cases:
        with pytest.raises(H.ValidationError, match=msg):
            H.CipherTensor.deserialize(ctx, bytes(b))
        with pytest.raises(Exception, match=msg):
            env["ref"].get_tensor(bytes(b))


@pytest.mark.parametrize("ct_len", [2 ** 64 - 1, 2 ** 64 - 8, None])
def test_wire_rejects_oversized_ciphertext_length(env, ct_len):
    """A ciphertext length field past the end of the message (or near 2^64, where pos + len
    would wrap) is 'truncated', never a read outside the buffer."""
    data, _ = _msg(env)
    hdr = 1 + 4 + 4  # ndims, dims[0], count
    bad = bytearray(data)
    remaining = len(data) - hdr - 8
    struct.pack_into("<Q", bad, hdr, ct_len if ct_len is not None else remaining + 1)
    with pytest.raises(H.ValidationError, match="truncated"):
        H.CipherTensor.deserialize(env["ctx"], bytes(bad))
