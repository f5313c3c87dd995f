# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE ONLY -- ctypes binding of oracle/liboracle.so, the plain-C
restatement of the reference algorithms (oracle/henet_oracle.c).  Imported only by
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.  If the shared
object is missing it is rebuilt from source with the system C compiler (the
restatement has no dependency on /root/reference).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "liboracle.so")
vp = C.c_void_p
u64p = C.POINTER(C.c_uint64)

_PROTOS = {
    "oc_ctx_create": (vp, [C.c_uint32, u64p, C.c_uint32, C.c_uint64, C.c_double]),
    "oc_ctx_destroy": (None, [vp]),
    "oc_ntt_root": (C.c_uint64, [vp, C.c_uint32]),
    "oc_barrett_reduce_128": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64]),
    "oc_barrett_reduce_64": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "oc_ntt_forward": (None, [vp, C.c_uint32, vp]),
    "oc_ntt_inverse": (None, [vp, C.c_uint32, vp]),
    "oc_encode_scalar": (C.c_int, [vp, C.c_double, C.c_uint32, C.c_double, vp]),
    "oc_encode_vector": (C.c_int, [vp, vp, C.c_uint32, C.c_uint32, C.c_double, vp]),
    "oc_decode": (None, [vp, vp, C.c_uint32, C.c_double, vp]),
    "oc_add_ct_ct": (None, [vp, vp, vp, C.c_uint32, C.c_uint32, vp]),
    "oc_mul_ct_pt_scalar": (None, [vp, vp, C.c_uint32, C.c_uint32, vp, vp]),
    "oc_add_ct_pt_vector": (None, [vp, vp, C.c_uint32, C.c_uint32, vp, vp]),
    "oc_square": (None, [vp, vp, C.c_uint32, vp]),
    "oc_mul_ct_ct": (None, [vp, vp, vp, C.c_uint32, vp]),
    "oc_relinearize": (None, [vp, vp, C.c_uint32, vp, vp]),
    "oc_rescale": (C.c_int, [vp, vp, C.c_uint32, C.c_uint32, C.c_uint32, vp]),
    "oc_derive_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "oc_keygen": (None, [vp, C.c_uint64, vp, vp]),
    "oc_encrypt_batch": (C.c_int, [vp, vp, vp, C.c_uint32, C.c_int, C.c_uint64, vp]),
    "oc_decrypt": (None, [vp, vp, vp, C.c_uint32, C.c_uint32, C.c_double, vp]),
    "oc_dense": (C.c_int, [vp, vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, vp, vp, C.c_int, C.c_int, vp,
                           C.c_uint32, vp]),
    "oc_conv": (C.c_int, [vp, vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                          C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, vp, vp, C.c_int,
                          C.c_int, vp, C.c_uint32, vp]),
    "oc_square_layer": (None, [vp, vp, C.c_uint64, C.c_uint32, vp, C.c_int, vp]),
    "oc_dense_lazy": (C.c_int, [vp, vp, C.c_uint32, C.c_uint32, C.c_uint32, vp, C.c_int, vp]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            subprocess.run(["make", "-C", HERE, "liboracle.so"], check=True, capture_output=True)
        _lib = C.CDLL(SO)
        for k, (r, a) in _PROTOS.items():
            f = getattr(_lib, k)
            f.restype = r
            f.argtypes = a
    return _lib


def _p(a):
    return C.c_void_p(a.ctypes.data)


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


class OracleError(RuntimeError):
    """The restatement's counterpart of henet::ValidationError."""


class OracleContext:
    def __init__(self, n: int, chain: Sequence[int], special: int, scale: float):
        arr = (C.c_uint64 * len(chain))(*chain)
        self._h = lib().oc_ctx_create(n, arr, len(chain), special, float(scale))
        self.n, self.chain, self.special, self.scale = n, list(chain), special, float(scale)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.oc_ctx_destroy(self._h)
            self._h = None

    @property
    def L(self):
        return len(self.chain)

    @property
    def full(self):
        return self.L + (1 if self.special else 0)

    def ntt_root(self, i):
        return int(lib().oc_ntt_root(self._h, i))

    def ntt(self, basis_index, limb, inverse=False):
        a = _u64(limb).copy()
        (lib().oc_ntt_inverse if inverse else lib().oc_ntt_forward)(self._h, basis_index, _p(a))
        return a

    def encode_scalar(self, value, level, scale):
        out = np.empty(level, dtype=np.uint64)
        if lib().oc_encode_scalar(self._h, float(value), level, float(scale), _p(out)):
            raise OracleError("encode_scalar: scaled magnitude out of range")
        return out

    def encode_scalars(self, values, level, scale):
        return np.stack([self.encode_scalar(v, level, scale) for v in np.asarray(values).reshape(-1)])

    def encode_vector(self, slots, level, scale):
        s = np.asarray(slots, dtype=np.complex128)
        ri = np.ascontiguousarray(np.stack([s.real, s.imag], -1).reshape(-1))
        out = np.empty((level, self.n), dtype=np.uint64)
        if lib().oc_encode_vector(self._h, _p(ri), s.size, level, float(scale), _p(out)):
            raise OracleError("encode_vector: scaled magnitude out of range")
        return out

    def decode(self, words, scale):
        w = _u64(words)
        out = np.empty(self.n, dtype=np.float64)
        lib().oc_decode(self._h, _p(w), w.shape[0], float(scale), _p(out))
        return out[0::2] + 1j * out[1::2]

    # ---- ciphertext ops; inputs (count, polys, level, N) ----
    def _each(self, words, fn, out_shape):
        w = _u64(words)
        out = np.empty((w.shape[0],) + out_shape, dtype=np.uint64)
        for e in range(w.shape[0]):
            fn(w[e], out[e])
        return out

    def mul_ct_pt_scalar(self, words, residues):
        w = _u64(words)
        r = _u64(residues)
        _, polys, level, n = w.shape
        return self._each(w, lambda a, o: lib().oc_mul_ct_pt_scalar(self._h, _p(a), polys, level, _p(r), _p(o)),
                          (polys, level, n))

    def add_ct_ct(self, a, b):
        a = _u64(a)
        b = _u64(b)
        cnt, polys, level, n = a.shape
        out = np.empty_like(a)
        for e in range(cnt):
            lib().oc_add_ct_ct(self._h, _p(a[e]), _p(b[e]), polys, level, _p(out[e]))
        return out

    def add_ct_pt_vector(self, words, pt):
        w = _u64(words)
        p = _u64(pt)
        _, polys, level, n = w.shape
        return self._each(w, lambda a, o: lib().oc_add_ct_pt_vector(self._h, _p(a), polys, level, _p(p), _p(o)),
                          (polys, level, n))

    def square(self, words):
        w = _u64(words)
        _, _, level, n = w.shape
        return self._each(w, lambda a, o: lib().oc_square(self._h, _p(a), level, _p(o)), (3, level, n))

    def mul_ct_ct(self, a, b):
        a = _u64(a)
        b = _u64(b)
        cnt, _, level, n = a.shape
        out = np.empty((cnt, 3, level, n), dtype=np.uint64)
        for e in range(cnt):
            lib().oc_mul_ct_ct(self._h, _p(a[e]), _p(b[e]), level, _p(out[e]))
        return out

    def relinearize(self, words3, rk):
        w = _u64(words3)
        k = _u64(rk)
        _, _, level, n = w.shape
        return self._each(w, lambda a, o: lib().oc_relinearize(self._h, _p(a), level, _p(k), _p(o)), (2, level, n))

    def rescale(self, words, target):
        w = _u64(words)
        _, polys, level, n = w.shape
        out = np.empty((w.shape[0], polys, target, n), dtype=np.uint64)
        for e in range(w.shape[0]):
            if lib().oc_rescale(self._h, _p(w[e]), polys, level, target, _p(out[e])):
                raise OracleError("bad rescale target")
        return out

    # ---- client side ----
    def derive_seed(self, seed, tag):
        return int(lib().oc_derive_seed(seed, tag))

    def keygen(self, seed, with_relin=True):
        sk = np.empty((self.full, self.n), dtype=np.uint64)
        rk = np.empty((self.L, 2, self.L + 1, self.n), dtype=np.uint64) if with_relin and self.special else None
        lib().oc_keygen(self._h, seed, _p(sk), _p(rk) if rk is not None else None)
        return sk, rk

    def encrypt_tensor(self, sk, samples, seed, packing=0):
        """encrypt_tensor (henet/graph.hpp:68-91): samples (batch, count)."""
        s = np.asarray(samples, dtype=np.float64)
        batch, count = s.shape
        out = np.empty((count, 2, self.L, self.n), dtype=np.uint64)
        skw = _u64(sk)
        for e in range(count):
            vals = np.ascontiguousarray(s[:, e])
            if lib().oc_encrypt_batch(self._h, _p(skw), _p(vals), batch, packing, self.derive_seed(seed, e),
                                      _p(out[e])):
                raise OracleError("encrypt: encode failed")
        return out

    def decrypt_tensor(self, sk, words, scale, packing, batch):
        w = _u64(words)
        cnt, polys, level, n = w.shape
        out = np.empty((batch, cnt))
        buf = np.empty(self.n, dtype=np.float64)
        skw = _u64(sk)
        for e in range(cnt):
            lib().oc_decrypt(self._h, _p(skw), _p(w[e]), polys, level, float(scale), _p(buf))
            slots = buf[0::2] + 1j * buf[1::2]
            if packing == 0:
                out[:, e] = slots[:batch].real
            else:
                k = batch // 2
                out[:k, e] = slots[:k].real
                out[k:, e] = slots[:k].imag
        return out

    # ---- graph layers ----
    def dense(self, x, w, level, x_scale, bias=None, packing=0, rescale=True, outputs=None):
        x = _u64(x)
        w = np.ascontiguousarray(w, dtype=np.float32)
        K, M = w.shape
        b = np.ascontiguousarray(bias, dtype=np.float32) if bias is not None else None
        outs = np.ascontiguousarray(outputs, dtype=np.uint32) if outputs is not None else None
        cnt = len(outs) if outs is not None else M
        lo = level - 1 if rescale else level
        out = np.empty((cnt, 2, lo, self.n), dtype=np.uint64)
        if lib().oc_dense(self._h, _p(x), K, M, level, float(x_scale), _p(w), _p(b) if b is not None else None,
                          packing, int(rescale), _p(outs) if outs is not None else None, cnt, _p(out)):
            raise OracleError("dense: validation error")
        return out

    def dense_lazy(self, x, w, level, rescale=True):
        """oc_dense without a bias, 128-bit sums reduced once (large-K checks)."""
        x = _u64(x)
        w = np.ascontiguousarray(w, dtype=np.float32)
        K, M = w.shape
        lo = level - 1 if rescale else level
        out = np.empty((M, 2, lo, self.n), dtype=np.uint64)
        if lib().oc_dense_lazy(self._h, _p(x), K, M, level, _p(w), int(rescale), _p(out)):
            raise OracleError("dense_lazy: validation error")
        return out

    def conv(self, x, w, in_shape, stride, pad, level, x_scale, bias=None, packing=0, rescale=True, outputs=None):
        x = _u64(x)
        w = np.ascontiguousarray(w, dtype=np.float32)
        F, Cc, win, _ = w.shape
        _, IH, IW = in_shape
        OH = (IH + pad[0] + pad[2] - win) // stride + 1
        OW = (IW + pad[1] + pad[3] - win) // stride + 1
        b = np.ascontiguousarray(bias, dtype=np.float32) if bias is not None else None
        outs = np.ascontiguousarray(outputs, dtype=np.uint32) if outputs is not None else None
        cnt = len(outs) if outs is not None else F * OH * OW
        lo = level - 1 if rescale else level
        out = np.empty((cnt, 2, lo, self.n), dtype=np.uint64)
        if lib().oc_conv(self._h, _p(x), Cc, IH, IW, F, win, stride, pad[0], pad[1], OH, OW, level, float(x_scale),
                         _p(w), _p(b) if b is not None else None, packing, int(rescale),
                         _p(outs) if outs is not None else None, cnt, _p(out)):
            raise OracleError("conv: validation error")
        return out

    def square_layer(self, x, rk, rescale=True):
        x = _u64(x)
        cnt, _, level, n = x.shape
        lo = level - 1 if rescale else level
        out = np.empty((cnt, 2, lo, n), dtype=np.uint64)
        lib().oc_square_layer(self._h, _p(x), cnt, level, _p(_u64(rk)), int(rescale), _p(out))
        return out


def barrett_128(lo, hi, q):
    return int(lib().oc_barrett_reduce_128(lo, hi, q))


def barrett_64(z, q):
    return int(lib().oc_barrett_reduce_64(z, q))
