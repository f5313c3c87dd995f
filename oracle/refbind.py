# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE ONLY -- ctypes binding of oracle/_ref/libhenet_ref.so,
the unmodified reference library (/root/reference/proj/include/henet)
compiled by oracle/Makefile.  Imported only by tests/, __graft_entry__.smoke()
and bench.py's reference / cpu_baseline legs; never by the product package.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libhenet_ref.so")

vp = C.c_void_p
u64p = C.POINTER(C.c_uint64)


def available() -> bool:
    return os.path.exists(REF_SO)


def _p(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


_PROTOS = {
    "ref_last_error": (C.c_char_p, []),
    "ref_ctx_create": (vp, [C.c_uint32, u64p, C.c_uint32, C.c_uint64, C.c_double]),
    "ref_ctx_destroy": (None, [vp]),
    "ref_ntt_root": (C.c_uint64, [vp, C.c_uint32]),
    "ref_ntt": (C.c_int, [vp, C.c_uint32, vp, C.c_int]),
    "ref_barrett": (C.c_int, [vp, C.c_uint32, vp, vp, C.c_uint64, C.c_int, vp]),
    "ref_keygen": (vp, [vp, C.c_uint64, C.c_int]),
    "ref_keys_destroy": (None, [vp]),
    "ref_sk_words": (C.c_int, [vp, vp]),
    "ref_rk_words": (C.c_int, [vp, vp]),
    "ref_encrypt_tensor": (C.c_int, [vp, vp, vp, C.c_uint32, C.c_uint64, C.c_uint64, C.c_int, C.c_uint, vp,
                                     C.POINTER(C.c_double)]),
    "ref_decrypt_tensor": (C.c_int, [vp, vp, vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double, C.c_int,
                                     C.c_uint32, vp]),
    "ref_encode_scalar": (C.c_int, [vp, C.c_double, C.c_uint32, C.c_double, vp]),
    "ref_encode_vector": (C.c_int, [vp, vp, C.c_uint32, C.c_uint32, C.c_double, vp]),
    "ref_decode": (C.c_int, [vp, vp, C.c_uint32, C.c_double, vp]),
    "ref_mul_ct_pt_scalar": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double, C.c_int, vp,
                                       C.c_double, vp, C.POINTER(C.c_double)]),
    "ref_add_ct_ct": (C.c_int, [vp, vp, vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double, C.c_int, vp]),
    "ref_add_ct_pt_vector": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double, C.c_int, vp,
                                       C.c_double, vp]),
    "ref_rescale": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double, C.c_int, C.c_uint32, vp,
                              C.POINTER(C.c_double)]),
    "ref_square": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, C.c_double, C.c_int, vp, C.POINTER(C.c_double)]),
    "ref_mul_ct_ct": (C.c_int, [vp, vp, vp, C.c_uint64, C.c_uint32, C.c_double, C.c_double, C.c_int, vp,
                                C.POINTER(C.c_double)]),
    "ref_relinearize": (C.c_int, [vp, vp, vp, C.c_uint64, C.c_uint32, C.c_double, C.c_int, vp]),
    "ref_plan_json": (C.c_int, [vp, C.c_char_p, vp, C.c_uint64, C.c_int, C.c_int, vp, C.c_uint64]),
    "ref_execute": (C.c_int, [vp, vp, C.c_char_p, vp, C.c_uint64, C.c_int, C.c_int, vp, C.c_uint64, C.c_double,
                              C.c_uint, C.c_uint64, vp, C.c_uint64, u64p, C.POINTER(C.c_uint32),
                              C.POINTER(C.c_double), C.POINTER(C.c_double), u64p, u64p]),
    "ref_set_relu_clip": (None, [C.c_double]),
    "ref_put_tensor": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double, C.c_int, vp, C.c_uint32,
                                 vp, C.c_uint64, u64p]),
    "ref_get_tensor": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, u64p, C.POINTER(C.c_uint32),
                                 C.POINTER(C.c_uint32), C.POINTER(C.c_double)]),
    "ref_nonlin_apply": (C.c_int, [vp, vp, C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, vp, C.c_uint64, C.c_uint32,
                                   C.c_double, C.c_int, vp]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(REF_SO + " not built (needs /root/reference; run oracle/Makefile)")
        _lib = C.CDLL(REF_SO)
        for k, (r, a) in _PROTOS.items():
            f = getattr(_lib, k)
            f.restype = r
            f.argtypes = a
    return _lib


class RefError(RuntimeError):
    pass


def _chk(rc):
    if rc != 0:
        raise RefError(lib().ref_last_error().decode())


class RefContext:
    """The reference CkksContext built by field assignment."""

    def __init__(self, n: int, chain: Sequence[int], special: int, scale: float):
        L = lib()
        arr = (C.c_uint64 * len(chain))(*chain)
        self._h = L.ref_ctx_create(n, arr, len(chain), special, float(scale))
        if not self._h:
            raise RefError(L.ref_last_error().decode())
        self.n, self.chain, self.special, self.scale = n, list(chain), special, float(scale)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ref_ctx_destroy(self._h)
            self._h = None

    @property
    def L(self):
        return len(self.chain)

    def ntt_root(self, i):
        return int(lib().ref_ntt_root(self._h, i))

    def ntt(self, basis_index: int, limb: np.ndarray, inverse=False) -> np.ndarray:
        a = np.ascontiguousarray(limb, dtype=np.uint64).copy()
        _chk(lib().ref_ntt(self._h, basis_index, _p(a), int(inverse)))
        return a

    def barrett(self, basis_index, lo, hi=None, b64=False):
        lo = np.ascontiguousarray(lo, dtype=np.uint64)
        hi = np.ascontiguousarray(hi if hi is not None else np.zeros_like(lo), dtype=np.uint64)
        out = np.empty_like(lo)
        _chk(lib().ref_barrett(self._h, basis_index, _p(lo), _p(hi), lo.size, int(b64), _p(out)))
        return out

    def keygen(self, seed: int, with_relin=True) -> "RefKeys":
        h = lib().ref_keygen(self._h, seed, int(with_relin))
        if not h:
            raise RefError(lib().ref_last_error().decode())
        return RefKeys(self, h, with_relin)

    def encrypt_tensor(self, keys, samples: np.ndarray, seed: int, packing=0, threads=0):
        """samples: (batch, count) -> words (count, 2, L, N), scale"""
        s = np.ascontiguousarray(samples, dtype=np.float64)
        batch, count = s.shape
        out = np.empty((count, 2, self.L, self.n), dtype=np.uint64)
        sc = C.c_double()
        _chk(lib().ref_encrypt_tensor(self._h, keys._h, _p(s), batch, count, seed, packing,
                                      threads or os.cpu_count() or 1, _p(out), C.byref(sc)))
        return out, sc.value

    def decrypt_tensor(self, keys, words: np.ndarray, scale: float, packing: int, batch: int) -> np.ndarray:
        w = np.ascontiguousarray(words, dtype=np.uint64)
        count, polys, level, _ = w.shape
        out = np.empty((batch, count), dtype=np.float64)
        _chk(lib().ref_decrypt_tensor(self._h, keys._h, _p(w), count, polys, level, scale, packing, batch, _p(out)))
        return out

    def encode_scalar(self, value, level, scale):
        out = np.empty(level, dtype=np.uint64)
        _chk(lib().ref_encode_scalar(self._h, float(value), level, float(scale), _p(out)))
        return out

    def encode_vector(self, slots, level, scale):
        s = np.asarray(slots, dtype=np.complex128)
        ri = np.ascontiguousarray(np.stack([s.real, s.imag], axis=-1).reshape(-1))
        out = np.empty((level, self.n), dtype=np.uint64)
        _chk(lib().ref_encode_vector(self._h, _p(ri), s.size, level, float(scale), _p(out)))
        return out

    def decode(self, words, scale):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        out = np.empty(self.n, dtype=np.float64)
        _chk(lib().ref_decode(self._h, _p(w), w.shape[0], float(scale), _p(out)))
        return out[0::2] + 1j * out[1::2]

    def mul_ct_pt_scalar(self, words, scale, residues, pt_scale, packing=0):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        count, polys, level, _ = w.shape
        r = np.ascontiguousarray(residues, dtype=np.uint64)
        out = np.empty_like(w)
        sc = C.c_double()
        _chk(lib().ref_mul_ct_pt_scalar(self._h, _p(w), count, polys, level, scale, packing, _p(r), pt_scale,
                                        _p(out), C.byref(sc)))
        return out, sc.value

    def add_ct_ct(self, a, b, scale, packing=0):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        b = np.ascontiguousarray(b, dtype=np.uint64)
        count, polys, level, _ = a.shape
        out = np.empty_like(a)
        _chk(lib().ref_add_ct_ct(self._h, _p(a), _p(b), count, polys, level, scale, packing, _p(out)))
        return out

    def add_ct_pt_vector(self, words, scale, pt_words, pt_scale, packing=0):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        count, polys, level, _ = w.shape
        p = np.ascontiguousarray(pt_words, dtype=np.uint64)
        out = np.empty_like(w)
        _chk(lib().ref_add_ct_pt_vector(self._h, _p(w), count, polys, level, scale, packing, _p(p), pt_scale, _p(out)))
        return out

    def rescale(self, words, scale, target, packing=0):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        count, polys, level, n = w.shape
        out = np.empty((count, polys, target, n), dtype=np.uint64)
        sc = C.c_double()
        _chk(lib().ref_rescale(self._h, _p(w), count, polys, level, scale, packing, target, _p(out), C.byref(sc)))
        return out, sc.value

    def square(self, words, scale, packing=0):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        count, _, level, n = w.shape
        out = np.empty((count, 3, level, n), dtype=np.uint64)
        sc = C.c_double()
        _chk(lib().ref_square(self._h, _p(w), count, level, scale, packing, _p(out), C.byref(sc)))
        return out, sc.value

    def mul_ct_ct(self, a, b, scale_a, scale_b, packing=0):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        b = np.ascontiguousarray(b, dtype=np.uint64)
        count, _, level, n = a.shape
        out = np.empty((count, 3, level, n), dtype=np.uint64)
        sc = C.c_double()
        _chk(lib().ref_mul_ct_ct(self._h, _p(a), _p(b), count, level, scale_a, scale_b, packing, _p(out), C.byref(sc)))
        return out, sc.value

    def relinearize(self, keys, words, scale, packing=0):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        count, _, level, n = w.shape
        out = np.empty((count, 2, level, n), dtype=np.uint64)
        _chk(lib().ref_relinearize(self._h, keys._h, _p(w), count, level, scale, packing, _p(out)))
        return out

    def plan(self, manifest: str, blob: bytes, mode=0, patch=False) -> dict:
        buf = C.create_string_buffer(1 << 20)
        b = np.frombuffer(blob, dtype=np.uint8) if blob else np.zeros(1, np.uint8)
        _chk(lib().ref_plan_json(self._h, manifest.encode(), _p(b), len(blob), mode, int(patch), buf, len(buf)))
        return json.loads(buf.value.decode())

    def execute(self, keys, manifest: str, blob: bytes, in_words: np.ndarray, in_scale: float, mode=0, patch=False,
                threads=0, refresh_seed=0, out_capacity=None):
        w = np.ascontiguousarray(in_words, dtype=np.uint64)
        count = w.shape[0]
        cap = out_capacity or (w.size * 4)
        out = np.empty(cap, dtype=np.uint64)
        b = np.frombuffer(blob, dtype=np.uint8) if blob else np.zeros(1, np.uint8)
        oc, ol, osc, ms, rs, rl = C.c_uint64(), C.c_uint32(), C.c_double(), C.c_double(), C.c_uint64(), C.c_uint64()
        _chk(lib().ref_execute(self._h, keys._h if keys else None, manifest.encode(), _p(b), len(blob), mode,
                               int(patch), _p(w), count, in_scale, threads, refresh_seed, _p(out), cap,
                               C.byref(oc), C.byref(ol), C.byref(osc), C.byref(ms), C.byref(rs), C.byref(rl)))
        n_words = oc.value * 2 * ol.value * self.n
        res = out[:n_words].reshape(oc.value, 2, ol.value, self.n).copy()
        return res, osc.value, dict(exec_ms=ms.value, rescale_ops=rs.value, relin_ops=rl.value)

    def put_tensor(self, words, scale, packing=0, dims=None) -> bytes:
        """detail::put_tensor (henet/protocol.hpp:335-344): the wire bytes of a CipherTensor."""
        w = np.ascontiguousarray(words, dtype=np.uint64)
        count, polys, level, _ = w.shape
        d = np.ascontiguousarray(dims if dims is not None else [count], dtype=np.uint32)
        n = C.c_uint64()
        _chk(lib().ref_put_tensor(self._h, _p(w), count, polys, level, scale, packing, _p(d), d.size, None, 0,
                                  C.byref(n)))
        out = np.empty(n.value, dtype=np.uint8)
        _chk(lib().ref_put_tensor(self._h, _p(w), count, polys, level, scale, packing, _p(d), d.size, _p(out),
                                  out.size, C.byref(n)))
        return out.tobytes()

    def get_tensor(self, data: bytes):
        """detail::get_tensor (henet/protocol.hpp:346-358) -> (words, scale)."""
        b = np.frombuffer(data, dtype=np.uint8)
        cap = b.size // 8 + 1
        out = np.empty(cap, dtype=np.uint64)
        cnt, polys, level, sc = C.c_uint64(), C.c_uint32(), C.c_uint32(), C.c_double()
        _chk(lib().ref_get_tensor(self._h, _p(b), b.size, _p(out), cap, C.byref(cnt), C.byref(polys), C.byref(level),
                                  C.byref(sc)))
        nw = cnt.value * polys.value * level.value * self.n
        return out[:nw].reshape(cnt.value, polys.value, level.value, self.n).copy(), sc.value

    def nonlin_apply(self, keys, kind, window, layer_seq, refresh_seed, words, scale, packing):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        count, _, level, n = w.shape
        groups = count // window
        out = np.empty((groups, 2, self.L, n), dtype=np.uint64)
        _chk(lib().ref_nonlin_apply(self._h, keys._h, kind, window, layer_seq, refresh_seed, _p(w), count, level,
                                    scale, packing, _p(out)))
        return out


def set_relu_clip(hi: float) -> None:
    """Relu nodes clamp to [0, hi] in the reference-side providers (config 4's ReLU6,
    SURVEY H8); 0 restores plain ReLU."""
    lib().ref_set_relu_clip(float(hi))


class RefKeys:
    def __init__(self, ctx: RefContext, h, with_relin: bool):
        self.ctx, self._h, self.with_relin = ctx, h, with_relin

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ref_keys_destroy(self._h)
            self._h = None

    def sk_words(self) -> np.ndarray:
        full = self.ctx.L + (1 if self.ctx.special else 0)
        out = np.empty((full, self.ctx.n), dtype=np.uint64)
        _chk(lib().ref_sk_words(self._h, _p(out)))
        return out

    def rk_words(self) -> np.ndarray:
        L = self.ctx.L
        out = np.empty((L, 2, L + 1, self.ctx.n), dtype=np.uint64)
        _chk(lib().ref_rk_words(self._h, _p(out)))
        return out
