# SPDX-License-Identifier: Apache-2.0
"""Python mirror of the reference ``henet`` API for the encrypted-inference hot
path, over the C ABI (include/henet_b200.h).

Names, argument meaning and error behaviour follow the reference headers
(proj/include/henet/*.hpp, cited per function).  Ciphertexts live in HBM as
``CipherTensor`` batches; residues cross the boundary as numpy uint64 arrays
in the reference's RingElement word order ``[elem][poly][limb][N]``.

This module is host plumbing: all arithmetic runs in libhenet_b200.so.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np

from ._lib import NONLIN_FN, CudaError, HeError, UnsupportedError, ValidationError, check, hg_exec_stats, hg_node_desc, lib  # noqa: F401

PACKING_REAL, PACKING_COMPLEX = 0, 1
OPS = {
    "Input": 0, "ConstWeight": 1, "Add": 2, "Multiply": 3, "Square": 4, "Dot": 5,
    "Convolution": 6, "Reshape": 7, "Relu": 8, "MaxPool": 9, "Output": 10,
}
RESCALE_LAZY, RESCALE_NAIVE = 0, 1
SKIP, RESCALE_AFTER = 0, 1
NONLIN_RELU, NONLIN_MAXPOOL = 1, 2


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


class CkksContext:
    """CkksContext (henet/params.hpp:110-167) built from parameter fields, plus
    its device tables.  `special=0` means no key-switching prime."""

    def __init__(self, poly_degree: int, chain: Sequence[int], special: int, default_scale: float, device: int = 0):
        arr = (C.c_uint64 * len(chain))(*chain)
        h = C.c_void_p()
        check(lib.hg_ctx_create(poly_degree, arr, len(chain), special, float(default_scale), device, C.byref(h)))
        self._h = h
        self.n = int(poly_degree)
        self.chain = [int(q) for q in chain]
        self.special = int(special)
        self.default_scale = float(default_scale)
        self.device = device

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.hg_ctx_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def degree(self) -> int:
        return self.n

    def slot_count(self) -> int:
        return self.n // 2

    def chain_length(self) -> int:
        return len(self.chain)

    def modulus(self, i: int) -> int:
        return self.chain[i]

    def ntt_root(self, basis_index: int) -> int:
        r = C.c_uint64()
        check(lib.hg_ctx_ntt_root(self._h, basis_index, C.byref(r)))
        return r.value

    def stream(self) -> int:
        return lib.hg_ctx_stream(self._h)

    def synchronize(self) -> None:
        check(lib.hg_ctx_synchronize(self._h))

    def launch_count(self) -> int:
        return int(lib.hg_ctx_launch_count(self._h))


class CipherTensor:
    """Device-resident batch of ciphertexts (CipherTensor, henet/graph.hpp:50-60)."""

    def __init__(self, ctx: CkksContext, count: int, polys: int = 2, level: Optional[int] = None,
                 scale: float = 1.0, packing: int = PACKING_REAL, shape: Optional[Sequence[int]] = None,
                 _handle=None):
        self.ctx = ctx
        if _handle is not None:
            self._h = _handle
        else:
            h = C.c_void_p()
            check(lib.hg_tensor_create(ctx.handle, count, polys, level or ctx.chain_length(), float(scale), packing,
                                       C.byref(h)))
            self._h = h
        if shape is not None:
            self.set_shape(shape)

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.hg_tensor_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def info(self):
        cnt, polys, level, scale, packing = C.c_uint64(), C.c_uint32(), C.c_uint32(), C.c_double(), C.c_int()
        check(lib.hg_tensor_info(self._h, C.byref(cnt), C.byref(polys), C.byref(level), C.byref(scale), C.byref(packing)))
        return cnt.value, polys.value, level.value, scale.value, packing.value

    @property
    def count(self) -> int:
        return self.info()[0]

    @property
    def polys(self) -> int:
        return self.info()[1]

    @property
    def level(self) -> int:
        return self.info()[2]

    @property
    def scale(self) -> float:
        return self.info()[3]

    @property
    def packing(self) -> int:
        return self.info()[4]

    @property
    def shape(self) -> List[int]:
        dims = (C.c_uint32 * 8)()
        n = C.c_uint32(8)
        check(lib.hg_tensor_get_shape(self._h, dims, C.byref(n)))
        return [dims[i] for i in range(n.value)]

    def set_shape(self, shape: Sequence[int]) -> None:
        arr = (C.c_uint32 * len(shape))(*shape)
        check(lib.hg_tensor_set_shape(self._h, arr, len(shape)))

    def set_scale(self, scale: float) -> None:
        check(lib.hg_tensor_set_scale(self._h, float(scale)))

    @classmethod
    def from_words(cls, ctx: CkksContext, words: np.ndarray, scale: float, packing: int = PACKING_REAL,
                   shape: Optional[Sequence[int]] = None, polys: Optional[int] = None) -> "CipherTensor":
        """words: uint64 array reshapeable to (count, polys, level, N)."""
        w = np.ascontiguousarray(words, dtype=np.uint64)
        n = ctx.n
        if polys is None:
            polys = w.shape[1] if w.ndim == 4 else 2
        level = w.shape[2] if w.ndim == 4 else None
        if level is None:
            raise ValueError("words must have shape (count, polys, level, N)")
        count = w.size // (polys * level * n)
        t = cls(ctx, count, polys, level, scale, packing, shape=shape or [count])
        check(lib.hg_tensor_upload(t.handle, _ptr(w), None))
        return t

    def to_words(self) -> np.ndarray:
        cnt, polys, level, _, _ = self.info()
        out = np.empty((cnt, polys, level, self.ctx.n), dtype=np.uint64)
        check(lib.hg_tensor_download(self._h, _ptr(out), None))
        return out

    @classmethod
    def deserialize(cls, ctx: CkksContext, data: bytes) -> "CipherTensor":
        """get_tensor (henet/protocol.hpp:346-358): wire bytes straight into a device tensor."""
        b = np.frombuffer(data, dtype=np.uint8)
        h = C.c_void_p()
        used = C.c_uint64()
        check(lib.hg_tensor_deserialize(ctx.handle, _ptr(b), b.size, C.byref(used), C.byref(h), None))
        return cls(ctx, 0, _handle=h)

    def serialize(self) -> bytes:
        """put_tensor (henet/protocol.hpp:335-344)."""
        out = np.empty(lib.hg_tensor_serialized_size(self._h), dtype=np.uint8)
        check(lib.hg_tensor_serialize(self._h, _ptr(out), out.size, None))
        return out.tobytes()

    def upload_u32(self, words: np.ndarray) -> None:
        w = np.ascontiguousarray(words, dtype=np.uint32)
        check(lib.hg_tensor_upload_u32(self._h, _ptr(w), None))

    def to_u32(self) -> np.ndarray:
        cnt, polys, level, _, _ = self.info()
        out = np.empty((cnt, polys, level, self.ctx.n), dtype=np.uint32)
        check(lib.hg_tensor_download_u32(self._h, _ptr(out), None))
        return out

    def device_ptr(self) -> int:
        return lib.hg_tensor_device_ptr(self._h)

    @property
    def word_bytes(self) -> int:
        """4 (u32 residues) or 8 (u64, contexts with a prime >= 2^30)."""
        return int(lib.hg_tensor_word_bytes(self._h))

    def torch_view(self, device: Optional[int] = None):
        """Zero-copy torch view (count, polys * level * N) of the device residues, int32 or
        int64 by word size (bit patterns; residues are < 2^63).  The view keeps this tensor
        alive.  Work queued on the context stream must be synchronised before the view is
        used on another stream (CkksContext.synchronize())."""
        import torch
        cnt, polys, level, _, _ = self.info()
        wb = self.word_bytes

        class _Cai:
            pass

        cai = _Cai()
        cai.owner = self
        cai.__cuda_array_interface__ = {"shape": (cnt, polys * level * self.ctx.n),
                                        "typestr": "<i8" if wb == 8 else "<i4",
                                        "data": (int(self.device_ptr() or 0), False), "version": 3}
        dev = torch.cuda.current_device() if device is None else device
        return torch.as_tensor(cai, device=f"cuda:{dev}")


class RelinKey:
    """RelinKey (henet/ckks.hpp:25-27) uploaded from serialize_relin_key word order."""

    def __init__(self, ctx: CkksContext, words: np.ndarray):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        h = C.c_void_p()
        check(lib.hg_relin_key_upload(ctx.handle, _ptr(w), w.size, C.byref(h)))
        self._h = h
        self.ctx = ctx

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.hg_relin_key_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h


class SecretKey:
    """SecretKey (henet/ckks.hpp:21-23): s in NTT form over the full basis (chain limbs,
    then the special limb), serialize_secret_key word order; on the device for the GPU
    client side (encrypt_tensor / decrypt / decrypt_tensor)."""

    def __init__(self, ctx: CkksContext, words: np.ndarray):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        h = C.c_void_p()
        check(lib.hg_secret_key_upload(ctx.handle, _ptr(w), w.size, C.byref(h)))
        self._h = h
        self.ctx = ctx

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.hg_secret_key_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h


def encrypt_tensor(ctx: CkksContext, sk: SecretKey, samples: np.ndarray, seed: int, packing: int = PACKING_REAL,
                   shape: Optional[Sequence[int]] = None) -> "CipherTensor":
    """encrypt_tensor (henet/graph.hpp:68-91) on the GPU: samples (batch, count), one
    ciphertext per element, encrypt_batch with derive_seed(seed, e)."""
    s = np.ascontiguousarray(samples, dtype=np.float64)
    batch, count = s.shape
    out = CipherTensor(ctx, count, 2, len(ctx.chain), ctx.default_scale, packing)
    check(lib.hg_encrypt_tensor(ctx.handle, sk.handle, _ptr(s), batch, count, seed, packing, out.handle, None))
    if shape is not None:
        out.set_shape(shape)
    return out


def decrypt(ctx: CkksContext, sk: SecretKey, ct: "CipherTensor") -> np.ndarray:
    """decrypt (henet/ckks.hpp:256-268): plaintext words (count, level, N), NTT domain."""
    out = np.empty((ct.count, ct.level, ctx.n), dtype=np.uint64)
    check(lib.hg_decrypt(ctx.handle, sk.handle, ct.handle, _ptr(out), None))
    return out


def decrypt_tensor(ctx: CkksContext, sk: SecretKey, ct: "CipherTensor", batch: int) -> np.ndarray:
    """decrypt_tensor (henet/graph.hpp:93-103): (batch, count) decoded values."""
    out = np.empty((batch, ct.count), dtype=np.float64)
    check(lib.hg_decrypt_tensor(ctx.handle, sk.handle, ct.handle, batch, _ptr(out), None))
    return out


def shard_range(total: int, rank: int, nranks: int) -> range:
    """hg_shard_range: rank's contiguous block of `total` items (sizes differ by <= 1)."""
    b, c = C.c_uint64(), C.c_uint64()
    check(lib.hg_shard_range(int(total), int(rank), int(nranks), C.byref(b), C.byref(c)))
    return range(b.value, b.value + c.value)


def _load_torch_nccl() -> None:
    """The library resolves NCCL at run time and prefers a copy already in the process:
    load torch's (newer, and the one torch.distributed needs) before the first hg_comm call."""
    try:
        import torch  # noqa: F401  (libtorch_cuda links its bundled libnccl.so.2)
    except Exception:  # pragma: no cover - torch absent: the system NCCL is used
        pass


def comm_unique_id() -> bytes:
    """hg_comm_unique_id (ncclGetUniqueId): create on one rank, send to all."""
    _load_torch_nccl()
    buf = (C.c_uint8 * 128)()
    check(lib.hg_comm_unique_id(buf))
    return bytes(buf)


class Communicator:
    """hg_comm: an NCCL communicator bound to a context's device, one process per GPU."""

    def __init__(self, ctx: CkksContext, unique_id: bytes, nranks: int, rank: int):
        assert len(unique_id) == 128
        _load_torch_nccl()
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        check(lib.hg_comm_create(ctx.handle, buf, int(nranks), int(rank), C.byref(h)))
        self._h, self.ctx, self.nranks, self.rank = h, ctx, nranks, rank

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.hg_comm_destroy(self._h)
            self._h = None

    def allgather(self, local: CipherTensor, total: int) -> CipherTensor:
        """hg_allgather_tensor: every rank's block (shard_range(total, r, n)) of the output
        ciphertexts, gathered in place on the context stream."""
        h = C.c_void_p()
        check(lib.hg_allgather_tensor(self._h, local.handle, int(total), C.byref(h), None))
        return CipherTensor(self.ctx, 0, _handle=h)

    def broadcast(self, t: CipherTensor, root: int = 0) -> None:
        check(lib.hg_broadcast_tensor(self._h, t.handle, int(root), None))


class RefreshEngine:
    """NonlinearityEngine + LocalProvider (henet/graph.hpp:699-752) on the GPU: pass it as
    execute()'s provider; the request never leaves the device."""

    def __init__(self, ctx: CkksContext, sk: SecretKey, seed: int):
        h = C.c_void_p()
        check(lib.hg_refresh_engine_create(ctx.handle, sk.handle, seed, C.byref(h)))
        self._h = h
        self.ctx = ctx
        self.sk = sk

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.hg_refresh_engine_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def set_relu_clip(self, hi: float) -> None:
        """hi > 0: ReLU refreshes clamp to [0, hi] (the client-aided ReLU6 of BASELINE c4)."""
        check(lib.hg_refresh_engine_set_relu_clip(self._h, float(hi)))

    def apply(self, kind: int, window: int, layer_seq: int, request: "CipherTensor") -> "CipherTensor":
        """NonlinearityEngine::apply on a device tensor; returns the fresh encryptions."""
        out = CipherTensor(self.ctx, request.count // window, 2, len(self.ctx.chain), self.ctx.default_scale,
                           request.info()[4])
        check(lib.hg_refresh_engine_apply(self._h, kind, window, layer_seq, request.handle, out.handle))
        return out


def _empty_like(ctx: CkksContext, ct: CipherTensor) -> CipherTensor:
    return CipherTensor(ctx, 0, 2, 1, 1.0)


# ---------------------------------------------------------------------------
# Op level (henet/ckks.hpp)
# ---------------------------------------------------------------------------
def add_ct_ct(ctx, a, b):
    """henet/ckks.hpp:286-290"""
    out = _empty_like(ctx, a)
    check(lib.hg_add_ct_ct(ctx.handle, a.handle, b.handle, out.handle, None))
    return out


def mul_ct_pt_scalar(ctx, ct, residues, pt_scale, per_element=False):
    """henet/ckks.hpp:387-392; residues: (level,) or (count, level) canonical."""
    r = np.ascontiguousarray(residues, dtype=np.uint64)
    out = _empty_like(ctx, ct)
    check(lib.hg_mul_ct_pt_scalar(ctx.handle, ct.handle, _ptr(r), int(per_element), float(pt_scale), out.handle, None))
    return out


def add_ct_pt_scalar(ctx, ct, residues, pt_scale, per_element=False):
    """henet/ckks.hpp:325-330"""
    r = np.ascontiguousarray(residues, dtype=np.uint64)
    out = _empty_like(ctx, ct)
    check(lib.hg_add_ct_pt_scalar(ctx.handle, ct.handle, _ptr(r), int(per_element), float(pt_scale), out.handle, None))
    return out


def add_ct_pt_vector(ctx, ct, pt_words, pt_scale, per_element=False):
    """henet/ckks.hpp:306-311"""
    w = np.ascontiguousarray(pt_words, dtype=np.uint64)
    out = _empty_like(ctx, ct)
    check(lib.hg_add_ct_pt_vector(ctx.handle, ct.handle, _ptr(w), int(per_element), float(pt_scale), out.handle, None))
    return out


def square(ctx, ct):
    """henet/ckks.hpp:424-437"""
    out = _empty_like(ctx, ct)
    check(lib.hg_square(ctx.handle, ct.handle, out.handle, None))
    return out


def mul_ct_ct(ctx, a, b):
    """henet/ckks.hpp:407-422"""
    out = _empty_like(ctx, a)
    check(lib.hg_mul_ct_ct(ctx.handle, a.handle, b.handle, out.handle, None))
    return out


def relinearize(ctx, ct, rk: RelinKey):
    """henet/ckks.hpp:442-499"""
    out = _empty_like(ctx, ct)
    check(lib.hg_relinearize(ctx.handle, ct.handle, rk.handle, out.handle, None))
    return out


def square_relin(ctx, ct, rk: RelinKey, rescale: bool = False):
    """eval_square body, henet/graph.hpp:1003-1004"""
    out = _empty_like(ctx, ct)
    check(lib.hg_square_relin(ctx.handle, ct.handle, rk.handle, int(rescale), out.handle, None))
    return out


def rescale(ctx, ct, target_level):
    """henet/ckks.hpp:504-519"""
    out = _empty_like(ctx, ct)
    check(lib.hg_rescale(ctx.handle, ct.handle, int(target_level), out.handle, None))
    return out


def rescale_next(ctx, ct):
    """henet/ckks.hpp:521-524"""
    if ct.level < 2:
        raise ValidationError("cannot rescale below level 1")
    return rescale(ctx, ct, ct.level - 1)


def ntt_forward(ctx, t: CipherTensor):
    check(lib.hg_ntt_forward(ctx.handle, t.handle, None))


def ntt_inverse(ctx, t: CipherTensor):
    check(lib.hg_ntt_inverse(ctx.handle, t.handle, None))


# ---------------------------------------------------------------------------
# Encoding (henet/encoding.hpp)
# ---------------------------------------------------------------------------
def encode_scalars(ctx, values, level, scale) -> np.ndarray:
    """encode_scalar (henet/encoding.hpp:180-197) for many values: (count, level) residues."""
    v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
    out = np.empty((v.size, level), dtype=np.uint64)
    check(lib.hg_encode_scalars(ctx.handle, _ptr(v), v.size, level, float(scale), _ptr(out)))
    return out


def encode_scalar(ctx, value, level, scale) -> np.ndarray:
    return encode_scalars(ctx, [value], level, scale)[0]


def encode_vectors(ctx, slots: np.ndarray, level, scale) -> np.ndarray:
    """encode_vector (henet/encoding.hpp:144-171) for a (count, n_slots) complex array:
    returns (count, level, N) NTT-domain words."""
    s = np.asarray(slots, dtype=np.complex128)
    if s.ndim == 1:
        s = s[None, :]
    count, n_slots = s.shape
    ri = np.ascontiguousarray(np.stack([s.real, s.imag], axis=-1).reshape(-1))
    out = np.empty((count, level, ctx.n), dtype=np.uint64)
    check(lib.hg_encode_vector(ctx.handle, _ptr(ri), n_slots, count, level, float(scale), _ptr(out)))
    return out


def encode_vector(ctx, slots, level, scale) -> np.ndarray:
    return encode_vectors(ctx, np.asarray(slots)[None, :], level, scale)[0]


def decode_vector(ctx, words: np.ndarray, scale: float) -> np.ndarray:
    """decode_slots (henet/encoding.hpp:223-264) of one (level, N) plaintext: N/2 complex slots."""
    w = np.ascontiguousarray(words, dtype=np.uint64)
    level = w.shape[0]
    out = np.empty(ctx.n, dtype=np.float64)
    check(lib.hg_decode_vector(ctx.handle, _ptr(w), 1, level, float(scale), _ptr(out)))
    return out[0::2] + 1j * out[1::2]


# ---------------------------------------------------------------------------
# Graph level (henet/graph.hpp)
# ---------------------------------------------------------------------------
class PlainModel:
    """PlainModel (henet/graph.hpp:154-182), loaded from the reference's JSON
    manifest + little-endian f32 blob format (load_model, henet/graph.hpp:236-437)."""

    def __init__(self, packing: int = PACKING_REAL):
        h = C.c_void_p()
        check(lib.hg_model_create(packing, C.byref(h)))
        self._h = h
        self.packing = packing
        self.node_ids: List[str] = []

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.hg_model_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def keep_encodings(self, on: bool = True) -> None:
        """Weight encodings persist across executes (the reference's shared WeightEncoder
        after precompile_weights, henet/graph.hpp:595-679); results are identical."""
        check(lib.hg_model_keep_encodings(self._h, int(on)))

    def add_weight(self, name: str, dims: Sequence[int], data: np.ndarray) -> None:
        d = np.ascontiguousarray(data, dtype=np.float32).reshape(-1)
        arr = (C.c_uint32 * len(dims))(*dims)
        check(lib.hg_model_add_weight(self._h, name.encode(), arr, len(dims), _ptr(d)))

    def add_node(self, nid: str, op: str, inputs: Sequence[str] = (), attrs: Optional[dict] = None,
                 weight_ref: str = "", bias_ref: str = "") -> None:
        attrs = attrs or {}
        d = hg_node_desc()
        d.id = nid.encode()
        d.op = OPS[op]
        ins = (C.c_char_p * max(len(inputs), 1))(*[i.encode() for i in inputs])
        d.inputs = ins
        d.n_inputs = len(inputs)
        shp = attrs.get("shape", [])
        sarr = (C.c_uint32 * max(len(shp), 1))(*shp)
        d.shape = sarr
        d.shape_len = len(shp)
        d.stride = attrs.get("stride", 1)
        d.window = attrs.get("window", 0)
        d.filters = attrs.get("filters", 0)
        pad = attrs.get("pad", [0, 0, 0, 0])
        if len(pad) != 4:
            raise ValidationError("pad must be [top, left, bottom, right]")
        for i in range(4):
            d.pad[i] = pad[i]
        d.pool_stride = attrs.get("pool_stride", 0)
        d.weight_ref = weight_ref.encode() if weight_ref else None
        d.bias_ref = bias_ref.encode() if bias_ref else None
        check(lib.hg_model_add_node(self._h, C.byref(d)))
        self.node_ids.append(nid)

    def finalize(self) -> None:
        check(lib.hg_model_finalize(self._h))

    def shape(self, nid: str) -> List[int]:
        dims = (C.c_uint32 * 8)()
        n = C.c_uint32(8)
        check(lib.hg_model_shape(self._h, nid.encode(), dims, C.byref(n)))
        return [dims[i] for i in range(n.value)]

    @classmethod
    def load(cls, manifest: str, blob: bytes) -> "PlainModel":
        j = json.loads(manifest)
        packing = {"real": PACKING_REAL, "complex": PACKING_COMPLEX}[j.get("packing", "real")]
        m = cls(packing)
        for name, entry in j.get("weights", {}).items():
            shape = [int(x) for x in entry["shape"]]
            off = int(entry["offset"])
            cnt = int(np.prod(shape)) if shape else 1
            if off % 4:
                raise ValidationError("weight offset must be 4-byte aligned")
            if off + 4 * cnt > len(blob):
                raise ValidationError("weight blob truncated for entry " + name)
            m.add_weight(name, shape, np.frombuffer(blob, dtype="<f4", count=cnt, offset=off))
        for n in j["nodes"]:
            m.add_node(n["id"], n["op"], n.get("inputs", []), n.get("attrs", {}), n.get("weight_ref", ""),
                       n.get("bias_ref", ""))
        m.finalize()
        return m


class RescalePlan:
    """RescalePlan (henet/graph.hpp:457-461)."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.hg_plan_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @classmethod
    def plan(cls, ctx: CkksContext, model: PlainModel, mode: int = RESCALE_LAZY) -> "RescalePlan":
        """plan_rescaling, henet/graph.hpp:504-584"""
        h = C.c_void_p()
        check(lib.hg_plan_rescaling(ctx.handle, model.handle, mode, C.byref(h)))
        return cls(h)

    @classmethod
    def plan_params(cls, chain: Sequence[int], default_scale: float, model: PlainModel,
                    mode: int = RESCALE_LAZY) -> "RescalePlan":
        """plan_rescaling from the parameter fields only (host logic, no GPU)."""
        arr = (C.c_uint64 * len(chain))(*chain)
        h = C.c_void_p()
        check(lib.hg_plan_rescaling_params(arr, len(chain), float(default_scale), model.handle, mode, C.byref(h)))
        return cls(h)

    @classmethod
    def from_nodes(cls, mode: int, planned: int, nodes: Dict[str, tuple]) -> "RescalePlan":
        """nodes: id -> (decision, level_in, level_out, scale_out)"""
        h = C.c_void_p()
        check(lib.hg_plan_create(mode, planned, C.byref(h)))
        for nid, (dec, lin, lout, sc) in nodes.items():
            check(lib.hg_plan_set_node(h, nid.encode(), dec, lin, lout, float(sc)))
        return cls(h)

    def node(self, nid: str):
        dec, lin, lout, sc = C.c_int(), C.c_uint32(), C.c_uint32(), C.c_double()
        check(lib.hg_plan_get_node(self._h, nid.encode(), C.byref(dec), C.byref(lin), C.byref(lout), C.byref(sc)))
        return dec.value, lin.value, lout.value, sc.value

    @property
    def planned_rescale_ops(self) -> int:
        return int(lib.hg_plan_planned_rescales(self._h))


@dataclass
class ExecutionStats:
    """ExecutionStats, henet/graph.hpp:776-782"""
    rescale_ops: int = 0
    relin_ops: int = 0
    nonlin_elements: int = 0
    wall_ms: float = 0.0
    kernel_launches: int = 0
    layer_ms: List = field(default_factory=list)  # [(node id, ms)] in execution order


# provider(kind, window, layer_seq, request: CipherTensor) -> uint64 words (groups, 2, L, N)
Provider = Callable[[int, int, int, CipherTensor], np.ndarray]


def execute(ctx: CkksContext, model: PlainModel, plan: RescalePlan, inp: CipherTensor,
            relin: Optional[RelinKey] = None, provider: "Optional[Provider | RefreshEngine]" = None,
            stats: Optional[ExecutionStats] = None) -> CipherTensor:
    """execute, henet/graph.hpp:1121-1126 -- the whole graph on the GPU."""
    errors: List[BaseException] = []

    def _cb(user, kind, window, layer_seq, req_h, resp_h):
        try:
            req = CipherTensor(ctx, 0, _handle=C.c_void_p(req_h))
            resp = CipherTensor(ctx, 0, _handle=C.c_void_p(resp_h))
            try:
                words = provider(kind, window, layer_seq, req)
                w = np.ascontiguousarray(words, dtype=np.uint64)
                check(lib.hg_tensor_upload(resp.handle, _ptr(w), None))
            finally:
                req._h = None  # borrowed handles
                resp._h = None
            return 0
        except BaseException as e:  # pragma: no cover - surfaced below
            errors.append(e)
            return 1

    user = None
    if isinstance(provider, RefreshEngine):  # native provider: hg_refresh_engine_apply on the engine
        cb = C.cast(lib.hg_refresh_engine_apply, NONLIN_FN)
        user = provider.handle
    else:
        cb = NONLIN_FN(_cb) if provider is not None else NONLIN_FN()
    out = C.c_void_p()
    st = hg_exec_stats()
    rc = lib.hg_execute(ctx.handle, model.handle, plan.handle, inp.handle, relin.handle if relin else None, cb, user,
                        C.byref(out), C.byref(st) if stats is not None else None, None)
    if errors:
        raise errors[0]
    check(rc)
    if stats is not None:
        stats.rescale_ops = st.rescale_ops
        stats.relin_ops = st.relin_ops
        stats.nonlin_elements = st.nonlin_elements
        stats.wall_ms = st.wall_ms
        stats.kernel_launches = st.kernel_launches
        n = C.c_uint32()
        check(lib.hg_last_exec_layer_count(C.byref(n)))
        stats.layer_ms = []
        for i in range(n.value):
            nid, ms = C.c_char_p(), C.c_double()
            check(lib.hg_last_exec_layer(i, C.byref(nid), C.byref(ms)))
            stats.layer_ms.append((nid.value.decode(), ms.value))
    return CipherTensor(ctx, 0, _handle=out)


def bench_int_peak(device: int = 0, kind: int = 0) -> float:
    """Measured integer-pipe peak, lane-ops/s (kind 0 IMAD, 1 IMAD.WIDE (= one 32x32->64 MAC), 2 IMAD.HI,
    3 Shoup lazy modular product = IMAD.HI + 2 IMAD, 4 int8 tensor-core MAC/s)."""
    v = C.c_double()
    check(lib.hg_bench_int_peak(device, kind, C.byref(v)))
    return v.value


def prof_enable(on: bool = True) -> None:
    """Bracket every kernel launch with CUDA events on its stream."""
    check(lib.hg_prof_enable(int(on)))


def prof_report() -> dict:
    """{kernel: {"ms": total_ms, "launches": n}} since the last report."""
    buf = C.create_string_buffer(1 << 16)
    check(lib.hg_prof_report(buf, len(buf)))
    return json.loads(buf.value.decode())
