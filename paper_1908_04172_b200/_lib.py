# SPDX-License-Identifier: Apache-2.0
"""ctypes binding of the in-tree C ABI library ``libhenet_b200.so``.

The library is the product: every numerical operation runs in its sm_100a
kernels.  There is no fallback -- if the shared library is missing or cannot
be loaded this module raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhenet_b200.so")
# Kernel-variant experiments (scripts/) may point at another build of the same library.
LIB_PATH = os.environ.get("HENET_B200_LIB", LIB_PATH)

HG_OK, HG_ERR_VALIDATION, HG_ERR_CUDA, HG_ERR_UNSUPPORTED, HG_ERR_ALLOC, HG_ERR_INTERNAL = range(6)

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
dblp = C.POINTER(C.c_double)
vp = C.c_void_p


class hg_node_desc(C.Structure):
    _fields_ = [
        ("id", C.c_char_p),
        ("op", C.c_int),
        ("inputs", C.POINTER(C.c_char_p)),
        ("n_inputs", C.c_uint32),
        ("shape", u32p),
        ("shape_len", C.c_uint32),
        ("stride", C.c_uint32),
        ("window", C.c_uint32),
        ("filters", C.c_uint32),
        ("pad", C.c_uint32 * 4),
        ("pool_stride", C.c_uint32),
        ("weight_ref", C.c_char_p),
        ("bias_ref", C.c_char_p),
    ]


class hg_exec_stats(C.Structure):
    _fields_ = [
        ("rescale_ops", C.c_uint64),
        ("relin_ops", C.c_uint64),
        ("nonlin_elements", C.c_uint64),
        ("wall_ms", C.c_double),
        ("kernel_launches", C.c_uint64),
    ]


NONLIN_FN = C.CFUNCTYPE(C.c_int, vp, C.c_int, C.c_uint32, C.c_uint32, vp, vp)

# name -> (restype, argtypes); mirrors include/henet_b200.h
PROTOTYPES = {
    "hg_last_error": (C.c_char_p, []),
    "hg_abi_version": (C.c_int, []),
    "hg_ctx_create": (C.c_int, [C.c_uint32, u64p, C.c_uint32, C.c_uint64, C.c_double, C.c_int, C.POINTER(vp)]),
    "hg_ctx_destroy": (None, [vp]),
    "hg_ctx_ntt_root": (C.c_int, [vp, C.c_uint32, u64p]),
    "hg_ctx_stream": (vp, [vp]),
    "hg_ctx_synchronize": (C.c_int, [vp]),
    "hg_ctx_launch_count": (C.c_uint64, [vp]),
    "hg_tensor_create": (C.c_int, [vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double, C.c_int, C.POINTER(vp)]),
    "hg_tensor_destroy": (None, [vp]),
    "hg_tensor_info": (C.c_int, [vp, u64p, u32p, u32p, dblp, C.POINTER(C.c_int)]),
    "hg_tensor_set_scale": (C.c_int, [vp, C.c_double]),
    "hg_tensor_set_shape": (C.c_int, [vp, u32p, C.c_uint32]),
    "hg_tensor_get_shape": (C.c_int, [vp, u32p, u32p]),
    "hg_tensor_upload": (C.c_int, [vp, vp, vp]),
    "hg_tensor_download": (C.c_int, [vp, vp, vp]),
    "hg_tensor_upload_segments": (C.c_int, [vp, vp, vp]),
    "hg_tensor_assign": (C.c_int, [vp, vp]),
    "hg_shard_range": (C.c_int, [C.c_uint64, C.c_int, C.c_int, u64p, u64p]),
    "hg_comm_unique_id": (C.c_int, [vp]),
    "hg_comm_create": (C.c_int, [vp, vp, C.c_int, C.c_int, C.POINTER(vp)]),
    "hg_comm_destroy": (None, [vp]),
    "hg_allgather_tensor": (C.c_int, [vp, vp, C.c_uint64, C.POINTER(vp), vp]),
    "hg_broadcast_tensor": (C.c_int, [vp, vp, C.c_int, vp]),
    "hg_tensor_download_segments": (C.c_int, [vp, vp, vp]),
    "hg_tensor_upload_u32": (C.c_int, [vp, vp, vp]),
    "hg_tensor_download_u32": (C.c_int, [vp, vp, vp]),
    "hg_tensor_device_ptr": (vp, [vp]),
    "hg_tensor_words": (C.c_uint64, [vp]),
    "hg_tensor_word_bytes": (C.c_uint32, [vp]),
    "hg_relin_key_upload": (C.c_int, [vp, vp, C.c_uint64, C.POINTER(vp)]),
    "hg_relin_key_destroy": (None, [vp]),
    "hg_add_ct_ct": (C.c_int, [vp, vp, vp, vp, vp]),
    "hg_mul_ct_pt_scalar": (C.c_int, [vp, vp, vp, C.c_int, C.c_double, vp, vp]),
    "hg_add_ct_pt_scalar": (C.c_int, [vp, vp, vp, C.c_int, C.c_double, vp, vp]),
    "hg_add_ct_pt_vector": (C.c_int, [vp, vp, vp, C.c_int, C.c_double, vp, vp]),
    "hg_square": (C.c_int, [vp, vp, vp, vp]),
    "hg_mul_ct_ct": (C.c_int, [vp, vp, vp, vp, vp]),
    "hg_relinearize": (C.c_int, [vp, vp, vp, vp, vp]),
    "hg_square_relin": (C.c_int, [vp, vp, vp, C.c_int, vp, vp]),
    "hg_rescale": (C.c_int, [vp, vp, C.c_uint32, vp, vp]),
    "hg_ntt_forward": (C.c_int, [vp, vp, vp]),
    "hg_ntt_inverse": (C.c_int, [vp, vp, vp]),
    "hg_encode_scalars": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, C.c_double, vp]),
    "hg_encode_vector": (C.c_int, [vp, vp, C.c_uint32, C.c_uint64, C.c_uint32, C.c_double, vp]),
    "hg_secret_key_upload": (C.c_int, [vp, vp, C.c_uint64, C.POINTER(vp)]),
    "hg_decode_vector": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, C.c_double, vp]),
    "hg_secret_key_destroy": (None, [vp]),
    "hg_encrypt_tensor": (C.c_int, [vp, vp, vp, C.c_uint32, C.c_uint64, C.c_uint64, C.c_int, vp, vp]),
    "hg_decrypt": (C.c_int, [vp, vp, vp, vp, vp]),
    "hg_decrypt_tensor": (C.c_int, [vp, vp, vp, C.c_uint32, vp, vp]),
    "hg_refresh_engine_create": (C.c_int, [vp, vp, C.c_uint64, C.POINTER(vp)]),
    "hg_model_keep_encodings": (C.c_int, [vp, C.c_int]),
    "hg_tensor_deserialize": (C.c_int, [vp, vp, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(vp), vp]),
    "hg_tensor_serialized_size": (C.c_uint64, [vp]),
    "hg_tensor_serialize": (C.c_int, [vp, vp, C.c_uint64, vp]),
    "hg_refresh_engine_destroy": (None, [vp]),
    "hg_refresh_engine_apply": (C.c_int, [vp, C.c_int, C.c_uint32, C.c_uint32, vp, vp]),
    "hg_refresh_engine_set_relu_clip": (C.c_int, [vp, C.c_double]),
    "hg_model_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "hg_model_destroy": (None, [vp]),
    "hg_model_add_weight": (C.c_int, [vp, C.c_char_p, u32p, C.c_uint32, vp]),
    "hg_model_add_node": (C.c_int, [vp, C.POINTER(hg_node_desc)]),
    "hg_model_finalize": (C.c_int, [vp]),
    "hg_model_node_count": (C.c_int, [vp, u32p]),
    "hg_model_shape": (C.c_int, [vp, C.c_char_p, u32p, u32p]),
    "hg_plan_rescaling": (C.c_int, [vp, vp, C.c_int, C.POINTER(vp)]),
    "hg_plan_rescaling_params": (C.c_int, [u64p, C.c_uint32, C.c_double, vp, C.c_int, C.POINTER(vp)]),
    "hg_plan_create": (C.c_int, [C.c_int, C.c_uint64, C.POINTER(vp)]),
    "hg_plan_set_node": (C.c_int, [vp, C.c_char_p, C.c_int, C.c_uint32, C.c_uint32, C.c_double]),
    "hg_plan_get_node": (C.c_int, [vp, C.c_char_p, C.POINTER(C.c_int), u32p, u32p, dblp]),
    "hg_plan_planned_rescales": (C.c_uint64, [vp]),
    "hg_plan_destroy": (None, [vp]),
    "hg_execute": (C.c_int, [vp, vp, vp, vp, vp, NONLIN_FN, vp, C.POINTER(vp), C.POINTER(hg_exec_stats), vp]),
    "hg_bench_int_peak": (C.c_int, [C.c_int, C.c_int, dblp]),
    "hg_last_exec_node_ms": (C.c_int, [vp, dblp]),
    "hg_last_exec_layer_count": (C.c_int, [u32p]),
    "hg_last_exec_layer": (C.c_int, [C.c_uint32, C.POINTER(C.c_char_p), dblp]),
    "hg_last_upload_h2d_bytes": (C.c_int, [u64p]),
    "hg_prof_enable": (C.c_int, [C.c_int]),
    "hg_prof_report": (C.c_int, [C.c_char_p, C.c_uint64]),
}


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no CPU fallback)"
        )
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class HeError(RuntimeError):
    """Base error of the B200 path."""


class ValidationError(HeError):
    """Mirror of henet::ValidationError (henet/common.hpp:25-28)."""


class CudaError(HeError):
    pass


class UnsupportedError(HeError):
    pass


def check(rc: int) -> None:
    if rc == HG_OK:
        return
    msg = (lib.hg_last_error() or b"").decode()
    if rc == HG_ERR_VALIDATION:
        raise ValidationError(msg)
    if rc == HG_ERR_CUDA:
        raise CudaError(msg)
    if rc == HG_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    raise HeError(f"error {rc}: {msg}")
