"""ctypes binding of the C ABI declared in include/iolm_cuda.h.

The product path has exactly one implementation: libiolm_cuda.so (sm_100a). If the library is
missing or cannot be loaded this module raises - there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
ENGINE_SO = PKG / "libiolm_cuda.so"

IOLM_OK = 0
IOLM_E_CONTRACT = 1
IOLM_E_SEQ_TOO_LONG = 2
IOLM_E_UNSUPPORTED = 3
IOLM_E_CUDA = 4
IOLM_E_OOM = 5
IOLM_E_CORRUPT_HEADER = 6
IOLM_E_TRUNCATED_BLOB = 7
IOLM_E_UNKNOWN_ENCODING = 8
IOLM_E_STALE = 9

VOCAB, PAD, BOS, EOS = 131, 128, 129, 130
KCLASSES = ["embed_ln", "gemm_qkv", "attn_prefill", "attn_decode", "gemm_o", "ln", "gemm_in",
            "gemm_out", "head", "quant"]


class Opts(C.Structure):
    _fields_ = [
        ("max_tokens_per_step", C.c_int32),
        ("max_slots", C.c_int32),
        ("page_size", C.c_int32),
        ("act_quant", C.c_int32),
        ("prefix_sharing", C.c_int32),
        ("use_cuda_graph", C.c_int32),
        ("kernel_timing", C.c_int32),
        ("sparse_mma", C.c_int32),
        ("int4_mma", C.c_int32),
        ("prefill_tc", C.c_int32),
        ("reserved", C.c_int32 * 6),
    ]


class ModelConfigC(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("vocab_size", "d_model", "n_layers", "n_heads", "d_ff", "max_seq_len", "head_dim")]


class Stats(C.Structure):
    _fields_ = [
        ("steps", C.c_int64),
        ("tokens", C.c_int64),
        ("prefill_tokens", C.c_int64),
        ("decode_tokens", C.c_int64),
        ("prefix_tokens", C.c_int64),
        ("kernel_launches", C.c_int64),
        ("device_ms", C.c_double),
    ]


# name -> (restype, argtypes); the list is also what the symbol-export test checks.
SIGNATURES = {
    "iolm_cuda_create": (C.c_int, [C.c_void_p, C.c_size_t, C.c_int, C.POINTER(Opts), C.POINTER(C.c_void_p)]),
    "iolm_cuda_destroy": (None, [C.c_void_p]),
    "iolm_cuda_create_multi": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p, C.c_int32, C.POINTER(Opts),
                                         C.POINTER(C.c_void_p)]),
    "iolm_cuda_device_count": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    "iolm_cuda_save_image": (C.c_int, [C.c_void_p, C.c_char_p]),
    "iolm_cuda_create_from_image": (C.c_int, [C.c_char_p, C.c_uint64, C.c_int, C.POINTER(Opts),
                                              C.POINTER(C.c_void_p)]),
    "iolm_cuda_image_info": (C.c_int, [C.c_char_p, C.POINTER(C.c_uint64), C.POINTER(ModelConfigC)]),
    "iolm_cuda_bundle_hash": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    "iolm_cuda_config": (C.c_int, [C.c_void_p, C.POINTER(ModelConfigC)]),
    "iolm_cuda_layer_shape": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "iolm_cuda_layer_heads": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.POINTER(C.c_int32)]),
    "iolm_cuda_decode": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                   C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_int64)]),
    "iolm_cuda_decode_device_ids": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                              C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64),
                                              C.POINTER(C.c_int64)]),
    "iolm_cuda_forward_logits": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                           C.POINTER(C.c_uint64)]),
    "iolm_cuda_forward_capture": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                            C.POINTER(C.c_uint64)]),
    "iolm_cuda_forward_codes": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.POINTER(C.c_uint64)]),
    "iolm_cuda_gram": (C.c_int, [C.c_int, C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_void_p]),
    "iolm_cuda_last_stats": (C.c_int, [C.c_void_p, C.POINTER(Stats)]),
    "iolm_cuda_last_error": (C.c_char_p, []),
    "iolm_cuda_set_kernel_timing": (C.c_int, [C.c_void_p, C.c_int32]),
    "iolm_cuda_kernel_times": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32]),
    "iolm_cuda_debug_gemm_f16": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                            C.c_int32, C.c_int32, C.c_int32]),
    "iolm_cuda_debug_gemm_time": (C.c_int, [C.c_int32] * 7 + [C.POINTER(C.c_float)]),
    "iolm_cuda_debug_quant_rows_f16": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "iolm_cuda_debug_gemm_s8": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                          C.c_int32, C.c_int32]),
    "iolm_cuda_debug_gemm_sp24": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                            C.c_void_p, C.c_void_p, C.c_void_p]),
    "iolm_cuda_debug_gemm_w4": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                          C.c_int32]),
    "iolm_cuda_debug_partition": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.POINTER(C.c_int32)]),
    "iolm_cuda_debug_gemm_sp24_f16": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                                 C.c_void_p]),
    "iolm_cuda_debug_gemm_sp24_time": (C.c_int, [C.c_int32] * 5 + [C.POINTER(C.c_float)]),
    "iolm_cuda_debug_gemm_sp24_f16_time": (C.c_int, [C.c_int32] * 5 + [C.POINTER(C.c_float)]),
}

_LIB = None


def load() -> C.CDLL:
    """Load libiolm_cuda.so; raises if it is absent (no fallback path exists)."""
    global _LIB
    if _LIB is None:
        if not ENGINE_SO.exists():
            raise RuntimeError(
                f"{ENGINE_SO} is missing: build it with `python -m paper_2507_04967_b200.build` "
                "(the prompt() hot path has no CPU fallback)")
        lib = C.CDLL(str(ENGINE_SO))
        for name, (res, args) in SIGNATURES.items():
            if not hasattr(lib, name):
                continue  # tests/test_abi.py asserts every declared symbol is exported
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def last_error() -> str:
    msg = load().iolm_cuda_last_error()
    return msg.decode() if msg else ""
