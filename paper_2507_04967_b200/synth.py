"""Workload generator for the throughput harness and tests (ctypes over libiolm_synth.so).

`toy_bundle` reproduces ToyModelParams::init(...).to_bundle() + serialize_bundle byte-for-byte
(/root/reference/proj/src/train.cpp:45-75, proj/src/model.cpp:311-346); `rows` renders the
synthetic table of SURVEY.md §8d as token ids. Harness code: the engine never uses it.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
SYNTH_SO = PKG / "libiolm_synth.so"
INSTRUCTION = "summarize in five words, plain:"  # 31 chars: BOS + this = the 32-token prefix

_LIB = None


def _lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not SYNTH_SO.exists():
            from . import build
            build.build_synth()
        lib = C.CDLL(str(SYNTH_SO))
        lib.synth_toy_bundle.argtypes = [C.c_int] * 5 + [C.c_uint64, C.c_int, C.c_void_p, C.c_void_p,
                                                         C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]
        lib.synth_rows.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_void_p]
        lib.synth_fnv1a.restype = C.c_uint64
        lib.synth_fnv1a.argtypes = [C.c_void_p, C.c_size_t]
        lib.synth_free.argtypes = [C.c_void_p]
        _LIB = lib
    return _LIB


QUANT = {"dense": 0, "q8": 8, "q4": 4, "sparse24": 24}


def toy_bundle(d: int, L: int, H: int, F: int, S: int, seed: int = 42, quant: str = "dense",
               heads: list[int] | None = None, ffn: list[int] | None = None) -> bytes:
    """Random-init bundle; `heads`/`ffn` give per-layer pruned shapes (first-k survivors)."""
    lib = _lib()
    p, n = C.c_void_p(), C.c_size_t()
    hp = (C.c_int * L)(*heads) if heads is not None else None
    fp = (C.c_int * L)(*ffn) if ffn is not None else None
    st = lib.synth_toy_bundle(d, L, H, F, S, seed, QUANT[quant], hp, fp, C.byref(p), C.byref(n))
    if st:
        raise ValueError("synth_toy_bundle: unsupported shape for the requested encoding")
    data = C.string_at(p.value, n.value)
    lib.synth_free(p)
    return data


def fnv1a(data: bytes) -> int:
    buf = (C.c_char * len(data)).from_buffer_copy(data)
    return _lib().synth_fnv1a(buf, len(data))


def rows(first_row: int, n_rows: int, row_chars: int = 64, instruction: str = INSTRUCTION):
    """Token-id rows ([BOS] + instruction + row chars) in CSR form: (ids int32, offsets int64)."""
    per = 1 + len(instruction) + row_chars
    ids = np.empty(n_rows * per, np.int32)
    offs = np.empty(n_rows + 1, np.int64)
    _lib().synth_rows(instruction.encode(), first_row, n_rows, row_chars, ids.ctypes.data, offs.ctypes.data)
    return ids, offs


def row_strings(first_row: int, n_rows: int, row_chars: int = 64, instruction: str = INSTRUCTION) -> list[str]:
    ids, offs = rows(first_row, n_rows, row_chars, instruction)
    return ["".join(chr(c) for c in ids[offs[i] + 1:offs[i + 1]]) for i in range(n_rows)]


def scale_token_embeddings(bundle: bytes, factors: dict[int, float]) -> bytes:
    """A copy of a dense_f32 bundle with rows of `tok_embed` scaled (f32 multiply). The head is tied
    (logits = y . tok_embed^T, /root/reference/proj/src/runtime.cpp:213-215), so scaling the EOS / PAD /
    BOS rows makes a random-init model emit those ids at varied steps - the stop and no-render paths
    of batch_decode (runtime.cpp:286-298) that plain random-init models never reach. Test harness."""
    import json

    hl = int.from_bytes(bundle[6:10], "little")
    header = json.loads(bundle[10:10 + hl].decode())
    rec = next(t for t in header["tensors"] if t["name"] == "tok_embed")
    if rec["encoding"] != 0:
        raise ValueError("tok_embed must be dense_f32")
    base = 10 + hl + rec["offset"]
    emb = np.frombuffer(bundle[base:base + rec["length"]], np.float32).reshape(rec["rows"], rec["cols"]).copy()
    for tok, f in factors.items():
        emb[tok] *= np.float32(f)
    out = bytearray(bundle)
    out[base:base + rec["length"]] = emb.tobytes()
    return bytes(out)
