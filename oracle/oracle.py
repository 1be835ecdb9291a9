"""TEST INFRASTRUCTURE ONLY - the checker, never the product.

Python side of the CPU oracle:
  * `OracleModel`  - the plain-C restatement (oracle/iolm_oracle.c -> oracle/_build/liboracle.so)
                     driven over a bundle decoded here with numpy (restating
                     ModelBundle::decode_tensor, /root/reference/proj/src/model.cpp:140-204);
  * `RefRuntime`   - the UNMODIFIED reference (oracle/_ref/libiolm_ref.so, built from
                     /root/reference by oracle/Makefile) through its own public API;
  * `ref_toy_bundle`, `ref_compress` - the reference's own model/compression generators.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs import
this module. The product path (paper_2507_04967_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "liboracle.so"
REF_SO = HERE / "_ref" / "libiolm_ref.so"
REFERENCE_SRC = Path("/root/reference/proj")

BOS, EOS, PAD, VOCAB = 129, 130, 128, 131


def build(ref: bool = True) -> None:
    """Compile the C restatement and (when the reference sources exist) the reference library."""
    targets = ["oracle"]
    if ref and REFERENCE_SRC.exists():
        targets += ["ref", "dropin", "resolver", "patched"]
    subprocess.run(["make", "-s", "-C", str(HERE), "-j8", *targets], check=True)


# ----------------------------------------------------------------------------- bundle decode
ENC_DENSE, ENC_Q8, ENC_Q4, ENC_SPARSE24 = 0, 1, 2, 3


def parse_bundle(data: bytes, with_codes: bool = False) -> dict:
    """deserialize_bundle (model.cpp:348-406) + decode_tensor (model.cpp:140-204) in numpy.
    with_codes: also return the integer codes and scales of quantized tensors (W8A8 restatement)."""
    if len(data) < 10 or data[:4] != b"IOLM":
        raise ValueError("bundle: bad magic")
    hl = int.from_bytes(data[6:10], "little")
    header = json.loads(data[10:10 + hl].decode())
    blob = memoryview(data)[10 + hl:]
    tensors = {}
    codes_all = {}
    for t in header["tensors"]:
        r, c, enc, off, ln = t["rows"], t["cols"], t["encoding"], t["offset"], t["length"]
        p = np.frombuffer(blob[off:off + ln], dtype=np.uint8)
        if enc == ENC_DENSE:
            v = p.view(np.float32).reshape(r, c).copy()
        elif enc == ENC_Q8:
            codes = p[: r * c].view(np.int8).reshape(r, c)
            scales = p[r * c: r * c + 4 * r].view(np.float32)
            v = codes.astype(np.float32) * scales[:, None]
            if with_codes:
                codes_all[t["name"]] = (codes.astype(np.int8), scales.copy())
        elif enc == ENC_Q4:
            rb = (c + 1) // 2
            packed = p[: r * rb].reshape(r, rb)
            scales = p[r * rb: r * rb + 4 * r].view(np.float32)
            nib = np.empty((r, rb * 2), np.int32)
            nib[:, 0::2] = packed & 0x0F
            nib[:, 1::2] = packed >> 4
            v = (nib[:, :c] - 8).astype(np.float32) * scales[:, None]
        elif enc == ENC_SPARSE24:
            g = c // 4
            irb = (g + 1) // 2
            codes = p[: r * g * 2].view(np.int8).reshape(r, g, 2)
            idx = p[r * g * 2: r * g * 2 + r * irb].reshape(r, irb)
            scales = p[r * g * 2 + r * irb: r * g * 2 + r * irb + 4 * r].view(np.float32)
            nibs = np.empty((r, irb * 2), np.uint8)
            nibs[:, 0::2] = idx & 0x0F
            nibs[:, 1::2] = idx >> 4
            nibs = nibs[:, :g]
            v = np.zeros((r, g, 4), np.float32)
            ri, gi = np.meshgrid(np.arange(r), np.arange(g), indexing="ij")
            v[ri, gi, nibs & 3] = codes[:, :, 0].astype(np.float32) * scales[:, None]
            v[ri, gi, (nibs >> 2) & 3] = codes[:, :, 1].astype(np.float32) * scales[:, None]
            v = v.reshape(r, c)
            if with_codes:
                cd = np.zeros((r, g, 4), np.int8)
                cd[ri, gi, nibs & 3] = codes[:, :, 0]
                cd[ri, gi, (nibs >> 2) & 3] = codes[:, :, 1]
                codes_all[t["name"]] = (cd.reshape(r, c), scales.copy())
        else:
            raise ValueError(f"unknown encoding {enc}")
        tensors[t["name"]] = np.ascontiguousarray(v, dtype=np.float32)
    return {"config": header["config"], "tensors": tensors, "header": header, "codes": codes_all}


# ----------------------------------------------------------------------------- C restatement
class _OrcModel(C.Structure):
    _fields_ = [
        ("V", C.c_int), ("d", C.c_int), ("L", C.c_int), ("H", C.c_int), ("S", C.c_int), ("hd", C.c_int),
        ("heads", C.POINTER(C.c_int)), ("ffn", C.POINTER(C.c_int)),
        ("tok", C.c_void_p), ("pos", C.c_void_p), ("lnf_g", C.c_void_p), ("lnf_b", C.c_void_p),
        ("ln1_g", C.POINTER(C.c_void_p)), ("ln1_b", C.POINTER(C.c_void_p)),
        ("ln2_g", C.POINTER(C.c_void_p)), ("ln2_b", C.POINTER(C.c_void_p)),
        ("tok_t", C.c_void_p),
        ("wq", C.POINTER(C.c_void_p)), ("wk", C.POINTER(C.c_void_p)), ("wv", C.POINTER(C.c_void_p)),
        ("wo", C.POINTER(C.c_void_p)), ("w_in", C.POINTER(C.c_void_p)), ("w_out", C.POINTER(C.c_void_p)),
        ("act_quant", C.c_int), ("wcodes_t", C.POINTER(C.c_void_p)), ("wscale", C.POINTER(C.c_void_p)),
        ("gpu_points", C.c_int),
    ]


_ORC = None


def load_oracle() -> C.CDLL:
    global _ORC
    if _ORC is None:
        if not ORACLE_SO.exists():
            build(ref=False)
        lib = C.CDLL(str(ORACLE_SO))
        lib.orc_forward.argtypes = [C.POINTER(_OrcModel), C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                    C.POINTER(C.c_uint64)]
        lib.orc_decode_row.argtypes = [C.POINTER(_OrcModel), C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                       C.c_void_p, C.POINTER(C.c_uint64)]
        lib.orc_decode_rows.argtypes = [C.POINTER(_OrcModel), C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                        C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.c_int]
        lib.orc_decode_rows_gaps.argtypes = [C.POINTER(_OrcModel), C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                             C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.c_int,
                                             C.c_void_p, C.c_void_p]
        lib.orc_forward_codes.argtypes = [C.POINTER(_OrcModel), C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                          C.c_void_p]
        lib.orc_init_dense_params.restype = C.c_size_t
        lib.orc_init_dense_params.argtypes = [C.c_int] * 6 + [C.c_uint64, C.c_void_p]
        lib.orc_quant_rows_s8.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        lib.orc_gemm_s8.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
        _ORC = lib
    return _ORC


class OracleModel:
    """The C restatement over a decoded bundle."""

    def __init__(self, bundle: bytes | dict, act_quant: bool = False, gpu_points: bool = False):
        """act_quant: the W8A8 restatement (per-token int8 activations, int8 weight codes, exact
        int32 accumulation) - requires q8 / sparse24_q8 encodings for every linear weight.
        gpu_points (W8A8 only): round q/k/v, the attention output and the GELU output to fp16 where
        the GPU engine stores them, before they are quantized (W8A8 semantics)."""
        b = parse_bundle(bundle, with_codes=act_quant) if isinstance(bundle, (bytes, bytearray)) else bundle
        cfg, T = b["config"], b["tensors"]
        self.cfg = cfg
        L = cfg["n_layers"]
        self._keep = []
        m = _OrcModel()
        m.V, m.d, m.L, m.H, m.S = cfg["vocab_size"], cfg["d_model"], L, cfg["n_heads"], cfg["max_seq_len"]
        m.hd = cfg["d_model"] // cfg["n_heads"]
        heads = (C.c_int * L)(*[len(h) for h in cfg["active_heads"]])
        ffn = (C.c_int * L)(*cfg["active_ffn"])
        m.heads, m.ffn = heads, ffn
        self._keep += [heads, ffn]

        def ptr(a):
            self._keep.append(a)
            return a.ctypes.data

        m.tok, m.pos = ptr(T["tok_embed"]), ptr(T["pos_embed"])
        m.lnf_g, m.lnf_b = ptr(T["final_norm.gain"]), ptr(T["final_norm.bias"])
        m.tok_t = ptr(np.ascontiguousarray(T["tok_embed"].T))
        for fld, name in [("ln1_g", "attn_norm.gain"), ("ln1_b", "attn_norm.bias"), ("ln2_g", "ffn_norm.gain"),
                          ("ln2_b", "ffn_norm.bias"), ("wq", "attn.wq"), ("wk", "attn.wk"), ("wv", "attn.wv"),
                          ("wo", "attn.wo"), ("w_in", "ffn.w_in"), ("w_out", "ffn.w_out")]:
            tr = name.startswith("attn.w") or name.startswith("ffn.w")  # weights go in transposed
            arr = (C.c_void_p * L)(*[ptr(np.ascontiguousarray(T[f"layers.{l}.{name}"].T) if tr
                                         else T[f"layers.{l}.{name}"]) for l in range(L)])
            self._keep.append(arr)
            setattr(m, fld, arr)
        m.act_quant = 1 if act_quant else 0
        m.gpu_points = 1 if (act_quant and gpu_points) else 0
        if act_quant:
            names = ["attn.wq", "attn.wk", "attn.wv", "attn.wo", "ffn.w_in", "ffn.w_out"]
            cw, cs = [], []
            for l in range(L):
                for nm in names:
                    key = f"layers.{l}.{nm}"
                    if key not in b["codes"]:
                        raise ValueError(f"W8A8 needs q8/sparse24 codes for {key}")
                    codes, scales = b["codes"][key]
                    cw.append(ptr(np.ascontiguousarray(codes.T)))
                    cs.append(ptr(np.ascontiguousarray(scales, dtype=np.float32)))
            m.wcodes_t = (C.c_void_p * len(cw))(*cw)
            m.wscale = (C.c_void_p * len(cs))(*cs)
            self._keep += [m.wcodes_t, m.wscale]
        self._m = m
        self.lib = load_oracle()

    def forward(self, ids, mask=None):
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        n = len(ids)
        out = np.zeros((n, self.cfg["vocab_size"]), np.float32)
        mk = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        madds = C.c_uint64()
        st = self.lib.orc_forward(C.byref(self._m), ids.ctypes.data, None if mk is None else mk.ctypes.data,
                                  n, out.ctypes.data, C.byref(madds))
        if st:
            raise RuntimeError(f"oracle forward status {st}")
        return out, madds.value

    def decode_ids(self, ids: np.ndarray, offsets: np.ndarray, max_new: int, threads: int = 1,
                   gaps: bool = False):
        """Greedy ids [n x max_new], lengths, madds; with gaps=True also the CPU top-1 - top-2 logit
        gap and max |logit| at every prediction ([n x (max_new + 1)] each, NaN past the row's end)."""
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        n = len(offsets) - 1
        out = np.zeros((n, max(max_new, 1)), np.int32)
        ln = np.zeros(n, np.int32)
        madds = C.c_uint64()
        gap = np.full((n, max_new + 1), np.nan, np.float32) if gaps else None
        amax = np.full((n, max_new + 1), np.nan, np.float32) if gaps else None
        st = self.lib.orc_decode_rows_gaps(C.byref(self._m), ids.ctypes.data, offsets.ctypes.data, n, max_new,
                                           out.ctypes.data, ln.ctypes.data, C.byref(madds), threads,
                                           None if gap is None else gap.ctypes.data,
                                           None if amax is None else amax.ctypes.data)
        if st:
            raise RuntimeError(f"oracle decode status {st}")
        if gaps:
            return out[:, :max_new], ln, madds.value, gap, amax
        return out[:, :max_new], ln, madds.value

    def forward_codes(self, ids):
        """W8A8 forward returning (logits, codes, scales): the int8 operand codes of every linear input,
        per layer [attn_in n x d][attn_out_in n x kh][ffn_in n x d][ffn_mid n x f], and their
        per-token scales, per layer [4 x n]."""
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        n, cfg = len(ids), self.cfg
        tot = sum(n * (2 * cfg["d_model"] + len(h) * (cfg["d_model"] // cfg["n_heads"]) + f)
                  for h, f in zip(cfg["active_heads"], cfg["active_ffn"]))
        codes = np.zeros(tot, np.int8)
        scales = np.zeros(4 * n * cfg["n_layers"], np.float32)
        out = np.zeros((n, cfg["vocab_size"]), np.float32)
        st = self.lib.orc_forward_codes(C.byref(self._m), ids.ctypes.data, n, out.ctypes.data, codes.ctypes.data,
                                        scales.ctypes.data)
        if st:
            raise RuntimeError(f"oracle forward_codes status {st}")
        return out, codes, scales


def render(ids_row, n) -> str:
    """Tokenizer::decode of emitted ids: 0..127 -> chars, PAD/BOS -> nothing (tokenizer.cpp:23-36)."""
    return "".join(chr(int(t)) for t in ids_row[:n] if 0 <= int(t) <= 127)


def quant_rows_s8(x: np.ndarray):
    x = np.ascontiguousarray(x, dtype=np.float32)
    n, d = x.shape
    codes = np.zeros((n, d), np.int8)
    scales = np.zeros(n, np.float32)
    load_oracle().orc_quant_rows_s8(x.ctypes.data, n, d, codes.ctypes.data, scales.ctypes.data)
    return codes, scales


def gemm_s8(a: np.ndarray, w: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.int8)
    w = np.ascontiguousarray(w, dtype=np.int8)
    M, K = a.shape
    N = w.shape[0]
    out = np.zeros((M, N), np.int32)
    load_oracle().orc_gemm_s8(a.ctypes.data, w.ctypes.data, M, N, K, out.ctypes.data)
    return out


# ----------------------------------------------------------------------------- the reference itself
_REF = None


def ref_available() -> bool:
    return REF_SO.exists()


def load_ref() -> C.CDLL:
    global _REF
    if _REF is None:
        if not REF_SO.exists():
            if REFERENCE_SRC.exists():
                build(ref=True)
            else:
                raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        lib = C.CDLL(str(REF_SO))
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_toy_bundle.argtypes = [C.c_int] * 5 + [C.c_uint64, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]
        lib.ref_compress.argtypes = [C.c_void_p, C.c_size_t, C.c_char_p, C.c_char_p, C.c_void_p, C.c_int,
                                     C.c_uint64, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]
        lib.ref_runtime_create.restype = C.c_void_p
        lib.ref_runtime_create.argtypes = [C.c_void_p, C.c_size_t]
        lib.ref_runtime_destroy.argtypes = [C.c_void_p]
        lib.ref_runtime_hash.restype = C.c_uint64
        lib.ref_runtime_hash.argtypes = [C.c_void_p]
        lib.ref_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_uint64)]
        lib.ref_batch_decode.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                         C.c_void_p, C.POINTER(C.c_uint64), C.c_int, C.c_int]
        lib.ref_free.argtypes = [C.c_void_p]
        _REF = lib
    return _REF


def _take(lib, p, n) -> bytes:
    data = C.string_at(p.value, n.value)
    lib.ref_free(p)
    return data


def ref_toy_bundle(d, L, H, F, S, seed=42) -> bytes:
    lib = load_ref()
    p, n = C.c_void_p(), C.c_size_t()
    st = lib.ref_toy_bundle(d, L, H, F, S, seed, C.byref(p), C.byref(n))
    if st:
        raise RuntimeError(lib.ref_last_error().decode())
    return _take(lib, p, n)


def ref_compress(bundle: bytes, recipe: dict, prompts: list[str], seed: int = 7) -> bytes:
    lib = load_ref()
    chars = "".join(prompts).encode()
    offs = np.zeros(len(prompts) + 1, np.int64)
    offs[1:] = np.cumsum([len(p) for p in prompts])
    p, n = C.c_void_p(), C.c_size_t()
    buf = C.create_string_buffer(bundle, len(bundle))
    st = lib.ref_compress(buf, len(bundle), json.dumps(recipe).encode(), chars, offs.ctypes.data, len(prompts),
                          seed, C.byref(p), C.byref(n))
    if st:
        raise RuntimeError(lib.ref_last_error().decode())
    return _take(lib, p, n)


class RefRuntime:
    """iolm::ModelRuntime (the reference, compiled unmodified)."""

    def __init__(self, bundle: bytes):
        self.lib = load_ref()
        self._buf = C.create_string_buffer(bytes(bundle), len(bundle))
        self.h = self.lib.ref_runtime_create(self._buf, len(bundle))
        if not self.h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        hl = int.from_bytes(bundle[6:10], "little")
        self.cfg = json.loads(bundle[10:10 + hl].decode())["config"]

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_runtime_destroy(self.h)
            self.h = None

    def bundle_hash(self) -> int:
        return self.lib.ref_runtime_hash(self.h)

    def forward(self, ids, mask=None):
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        out = np.zeros((len(ids), self.cfg["vocab_size"]), np.float32)
        mk = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        madds = C.c_uint64()
        st = self.lib.ref_forward(self.h, ids.ctypes.data, None if mk is None else mk.ctypes.data, len(ids),
                                  out.ctypes.data, C.byref(madds))
        if st:
            raise RuntimeError(f"{st}: {self.lib.ref_last_error().decode()}")
        return out, madds.value

    def batch_decode(self, prompts: list[str], max_new: int, threads: int = 1, batch_size: int = 16):
        chars = "".join(prompts).encode()
        offs = np.zeros(len(prompts) + 1, np.int64)
        offs[1:] = np.cumsum([len(p) for p in prompts])
        out = C.create_string_buffer(max(1, len(prompts) * max_new))
        ln = np.zeros(len(prompts), np.int32)
        madds = C.c_uint64()
        st = self.lib.ref_batch_decode(self.h, chars, offs.ctypes.data, len(prompts), max_new, out,
                                       ln.ctypes.data, C.byref(madds), threads, batch_size)
        if st:
            raise RuntimeError(f"{st}: {self.lib.ref_last_error().decode()}")
        raw = out.raw
        return [raw[i * max_new: i * max_new + ln[i]].decode() for i in range(len(prompts))], madds.value
