"""Python mirror of the reference's model-runtime interface over the C ABI.

`ModelRuntime` keeps the public surface of iolm::ModelRuntime
(/root/reference/proj/include/iolm/runtime.hpp:37-60): construction from a bundle, config(),
bundle_hash(), forward(ids, mask, counter), greedy_decode(prompt, n, counter),
batch_decode(prompts, n, counter) - same argument meaning, same outputs, same error classes
(proj/include/iolm/common.hpp:16-89). Every call runs on the sm_100a engine (libiolm_cuda.so);
there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib

# --------------------------------------------------------------------------- errors (common.hpp)


class Error(RuntimeError):
    """iolm::Error"""


class ContractViolation(Error):
    pass


class SequenceTooLong(Error):
    pass


class CorruptHeader(Error):
    pass


class TruncatedBlob(Error):
    pass


class UnknownEncoding(Error):
    pass


class UnsupportedOnGpu(Error):
    """A bundle/shape this GPU build cannot run (no CPU fallback exists)."""


class CudaError(Error):
    pass


class StaleImage(Error):
    """A device-layout image built from another bundle or with other weight options."""


class DeviceOutOfMemory(CudaError):
    pass


_STATUS = {
    _lib.IOLM_E_CONTRACT: ContractViolation,
    _lib.IOLM_E_SEQ_TOO_LONG: SequenceTooLong,
    _lib.IOLM_E_UNSUPPORTED: UnsupportedOnGpu,
    _lib.IOLM_E_CUDA: CudaError,
    _lib.IOLM_E_OOM: DeviceOutOfMemory,
    _lib.IOLM_E_CORRUPT_HEADER: CorruptHeader,
    _lib.IOLM_E_TRUNCATED_BLOB: TruncatedBlob,
    _lib.IOLM_E_UNKNOWN_ENCODING: UnknownEncoding,
    _lib.IOLM_E_STALE: StaleImage,
}


def _check(status: int) -> None:
    if status != _lib.IOLM_OK:
        raise _STATUS.get(status, Error)(_lib.last_error())


class FlopCounter:
    """iolm::FlopCounter (matrix.hpp:16-24): cumulative multiply-adds."""

    def __init__(self) -> None:
        self._t = 0

    def add(self, madds: int) -> None:
        self._t += int(madds)

    def total(self) -> int:
        return self._t

    def reset(self) -> None:
        self._t = 0


# --------------------------------------------------------------------------- tokenizer (tokenizer.cpp)
PAD, BOS, EOS, VOCAB = _lib.PAD, _lib.BOS, _lib.EOS, _lib.VOCAB


def encode(text: str | bytes) -> list[int]:
    """Tokenizer::encode: bytes 0..127 -> ids; non-ASCII raises ContractViolation."""
    b = text.encode("latin-1") if isinstance(text, str) else bytes(text)
    for i, c in enumerate(b):
        if c > 127:
            raise ContractViolation(f"Tokenizer: non-ASCII byte {c} at offset {i}")
    return list(b)


def decode_ids(ids) -> str:
    """Tokenizer::decode for emitted ids: 0..127 render, PAD/BOS render nothing."""
    return "".join(chr(int(t)) for t in ids if 0 <= int(t) <= 127)


@dataclass
class ModelConfig:
    vocab_size: int
    d_model: int
    n_layers: int
    n_heads: int
    d_ff: int
    max_seq_len: int
    active_heads: list = field(default_factory=list)
    active_ffn: list = field(default_factory=list)

    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    def layer_heads(self, l: int) -> int:
        return len(self.active_heads[l])

    def layer_ffn(self, l: int) -> int:
        return self.active_ffn[l]


def bundle_config(bundle: bytes) -> ModelConfig:
    hl = int.from_bytes(bundle[6:10], "little")
    c = json.loads(bundle[10:10 + hl].decode())["config"]
    return ModelConfig(**c)


def image_header(path) -> dict:
    """Header of a device-layout image (format: iolm_cuda.h, iolm_cuda_save_image): bundle hash,
    model config (with the active head ids), the weight options and per-layer weight forms."""
    with open(path, "rb") as f:
        if f.read(8) != b"IOLMDL02":
            raise CorruptHeader("device-layout image: bad magic")
        nw = int.from_bytes(f.read(8), "little")
        w = np.frombuffer(f.read(8 * nw), dtype="<i8").tolist()
    if len(w) != nw or nw < 10:
        raise TruncatedBlob("device-layout image: file ends early")
    cfg = ModelConfig(*w[1:7])
    at = 10
    for _ in range(cfg.n_layers):
        n = w[at]
        cfg.active_heads.append(w[at + 1:at + 1 + n])
        at += 1 + n
    cfg.active_ffn = w[at:at + cfg.n_layers]
    at += cfg.n_layers
    forms = ["values", "codes", "int8", "sp24", "int4", "sp24f"]
    return {"bundle_hash": w[0] & (2**64 - 1), "config": cfg,
            "act_quant": bool(w[7]), "sparse_mma": bool(w[8]), "int4_mma": bool(w[9]),
            "weight_forms": [forms[m] for m in w[at:at + 4 * cfg.n_layers]]}


# --------------------------------------------------------------------------- runtime
class ModelRuntime:
    """iolm::ModelRuntime on a B200. `bundle` is the serialize_bundle byte stream. `device` is one GPU
    index, or a list of them: one context over several GPUs (iolm_cuda_create_multi), whose
    batch_decode range-partitions the rows over full per-GPU replicas."""

    def __init__(self, bundle: bytes, device=0, max_tokens_per_step: int = 0, max_slots: int = 0,
                 prefix_sharing: bool = True, act_quant: bool = False, kernel_timing: bool = False,
                 sparse_mma: bool = True, int4_mma: bool = True, prefill_tc: bool | None = None):
        self._lib = _lib.load()
        opts = self._opts(max_tokens_per_step, max_slots, prefix_sharing, act_quant, kernel_timing, sparse_mma,
                          int4_mma, prefill_tc)
        h = C.c_void_p()
        buf = (C.c_char * len(bundle)).from_buffer_copy(bundle)
        if isinstance(device, (list, tuple)):
            devs = (C.c_int32 * len(device))(*device)
            _check(self._lib.iolm_cuda_create_multi(buf, len(bundle), devs, len(device), C.byref(opts), C.byref(h)))
        else:
            _check(self._lib.iolm_cuda_create(buf, len(bundle), device, C.byref(opts), C.byref(h)))
        self._h = h
        hl = int.from_bytes(bundle[6:10], "little")
        self._config = ModelConfig(**json.loads(bundle[10:10 + hl].decode())["config"])

    @staticmethod
    def _opts(max_tokens_per_step=0, max_slots=0, prefix_sharing=True, act_quant=False, kernel_timing=False,
              sparse_mma=True, int4_mma=True, prefill_tc=None) -> _lib.Opts:
        opts = _lib.Opts()
        opts.max_tokens_per_step = max_tokens_per_step
        opts.max_slots = max_slots
        opts.prefix_sharing = 0 if prefix_sharing else -1
        opts.act_quant = 1 if act_quant else 0
        opts.kernel_timing = 1 if kernel_timing else 0
        opts.sparse_mma = 0 if sparse_mma else -1
        opts.int4_mma = 0 if int4_mma else -1
        opts.prefill_tc = 0 if prefill_tc is None else (1 if prefill_tc else -1)
        return opts

    @classmethod
    def from_image(cls, path, expected_hash: int = 0, device: int = 0, **options) -> "ModelRuntime":
        """A runtime from a device-layout image (iolm_cuda_create_from_image): `options` take the
        constructor's keywords; the weight-shaping ones must match the saved runtime's (StaleImage)."""
        self = cls.__new__(cls)
        self._lib = _lib.load()
        opts = cls._opts(**options)
        h = C.c_void_p()
        _check(self._lib.iolm_cuda_create_from_image(os.fsencode(path), expected_hash, device, C.byref(opts),
                                                     C.byref(h)))
        self._h = h
        self._config = image_header(path)["config"]
        return self

    def save_image(self, path) -> None:
        """Writes this runtime's device layout (iolm_cuda_save_image)."""
        _check(self._lib.iolm_cuda_save_image(self._h, os.fsencode(path)))

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.iolm_cuda_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def config(self) -> ModelConfig:
        return self._config

    def device_count(self) -> int:
        v = C.c_int32()
        _check(self._lib.iolm_cuda_device_count(self._h, C.byref(v)))
        return v.value

    def bundle_hash(self) -> int:
        v = C.c_uint64()
        _check(self._lib.iolm_cuda_bundle_hash(self._h, C.byref(v)))
        return v.value

    def last_stats(self) -> dict:
        s = _lib.Stats()
        _check(self._lib.iolm_cuda_last_stats(self._h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in _lib.Stats._fields_}

    def set_kernel_timing(self, on: bool) -> None:
        _check(self._lib.iolm_cuda_set_kernel_timing(self._h, 1 if on else 0))

    def kernel_times(self) -> dict:
        """Per kernel class of the last call: {name: (ms, algorithmic work, launches)}."""
        n = len(_lib.KCLASSES)
        ms, work, cnt = (C.c_double * n)(), (C.c_double * n)(), (C.c_int64 * n)()
        _check(self._lib.iolm_cuda_kernel_times(self._h, ms, work, cnt, n))
        return {k: (ms[i], work[i], cnt[i]) for i, k in enumerate(_lib.KCLASSES)}

    # ---- forward (runtime.cpp:217-232)
    def forward(self, ids, mask=None, counter: FlopCounter | None = None) -> np.ndarray:
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        if ids.size == 0:
            raise ContractViolation("forward: empty sequence")
        mk = None
        if mask is not None and len(mask):
            if len(mask) != len(ids):
                raise ContractViolation("forward: mask length mismatch")
            mk = np.ascontiguousarray(mask, dtype=np.uint8)
        out = np.empty((len(ids), self._config.vocab_size), np.float32)
        madds = C.c_uint64()
        _check(self._lib.iolm_cuda_forward_logits(self._h, ids.ctypes.data, None if mk is None else mk.ctypes.data,
                                                  len(ids), out.ctypes.data, C.byref(madds)))
        if counter is not None:
            counter.add(madds.value)
        return out

    def forward_codes(self, ids):
        """W8A8 runtimes (act_quant): (logits, int8 operand codes, per-token scales) of every linear
        input - layout of iolm_cuda_forward_codes (include/iolm_cuda.h)."""
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        n, cfg = len(ids), self._config
        hd = cfg.d_model // cfg.n_heads
        tot = sum(n * (2 * cfg.d_model + cfg.layer_heads(l) * hd + cfg.layer_ffn(l)) for l in range(cfg.n_layers))
        codes = np.zeros(tot, np.int8)
        scales = np.zeros(4 * n * cfg.n_layers, np.float32)
        out = np.empty((n, cfg.vocab_size), np.float32)
        madds = C.c_uint64()
        _check(self._lib.iolm_cuda_forward_codes(self._h, ids.ctypes.data, n, out.ctypes.data, codes.ctypes.data,
                                                 scales.ctypes.data, C.byref(madds)))
        return out, codes, scales

    # ---- token-level throughput API
    def decode_token_rows(self, ids: np.ndarray, offsets: np.ndarray, max_new_tokens: int,
                          device_ids: int | None = None):
        """CSR token rows (already [BOS]+bytes) -> (out_ids [n x max_new], out_len [n], madds).
        `device_ids`: pointer to the same ids already resident in device memory."""
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        n = len(offsets) - 1
        out = np.zeros((n, max(1, max_new_tokens)), np.int32)
        ln = np.zeros(n, np.int32)
        madds = C.c_uint64()
        bad = C.c_int64(-1)
        if device_ids is None:
            ids = np.ascontiguousarray(ids, dtype=np.int32)
            st = self._lib.iolm_cuda_decode(self._h, ids.ctypes.data, offsets.ctypes.data, n, max_new_tokens,
                                            out.ctypes.data, ln.ctypes.data, C.byref(madds), C.byref(bad))
        else:
            st = self._lib.iolm_cuda_decode_device_ids(self._h, C.c_void_p(device_ids), offsets.ctypes.data, n,
                                                       max_new_tokens, out.ctypes.data, ln.ctypes.data,
                                                       C.byref(madds), C.byref(bad))
        _check(st)
        return out[:, :max_new_tokens], ln, madds.value

    # ---- batch_decode (runtime.cpp:241-309)
    def batch_decode(self, prompts, max_new_tokens: int, counter: FlopCounter | None = None) -> list[str]:
        prompts = list(prompts)
        if not prompts:
            raise ContractViolation("batch_decode: batch size must be >= 1")
        if max_new_tokens < 0:
            raise ContractViolation("batch_decode: max_new_tokens must be >= 0")
        if max_new_tokens == 0:
            return [""] * len(prompts)
        S = self._config.max_seq_len
        rows = []
        for i, p in enumerate(prompts):  # encode + length check in prompt order, like the reference
            ids = [BOS] + encode(p)
            if len(ids) > S:
                raise SequenceTooLong(f"batch_decode: prompt {i} needs {len(ids)} tokens, max_seq_len is {S}")
            rows.append(ids)
        offsets = np.zeros(len(rows) + 1, np.int64)
        offsets[1:] = np.cumsum([len(r) for r in rows])
        flat = np.fromiter((t for r in rows for t in r), dtype=np.int32, count=int(offsets[-1]))
        out, ln, madds = self.decode_token_rows(flat, offsets, max_new_tokens)
        if counter is not None:
            counter.add(madds)
        return [decode_ids(out[i, :ln[i]]) for i in range(len(rows))]

    def greedy_decode(self, prompt: str, max_new_tokens: int, counter: FlopCounter | None = None) -> str:
        return self.batch_decode([prompt], max_new_tokens, counter)[0]


def full_forward_flops(cfg: ModelConfig, seq_len: int) -> int:
    """runtime.cpp:311-325"""
    t, d, hd = seq_len, cfg.d_model, cfg.head_dim()
    total = 0
    for l in range(cfg.n_layers):
        kh, f = cfg.layer_heads(l) * hd, cfg.layer_ffn(l)
        total += 4 * t * d * kh + kh * t * (t + 1) + 2 * t * d * f
    return total + t * d * cfg.vocab_size


def decode_flops(cfg: ModelConfig, prompt_len: int, new_tokens: int) -> int:
    """runtime.cpp:327-345"""
    d, hd, v = cfg.d_model, cfg.head_dim(), cfg.vocab_size
    s0 = prompt_len + 1
    if new_tokens == 0:
        return 0
    total = 0
    for l in range(cfg.n_layers):
        kh, f = cfg.layer_heads(l) * hd, cfg.layer_ffn(l)
        total += 4 * s0 * d * kh + kh * s0 * (s0 + 1) + 2 * s0 * d * f
        for i in range(1, new_tokens + 1):
            total += 4 * d * kh + 2 * d * f + 2 * kh * (s0 + i)
    return total + d * v + new_tokens * d * v
