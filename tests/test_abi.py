"""CPU-only checks of the drop-in boundary: the C ABI library loads and exports every entry point
include/iolm_cuda.h declares; bundle validation errors map to the reference's exception classes
(proj/src/model.cpp:348-406, proj/include/iolm/common.hpp) before any device work; the product
path fails loudly (no CPU fallback) on a machine without a GPU; the C++ shim compiles."""
import ctypes as C
import json
import re
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2507_04967_b200 import _lib
from paper_2507_04967_b200 import runtime as R
from paper_2507_04967_b200 import synth

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "iolm_cuda.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(iolm_cuda_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_expected_surface():
    syms = declared_symbols()
    for s in ["iolm_cuda_create", "iolm_cuda_destroy", "iolm_cuda_decode", "iolm_cuda_forward_logits",
              "iolm_cuda_bundle_hash", "iolm_cuda_config", "iolm_cuda_last_error", "iolm_cuda_decode_device_ids"]:
        assert s in syms


def test_library_exports_every_declared_symbol(engine_lib):
    missing = [s for s in declared_symbols() if not hasattr(engine_lib, s)]
    assert not missing, missing
    assert set(declared_symbols()) <= set(_lib.SIGNATURES)


def _create(data: bytes):
    lib = _lib.load()
    h = C.c_void_p()
    buf = (C.c_char * max(1, len(data))).from_buffer_copy(data or b"\0")
    st = lib.iolm_cuda_create(buf, len(data), 0, None, C.byref(h))
    if st == 0:
        lib.iolm_cuda_destroy(h)
    return st, _lib.last_error()


def _rewrite_header(b: bytes, fn) -> bytes:
    hl = int.from_bytes(b[6:10], "little")
    hdr = json.loads(b[10:10 + hl])
    fn(hdr)
    h2 = json.dumps(hdr, separators=(",", ":")).encode()
    return b[:6] + len(h2).to_bytes(4, "little") + h2 + b[10 + hl:]


@pytest.fixture(scope="module")
def tiny():
    return synth.toy_bundle(32, 2, 2, 64, 128, seed=42)


def test_bundle_errors_map_to_reference_classes(tiny):
    assert _create(b"XXXX" + tiny[4:])[0] == _lib.IOLM_E_CORRUPT_HEADER            # bad magic
    assert _create(tiny[:4] + b"\x02\x00" + tiny[6:])[0] == _lib.IOLM_E_CORRUPT_HEADER  # version
    assert _create(tiny[:-100])[0] == _lib.IOLM_E_TRUNCATED_BLOB                     # truncated blob
    assert _create(tiny[:10] + b"[" + tiny[11:])[0] == _lib.IOLM_E_CORRUPT_HEADER     # bad JSON
    bad_enc = _rewrite_header(tiny, lambda h: h["tensors"][4].__setitem__("encoding", 7))
    assert _create(bad_enc)[0] == _lib.IOLM_E_UNKNOWN_ENCODING
    bad_cfg_ffn = _rewrite_header(tiny, lambda h: h["config"].__setitem__("d_ff", 32))
    assert _create(bad_cfg_ffn)[0] == _lib.IOLM_E_CONTRACT  # active_ffn > d_ff

    def swap_dims(h):  # wq stored as [d x kh] instead of [kh x d]: same length, wrong shape
        t = next(t for t in h["tensors"] if t["name"] == "layers.0.attn.wo")
        t["rows"], t["cols"] = 16, 64
    st, msg = _create(_rewrite_header(tiny, swap_dims))
    assert st == _lib.IOLM_E_CONTRACT and "shape" in msg
    no_tensor = _rewrite_header(tiny, lambda h: h["tensors"].pop())
    assert _create(no_tensor)[0] == _lib.IOLM_E_CONTRACT
    bad_cfg = _rewrite_header(tiny, lambda h: h["config"].__setitem__("active_ffn", [0, 64]))
    assert _create(bad_cfg)[0] == _lib.IOLM_E_CONTRACT
    assert _create(b"")[0] == _lib.IOLM_E_CONTRACT


def test_unsupported_shapes_are_rejected_not_run(tiny):
    odd = synth.toy_bundle(36, 1, 3, 24, 16, seed=1)  # head_dim 12
    st, msg = _create(odd)
    assert st == _lib.IOLM_E_UNSUPPORTED, msg


def test_no_gpu_fails_loudly(tiny):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    st, msg = _create(tiny)
    assert st == _lib.IOLM_E_CUDA and msg
    with pytest.raises(R.CudaError):
        R.ModelRuntime(tiny)


def test_tokenizer_and_flop_formulas():
    assert R.encode("Hi!") == [72, 105, 33]
    with pytest.raises(R.ContractViolation):
        R.encode("caf\xe9")
    assert R.decode_ids([72, 128, 129, 105]) == "Hi"
    meta = json.loads((ROOT / "tests" / "golden" / "tiny.json").read_text())
    cfg = R.bundle_config(synth.toy_bundle(*meta["dims"]))
    # every golden row is BOS + 31 + 64 chars and emits 8 tokens: decode_flops closed form
    # (runtime.cpp:327-345) summed over rows equals the reference FlopCounter total
    per_row = R.decode_flops(cfg, 31 + 64, 8)
    assert per_row * meta["decode_rows"] == meta["decode_madds"]
    assert R.full_forward_flops(cfg, 96) == meta["forward_madds"][0]


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
@pytest.mark.parametrize("with_ref", [False, True])
def test_cpp_shim_compiles(with_ref, tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text('#include "iolm_cuda_runtime.hpp"\nint main(){ return 0; }\n')
    cmd = ["g++", "-std=c++20", "-fsyntax-only", f"-I{ROOT / 'include'}", str(src)]
    if with_ref:
        ref_inc = Path("/root/reference/proj/include")
        json_dir = Path("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann")
        if not ref_inc.exists():
            pytest.skip("reference headers absent")
        cmd += ["-DIOLM_CUDA_WITH_REFERENCE_TYPES", f"-I{ref_inc}", f"-I{json_dir}"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr


def _image_bytes(words, arrays=b""):
    w = np.asarray(words, dtype="<i8")
    return b"IOLMDL02" + len(w).to_bytes(8, "little") + w.tobytes() + arrays


def _image_info(path):
    lib = _lib.load()
    h, cfg = C.c_uint64(), _lib.ModelConfigC()
    st = lib.iolm_cuda_image_info(str(path).encode(), C.byref(h), C.byref(cfg))
    return st, h.value, cfg


def test_device_image_header_validation(tmp_path):
    """iolm_cuda_image_info parses and validates a device-layout image header without device work
    (the registry can check an image's bundle hash before loading it)."""
    # hash, vocab, d, L, n_heads, d_ff, S, act_quant, sparse_mma, int4_mma | heads | ffn | forms
    words = [-7, 131, 64, 2, 4, 256, 128, 0, 1, 1, 2, 0, 1, 4, 0, 1, 2, 3, 256, 128, 0, 0, 0, 0, 1, 1, 1, 1]
    p = tmp_path / "ok.iolmdev"
    p.write_bytes(_image_bytes(words))
    st, h, cfg = _image_info(p)
    assert st == _lib.IOLM_OK, _lib.last_error()
    assert h == 2**64 - 7 and (cfg.d_model, cfg.n_layers, cfg.head_dim, cfg.max_seq_len) == (64, 2, 16, 128)
    hdr = R.image_header(p)
    assert hdr["bundle_hash"] == h and hdr["config"].active_heads == [[0, 1], [0, 1, 2, 3]]
    assert hdr["config"].active_ffn == [256, 128] and hdr["weight_forms"] == ["values"] * 4 + ["codes"] * 4

    def status(data):
        q = tmp_path / "x.iolmdev"
        q.write_bytes(data)
        return _image_info(q)[0]

    assert status(b"IOLMDL01" + _image_bytes(words)[8:]) == _lib.IOLM_E_CORRUPT_HEADER      # magic (v01: bf16 arrays)
    assert status(_image_bytes(words)[:40]) == _lib.IOLM_E_TRUNCATED_BLOB                   # short
    assert status(_image_bytes(words[:-1])) == _lib.IOLM_E_CORRUPT_HEADER                   # words
    assert status(_image_bytes(words + [0])) == _lib.IOLM_E_CORRUPT_HEADER                  # trailing
    bad_heads = list(words)
    bad_heads[11], bad_heads[12] = 1, 0                                                     # descending
    assert status(_image_bytes(bad_heads)) == _lib.IOLM_E_CORRUPT_HEADER
    bad_form = list(words)
    bad_form[-1] = 9                                                                        # form tag
    assert status(_image_bytes(bad_form)) == _lib.IOLM_E_CORRUPT_HEADER
    bad_ffn = list(words)
    bad_ffn[18] = 512                                                                       # > d_ff
    assert status(_image_bytes(bad_ffn)) == _lib.IOLM_E_CORRUPT_HEADER
    st, _, _ = _image_info(tmp_path / "missing.iolmdev")
    assert st == _lib.IOLM_E_CONTRACT
