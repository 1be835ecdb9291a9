"""W4A16 with int4 weights in HBM, expanded to fp16 inside the tcgen05 GEMM (shared memory).

The kernel consumes the bundle's q4_perchannel payload as stored (nibble rows, low nibble = even
column, code = nibble - 8, f32 scale per row; proj/src/model.cpp:164-176). Checks:
* the GEMM equals an fp64 restatement of decode_tensor's semantics on the same fp16 activations
  (rel. error <= 1e-5: fp32 accumulation of exact fp16 products);
* the whole engine with native int4 weights is bitwise identical (logits and greedy ids) to the
  same engine holding the codes as fp16 in HBM (int4_mma off): the MMA sees identical operands;
  pruned / odd widths included.
"""
import numpy as np
import pytest

from paper_2507_04967_b200 import runtime as R
from paper_2507_04967_b200 import synth

pytestmark = pytest.mark.gpu
TOY = (128, 4, 4, 512, 160)


def h16_bits(x):
    return np.ascontiguousarray(x, np.float32).astype(np.float16).view(np.uint16)


def make_q4(rng, N, K):
    codes = rng.integers(-7, 8, size=(N, K)).astype(np.int8)
    nib = (codes + 8).astype(np.uint8)
    if K % 2:
        nib = np.concatenate([nib, np.full((N, 1), 0, np.uint8)], axis=1)
    packed = (nib[:, 0::2] | (nib[:, 1::2] << 4)).astype(np.uint8)
    scales = rng.uniform(1e-3, 2e-2, size=N).astype(np.float32)
    return np.frombuffer(packed.tobytes() + scales.tobytes(), np.uint8).copy(), codes, scales


@pytest.mark.parametrize("M,N,K,pair", [(300, 3840, 1280, 1), (1000, 1280, 5120, 1), (77, 136, 1280, 0),
                                        (513, 2560, 2504, 1), (40, 64, 64, 0)])
def test_w4_gemm(engine_lib, M, N, K, pair):
    rng = np.random.default_rng(M + N + K)
    payload, codes, scales = make_q4(rng, N, K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    a = np.ascontiguousarray(h16_bits(A))
    out = np.zeros((M, N), np.float32)
    st = engine_lib.iolm_cuda_debug_gemm_w4(a.ctypes.data, payload.ctypes.data, out.ctypes.data, M, N, K, pair)
    assert st == 0, engine_lib.iolm_cuda_last_error()
    af = a.view(np.float16).astype(np.float64)
    ref = (af @ codes.astype(np.float64).T) * scales.astype(np.float64)[None, :]
    err = np.abs(out - ref).max() / (np.abs(ref).max() + 1e-30)
    assert err < 1e-5, err


@pytest.mark.parametrize("heads,ffn", [(None, None), ([1, 3, 2, 4], [77, 250, 130, 512])])
def test_engine_int4_equals_codes(heads, ffn):
    b = synth.toy_bundle(*TOY, seed=42, quant="q4", heads=heads, ffn=ffn)
    w4 = R.ModelRuntime(b)
    cd = R.ModelRuntime(b, int4_mma=False)
    ids, offs = synth.rows(80, 3, 64)
    for r in range(3):
        row = ids[offs[r]:offs[r + 1]]
        assert np.array_equal(w4.forward(row), cd.forward(row))
    ids, offs = synth.rows(0, 64, 64)
    gi, gl, gm = w4.decode_token_rows(ids, offs, 8)
    di, dl, dm = cd.decode_token_rows(ids, offs, 8)
    assert gm == dm and np.array_equal(gl, dl) and np.array_equal(gi, di)
