"""2:4 structured-sparse W8A8 on the sparse tensor cores (tcgen05.mma.sp kind::i8).

The sparse kernel consumes the bundle's sparse24_q8 payload as stored (kept codes + position
nibbles, proj/src/model.cpp:255-290; decode semantics :177-199). Checks:
* integer accumulators are bit-exact against X_s8 . dense(W)^T (the CPU restatement of
  decode_tensor's expansion with exact integer sums) over regular, tail and irregular shapes;
* the scaled epilogue (acc * s_a[token]) * s_w[channel] equals the f32 restatement bit-for-bit;
* the whole engine with sparse MMAs is bitwise identical (logits and greedy ids) to the same
  W8A8 engine with the weights expanded to dense int8 (sparse_mma off), including pruned and
  irregular shapes (C3/C3b), and batch invariance holds.
"""
import numpy as np
import pytest

from paper_2507_04967_b200 import runtime as R
from paper_2507_04967_b200 import synth

pytestmark = pytest.mark.gpu
TOY = (128, 4, 4, 512, 160)
PAIRS = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]


def make_sparse24(rng, N, K):
    """A sparse24_q8 tensor payload (codes, position nibbles, scales) and its dense int8 twin."""
    G = K // 4
    sel = rng.integers(0, 6, size=(N, G))
    pos = np.array(PAIRS, np.uint8)[sel]                              # [N, G, 2] ascending
    codes = rng.integers(-127, 128, size=(N, G, 2)).astype(np.int8)
    nib = (pos[..., 0] | (pos[..., 1] << 2)).astype(np.uint8)         # [N, G]
    if G % 2:
        nib = np.concatenate([nib, np.zeros((N, 1), np.uint8)], axis=1)
    idx = (nib[:, 0::2] | (nib[:, 1::2] << 4)).astype(np.uint8)        # low nibble = even group
    scales = rng.uniform(1e-3, 2e-2, size=N).astype(np.float32)
    payload = codes.tobytes() + idx.tobytes() + scales.tobytes()
    dense = np.zeros((N, G, 4), np.int8)
    n_i, g_i = np.meshgrid(np.arange(N), np.arange(G), indexing="ij")
    dense[n_i, g_i, pos[..., 0]] = codes[..., 0]
    dense[n_i, g_i, pos[..., 1]] = codes[..., 1]
    return np.frombuffer(payload, np.uint8).copy(), dense.reshape(N, K), scales


def run_sp(lib, X, payload, N, epi=5, a_scale=None):
    T, K = X.shape
    out_i = np.zeros((T, N), np.int32)
    out_f = np.zeros((T, N), np.float32)
    a = np.zeros(T, np.float32) if a_scale is None else np.ascontiguousarray(a_scale, np.float32)
    st = lib.iolm_cuda_debug_gemm_sp24(np.ascontiguousarray(X).ctypes.data, payload.ctypes.data, T, N, K, epi,
                                       a.ctypes.data, out_i.ctypes.data, out_f.ctypes.data)
    assert st == 0, lib.iolm_cuda_last_error()
    return out_i if epi == 5 else out_f


@pytest.mark.parametrize("T,N,K", [
    (224, 256, 256), (300, 1920, 1280), (1000, 2560, 1280), (77, 1280, 2560), (18944, 384, 640),
    (513, 130, 2512), (5, 16, 16),
])
def test_sp24_s32_bitexact(engine_lib, T, N, K):
    rng = np.random.default_rng(T + 3 * N + 7 * K)
    payload, Wd, _ = make_sparse24(rng, N, K)
    X = rng.integers(-127, 128, size=(T, K)).astype(np.int8)
    got = run_sp(engine_lib, X, payload, N)
    want = (X.astype(np.float64) @ Wd.astype(np.float64).T).astype(np.int64)  # exact: |sum| < 2^53
    assert np.array_equal(got.astype(np.int64), want)


def test_sp24_scaled_epilogue_bitexact(engine_lib):
    rng = np.random.default_rng(11)
    T, N, K = 450, 640, 1280
    payload, Wd, scales = make_sparse24(rng, N, K)
    X = rng.integers(-127, 128, size=(T, K)).astype(np.int8)
    a = rng.uniform(1e-3, 5e-2, size=T).astype(np.float32)
    got = run_sp(engine_lib, X, payload, N, epi=0, a_scale=a)
    acc = (X.astype(np.float64) @ Wd.astype(np.float64).T).astype(np.int64).astype(np.float32)
    want = (acc * a[:, None]).astype(np.float32) * scales[None, :]
    assert np.array_equal(got, want.astype(np.float32))


def test_sp24_rejects_unordered_positions(engine_lib):
    rng = np.random.default_rng(5)
    payload, _, _ = make_sparse24(rng, 16, 64)
    G = 16
    payload[16 * G * 2] = 0x01 | (0x4 << 4)  # row 0 group 0: p0 = 1, p1 = 0 (descending)
    X = np.zeros((8, 64), np.int8)
    out = np.zeros((8, 16), np.int32)
    st = engine_lib.iolm_cuda_debug_gemm_sp24(X.ctypes.data, payload.ctypes.data, 8, 16, 64, 5, None,
                                              out.ctypes.data, None)
    assert st == 3


@pytest.mark.parametrize("heads,ffn", [
    (None, None),                               # dense shapes
    ([2, 2, 2, 2], [256, 256, 256, 256]),      # C3-style 50% pruning
    ([1, 3, 2, 4], [124, 500, 260, 388]),      # C3b irregular (FFN widths % 4 == 0, odd group counts)
])
def test_engine_sparse_equals_dense_int8(heads, ffn):
    b = synth.toy_bundle(*TOY, seed=42, quant="sparse24", heads=heads, ffn=ffn)
    sp = R.ModelRuntime(b, act_quant=True)
    dn = R.ModelRuntime(b, act_quant=True, sparse_mma=False)
    ids, offs = synth.rows(60, 3, 64)
    for r in range(3):
        row = ids[offs[r]:offs[r + 1]]
        assert np.array_equal(sp.forward(row), dn.forward(row))
    ids, offs = synth.rows(0, 64, 64)
    gi, gl, gm = sp.decode_token_rows(ids, offs, 8)
    di, dl, dm = dn.decode_token_rows(ids, offs, 8)
    assert gm == dm and np.array_equal(gl, dl) and np.array_equal(gi, di)


def test_engine_sparse_batch_invariance():
    b = synth.toy_bundle(*TOY, seed=42, quant="sparse24", heads=[2, 2, 2, 2], ffn=[256] * 4)
    rt = R.ModelRuntime(b, act_quant=True)
    prompts = synth.row_strings(900, 16, 64)
    full = rt.batch_decode(prompts, 8)
    for i in [0, 7, 15]:
        assert rt.batch_decode([prompts[i]], 8) == [full[i]]


def test_engine_sparse_long_rows_hd128():
    """C4 attention shapes (hd 128, 544-token prompts) with 2:4 W8A8 weights: sparse MMAs are bitwise
    equal to the dense-int8 engine, and track the W8A8 restatement (oracle) within tolerance."""
    from oracle import oracle as O
    cfg = (256, 2, 2, 1024, 576)
    b = synth.toy_bundle(*cfg, seed=42, quant="sparse24", heads=[1, 2], ffn=[512, 516])
    sp = R.ModelRuntime(b, act_quant=True)
    dn = R.ModelRuntime(b, act_quant=True, sparse_mma=False)
    ids, offs = synth.rows(4000, 3, 512)
    row = ids[offs[0]:offs[1]]
    got = sp.forward(row)
    assert np.array_equal(got, dn.forward(row))
    ref = O.OracleModel(b, act_quant=True, gpu_points=True).forward(row)[0]
    rel = np.linalg.norm(got - ref, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-30)
    assert rel.max() <= 2.5e-2 and rel.mean() <= 5e-3, (rel.max(), rel.mean())  # W8A8 tolerance
    gi, gl, _ = sp.decode_token_rows(ids, offs, 8)
    di, dl, _ = dn.decode_token_rows(ids, offs, 8)
    assert np.array_equal(gl, dl) and np.array_equal(gi, di)


# ---------------------------------------------------------------- fp16 activations (kind::f16 .sp)

def h16_bits(x):
    h = np.ascontiguousarray(x, np.float32).astype(np.float16)
    return h.view(np.uint16), h.astype(np.float32)


@pytest.mark.parametrize("T,N,K", [(224, 256, 256), (300, 1920, 1280), (77, 1280, 2560), (513, 130, 2512), (5, 16, 16)])
def test_sp24_f16_gemm(engine_lib, T, N, K):
    """tcgen05.mma.sp kind::f16 over the payload's kept codes as exact fp16 and fp16 activations,
    epilogue acc * s_w: against an f64 product of the same fp16 values (fp32 accumulation bound)."""
    rng = np.random.default_rng(T + 5 * N + 11 * K)
    payload, Wd, scales = make_sparse24(rng, N, K)
    xb, xf = h16_bits(rng.standard_normal((T, K)).astype(np.float32))
    out = np.zeros((T, N), np.float32)
    st = engine_lib.iolm_cuda_debug_gemm_sp24_f16(xb.ctypes.data, payload.ctypes.data, T, N, K, out.ctypes.data)
    assert st == 0, engine_lib.iolm_cuda_last_error()
    want = (xf.astype(np.float64) @ Wd.astype(np.float64).T) * scales[None, :].astype(np.float64)
    bound = (np.abs(xf).astype(np.float64) @ np.abs(Wd).astype(np.float64).T) * scales[None, :] * 4e-6 + 1e-30
    assert np.all(np.abs(out - want) <= bound), float(np.max(np.abs(out - want) / bound))


@pytest.mark.parametrize("heads,ffn", [(None, None), ([2, 2, 2, 2], [256, 256, 256, 256]),
                                       ([1, 3, 2, 4], [124, 500, 260, 388])])
def test_engine_sparse_f16_matches_dense_codes(heads, ffn):
    """sparse24_q8 WITHOUT act_quant (the drop-in default): the 2:4 sparse tensor cores on fp16
    activations (W_SP24F) against the same engine with the codes expanded to dense fp16 (sparse_mma
    off): logits to fp32-accumulation-order rounding, greedy ids identical but for near-ties, and the
    reference semantics (f32 oracle) within the fp16 tolerance."""
    from oracle import oracle as O
    from parity import check_agreement
    b = synth.toy_bundle(*TOY, seed=42, quant="sparse24", heads=heads, ffn=ffn)
    sp = R.ModelRuntime(b)
    dn = R.ModelRuntime(b, sparse_mma=False)
    om = O.OracleModel(b)
    ids, offs = synth.rows(60, 3, 64)
    for r in range(3):
        row = ids[offs[r]:offs[r + 1]]
        a, d, ref = sp.forward(row), dn.forward(row), om.forward(row)[0]
        assert np.max(np.abs(a - d)) <= 1e-3 * np.max(np.abs(d)), np.max(np.abs(a - d))
        rel = np.linalg.norm(a - ref, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-30)
        assert rel.max() <= 1e-2, rel.max()
    ids, offs = synth.rows(0, 64, 64)
    gi, gl, gm = sp.decode_token_rows(ids, offs, 8)
    oi, ol, om_m = om.decode_ids(ids, offs, 8, threads=8)
    check_agreement(om, ids, offs, gi, gl, oi, ol, label="sp24 fp16")
    one, l1, _ = sp.decode_token_rows(ids[offs[5]:offs[6]], np.array([0, offs[6] - offs[5]]), 8)
    assert l1[0] == gl[5] and np.array_equal(one[0, :l1[0]], gi[5, :gl[5]])  # batch invariance
