"""C4-shaped execution at toy scale: head_dim 128, 576-position context, 512-character rows
(each row is 8 prefill query chunks of 64 and 36 KV pages), W8A8 over pruned 2:4 weights."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2507_04967_b200 import runtime as R
from paper_2507_04967_b200 import synth

pytestmark = pytest.mark.gpu
DIMS = (256, 2, 2, 512, 576)  # head_dim 128


def rel_l2_rows(a, b):
    return np.linalg.norm(a - b, axis=1) / np.maximum(np.linalg.norm(b, axis=1), 1e-30)


def test_hd128_long_rows_logits_and_decode():
    b = synth.toy_bundle(*DIMS, seed=4)
    rt, om = R.ModelRuntime(b), O.OracleModel(b)
    ids, offs = synth.rows(0, 6, 512)
    row = ids[offs[0]:offs[1]]
    assert len(row) == 544
    assert rel_l2_rows(rt.forward(row), om.forward(row)[0]).max() <= 1e-2
    gi, gl, gm = rt.decode_token_rows(ids, offs, 8)
    oi, ol, omm = om.decode_ids(ids, offs, 8, threads=6)
    assert gm == omm
    same = sum(gl[i] == ol[i] and np.array_equal(gi[i, :gl[i]], oi[i, :ol[i]]) for i in range(6))
    assert same >= 5


def test_hd128_pruned_sparse24_w8a8():
    b = synth.toy_bundle(*DIMS, seed=4, quant="sparse24", heads=[1, 2], ffn=[256, 384])
    rt = R.ModelRuntime(b, act_quant=True)
    oq = O.OracleModel(b, act_quant=True)
    ids, offs = synth.rows(10, 2, 512)
    row = ids[offs[0]:offs[1]]
    assert rel_l2_rows(rt.forward(row), oq.forward(row)[0]).max() <= 2.5e-2
    full = rt.batch_decode(synth.row_strings(10, 4, 512), 8)
    assert rt.batch_decode(synth.row_strings(12, 1, 512), 8) == [full[2]]
