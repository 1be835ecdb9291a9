"""Last-layer head-row compaction (engine.cu, Engine::launch_step): after the last layer's QKV GEMM
(K/V of every token) and attention, only the step's head rows - the tokens whose logits the argmax
reads - go through Wo, LN2, W_in and W_out. Every op after the gather is row-wise, so greedy ids,
lengths and madds must be BITWISE those of the uncompacted engine (IOLM_LAST_COMPACT=0) for every
weight form: fp16 dense, W8A8 (per-token scales of the compacted rows), W4A16, 2:4 sparse with int8
and fp16 activations, irregular pruning; with step budgets that split prompts across steps (prompt
chunks without a head row) and with the shared-prefix K/V-only step (no head rows at all)."""
import os

import numpy as np
import pytest

from paper_2507_04967_b200 import runtime as R
from paper_2507_04967_b200 import synth

pytestmark = pytest.mark.gpu

CASES = {
    "f16-hd64": dict(dims=(1280, 2, 20, 5120, 128), quant="dense"),
    "w8a8": dict(dims=(256, 3, 4, 1024, 160), quant="q8", act_quant=True),
    "w4a16": dict(dims=(256, 2, 4, 1024, 160), quant="q4"),
    "sp24-w8a8-pruned": dict(dims=(256, 3, 4, 1024, 160), quant="sparse24", act_quant=True, heads=[2, 3, 2],
                             ffn=[512, 384, 640]),
    "sp24-f16": dict(dims=(256, 2, 4, 1024, 160), quant="sparse24", heads=[2, 2], ffn=[512, 512]),
    "hd128-long": dict(dims=(256, 2, 2, 1024, 576), quant="dense", row_chars=400),
}


def _runtime(b, compact, **kw):
    old = os.environ.get("IOLM_LAST_COMPACT")
    try:
        if compact:
            os.environ.pop("IOLM_LAST_COMPACT", None)
        else:
            os.environ["IOLM_LAST_COMPACT"] = "0"
        return R.ModelRuntime(b, **kw)
    finally:
        if old is None:
            os.environ.pop("IOLM_LAST_COMPACT", None)
        else:
            os.environ["IOLM_LAST_COMPACT"] = old


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("budget", [1, 8])
def test_compacted_last_layer_is_bitwise(name, budget):
    c = CASES[name]
    b = synth.toy_bundle(*c["dims"], seed=42, quant=c["quant"], heads=c.get("heads"), ffn=c.get("ffn"))
    kw = dict(act_quant=c.get("act_quant", False))
    ids, offs = synth.rows(100, 40, c.get("row_chars", 64))
    for step_kw in [{}, dict(max_tokens_per_step=256, max_slots=8)]:
        on, off = _runtime(b, True, **kw, **step_kw), _runtime(b, False, **kw, **step_kw)
        try:
            gi, gl, gm = on.decode_token_rows(ids, offs, budget)
            ri, rl, rm = off.decode_token_rows(ids, offs, budget)
            assert gm == rm
            assert np.array_equal(gl, rl)
            for i in range(len(gl)):
                assert np.array_equal(gi[i, :gl[i]], ri[i, :rl[i]]), (name, step_kw, i)
            # forward() (all positions' logits) never compacts; its last position agrees with the
            # compacted decode's first token
            row = ids[offs[0]:offs[1]]
            assert int(np.argmax(on.forward(row)[-1])) == int(gi[0, 0]) or gl[0] == 0
        finally:
            on.close()
            off.close()
