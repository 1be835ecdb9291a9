"""GPU parity of batch_decode's stop and no-render paths (SURVEY.md Appendix A items 11-12,
/root/reference/proj/src/runtime.cpp:286-298): EOS stops a row before emitting (also on the very
first prediction, right after admission), PAD / BOS are emitted, fed back and render nothing, the
budget and full-context stops, and the reference FlopCounter madds of early stops.

The bundles scale the tok_embed rows of EOS / PAD / BOS (tied head, runtime.cpp:213-215) so a
random-init model emits them at varied steps; the expected outputs are the REFERENCE's own
(tests/golden/*_stops.json, made by tests/golden/make_golden.py over oracle/_ref), and token ids are
compared with the C restatement, which matches those fixtures exactly (tests/test_oracle.py).
The GPU engine pipelines steps: a row that hits EOS still gets one speculative token in the next
step, which must be discarded (engine.cu, Engine::decode)."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_2507_04967_b200 import runtime as R
from paper_2507_04967_b200 import synth
from parity import check_agreement, same_row

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def load_case(name, var):
    meta = json.loads((GOLD / f"{name}.json").read_text())
    e = meta["variants"][var]
    b = synth.scale_token_embeddings(synth.toy_bundle(*meta["dims"], seed=meta["seed"]),
                                     {int(k): v for k, v in e["factors"].items()})
    prompts = meta["rows"]
    ids = np.concatenate([np.array([R.BOS] + R.encode(p), np.int32) for p in prompts])
    offs = np.concatenate([[0], np.cumsum([len(p) + 1 for p in prompts])]).astype(np.int64)
    return b, prompts, ids, offs, e


@pytest.fixture(scope="module", params=[(n, v) for n in ["tiny_stops", "toy_stops"]
                                        for v in ["eos", "pad", "bos", "mix"]],
                ids=lambda p: f"{p[0]}-{p[1]}")
def case(request):
    name, var = request.param
    b, prompts, ids, offs, e = load_case(name, var)
    rt = R.ModelRuntime(b)
    small = R.ModelRuntime(b, max_tokens_per_step=256, max_slots=8)  # many steps, slots recycled
    yield name, var, b, prompts, ids, offs, e, rt, small
    rt.close()
    small.close()


@pytest.mark.parametrize("budget", [1, 3, 8])
def test_stop_paths_match_reference(case, budget):
    name, var, b, prompts, ids, offs, e, rt, small = case
    want = e[str(budget)]
    om = O.OracleModel(b)
    oi, ol, omm = om.decode_ids(ids, offs, budget, threads=8)
    assert [O.render(oi[i], ol[i]) for i in range(len(prompts))] == want["outputs"]  # oracle pinned
    gi, gl, gm = rt.decode_token_rows(ids, offs, budget)
    div = check_agreement(om, ids, offs, gi, gl, oi, ol, label=f"{name}/{var}/{budget}")
    # madds: the reference's per-row count (advances differ per stop reason) summed over the call
    want_madds = sum(want["row_madds"][i] for i in range(len(prompts)) if all(d[0] != i for d in div))
    got_madds = gm - sum(rt.decode_token_rows(ids[offs[i]:offs[i + 1]], np.array([0, offs[i + 1] - offs[i]]),
                                              budget)[2] for i, *_ in div)
    assert got_madds == want_madds
    # the rendered strings through the shim surface (ModelRuntime.batch_decode) equal the reference's
    c = R.FlopCounter()
    got = rt.batch_decode(prompts, budget, c)
    assert c.total() == gm
    for i in range(len(prompts)):
        if all(d[0] != i for d in div):
            assert got[i] == want["outputs"][i], (i, got[i], want["outputs"][i])
    # the same ids with a tiny token budget / 8 slots (rows admitted while EOS rows free slots)
    si, sl, sm = small.decode_token_rows(ids, offs, budget)
    assert sm == gm and all(same_row(si, sl, gi, gl, i) for i in range(len(prompts)))
    # a row stopping on its first prediction, and other early stops, alone in a call
    for i in [i for i in range(len(prompts)) if gl[i] < budget][:4]:
        one, l1, _ = rt.decode_token_rows(ids[offs[i]:offs[i + 1]], np.array([0, offs[i + 1] - offs[i]]), budget)
        assert l1[0] == gl[i] and np.array_equal(one[0, :l1[0]], gi[i, :gl[i]])
    if var in ("eos", "mix"):
        assert (gl == 0).any()  # EOS right after admission
    if var in ("pad", "bos", "mix"):
        assert any(np.isin(gi[i, :gl[i]], [R.PAD, R.BOS]).any() for i in range(len(prompts)))
