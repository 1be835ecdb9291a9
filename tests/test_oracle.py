"""CPU-only: pins the oracle (C restatement + numpy bundle decode) and the workload generator
against the committed golden fixtures, which were produced by the reference itself
(tests/golden/make_golden.py over oracle/_ref). When the compiled reference is present it is also
compared directly."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_2507_04967_b200 import synth

GOLD = Path(__file__).resolve().parent / "golden"


def load(name):
    meta = json.loads((GOLD / f"{name}.json").read_text())
    logits = np.load(GOLD / f"{name}_logits.npz")
    return meta, logits


@pytest.mark.parametrize("name", ["tiny", "toy"])
def test_synth_bundle_matches_reference_hash(name):
    meta, _ = load(name)
    b = synth.toy_bundle(*meta["dims"], seed=meta["seed"])
    assert f"{synth.fnv1a(b):016x}" == meta["bundle_hash"]
    assert len(b) == meta["bundle_bytes"]


@pytest.mark.parametrize("name", ["tiny", "toy"])
def test_oracle_forward_bitexact_vs_golden(name):
    meta, logits = load(name)
    om = O.OracleModel(synth.toy_bundle(*meta["dims"], seed=meta["seed"]))
    ids, offs = synth.rows(meta["logit_first_row"], meta["logit_rows"], meta["row_chars"])
    for r in range(meta["logit_rows"]):
        got, madds = om.forward(ids[offs[r]:offs[r + 1]])
        assert np.array_equal(got.view(np.uint32), logits[f"row{r}"].view(np.uint32))
        assert madds == meta["forward_madds"][r]


@pytest.mark.parametrize("name", ["tiny", "toy"])
def test_oracle_decode_matches_golden(name):
    meta, _ = load(name)
    om = O.OracleModel(synth.toy_bundle(*meta["dims"], seed=meta["seed"]))
    ids, offs = synth.rows(meta["decode_first_row"], meta["decode_rows"], meta["row_chars"])
    oi, ol, madds = om.decode_ids(ids, offs, meta["max_new_tokens"], threads=4)
    assert [O.render(oi[i], ol[i]) for i in range(len(ol))] == meta["decode_outputs"]
    assert madds == meta["decode_madds"]


@pytest.mark.parametrize("name,quant", [("toy_q8", "q8"), ("toy_q4", "q4"), ("toy_sparse24", "sparse24")])
def test_compressed_payloads_and_decode(name, quant):
    """synth's RTN / magnitude-2:4 encoders write the same tensor payloads as the reference's
    apply_recipe; the numpy decode_tensor restatement + C oracle reproduce the reference logits
    bit-for-bit on them."""
    meta, logits = load(name)
    b = synth.toy_bundle(*meta["dims"], seed=meta["seed"], quant=quant)
    om = O.OracleModel(b)
    ids, offs = synth.rows(meta["logit_first_row"], meta["logit_rows"], meta["row_chars"])
    got, _ = om.forward(ids[offs[0]:offs[1]])
    assert np.array_equal(got.view(np.uint32), logits["row0"].view(np.uint32))
    ids, offs = synth.rows(0, meta["decode_rows"], meta["row_chars"])
    oi, ol, madds = om.decode_ids(ids, offs, 8, threads=4)
    assert [O.render(oi[i], ol[i]) for i in range(len(ol))] == meta["decode_outputs"]
    assert madds == meta["decode_madds"]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("name", ["toy_q8", "toy_q4", "toy_sparse24", "toy_pruned_sparse24"])
def test_reference_compress_reproduces_golden(name):
    meta, logits = load(name)
    base = O.ref_toy_bundle(*meta["dims"], seed=meta["seed"])
    b = O.ref_compress(base, meta["recipe"], synth.row_strings(0, meta["calibration_rows"], 64),
                       seed=meta["calibration_seed"])
    assert f"{synth.fnv1a(b):016x}" == meta["bundle_hash"]
    om = O.OracleModel(b)
    ids, offs = synth.rows(meta["logit_first_row"], 1, meta["row_chars"])
    got, _ = om.forward(ids[offs[0]:offs[1]])
    assert np.array_equal(got.view(np.uint32), logits["row0"].view(np.uint32))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_vs_reference_random_masks():
    b = O.ref_toy_bundle(48, 2, 3, 80, 64, seed=5)
    ref, om = O.RefRuntime(b), O.OracleModel(b)
    rng = np.random.default_rng(0)
    for _ in range(6):
        n = int(rng.integers(1, 64))
        ids = rng.integers(0, 131, size=n).astype(np.int32)
        mask = (rng.random(n) > 0.2).astype(np.uint8)
        mask[0] = 1
        a, ma = ref.forward(ids, mask)
        c, mc = om.forward(ids, mask)
        v = mask.astype(bool)
        assert np.array_equal(a[v].view(np.uint32), c[v].view(np.uint32)) and ma == mc


def test_c1_generator_and_forward_golden():
    """The 0.5B-class bundle (BASELINE configs[1]): generator hash + oracle last-position logits."""
    meta, logits = load("c1")
    b = synth.toy_bundle(*meta["dims"], seed=meta["seed"])
    assert f"{synth.fnv1a(b):016x}" == meta["bundle_hash"]
    om = O.OracleModel(b)
    del b
    ids, offs = synth.rows(meta["logit_first_row"], 1, meta["row_chars"])
    got, madds = om.forward(ids[offs[0]:offs[1]])
    assert np.array_equal(got.view(np.uint32), logits["row0"].view(np.uint32))
    assert madds == meta["forward_madds"][0]


def test_rtn_activation_quantizer_kats():
    """SPEC.md quantize_rtn examples (round-half-even, zero row -> scale 1), applied per token with
    the pinned W8A8 form q = rint(x * (1/s))."""
    codes, scales = O.quant_rows_s8(np.array([[0, 0, 0], [1.0, -2.0, 0.5]], np.float32))
    assert scales[0] == 1.0 and codes[0].tolist() == [0, 0, 0]
    assert scales[1] == np.float32(2.0) / np.float32(127.0)
    assert codes[1].tolist() == [64, -127, 32]
    x = np.random.default_rng(1).standard_normal((64, 257)).astype(np.float32)
    c, s = O.quant_rows_s8(x)
    assert np.all(np.abs(c.astype(np.float32) * s[:, None] - x) <= s[:, None] / 2 + 1e-7)


def test_gemm_s8_restatement():
    rng = np.random.default_rng(2)
    a = rng.integers(-127, 128, size=(7, 33), dtype=np.int8)
    w = rng.integers(-127, 128, size=(5, 33), dtype=np.int8)
    assert np.array_equal(O.gemm_s8(a, w), a.astype(np.int64) @ w.astype(np.int64).T)


def test_oracle_edge_semantics():
    """max_new 0, context-full stop, EOS never emitted, PAD/BOS rendering."""
    b = synth.toy_bundle(32, 2, 2, 64, 16, seed=3)
    om = O.OracleModel(b)
    ids = np.array([129] + [65] * 14, np.int32)  # 15 tokens, max_seq 16
    oi, ol, _ = om.decode_ids(ids, np.array([0, 15]), 8)
    assert ol[0] == 2  # emit, advance to 16 (full), emit, stop
    oi0, ol0, m0 = om.decode_ids(ids, np.array([0, 15]), 0)
    assert ol0[0] == 0 and m0 == 0
    assert O.render([65, 128, 129, 66], 4) == "AB"


def stop_case(name, var, budget):
    meta = json.loads((GOLD / f"{name}.json").read_text())
    e = meta["variants"][var]
    b = synth.scale_token_embeddings(synth.toy_bundle(*meta["dims"], seed=meta["seed"]),
                                     {int(k): v for k, v in e["factors"].items()})
    assert f"{synth.fnv1a(b):016x}" == e["bundle_hash"]
    prompts = meta["rows"]
    ids = np.concatenate([np.array([O.BOS] + [ord(c) for c in p], np.int32) for p in prompts])
    offs = np.concatenate([[0], np.cumsum([len(p) + 1 for p in prompts])]).astype(np.int64)
    return b, prompts, ids, offs, e[str(budget)]


@pytest.mark.parametrize("name", ["tiny_stops", "toy_stops"])
@pytest.mark.parametrize("var", ["eos", "pad", "bos", "mix"])
@pytest.mark.parametrize("budget", [1, 3, 8])
def test_oracle_stop_paths_vs_golden(name, var, budget):
    """EOS / PAD / BOS emission (runtime.cpp:286-298) on bundles whose tied-head rows for those ids
    are scaled up: the restatement's rendered outputs, per-row madds (= each row's number of
    advances, runtime.cpp:327-345) and the call total equal the reference's (golden fixtures)."""
    b, prompts, ids, offs, want = stop_case(name, var, budget)
    om = O.OracleModel(b)
    oi, ol, madds = om.decode_ids(ids, offs, budget, threads=8)
    assert [O.render(oi[i], ol[i]) for i in range(len(prompts))] == want["outputs"]
    assert madds == want["madds"]
    if name == "tiny_stops":
        for i in range(len(prompts)):
            _, _, m1 = om.decode_ids(ids[offs[i]:offs[i + 1]], np.array([0, offs[i + 1] - offs[i]]), budget)
            assert m1 == want["row_madds"][i], i
    # the fixture really exercises the path: some rows stop on EOS or emit PAD/BOS
    if var in ("eos", "mix"):
        assert any(ol[i] < budget and 0 < ol[i] for i in range(len(prompts))) or budget == 1
        assert any(ol[i] == 0 for i in range(len(prompts)))  # EOS on the first prediction
    if var in ("pad", "bos", "mix"):
        assert any(np.isin(oi[i, :ol[i]], [O.PAD, O.BOS]).any() for i in range(len(prompts)))
