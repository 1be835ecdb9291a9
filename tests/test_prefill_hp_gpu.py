"""tcgen05 prefill attention with O in TMEM (attn_tc.cu attn_prefill_hp_kernel: head-pair tiles for
hd 64, one head x 128 queries for hd 128 - the defaults) against the mma.sync kernel
(`prefill_tc=False`) and the CPU oracle.

Both kernels walk keys in 32-position blocks aligned to absolute positions, so they differ only in
fp32 summation order inside a block: logits agree to fp16 rounding (<= 5e-3 rel-L2), both stay within
the oracle tolerance (1e-2), and the head-pair kernel keeps batch invariance. Covers an even head
count (C1 shape, 20 heads), an odd one (7 heads: the last pair has one live head), hd 128 with rows up
to 590 tokens (several 128-query chunks), rows longer than one chunk, rows shorter than a page and
rows whose last block is partial."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2507_04967_b200 import runtime as R
from paper_2507_04967_b200 import synth

from parity import check_agreement

pytestmark = pytest.mark.gpu


def _rows(lens, seed):
    rng = np.random.default_rng(seed)
    rows = ["".join(chr(32 + int(c)) for c in rng.integers(0, 95, n)) for n in lens]
    ids = np.concatenate([np.array([R.BOS] + R.encode(r), np.int32) for r in rows])
    offs = np.concatenate([[0], np.cumsum([len(r) + 1 for r in rows])]).astype(np.int64)
    return ids, offs


@pytest.mark.parametrize("cfg", [(1280, 2, 20, 5120, 160), (448, 2, 7, 1024, 200), (512, 2, 4, 1024, 600)],
                         ids=["h20", "h7", "hd128"])
def test_prefill_hp_matches_mma_sync_and_oracle(cfg):
    b = synth.toy_bundle(*cfg, seed=42)
    hp, mm = R.ModelRuntime(b), R.ModelRuntime(b, prefill_tc=False)
    S = cfg[4]
    lens = [0, 1, 14, 15, 16, 31, 32, 47, 63, 64, 65, 96, 127, 128, 150, S - 10]
    ids, offs = _rows(lens, 3)
    om = O.OracleModel(b)
    for r in (2, 8, 10, 13, 15):  # forward logits: every position, both kernels and the oracle
        row = ids[offs[r]:offs[r + 1]]
        a, m = hp.forward(row), mm.forward(row)
        ref, _ = om.forward(row)
        rel = np.linalg.norm(a - m, axis=1) / np.maximum(np.linalg.norm(m, axis=1), 1e-30)
        assert rel.max() <= 5e-3, (r, rel.max())
        relo = np.linalg.norm(a - ref, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-30)
        assert relo.max() <= 1e-2, (r, relo.max())
    gi, gl, gm = hp.decode_token_rows(ids, offs, 6)
    mi, ml, mmad = mm.decode_token_rows(ids, offs, 6)
    oi, ol, omad = om.decode_ids(ids, offs, 6, threads=8)
    assert gm == mmad == omad
    check_agreement(om, ids, offs, gi, gl, oi, ol, label=f"hp {cfg}")
    # batch invariance: every row equals its own single-row call
    for i in (1, 9, 13, 15):
        one, onel, _ = hp.decode_token_rows(ids[offs[i]:offs[i + 1]], np.array([0, offs[i + 1] - offs[i]]), 6)
        assert onel[0] == gl[i] and np.array_equal(one[0, :onel[0]], gi[i, :gl[i]]), i
    hp.close()
    mm.close()
