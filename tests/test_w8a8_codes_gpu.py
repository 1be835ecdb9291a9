"""W8A8 against its GPU-faithful restatement (oracle/iolm_oracle.c with gpu_points: q/k/v, the
attention output and the GELU output rounded to fp16 where the engine stores them, before they are
quantized). The reference has no activation quantization; DESIGN.md §5 pins the rule.

Checked per GEMM input: the int8 operand codes the GPU fed every kind::i8 / 2:4 GEMM
(iolm_cuda_forward_codes) against the restatement's codes for the same rows, and the logits.
Remaining GPU/CPU differences are the fp32 summation order of LayerNorm and attention, the fp16
probabilities of the attention PV product and the SFU tanh of GELU: each can move a value across an
int8 rounding boundary, so codes are required equal on most elements and within +-1 everywhere in
the first layer, and the logits within W8A8_REL_TOL.

Measured (profiles/r02_w8a8_codes.txt): layer 0 of every model is >= 99.9% equal (its attention
input exactly); deeper layers drift because a single flipped code moves a token's amax, hence its
scale, hence all of its codes (a per-token-scale cascade, not an arithmetic difference). Two valid GPU
attention kernels that differ only in fp32 summation order disagree with EACH OTHER at least as much
(test_w8a8_cascade_is_kernel_independent), so the deeper-layer floor is a property of dynamic int8
activations, not of this engine."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2507_04967_b200 import runtime as R
from paper_2507_04967_b200 import synth
from parity import check_agreement

pytestmark = pytest.mark.gpu
W8A8_REL_TOL = 2.5e-2     # per-position logits rel-L2, toy model (max; the mean must stay <= 5e-3)
W8A8_REL_TOL_WIDE = 2.5e-2  # C2-C4 widths: max over positions; the mean must stay <= 1.5e-2
LAYER0_EQ = {"attn_in": 0.999, "attn_out_in": 0.995, "ffn_in": 0.98, "ffn_mid": 0.95}


def split_points(cfg, n, codes, scales):
    """-> list over layers of 4 (codes [n x cols], scales [n]) pairs."""
    hd = cfg["d_model"] // cfg["n_heads"] if isinstance(cfg, dict) else cfg.d_model // cfg.n_heads
    d = cfg["d_model"] if isinstance(cfg, dict) else cfg.d_model
    heads = cfg["active_heads"] if isinstance(cfg, dict) else cfg.active_heads
    ffn = cfg["active_ffn"] if isinstance(cfg, dict) else cfg.active_ffn
    out, off, so = [], 0, 0
    for l in range(len(heads)):
        pts = []
        for cols in (d, len(heads[l]) * hd, d, ffn[l]):
            pts.append((codes[off:off + n * cols].reshape(n, cols), scales[so:so + n]))
            off += n * cols
            so += n
        out.append(pts)
    return out


CASES = {
    "toy-q8": dict(dims=(128, 4, 4, 512, 160), quant="q8"),
    "toy-sparse24": dict(dims=(128, 4, 4, 512, 160), quant="sparse24"),
    "c2-2layer": dict(dims=(1280, 2, 20, 5120, 128), quant="q8"),
    "c3-2layer": dict(dims=(1280, 2, 20, 5120, 128), quant="sparse24", heads=[10, 10], ffn=[2560, 2560]),
    "c4-1layer": dict(dims=(2048, 1, 16, 8192, 576), quant="sparse24", heads=[8], ffn=[4096], row_chars=512),
}


@pytest.mark.parametrize("name", list(CASES))
def test_w8a8_codes_and_logits(name):
    c = CASES[name]
    b = synth.toy_bundle(*c["dims"], seed=42, quant=c["quant"], heads=c.get("heads"), ffn=c.get("ffn"))
    rt = R.ModelRuntime(b, act_quant=True)
    om = O.OracleModel(b, act_quant=True, gpu_points=True)
    ids, offs = synth.rows(300, 2, c.get("row_chars", 64))
    for r in range(2):
        row = ids[offs[r]:offs[r + 1]]
        n = len(row)
        g_logits, g_codes, g_sc = rt.forward_codes(row)
        o_logits, o_codes, o_sc = om.forward_codes(row)
        rel = np.linalg.norm(g_logits - o_logits, axis=1) / np.linalg.norm(o_logits, axis=1)
        gp, op = split_points(om.cfg, n, g_codes, g_sc), split_points(om.cfg, n, o_codes, o_sc)
        stats = []
        for l in range(len(gp)):
            for p, pname in enumerate(["attn_in", "attn_out_in", "ffn_in", "ffn_mid"]):
                gc, gs = gp[l][p]
                oc, os_ = op[l][p]
                diff = np.abs(gc.astype(np.int32) - oc.astype(np.int32))
                eq = float((diff == 0).mean())
                stats.append((l, pname, eq, int(diff.max()), float(np.abs(gs / os_ - 1).max())))
        print(name, r, f"logits rel-L2 max {rel.max():.3e} mean {rel.mean():.3e}",
              " ".join(f"L{l}.{p}:{e:.5f}/{m}/{s:.1e}" for l, p, e, m, s in stats))
        toy = name.startswith("toy")
        for l, pname, eq, mx, _ in stats:
            if toy and l == 0:
                assert eq >= 0.999 and mx <= 1, (l, pname, eq, mx)
            elif toy:
                assert eq >= 0.85, (l, pname, eq)
            elif l == 0:
                assert eq >= LAYER0_EQ[pname] and mx <= 2, (l, pname, eq, mx)
            else:
                assert eq >= 0.8, (l, pname, eq)
        if toy:
            assert rel.max() <= W8A8_REL_TOL and rel.mean() <= 5e-3, (rel.max(), rel.mean())
        else:
            assert rel.max() <= W8A8_REL_TOL_WIDE and rel.mean() <= 1.5e-2, (rel.max(), rel.mean())


@pytest.mark.parametrize("name", ["toy-q8", "toy-sparse24"])
def test_w8a8_decode_vs_gpu_points_restatement(name):
    c = CASES[name]
    b = synth.toy_bundle(*c["dims"], seed=42, quant=c["quant"])
    rt = R.ModelRuntime(b, act_quant=True)
    om = O.OracleModel(b, act_quant=True, gpu_points=True)
    ids, offs = synth.rows(0, 64, 64)
    gi, gl, gm = rt.decode_token_rows(ids, offs, 8)
    oi, ol, omm = om.decode_ids(ids, offs, 8, threads=8)
    assert gm == omm
    div = check_agreement(om, ids, offs, gi, gl, oi, ol, label=name)
    print(name, "divergences", div)


def _point_eq(cfg, n, a, b):
    """per (layer, point): fraction of equal int8 codes between two forward_codes captures."""
    pa, pb = split_points(cfg, n, a[1], a[2]), split_points(cfg, n, b[1], b[2])
    return [[float((pa[l][p][0] == pb[l][p][0]).mean()) for p in range(4)] for l in range(len(pa))]


@pytest.mark.parametrize("name", ["c2-2layer", "c3-2layer"])
def test_w8a8_cascade_is_kernel_independent(name):
    """The per-token-scale cascade is a property of dynamic int8 activations, not of this engine's
    arithmetic: two valid GPU attention kernels (head-pair tcgen05 vs mma.sync; same 32-key blocks,
    different fp32 summation order) disagree with EACH OTHER on the same order of codes as the GPU
    does with the CPU restatement. Asserted: layer-0 attention inputs identical in all three, and
    GPU-vs-restatement equality at every (layer, point) no worse than GPU-vs-GPU minus 5 points."""
    c = CASES[name]
    b = synth.toy_bundle(*c["dims"], seed=42, quant=c["quant"], heads=c.get("heads"), ffn=c.get("ffn"))
    hp, mm = R.ModelRuntime(b, act_quant=True), R.ModelRuntime(b, act_quant=True, prefill_tc=False)
    om = O.OracleModel(b, act_quant=True, gpu_points=True)
    ids, offs = synth.rows(300, 2, c.get("row_chars", 64))
    for r in range(2):
        row = ids[offs[r]:offs[r + 1]]
        a, m, o = hp.forward_codes(row), mm.forward_codes(row), om.forward_codes(row)
        gg, go = _point_eq(om.cfg, len(row), a, m), _point_eq(om.cfg, len(row), a, o)
        print(name, r, "GPU-vs-GPU", [[round(x, 4) for x in l] for l in gg],
              "GPU-vs-restatement", [[round(x, 4) for x in l] for l in go])
        assert gg[0][0] == 1.0 and go[0][0] == 1.0
        for l in range(len(gg)):
            for p in range(4):
                assert go[l][p] >= gg[l][p] - 0.05, (l, p, go[l][p], gg[l][p])
    hp.close()
    mm.close()
