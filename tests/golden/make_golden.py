"""Generates the committed golden fixtures in tests/golden/ from the REFERENCE ITSELF
(oracle/_ref/libiolm_ref.so = /root/reference/proj/src compiled unmodified by oracle/Makefile).

    python tests/golden/make_golden.py            # tiny, toy, compressed toy twins
    python tests/golden/make_golden.py --c1       # + the 0.5B-class config (about 2 minutes)

Every fixture records: the bundle FNV hash (pins the random-init weight generator), full logits of
a few rows (ModelRuntime::forward), greedy outputs + FlopCounter madds of synthetic rows
(ModelRuntime::batch_decode). Rows are the synthetic table of SURVEY.md §8d.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_2507_04967_b200 import synth  # noqa: E402

HERE = Path(__file__).resolve().parent

CONFIGS = {
    "tiny": dict(dims=(32, 2, 2, 64, 128), rows=64, logit_rows=3),
    "toy": dict(dims=(128, 4, 4, 512, 160), rows=48, logit_rows=2),
}
RECIPES = {
    "q8": {"steps": [{"op": "quantize", "bits": 8, "method": "rtn"}]},
    "q4": {"steps": [{"op": "quantize", "bits": 4, "method": "rtn"}]},
    "sparse24": {"steps": [{"op": "sparsify", "pattern": "two_of_four", "method": "magnitude"},
                           {"op": "quantize", "bits": 8, "method": "rtn"}]},
    "pruned_sparse24": {"steps": [{"op": "prune", "head_ratio": 0.5, "ffn_ratio": 0.5},
                                  {"op": "sparsify", "pattern": "two_of_four", "method": "magnitude"},
                                  {"op": "quantize", "bits": 8, "method": "rtn"}]},
}


def fixture(name: str, bundle: bytes, n_rows: int, logit_rows: int, row_chars: int = 64, extra=None) -> None:
    rt = O.RefRuntime(bundle)
    prompts = synth.row_strings(0, n_rows, row_chars)
    outs, madds = rt.batch_decode(prompts, 8, threads=8)
    ids, offs = synth.rows(1000, logit_rows, row_chars)
    logits = {}
    fmadds = []
    for r in range(logit_rows):
        lg, m = rt.forward(ids[offs[r]:offs[r + 1]])
        logits[f"row{r}"] = lg
        fmadds.append(m)
    np.savez_compressed(HERE / f"{name}_logits.npz", **logits)
    meta = {
        "name": name, "bundle_hash": f"{rt.bundle_hash():016x}", "bundle_bytes": len(bundle),
        "decode_first_row": 0, "decode_rows": n_rows, "row_chars": row_chars, "max_new_tokens": 8,
        "decode_outputs": outs, "decode_madds": madds,
        "logit_first_row": 1000, "logit_rows": logit_rows, "forward_madds": fmadds,
        "instruction": synth.INSTRUCTION, "seed": 42,
    }
    if extra:
        meta.update(extra)
    (HERE / f"{name}.json").write_text(json.dumps(meta, indent=1))
    print(f"{name}: hash {meta['bundle_hash']}, {n_rows} rows, madds {madds}")


# Stop-path fixtures: the tied head makes a scaled tok_embed row
# win the argmax, so these bundles emit EOS (stop before emitting), PAD / BOS (emitted, fed back,
# rendered as nothing) at varied steps. Per-row FlopCounter madds pin each row's number of advances.
STOP_VARIANTS = {"eos": {130: 8.0}, "pad": {128: 8.0}, "bos": {129: 12.0}, "mix": {130: 6.0, 128: 6.0, 129: 6.0}}
STOP_BUDGETS = (1, 3, 8)


def stop_rows(max_seq: int) -> list[str]:
    rng = np.random.default_rng(11)
    lens = [0, 1, 2, 15, 16, 17, 31, 33, 63, max_seq - 4, max_seq - 3, max_seq - 2] + \
        [int(x) for x in rng.integers(0, max_seq - 1, 4)]
    ragged = ["".join(chr(32 + int(c)) for c in rng.integers(0, 95, n)) for n in lens]
    return synth.row_strings(0, 32, 64) + ragged


def stop_fixture(name: str, dims) -> None:
    base = O.ref_toy_bundle(*dims, seed=42)
    prompts = stop_rows(dims[4])
    meta = {"name": name, "dims": dims, "seed": 42, "rows": prompts, "variants": {}}
    for var, factors in STOP_VARIANTS.items():
        b = synth.scale_token_embeddings(base, factors)
        rt = O.RefRuntime(b)
        entry = {"factors": {str(k): v for k, v in factors.items()}, "bundle_hash": f"{rt.bundle_hash():016x}"}
        for n in STOP_BUDGETS:
            outs, total = rt.batch_decode(prompts, n, threads=8)
            per_row = [rt.batch_decode([p], n)[1] for p in prompts]
            assert sum(per_row) == total
            entry[str(n)] = {"outputs": outs, "row_madds": per_row, "madds": total}
        meta["variants"][var] = entry
    (HERE / f"{name}.json").write_text(json.dumps(meta, indent=1))
    print(f"{name}: {len(prompts)} rows x {len(STOP_VARIANTS)} variants x budgets {STOP_BUDGETS}")


def main() -> None:
    for name, c in CONFIGS.items():
        b = O.ref_toy_bundle(*c["dims"], seed=42)
        fixture(name, b, c["rows"], c["logit_rows"], extra={"dims": c["dims"]})
    base = O.ref_toy_bundle(*CONFIGS["toy"]["dims"], seed=42)
    calib = synth.row_strings(0, 8, 64)  # calibration = the first 8 rows
    for name, recipe in RECIPES.items():
        b = O.ref_compress(base, recipe, calib, seed=7)
        fixture(f"toy_{name}", b, 32, 1, extra={"dims": CONFIGS["toy"]["dims"], "recipe": recipe,
                                                "calibration_rows": 8, "calibration_seed": 7})
    stop_fixture("tiny_stops", CONFIGS["tiny"]["dims"])
    stop_fixture("toy_stops", CONFIGS["toy"]["dims"])
    if "--c1" in sys.argv:
        b = O.ref_toy_bundle(1280, 24, 20, 5120, 128, seed=42)
        fixture("c1", b, 16, 2, extra={"dims": (1280, 24, 20, 5120, 128)})


if __name__ == "__main__":
    main()
