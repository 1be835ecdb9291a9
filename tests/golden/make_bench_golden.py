"""Benchmark-size parity fixtures: the CPU oracle's greedy decode of the
FIRST rows of every bench.py workload (C1, C2-W8A8, C2-W4A16, C3, C3b, C4 - the full 24/28-layer
models, seed-42 weights, the benchmark's own synthetic rows), with the CPU top-1/top-2 logit gap and
max |logit| at every prediction, so tests/test_bench_parity_gpu.py can check the GPU against them in
seconds and trace every divergence to an fp near-tie.

    python tests/golden/make_bench_golden.py [config ...]     # ~30 min on 8 cores for all

Checkers (test infrastructure, oracle/):
  * dense / q4 weight-only configs: the C restatement in f32 (oracle/iolm_oracle.c), which is
    bit-exact with the reference on forward logits, greedy decode and madds (tests/test_oracle.py;
    C1 additionally pinned by tests/golden/c1.json, made by the reference itself);
  * W8A8 configs: the W8A8 restatement at the GPU engine's rounding points (gpu_points).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2507_04967_b200 import synth  # noqa: E402

HERE = Path(__file__).resolve().parent
ROWS = {"c1": 100, "c2-w8a8": 100, "c2-w4a16": 100, "c3": 100, "c3b": 100, "c4": 16, "c3-f16": 100}
FIRST_ROW = 0
MAX_NEW = 8


def bundle_digest(data: bytes) -> str:
    """sha256 of the serialized bundle: pins the random-init weights the fixture was made with."""
    return hashlib.sha256(data).hexdigest()


def make(name: str) -> None:
    cfg = bench.CONFIGS[name]
    n = ROWS[name]
    t0 = time.time()
    b = synth.toy_bundle(*cfg["dims"], seed=42, quant=cfg["quant"], heads=cfg.get("heads"), ffn=cfg.get("ffn"))
    aq = bool(cfg.get("act_quant"))
    om = O.OracleModel(b, act_quant=aq, gpu_points=aq)
    ids, offs = synth.rows(FIRST_ROW, n, cfg["row_chars"])
    oi, ol, madds, gap, amax = om.decode_ids(ids, offs, MAX_NEW, threads=os.cpu_count() or 1, gaps=True)
    fx = {
        "config": name, "workload": cfg["desc"], "bundle_sha256": bundle_digest(b),
        "checker": "W8A8 restatement, GPU rounding points (oracle/iolm_oracle.c gpu_points)" if aq
        else "f32 restatement (bit-exact with the reference)",
        "first_row": FIRST_ROW, "rows": n, "row_chars": cfg["row_chars"], "max_new_tokens": MAX_NEW,
        "ids": oi.tolist(), "len": ol.tolist(), "madds": int(madds),
        "gap": [[None if np.isnan(v) else float(v) for v in r] for r in gap],
        "amax": [[None if np.isnan(v) else float(v) for v in r] for r in amax],
        "seconds": round(time.time() - t0, 1),
    }
    (HERE / f"bench_{name}.json").write_text(json.dumps(fx))
    print(f"{name}: {n} rows in {fx['seconds']} s", flush=True)


if __name__ == "__main__":
    for name in sys.argv[1:] or list(ROWS):
        make(name)
