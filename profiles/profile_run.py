"""Driver for ncu captures (never a bench number): builds the engine of one bench.py config and runs
`--calls` decode calls of `--rows` synthetic rows with device-resident ids.

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -s 3000 -c 400 --csv --log-file gpurun_out/c1_launches.csv python profiles/profile_run.py --config c1
  ncu --set full --clock-control none --import-source on -k regex:gemm_tn -s 300 -c 2 \
      -o gpurun_out/gemm python profiles/profile_run.py --config c1
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2507_04967_b200 import runtime as R  # noqa: E402
from paper_2507_04967_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1", choices=sorted(CONFIGS))
ap.add_argument("--rows", type=int, default=16384)
ap.add_argument("--calls", type=int, default=1)
args = ap.parse_args()
cfg = CONFIGS[args.config]
b = synth.toy_bundle(*cfg["dims"], seed=42, quant=cfg["quant"], heads=cfg.get("heads"), ffn=cfg.get("ffn"))
rt = R.ModelRuntime(b, act_quant=cfg.get("act_quant", False))
ids, offs = synth.rows(0, args.rows, cfg["row_chars"])
d = torch.from_numpy(ids).cuda()
torch.cuda.synchronize()
for _ in range(args.calls):
    o, ln, _ = rt.decode_token_rows(None, offs, 8, device_ids=d.data_ptr())
print("config", args.config, "rows", args.rows, "stats", rt.last_stats())
