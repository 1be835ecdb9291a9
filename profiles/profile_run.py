"""Driver for ncu captures (never a bench number): builds the C1 engine and runs `--calls` decode
calls of `--rows` synthetic rows with device-resident ids.

  ncu --metrics gpu__time_duration.sum --clock-control none -s 4000 -c 600 --csv \
      --log-file gpurun_out/launches.csv python profiles/profile_run.py
  ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 300 -c 2 \
      -o gpurun_out/gemm python profiles/profile_run.py
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2507_04967_b200 import runtime as R  # noqa: E402
from paper_2507_04967_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=4096)
ap.add_argument("--calls", type=int, default=2)
ap.add_argument("--dims", default="1280,24,20,5120,128")
ap.add_argument("--quant", default="dense")
ap.add_argument("--act-quant", action="store_true")
args = ap.parse_args()
dims = tuple(int(x) for x in args.dims.split(","))
b = synth.toy_bundle(*dims, seed=42, quant=args.quant)
rt = R.ModelRuntime(b, act_quant=args.act_quant)
ids, offs = synth.rows(0, args.rows, 64)
d = torch.from_numpy(ids).cuda()
torch.cuda.synchronize()
for _ in range(args.calls):
    o, ln, _ = rt.decode_token_rows(None, offs, 8, device_ids=d.data_ptr())
print("rows", args.rows, "stats", rt.last_stats())
