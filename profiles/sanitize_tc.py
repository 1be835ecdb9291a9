"""Small forwards through the tcgen05 prefill attention (hd 128) and the 2:4 sparse / W4A16 GEMMs,
for compute-sanitizer runs (racecheck / synccheck)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_04967_b200 import runtime as R  # noqa: E402
from paper_2507_04967_b200 import synth  # noqa: E402

ids, offs = synth.rows(0, 2, 200)
row = ids[offs[0]:offs[1]]
b = synth.toy_bundle(256, 1, 2, 512, 256, seed=1)
R.ModelRuntime(b).forward(row)  # hd 128 -> tcgen05 prefill
b = synth.toy_bundle(256, 1, 2, 512, 256, seed=1, quant="sparse24")
R.ModelRuntime(b, act_quant=True).forward(row)  # 2:4 sparse W8A8
b = synth.toy_bundle(256, 1, 2, 512, 256, seed=1, quant="q4")
R.ModelRuntime(b).forward(row)  # W4A16 converters
print("sanitize_tc ok")
