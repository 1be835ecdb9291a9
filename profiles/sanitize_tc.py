"""Small forwards through the tcgen05 prefill attention (hd 128 one-head tiles, hd 64 head-pair tiles
with an odd head count, P in TMEM) and the 2:4 sparse (TMA reduce-add residual epilogue) / W4A16
GEMMs, plus a short decode, for compute-sanitizer runs (memcheck / racecheck / synccheck)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_04967_b200 import runtime as R  # noqa: E402
from paper_2507_04967_b200 import synth  # noqa: E402

ids, offs = synth.rows(0, 2, 200)
row = ids[offs[0]:offs[1]]
b = synth.toy_bundle(256, 1, 2, 512, 256, seed=1)
R.ModelRuntime(b).forward(row)  # hd 128 -> tcgen05 prefill (one head x 128 queries)
b = synth.toy_bundle(448, 1, 7, 512, 256, seed=1)
rt = R.ModelRuntime(b)
rt.forward(row)  # hd 64, 7 heads -> head-pair tiles, last pair half live
rt.decode_token_rows(ids, offs, 3)
b = synth.toy_bundle(256, 1, 2, 512, 256, seed=1, quant="sparse24")
R.ModelRuntime(b, act_quant=True).forward(row)  # 2:4 sparse W8A8 (residual via TMA reduce-add)
R.ModelRuntime(b).forward(row)  # 2:4 sparse kind::f16 (fp16 activations)
b = synth.toy_bundle(256, 1, 2, 512, 256, seed=1, quant="q4")
R.ModelRuntime(b).forward(row)  # W4A16 converters
print("sanitize_tc ok")
