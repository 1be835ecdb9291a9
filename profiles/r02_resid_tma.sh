# Dense residual GEMMs through TMA reduce-add (IOLM_RESID_TMA=1) vs the coalesced RMW: bitwise check + C1 / C2-W8A8 A/B.
mkdir -p gpurun_out
cat > /tmp/rt_eq.py <<'PY'
import os, sys, numpy as np
sys.path.insert(0, '.')
from paper_2507_04967_b200 import runtime as R, synth
res = []
for quant, aq in [("dense", False), ("q8", True), ("q8", False)]:
    b = synth.toy_bundle(1280, 2, 20, 5120, 128, seed=42, quant=quant)
    ids, offs = synth.rows(300, 200, 64)
    outs = []
    for v in ("0", "1"):
        os.environ["IOLM_RESID_TMA"] = v
        rt = R.ModelRuntime(b, act_quant=aq)
        gi, gl, gm = rt.decode_token_rows(ids, offs, 8)
        outs.append((gi.copy(), gl.copy(), gm, rt.forward(ids[offs[0]:offs[1]])))
        rt.close()
    same = np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1]) and outs[0][2] == outs[1][2] and np.array_equal(outs[0][3], outs[1][3])
    res.append((quant, aq, same))
print("resid TMA bitwise:", res)
PY
timeout 600 python /tmp/rt_eq.py 2>&1 | tail -2
for c in c1 c2-w8a8; do
  for m in 0 1 0 1; do
    IOLM_RESID_TMA=$m timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/r_${m}_$c.json
    python -c "
import json; d=json.load(open('gpurun_out/r_${m}_$c.json')); print('$c tma=$m', round(d['value'],1), d['clocks']['sm_mhz'], d['kernels']['gemm_o']['ms'], d['kernels']['gemm_out']['ms'])"
  done
done
