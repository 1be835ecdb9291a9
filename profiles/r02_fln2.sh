# Fused LayerNorm, per-slice claims (v2): bitwise tests + C1 / C2-W8A8 A/B (0 / 1 / 2).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fused_ln_gpu.py -m gpu -x -q -rf > gpurun_out/g_fln.log 2>&1; echo "fln tests rc=$?"; tail -3 gpurun_out/g_fln.log
for c in c1; do
  for m in 0 1 2; do
    IOLM_FUSED_LN=$m timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/g_${m}_$c.json
    python -c "
import json; d=json.load(open('gpurun_out/g_${m}_$c.json')); print('$c fln=$m', round(d['value'],1), d['clocks']['sm_mhz'], {k: v['ms'] for k, v in d['kernels'].items()})"
  done
done
