# P in TMEM (IOLM_HP_PT=1) vs the smem-P kernel: parity with PT on, then C1 / C4 A/B on one box
mkdir -p gpurun_out
IOLM_HP_PT=1 timeout 900 python -m pytest tests/test_prefill_hp_gpu.py tests/test_runtime_gpu.py tests/test_longrows_gpu.py -q -x -rf > gpurun_out/pt_tests.log 2>&1; tail -3 gpurun_out/pt_tests.log
for c in c1 c4; do
  for v in 0 1 0 1; do
    IOLM_HP_PT=$v timeout 900 python bench.py --config $c --steps 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/pt_${c}_$v.json
    python -c "
import json; d=json.load(open('gpurun_out/pt_${c}_$v.json')); k=d['kernels']
print('$c pt=$v', round(d['value']), d['clocks']['sm_mhz'], k['attn_prefill'])"
  done
done
