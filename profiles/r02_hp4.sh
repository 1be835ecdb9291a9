# hp v4 / tc: early S release. parity + C1 / C4 A/B + ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_prefill_hp_gpu.py tests/test_runtime_gpu.py tests/test_longrows_gpu.py -q -x -rf > gpurun_out/hp4_tests.log 2>&1; tail -2 gpurun_out/hp4_tests.log
for c in c1 c4; do
  for pf in auto off; do
    timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline --prefill-tc $pf 2>/dev/null | tail -1 > gpurun_out/hp4_${c}_${pf}.json
    python -c "
import json; d=json.load(open('gpurun_out/hp4_${c}_${pf}.json')); k=d['kernels']
print('$c $pf', round(d['value']), d['clocks']['sm_mhz'], k['attn_prefill'])"
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_prefill -s 30 -c 1 \
  -o gpurun_out/hp4_c1_pf python profiles/profile_run.py --config c1 --rows 2048 > gpurun_out/hp4_ncu.log 2>&1; tail -1 gpurun_out/hp4_ncu.log
