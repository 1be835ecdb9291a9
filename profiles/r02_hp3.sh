# hp v3 (metadata prefetch + deferred epilogue): parity, C1 A/B, ncu; bf16-vs-fp16 A/B on one box
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_prefill_hp_gpu.py tests/test_runtime_gpu.py -q -x -rf > gpurun_out/hp3_tests.log 2>&1; tail -2 gpurun_out/hp3_tests.log
timeout 900 python -m pytest tests/test_w8a8_codes_gpu.py -q -rf -s -k cascade > gpurun_out/hp3_cascade.log 2>&1; grep -E "GPU-vs|passed|failed" gpurun_out/hp3_cascade.log | cut -c1-600
for pf in auto off; do
  timeout 600 python bench.py --config c1 --steps 3 --no-cpu-baseline --prefill-tc $pf 2>/dev/null | tail -1 > gpurun_out/hp3_c1_${pf}.json
  python -c "
import json; d=json.load(open('gpurun_out/hp3_c1_${pf}.json')); k=d['kernels']
print('c1 $pf', round(d['value']), d['clocks']['sm_mhz'], k['attn_prefill'])"
done
for i in 1 2; do
  (cd .ab_bf16 && timeout 600 python bench.py --config c1 --steps 3 --no-cpu-baseline 2>/dev/null | tail -1) > gpurun_out/ab_bf16_$i.json
  timeout 600 python bench.py --config c1 --steps 3 --no-cpu-baseline --prefill-tc off 2>/dev/null | tail -1 > gpurun_out/ab_f16_$i.json
  python -c "
import json
for n in ['ab_bf16_$i','ab_f16_$i']:
    d=json.load(open('gpurun_out/'+n+'.json')); k=d['kernels']
    print(n, round(d['value']), d['clocks']['sm_mhz'], {x:k[x]['ms'] for x in ['gemm_qkv','gemm_in','gemm_out','ln','attn_decode']})"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_prefill -s 30 -c 1 \
  -o gpurun_out/hp3_c1_pf python profiles/profile_run.py --config c1 --rows 2048 > gpurun_out/hp3_ncu.log 2>&1; tail -1 gpurun_out/hp3_ncu.log
