# head kernel (8 rows / CTA) + FMA-pipe int8 rounding: parity + C1 / C3 / C4 lines
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gemm_gpu.py tests/test_runtime_gpu.py tests/test_compressed_gpu.py tests/test_w8a8_codes_gpu.py tests/test_stops_gpu.py -q -rf > gpurun_out/q8_tests.log 2>&1; tail -2 gpurun_out/q8_tests.log; grep FAILED gpurun_out/q8_tests.log | head
for c in c1 c3 c4; do
  timeout 900 python bench.py --config $c --steps 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/q8_${c}.json
  python -c "
import json; d=json.load(open('gpurun_out/q8_${c}.json')); k=d['kernels']
print('$c', round(d['value']), d['clocks']['sm_mhz'], {x:k[x]['ms'] for x in ['head','ln','quant','embed_ln'] if x in k})"
done
