# 2:4 GEMM fp16 / QKV epilogues through staged bulk copies: parity + C3 / C3b / C3-f16 / C4 bench lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_sparse_gpu.py tests/test_compressed_gpu.py tests/test_w8a8_codes_gpu.py tests/test_bench_parity_gpu.py -q -rf -s > gpurun_out/h16s_tests.log 2>&1; tail -2 gpurun_out/h16s_tests.log; grep -E "^FAILED|rows identical" gpurun_out/h16s_tests.log | cut -c1-120
for c in c3 c4 c3-f16; do
  timeout 900 python bench.py --config $c --steps 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/h16s_${c}.json
  python -c "
import json; d=json.load(open('gpurun_out/h16s_${c}.json')); k=d['kernels']
print('$c', round(d['value']), d['clocks']['sm_mhz'], {x:(k[x]['ms'],round(k[x].get('TFLOP/s',0))) for x in ['gemm_qkv','gemm_in','gemm_o','gemm_out']})"
done
