mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_w8a8_codes_gpu.py tests/test_sparse_gpu.py tests/test_compressed_gpu.py -m gpu -q -x > gpurun_out/v15_tests.log 2>&1; tail -2 gpurun_out/v15_tests.log
for cfg in c2-w8a8 c3 c4; do for ga in 0 1; do
  IOLM_GELU_AMAX=$ga timeout 400 python bench.py --config $cfg --steps 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/v15_${cfg}_$ga.json
  python -c "
import json; d=json.load(open('gpurun_out/v15_${cfg}_$ga.json')); k=d['kernels']
print('$cfg amax=$ga', round(d['value']), d['clocks']['sm_mhz'], {n:(v['ms'], v.get('GB/s') or v.get('TFLOP/s')) for n,v in k.items() if n in ('quant','gemm_in','gemm_out')})"
done; done
