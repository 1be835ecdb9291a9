mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_runtime_gpu.py -m gpu -q -x > gpurun_out/v14_tests.log 2>&1; tail -1 gpurun_out/v14_tests.log
for cfg in c1 c3 c4; do for gb in 0 1; do
  IOLM_LN_GB_SMEM=$gb timeout 400 python bench.py --config $cfg --steps 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/v14_${cfg}_$gb.json
  python -c "
import json; d=json.load(open('gpurun_out/v14_${cfg}_$gb.json')); k=d['kernels']
print('$cfg gb=$gb', round(d['value']), d['clocks']['sm_mhz'], {n:(v['ms'], v.get('GB/s') or v.get('TFLOP/s')) for n,v in k.items() if n in ('ln','quant','embed_ln')})"
done; done
