mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sparse_gpu.py -m gpu -q > gpurun_out/v9_tests.log 2>&1; tail -2 gpurun_out/v9_tests.log
for cfg in c3 c4; do
  timeout 400 python bench.py --config $cfg --steps 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/v9_$cfg.json
  python -c "
import json; d=json.load(open('gpurun_out/v9_$cfg.json')); k=d['kernels']
print('$cfg', round(d['value']), d['clocks']['sm_mhz'], {n:(v['ms'], v.get('GB/s') or v.get('TFLOP/s')) for n,v in k.items()})"
done
