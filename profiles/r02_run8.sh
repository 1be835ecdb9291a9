mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_runtime_gpu.py -m gpu -q -k "persistent or prefill_tc or production" -s > gpurun_out/v8_tests.log 2>&1; tail -3 gpurun_out/v8_tests.log
for pf in 0 1; do
  IOLM_PF_PERSIST=$pf timeout 300 python bench.py --config c1 --steps 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/v8_c1_$pf.json
  python -c "
import json; d=json.load(open('gpurun_out/v8_c1_$pf.json')); k=d['kernels']
print('c1 pf=$pf', round(d['value']), d['clocks']['sm_mhz'], {n:(v['ms'], v.get('GB/s') or v.get('TFLOP/s')) for n,v in k.items() if 'attn' in n})"
done
IOLM_PF_PERSIST=1 timeout 300 python bench.py --config c3 --steps 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/v8_c3_1.json
python -c "
import json; d=json.load(open('gpurun_out/v8_c3_1.json')); k=d['kernels']
print('c3 pf=1', round(d['value']), d['clocks']['sm_mhz'], {n:(v['ms'], v.get('GB/s') or v.get('TFLOP/s')) for n,v in k.items() if 'attn' in n})"
