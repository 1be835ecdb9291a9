# hp kernel MMA issuer (incremental ring state, precomputed descriptors): parity + C1 / C4 prefill
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_prefill_hp_gpu.py tests/test_runtime_gpu.py tests/test_longrows_gpu.py -q -x -rf > gpurun_out/mi_tests.log 2>&1; tail -2 gpurun_out/mi_tests.log
for c in c1 c4; do
  timeout 900 python bench.py --config $c --steps 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/mi_${c}.json
  python -c "
import json; d=json.load(open('gpurun_out/mi_${c}.json')); k=d['kernels']
print('$c', round(d['value']), d['clocks']['sm_mhz'], k['attn_prefill'])"
done
