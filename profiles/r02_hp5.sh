# hp ring-depth / L2-prefetch variants (C1, same box, alternating) + full GPU suite with the regenerated fixtures
mkdir -p gpurun_out
for v in 0 1 2 3 0 2; do
  IOLM_HP_VARIANT=$v timeout 600 python bench.py --config c1 --steps 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/hp5_v$v.json
  python -c "
import json; d=json.load(open('gpurun_out/hp5_v$v.json')); k=d['kernels']
print('v$v', round(d['value']), d['clocks']['sm_mhz'], k['attn_prefill'])"
done
timeout 2400 python -m pytest tests -m gpu -q -rf -s > gpurun_out/hp5_tests.log 2>&1; tail -3 gpurun_out/hp5_tests.log
grep -E "rows identical|^FAILED" gpurun_out/hp5_tests.log | cut -c1-400
