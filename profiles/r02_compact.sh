# Last-layer head-row compaction: bitwise test + the suites that exercise the engine paths, then A/B benches.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_compact_gpu.py -m gpu -x -q -rf > gpurun_out/c_compact.log 2>&1; tail -3 gpurun_out/c_compact.log
timeout 1800 python -m pytest tests/test_runtime_gpu.py tests/test_stops_gpu.py tests/test_sparse_gpu.py tests/test_multi_gpu.py tests/test_w4_gpu.py tests/test_compressed_gpu.py -m gpu -q -rf > gpurun_out/c_suites.log 2>&1; tail -3 gpurun_out/c_suites.log
for c in c1 c3 c4; do
  IOLM_LAST_COMPACT=0 timeout 900 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/c_off_$c.json
  timeout 900 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/c_on_$c.json
  for f in gpurun_out/c_off_$c.json gpurun_out/c_on_$c.json; do python -c "
import json; d=json.load(open('$f')); print('$f', round(d['value'],1), d['clocks']['sm_mhz'], {k: v['ms'] for k, v in d['kernels'].items()})"; done
done
