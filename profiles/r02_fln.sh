# LayerNorm fused into the residual GEMM epilogue: bitwise tests, the engine suites, A/B benches (0 / 1 / 2).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fused_ln_gpu.py -m gpu -x -q -rf > gpurun_out/f_fln.log 2>&1; echo "fln tests rc=$?"; tail -3 gpurun_out/f_fln.log
timeout 1800 python -m pytest tests/test_compact_gpu.py tests/test_runtime_gpu.py tests/test_stops_gpu.py tests/test_multi_gpu.py tests/test_w8a8_codes_gpu.py tests/test_compressed_gpu.py tests/test_w4_gpu.py -m gpu -q -rf > gpurun_out/f_suites.log 2>&1; echo "suites rc=$?"; tail -3 gpurun_out/f_suites.log
for c in c1 c2-w8a8; do
  for m in 0 1 2; do
    IOLM_FUSED_LN=$m timeout 900 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/f_${m}_$c.json
    python -c "
import json; d=json.load(open('gpurun_out/f_${m}_$c.json')); print('$c fln=$m', round(d['value'],1), d['clocks']['sm_mhz'], {k: v['ms'] for k, v in d['kernels'].items()})"
  done
done
