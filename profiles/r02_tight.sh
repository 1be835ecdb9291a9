# Tightened parity tests (tie-traced C1 full model, C1-shaped, ragged, prefill kernels; C++ drop-in) + C1 bench.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_runtime_gpu.py -m gpu -q -rf -s > gpurun_out/t_runtime.log 2>&1; tail -3 gpurun_out/t_runtime.log
timeout 600 python -m pytest tests/test_dropin_gpu.py -m gpu -q -rf -s > gpurun_out/t_dropin.log 2>&1; tail -3 gpurun_out/t_dropin.log
grep -E "diverges|identical|agree" gpurun_out/t_dropin.log gpurun_out/t_runtime.log | head -20
timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/t_bench_c1.json; cut -c1-400 gpurun_out/t_bench_c1.json
