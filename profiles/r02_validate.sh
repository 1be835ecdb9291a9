mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v1_gpu.txt
lscpu | head -20 > gpurun_out/v1_cpu.txt
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/v1_tests.log 2>&1; tail -15 gpurun_out/v1_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 500 python bench.py 2>gpurun_out/v1_c1.err | tail -1 > gpurun_out/v1_c1.json; cat gpurun_out/v1_c1.json | head -c 600
