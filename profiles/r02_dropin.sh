mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_dropin_gpu.py tests/test_resolver.py tests/test_stops_gpu.py -m gpu -q -rf -s > gpurun_out/v2_dropin.log 2>&1; tail -40 gpurun_out/v2_dropin.log
