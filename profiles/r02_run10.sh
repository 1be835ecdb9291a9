mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gram_gpu.py tests/test_dropin_gpu.py tests/test_compressed_gpu.py -m gpu -q -rf -s > gpurun_out/v10_tests.log 2>&1; tail -3 gpurun_out/v10_tests.log; grep -E "build_hessian|apply_recipe|W8A8|FAIL|semantic|specialize|validate|multi-device" gpurun_out/v10_tests.log | head -30
