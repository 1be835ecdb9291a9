mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sparse_gpu.py tests/test_compressed_gpu.py tests/test_image_gpu.py -m gpu -q -rf -x > gpurun_out/v11_tests.log 2>&1; tail -15 gpurun_out/v11_tests.log
