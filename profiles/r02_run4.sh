mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multi_gpu.py tests/test_w8a8_codes_gpu.py tests/test_dropin_gpu.py -m gpu -q -rf -s > gpurun_out/v4_tests.log 2>&1; tail -3 gpurun_out/v4_tests.log; grep -E "rel-L2 max|divergences|semantic join|multi-device|FAIL|passed|failed" gpurun_out/v4_tests.log | head -30
timeout 400 python bench.py 2>/dev/null | tail -1 > gpurun_out/v4_c1.json; head -c 200 gpurun_out/v4_c1.json; echo
timeout 400 python bench.py --config c2-w8a8 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/v4_c2.json; head -c 200 gpurun_out/v4_c2.json; echo
timeout 600 python profiles/peaks.py > gpurun_out/v4_peaks.log 2>&1; tail -30 gpurun_out/v4_peaks.log
