mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_w8a8_codes_gpu.py tests/test_dropin_gpu.py -m gpu -q -rf -s > gpurun_out/v3_w8a8.log 2>&1; tail -5 gpurun_out/v3_w8a8.log; grep -E "rel-L2 max|divergences|semantic join|FAIL" gpurun_out/v3_w8a8.log | head -30
timeout 400 python bench.py 2>/dev/null | tail -1 > gpurun_out/v3_c1.json; head -c 300 gpurun_out/v3_c1.json; echo
timeout 400 python bench.py --config c2-w8a8 2>/dev/null | tail -1 > gpurun_out/v3_c2.json; head -c 300 gpurun_out/v3_c2.json
