# register-resident quantizer rows up to 2560 columns (IOLM_QUANT_REG=1) vs the two-pass kernel
mkdir -p gpurun_out
IOLM_QUANT_REG=1 timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_compressed_gpu.py -q -x -rf > gpurun_out/qr_tests.log 2>&1; tail -1 gpurun_out/qr_tests.log
for c in c2-w8a8 c3; do
  for v in 0 1 0 1; do
    IOLM_QUANT_REG=$v timeout 900 python bench.py --config $c --steps 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/qr_${c}_$v.json
    python -c "
import json; d=json.load(open('gpurun_out/qr_${c}_$v.json')); k=d['kernels']
print('$c reg=$v', round(d['value']), d['clocks']['sm_mhz'], k['quant'])"
  done
done
