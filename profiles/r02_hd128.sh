# hd-128 prompt chunks on attn_prefill_hp_kernel<128>: parity + C4 A/B (hp vs round-1 tcgen05 vs mma.sync)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_prefill_hp_gpu.py tests/test_runtime_gpu.py tests/test_longrows_gpu.py tests/test_sparse_gpu.py tests/test_stops_gpu.py -q -rf > gpurun_out/hd128_tests.log 2>&1; tail -3 gpurun_out/hd128_tests.log; grep FAILED gpurun_out/hd128_tests.log
timeout 600 python -m pytest tests/test_w8a8_codes_gpu.py -q -rf -s -k c4 > gpurun_out/hd128_w8a8.log 2>&1; grep -E "c4-1layer|passed|failed" gpurun_out/hd128_w8a8.log | cut -c1-400
for pf in auto on off; do
  timeout 900 python bench.py --config c4 --steps 3 --no-cpu-baseline --prefill-tc $pf 2>/dev/null | tail -1 > gpurun_out/hd128_c4_${pf}.json
  python -c "
import json; d=json.load(open('gpurun_out/hd128_c4_${pf}.json')); k=d['kernels']
print('c4 $pf', round(d['value']), d['clocks']['sm_mhz'], k['attn_prefill'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_prefill -s 30 -c 1 \
  -o gpurun_out/hd128_c4_pf python profiles/profile_run.py --config c4 --rows 256 > gpurun_out/hd128_ncu.log 2>&1; tail -1 gpurun_out/hd128_ncu.log
