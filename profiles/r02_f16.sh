# fp16 storage type + head-pair prefill v2 (O in TMEM): GPU test suite (bench-size W8A8 fixtures are
# regenerated separately), smoke, C1 / C3 / C2-W4A16 A/B, ncu of the hp kernel.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -s --deselect tests/test_bench_parity_gpu.py > gpurun_out/f16_tests.log 2>&1; tail -4 gpurun_out/f16_tests.log
grep -E "rows identical|^FAILED" gpurun_out/f16_tests.log | cut -c1-220
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_bench_parity_gpu.py -q -rf -s -k "c1 or w4a16 or bf16" > gpurun_out/f16_bparity.log 2>&1; grep -E "rows identical|passed|failed" gpurun_out/f16_bparity.log | cut -c1-300
for c in c1 c3; do
  for pf in auto off; do
    timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline --prefill-tc $pf 2>/dev/null | tail -1 > gpurun_out/f16_${c}_${pf}.json
    python -c "
import json; d=json.load(open('gpurun_out/f16_${c}_${pf}.json')); k=d['kernels']
print('$c $pf', round(d['value']), d['clocks']['sm_mhz'], k['attn_prefill'])"
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_prefill_hp -s 30 -c 1 \
  -o gpurun_out/f16_c1_pf python profiles/profile_run.py --config c1 --rows 2048 > gpurun_out/f16_ncu.log 2>&1; tail -1 gpurun_out/f16_ncu.log
