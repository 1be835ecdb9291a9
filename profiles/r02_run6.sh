mkdir -p gpurun_out
for cfg in c1 c2-w8a8 c3; do
  timeout 300 python bench.py --config $cfg --steps 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/v6_$cfg.json
  python -c "
import json; d=json.load(open('gpurun_out/v6_$cfg.json')); k=d['kernels']
print('$cfg', round(d['value']), d['clocks']['sm_mhz'], {n:(v['ms'], v.get('GB/s') or v.get('TFLOP/s')) for n,v in k.items()})"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_sp_kernel -s 40 -c 2 -o gpurun_out/v6_c3_sp python profiles/profile_run.py --config c3 --rows 2048 > gpurun_out/v6_ncu1.log 2>&1; tail -2 gpurun_out/v6_ncu1.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_prefill_kernel -s 20 -c 1 -o gpurun_out/v6_c1_pf python profiles/profile_run.py --config c1 --rows 2048 > gpurun_out/v6_ncu2.log 2>&1; tail -2 gpurun_out/v6_ncu2.log
