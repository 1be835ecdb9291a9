# Round-2 final validation after the last-layer head-row compaction and the TMA reduce-add residual epilogue: full GPU suite, smoke, every bench
# config, the reference arm, launch lists (C1 / C3) and a full ncu capture of the C1 GEMMs. Outputs: gpurun_out/f4_*.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/f4_gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -rf -s > gpurun_out/f4_tests.log 2>&1; tail -2 gpurun_out/f4_tests.log
grep -E "^FAILED" gpurun_out/f4_tests.log | cut -c1-200
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2>/dev/null | tail -1 > gpurun_out/f4_bench_c1.json
for c in c0 c2-w8a8 c2-w4a16 c3 c3b c3-f16 c4; do
  timeout 900 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/f4_bench_$c.json
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 2>/dev/null | tail -1 > gpurun_out/f4_ref_c1.json
for f in gpurun_out/f4_bench_*.json gpurun_out/f4_ref_c1.json; do python -c "
import json; d=json.load(open('$f')); r=d.get('roofline') or {}
print('$f', round(d['value'],1), (d.get('e2e') or {}).get('value'), (d.get('clocks') or {}).get('sm_mhz'), r.get('kernel'), r.get('frac'))"; done
for c in c1 c3; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 3000 -c 400 --csv --log-file gpurun_out/f4_${c}_launches.csv python profiles/profile_run.py --config $c > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tn" -s 200 -c 8 -o gpurun_out/f4_c1_full python profiles/profile_run.py --config c1 --rows 2048 > /dev/null 2>&1
ls -la gpurun_out/f4_*launches.csv gpurun_out/f4_*.ncu-rep
