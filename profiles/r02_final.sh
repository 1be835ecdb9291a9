# Round-2 validation on one B200: full GPU test suite, smoke, every bench config, the reference arm,
# ncu launch lists of C1 / C3 / C4. Outputs land in gpurun_out/r02f_*.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r02f_gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -rf -s > gpurun_out/r02f_tests.log 2>&1; tail -4 gpurun_out/r02f_tests.log
grep -E "rows identical to the oracle" gpurun_out/r02f_tests.log | cut -c1-200
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py 2>/dev/null | tail -1 > gpurun_out/r02f_bench_c1.json
for c in c0 c2-w8a8 c2-w4a16 c3 c3b c3-f16 c4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/r02f_bench_$c.json
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 2>/dev/null | tail -1 > gpurun_out/r02f_ref_c1.json
for f in gpurun_out/r02f_bench_*.json gpurun_out/r02f_ref_c1.json; do python -c "
import json; d=json.load(open('$f')); print('$f', round(d['value'],1), d.get('e2e',{}).get('value'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('roofline') or {}).get('kernel'), (d.get('roofline') or {}).get('frac'))"; done
for c in c1 c3 c4; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 3000 -c 400 --csv --log-file gpurun_out/r02f_${c}_launches.csv python profiles/profile_run.py --config $c > /dev/null 2>&1
done
ls -la gpurun_out/r02f_*launches.csv
