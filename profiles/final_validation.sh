set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final_tests.log 2>&1; tail -3 gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 400 python bench.py 2>/dev/null | tail -1 > gpurun_out/final_c1.json
for c in c0 c2-w8a8 c2-w4a16 c3 c3b c4; do timeout 400 python bench.py --config $c 2>/dev/null | tail -1 > gpurun_out/final_$c.json; done
for f in gpurun_out/final_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', round(d['value'],1), d['clocks']['sm_mhz'], d['roofline']['frac'])"; done
