#!/bin/bash
# A/B of an engine environment switch on a bench config: ab_env.sh VAR "v0 v1 v0 v1" [bench args...]
# Prints value and SM clock per run; full lines go to gpurun_out/ab_<VAR>.jsonl.
var=$1; vals=$2; shift 2
mkdir -p gpurun_out
for v in $vals; do
  line=$(env "$var=$v" timeout 400 python bench.py --no-kernel-timing "$@" 2>/dev/null | tail -1)
  echo "$line" >> "gpurun_out/ab_${var}.jsonl"
  echo "$line" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$var=$v', round(d['value'],1), d['unit'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
