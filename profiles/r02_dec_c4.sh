# C4 decode attention CTA shape A/B (heads per CTA, ring depth): bench.py --config c4, 3 steps each.
mkdir -p gpurun_out
for v in "0 3" "0 4" "2 3" "2 4" "8 3" "8 4"; do
  set -- $v
  IOLM_DEC_HG=$1 IOLM_DEC_STAGES=$2 timeout 600 python bench.py --config c4 --steps 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/d_$1_$2.json
  python -c "
import json; d=json.load(open('gpurun_out/d_$1_$2.json')); k=d['kernels']['attn_decode']; print('hg=$1 st=$2', round(d['value'],1), d['clocks']['sm_mhz'], k['ms'], k['GB/s'])"
done
