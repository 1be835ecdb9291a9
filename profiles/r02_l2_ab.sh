mkdir -p gpurun_out
for cfg in c3 c1; do
for mb in 0 60 90 120; do
  IOLM_L2_PERSIST=$mb IOLM_L2_VERBOSE=1 timeout 300 python bench.py --config $cfg --steps 3 --no-cpu-baseline 2>gpurun_out/l2_err_${cfg}_$mb.txt | tail -1 > gpurun_out/l2_${cfg}_$mb.json
  python -c "
import json; d=json.load(open('gpurun_out/l2_${cfg}_$mb.json')); k=d['kernels']
print('$cfg', $mb, round(d['value']), d['clocks']['sm_mhz'], {n:(v['ms'], v.get('GB/s') or v.get('TFLOP/s')) for n,v in k.items()})" 
  grep "L2 persist" gpurun_out/l2_err_${cfg}_$mb.txt | head -1
done; done
