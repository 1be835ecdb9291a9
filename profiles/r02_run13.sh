mkdir -p gpurun_out
for sp in on off; do
  timeout 400 python bench.py --config c3-bf16 --steps 3 --no-cpu-baseline --sparse-mma $sp 2>/dev/null | tail -1 > gpurun_out/v13_c3bf16_$sp.json
  python -c "
import json; d=json.load(open('gpurun_out/v13_c3bf16_$sp.json')); k=d['kernels']
print('c3-bf16 sparse=$sp', round(d['value']), d['clocks']['sm_mhz'], {n:(v['ms'], v.get('GB/s') or v.get('TFLOP/s')) for n,v in k.items()})"
done
timeout 900 python profiles/peaks.py > gpurun_out/v13_peaks.log 2>&1; python -c "
import json; d=json.load(open('gpurun_out/r02_peaks.json')); print(d['peaks_tops_sustained'], d['peaks_tops_burst'])"
