# compute-sanitizer over the round-2 kernels (hp prefill hd 64 / 128, P in TMEM; 2:4 GEMM TMA reduce-add)
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool python profiles/sanitize_tc.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool: $(tail -1 gpurun_out/san_$tool.log)"
done
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard" gpurun_out/san_*.log | head
