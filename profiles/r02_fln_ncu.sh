# Full ncu captures of 4 consecutive GEMM launches with the LN fused into W_out (C1, IOLM_FUSED_LN=1; diagnosis only).
mkdir -p gpurun_out
IOLM_FUSED_LN=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tn -s 100 -c 4 -o gpurun_out/h_fln2 python profiles/profile_run.py --config c1 --rows 4096 > gpurun_out/h_ncu.log 2>&1
tail -3 gpurun_out/h_ncu.log; ls -la gpurun_out/h_*
