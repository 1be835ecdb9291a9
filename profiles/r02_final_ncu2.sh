# Final-build full ncu captures of the non-GEMM kernels of C1 (attention prefill / decode, LayerNorm) and the C3 sparse GEMMs.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_|ln_stream" -s 120 -c 6 -o gpurun_out/f5_c1_nongemm python profiles/profile_run.py --config c1 --rows 2048 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_sp" -s 120 -c 4 -o gpurun_out/f5_c3_sp python profiles/profile_run.py --config c3 --rows 2048 > /dev/null 2>&1
ls -la gpurun_out/f5_*
