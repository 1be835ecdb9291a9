mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_sp_kernel -s 102 -c 2 -o gpurun_out/v7_c3_sp python profiles/profile_run.py --config c3 --rows 2048 > gpurun_out/v7_ncu1.log 2>&1; tail -1 gpurun_out/v7_ncu1.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_prefill_kernel -s 30 -c 1 -o gpurun_out/v7_c1_pf python profiles/profile_run.py --config c1 --rows 2048 > gpurun_out/v7_ncu2.log 2>&1; tail -1 gpurun_out/v7_ncu2.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tn_kernel -s 102 -c 2 -o gpurun_out/v7_c2_i8 python profiles/profile_run.py --config c2-w8a8 --rows 2048 > gpurun_out/v7_ncu3.log 2>&1; tail -1 gpurun_out/v7_ncu3.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ln_ -s 60 -c 1 -o gpurun_out/v7_c3_ln python profiles/profile_run.py --config c3 --rows 2048 > gpurun_out/v7_ncu4.log 2>&1; tail -1 gpurun_out/v7_ncu4.log
