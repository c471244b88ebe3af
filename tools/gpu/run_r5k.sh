set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 0 -c 2 -o gpurun_out/r5k_wide_gemms python tools/wide_time.py 4194304 > gpurun_out/r5k_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wide_tail -s 1 -c 1 -o gpurun_out/r5k_tail python tools/wide_time.py 4194304 >> gpurun_out/r5k_ncu.log 2>&1
tail -3 gpurun_out/r5k_ncu.log
