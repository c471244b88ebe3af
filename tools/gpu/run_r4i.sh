timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 12 -c 1 -o gpurun_out/r4i_dh python tools/bench_configs.py --which 5 > gpurun_out/r4i_ncu.log 2>&1; echo "rc=$?"
timeout 300 ncu -i gpurun_out/r4i_dh.ncu-rep --page raw --csv > gpurun_out/r4i_dh_raw.csv 2>&1
timeout 300 ncu -i gpurun_out/r4i_dh.ncu-rep --page details --csv > gpurun_out/r4i_dh_details.csv 2>&1
ls -la gpurun_out/r4i*
