set -x
true > gpurun_out/r4g_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r4g_tests.log
timeout 300 python tools/bench_configs.py --which 5 > gpurun_out/r4g_c5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tc_gemm -s 10 -c 10 --csv --log-file gpurun_out/r4g_c5_launches.csv python tools/bench_configs.py --which 5 > gpurun_out/r4g_ncu.log 2>&1
tail -n 3 gpurun_out/r4g_tests.log; tail -n 1 gpurun_out/r4g_c5.log | cut -c1-300
