set -x
timeout 300 python tools/bench_configs.py --which 5 > gpurun_out/r4f_c5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 120 --csv --log-file gpurun_out/r4f_c5_launches.csv python tools/bench_configs.py --which 5 > gpurun_out/r4f_ncu.log 2>&1
tail -n 3 gpurun_out/r4f_c5.log
