set -x
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/r5d_wide_launches.csv python tools/wide_time.py 4194304 > gpurun_out/r5d_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wide_tail -s 4 -c 1 -o gpurun_out/r5d_tail python tools/wide_time.py 4194304 > gpurun_out/r5d_ncu2.log 2>&1
ls -la gpurun_out
