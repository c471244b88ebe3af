set -x
timeout 900 python -m pytest tests/test_gpu_tc.py -q -s > gpurun_out/r5i_tc.log 2>&1; echo "rc=$?" >> gpurun_out/r5i_tc.log
grep -E "fused|passed|failed|rc=" gpurun_out/r5i_tc.log | tail -8
for v in 0 1; do GLX_WIDE_TAIL=$v timeout 300 python tools/wide_time.py 16777216; done > gpurun_out/r5i_time.log 2>&1
cat gpurun_out/r5i_time.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/r5i_wide_launches.csv python tools/wide_time.py 4194304 > gpurun_out/r5i_ncu1.log 2>&1
