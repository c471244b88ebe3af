set -x
timeout 240 python -m pytest tests/test_gpu_tc.py -q -k "fused_tail" -s > gpurun_out/r5n_tail.log 2>&1; echo "rc=$?" >> gpurun_out/r5n_tail.log
grep -E "N=|passed|failed|Error|rc=" gpurun_out/r5n_tail.log | tail -12
grep -q "rc=0" gpurun_out/r5n_tail.log || exit 1
for r in 1 2; do for v in 0 1; do GLX_WIDE_TAIL=$v timeout 200 python tools/wide_time.py 4194304; done; done > gpurun_out/r5n_time.log 2>&1
cat gpurun_out/r5n_time.log
timeout 900 python -m pytest tests/test_gpu_tc.py -q > gpurun_out/r5n_tc.log 2>&1; echo "rc=$?" >> gpurun_out/r5n_tc.log
tail -2 gpurun_out/r5n_tc.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 30 --csv --log-file gpurun_out/r5n_wide_launches.csv python tools/wide_time.py 4194304 > gpurun_out/r5n_ncu1.log 2>&1
