timeout 400 python -m pytest tests/test_gpu_tc.py -q -s -k "tf32" > gpurun_out/r5y_t.log 2>&1; echo "rc=$?" >> gpurun_out/r5y_t.log
grep -E "N=|tf32 wide|passed|failed|rc=|Error" gpurun_out/r5y_t.log | tail -14
grep -q "rc=0" gpurun_out/r5y_t.log || exit 1
for r in 1 2; do for v in tc cuda; do echo -n "$v "; GLX_WIDE_TAIL32=$v timeout 300 python tools/wide_time_tf32.py 2097152; done; done > gpurun_out/r5y_time.log 2>&1; cat gpurun_out/r5y_time.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:wide_tail32 -c 2 --csv --log-file gpurun_out/r5y_launches.csv python tools/wide_time_tf32.py 2097152 > gpurun_out/r5y_ncu.log 2>&1
