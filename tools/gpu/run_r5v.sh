timeout 400 python -m pytest tests/test_gpu_tc.py -q -s -k "tf32" > gpurun_out/r5v_t.log 2>&1; echo "rc=$?" >> gpurun_out/r5v_t.log
grep -E "N=|tf32 wide|passed|failed|rc=|Error" gpurun_out/r5v_t.log | tail -14
for v in 0 1; do GLX_WIDE_TAIL=$v timeout 300 python tools/wide_time_tf32.py 2097152; done > gpurun_out/r5v_time.log 2>&1; cat gpurun_out/r5v_time.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:wide_tail32 -c 3 --csv --log-file gpurun_out/r5v_launches.csv python tools/wide_time_tf32.py 2097152 > gpurun_out/r5v_ncu.log 2>&1
