timeout 400 python -m pytest tests/test_gpu_tc.py -q -s -k "tf32_fused" > gpurun_out/r5w_t.log 2>&1; echo "rc=$?" >> gpurun_out/r5w_t.log
grep -E "N=|passed|failed|rc=|Error" gpurun_out/r5w_t.log | tail -6
for r in 1 2; do for v in tpr2 tpr4; do echo -n "$v "; GLX_LIB=variants/lib_$v.so timeout 300 python tools/wide_time_tf32.py 2097152; done; done > gpurun_out/r5w_time.log 2>&1; cat gpurun_out/r5w_time.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:wide_tail32 -c 2 --csv --log-file gpurun_out/r5w_launches.csv python tools/wide_time_tf32.py 2097152 > gpurun_out/r5w_ncu.log 2>&1
