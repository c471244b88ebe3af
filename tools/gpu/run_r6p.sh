GLX_LIB=variants/lib_ht.so timeout 900 python -m pytest tests/test_gpu_tc.py -q -x -k "tf32" > gpurun_out/r6p_t.log 2>&1; echo "rc=$?" >> gpurun_out/r6p_t.log; tail -2 gpurun_out/r6p_t.log
grep -q "rc=0" gpurun_out/r6p_t.log || exit 1
for r in 1 2; do for v in base ht; do echo -n "$v tf32 "; GLX_LIB=variants/lib_$v.so timeout 200 python tools/wide_time_tf32.py 2097152; done; done > gpurun_out/r6p_ab.log 2>&1
cat gpurun_out/r6p_ab.log
