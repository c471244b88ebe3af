set -x
timeout 300 python -m pytest tests/test_gpu_tc.py -q -k "fused_tail" -s > gpurun_out/r5o_tail.log 2>&1; echo "rc=$?" >> gpurun_out/r5o_tail.log
GLX_LIB=variants/lib_sp18.so timeout 300 python -m pytest tests/test_gpu_tc.py -q -k "fused_tail and 1048704" -s > gpurun_out/r5o_tail18.log 2>&1; echo "rc=$?" >> gpurun_out/r5o_tail18.log
grep -E "N=|passed|failed|rc=" gpurun_out/r5o_tail.log gpurun_out/r5o_tail18.log
for r in 1 2; do for v in sp9 sp18; do echo -n "$v "; GLX_LIB=variants/lib_$v.so timeout 200 python tools/wide_time.py 4194304; done; GLX_WIDE_TAIL=0 timeout 200 python tools/wide_time.py 4194304; done > gpurun_out/r5o_time.log 2>&1
cat gpurun_out/r5o_time.log
