set -x
timeout 240 python -m pytest tests/test_gpu_tc.py -q -k "fused_tail" -s > gpurun_out/r5c_tail.log 2>&1; echo "rc=$?" >> gpurun_out/r5c_tail.log
grep -E "fused|unfused|passed|failed|Error" gpurun_out/r5c_tail.log | tail -12
grep -q "rc=0" gpurun_out/r5c_tail.log || exit 1
for v in 0 1; do GLX_WIDE_TAIL=$v timeout 200 python tools/wide_time.py 4194304; done > gpurun_out/r5c_time.log 2>&1
cat gpurun_out/r5c_time.log
timeout 900 python -m pytest tests/test_gpu_tc.py -q > gpurun_out/r5c_tc.log 2>&1; echo "rc=$?" >> gpurun_out/r5c_tc.log
tail -5 gpurun_out/r5c_tc.log
for v in 0 1; do GLX_WIDE_TAIL=$v timeout 300 python tools/wide_time.py 16777216; done >> gpurun_out/r5c_time.log 2>&1
cat gpurun_out/r5c_time.log
