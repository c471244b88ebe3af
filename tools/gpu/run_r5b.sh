set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x -k "fused_tail" > gpurun_out/r5b_tail.log 2>&1; echo "rc=$?" >> gpurun_out/r5b_tail.log
tail -30 gpurun_out/r5b_tail.log
timeout 900 python -m pytest tests/test_gpu_tc.py -q > gpurun_out/r5b_tc.log 2>&1; echo "rc=$?" >> gpurun_out/r5b_tc.log
tail -5 gpurun_out/r5b_tc.log
for v in 0 1; do GLX_WIDE_TAIL=$v timeout 300 python tools/wide_time.py 16777216; done > gpurun_out/r5b_time.log 2>&1
cat gpurun_out/r5b_time.log
