timeout 300 python -m pytest tests/test_gpu_tc.py -q -s > gpurun_out/r5q_tc.log 2>&1; echo "rc=$?" >> gpurun_out/r5q_tc.log
grep -E "N=|passed|failed|rc=" gpurun_out/r5q_tc.log
