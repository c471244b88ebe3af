timeout 900 python -m pytest tests/test_gpu_tc.py -q -s -m gpu > gpurun_out/r2p_tc.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_tc.log
