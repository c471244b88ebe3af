set -x
timeout 900 python -m pytest tests/test_gpu_generic.py tests/test_gpu_batch.py tests/test_gpu_online.py -q -x -m gpu > gpurun_out/r4b_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r4b_tests.log
tail -n 30 gpurun_out/r4b_tests.log
