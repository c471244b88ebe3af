set -x
timeout 900 python -m pytest tests/test_gpu_reference_backend.py tests/test_gpu_batch.py tests/test_gpu_generic.py -q -x -m gpu > gpurun_out/r4c_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r4c_tests.log
timeout 200 python tools/batch_epoch_time.py 256 > gpurun_out/r4c_time.log 2>&1
timeout 200 python tools/batch_epoch_time.py 33 >> gpurun_out/r4c_time.log 2>&1
tail -n 25 gpurun_out/r4c_tests.log; cat gpurun_out/r4c_time.log | tail -8
