set -x
nproc; free -g | head -2
python -m pytest tests/test_gpu_parity_fullsize.py -x -q -s -m gpu > gpurun_out/r2_parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/r2_parity.log
python -m pytest tests -x -q -m gpu > gpurun_out/r2_gputests.log 2>&1; echo "gpu rc=$?" >> gpurun_out/r2_gputests.log
tail -3 gpurun_out/r2_parity.log gpurun_out/r2_gputests.log
