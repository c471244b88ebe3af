set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests/test_gpu_parity_fullsize.py -x -q -s -m gpu > gpurun_out/r2_parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/r2_parity.log
python -m pytest tests -q -m gpu --deselect tests/test_gpu_parity_fullsize.py > gpurun_out/r2_gputests.log 2>&1; echo "gpu rc=$?" >> gpurun_out/r2_gputests.log
python bench.py --steps 20 --warmup 3 > gpurun_out/r2_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2_bench.log
tail -5 gpurun_out/r2_parity.log gpurun_out/r2_gputests.log gpurun_out/r2_bench.log
