timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r3b_gputests.log 2>&1; echo "gpu rc=$?" >> gpurun_out/r3b_gputests.log
timeout 900 python bench.py > gpurun_out/r3b_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r3b_bench.log
