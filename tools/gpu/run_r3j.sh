GLX_BATCH_KERNEL=rt timeout 200 python tools/batch_width_time.py 8 16 20 > gpurun_out/r3j_width.log 2>&1
timeout 200 python tools/batch_width_time.py 8 16 20 >> gpurun_out/r3j_width.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r3j_gputests.log 2>&1; echo "gpu rc=$?" >> gpurun_out/r3j_gputests.log
