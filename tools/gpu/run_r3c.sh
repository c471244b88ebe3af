timeout 400 python tools/btr_check.py > gpurun_out/r3c_check.log 2>&1 || echo "check failed rc=$?" >> gpurun_out/r3c_check.log
timeout 200 python tools/batch_width_time.py 24 33 48 64 > gpurun_out/r3c_width.log 2>&1
GLX_BATCH_KERNEL=rt timeout 200 python tools/batch_width_time.py 4 8 16 >> gpurun_out/r3c_width.log 2>&1
