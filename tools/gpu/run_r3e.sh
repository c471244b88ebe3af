GLX_LIB=variants/lib_dbg.so timeout 150 python tools/btr_one.py > gpurun_out/r3e_dbg.log 2>&1; echo rc=$? >> gpurun_out/r3e_dbg.log
timeout 400 python tools/btr_check.py > gpurun_out/r3e_check.log 2>&1 || echo "check failed rc=$?" >> gpurun_out/r3e_check.log
timeout 200 python tools/batch_width_time.py 24 33 48 64 > gpurun_out/r3e_width.log 2>&1
GLX_BATCH_KERNEL=rt timeout 200 python tools/batch_width_time.py 4 8 16 >> gpurun_out/r3e_width.log 2>&1
