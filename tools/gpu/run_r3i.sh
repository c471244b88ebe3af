GLX_LIB=variants/lib_dbg.so timeout 150 python tools/btr_one.py > gpurun_out/r3i_dbg.log 2>&1; echo rc=$? >> gpurun_out/r3i_dbg.log
timeout 400 python tools/btr_check.py > gpurun_out/r3i_check.log 2>&1 || echo "check failed rc=$?" >> gpurun_out/r3i_check.log
timeout 200 python tools/batch_width_time.py 24 33 48 64 > gpurun_out/r3i_width.log 2>&1
GLX_LIB=variants/lib_rtt.so timeout 150 python tools/btc_timeline.py 1000000 33 glx_btr_timing_dump > gpurun_out/r3i_tl.log 2>&1
