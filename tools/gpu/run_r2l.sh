timeout 300 python tools/btc_prec_check.py > gpurun_out/r2l_prec.log 2>&1 || { echo "prec check failed/hung rc=$?" >> gpurun_out/r2l_prec.log; exit 1; }
timeout 120 python tools/batch_epoch_time.py 256 > gpurun_out/r2l_ab.log 2>&1
timeout 400 bash tools/gpu/ab_variants.sh tok0 p0 p1 p2 p4 >> gpurun_out/r2l_ab.log 2>&1
GLX_LIB=variants/lib_timing.so timeout 120 python tools/btc_timeline.py > gpurun_out/r2l_timeline.log 2>&1
