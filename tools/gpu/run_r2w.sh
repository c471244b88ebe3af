timeout 500 bash tools/gpu/ab_variants.sh base osig > gpurun_out/r2w_ab.log 2>&1
GLX_LIB=variants/lib_osig.so timeout 300 python tools/btc_prec_check.py > gpurun_out/r2w_prec.log 2>&1
