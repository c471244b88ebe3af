timeout 500 bash tools/gpu/ab_variants.sh base sred > gpurun_out/r2v_ab.log 2>&1
GLX_LIB=variants/lib_sred.so GLX_BTC_PREC=fast timeout 300 python tools/btc_prec_check.py > gpurun_out/r2v_prec.log 2>&1
