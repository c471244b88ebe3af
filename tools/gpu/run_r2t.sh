timeout 300 python tools/btc_prec_check.py > gpurun_out/r2t_prec.log 2>&1
timeout 500 bash tools/gpu/ab_variants.sh base cvt0 rcp2p0 rcp2p1 > gpurun_out/r2t_ab.log 2>&1
