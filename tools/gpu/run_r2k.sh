timeout 300 python tools/btc_prec_check.py > gpurun_out/r2k_prec.log 2>&1 || { echo "prec check failed/hung rc=$?" >> gpurun_out/r2k_prec.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_parity_fullsize.py tests/test_gpu_eval_sweep_trainer.py tests/test_gpu_fullsize.py -q -m gpu > gpurun_out/r2k_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2k_tests.log
timeout 120 python tools/batch_epoch_time.py 256 > gpurun_out/r2k_ab.log 2>&1
timeout 300 bash tools/gpu/ab_variants.sh p2 p4 p5 >> gpurun_out/r2k_ab.log 2>&1
GLX_LIB=variants/lib_timing.so timeout 120 python tools/btc_timeline.py > gpurun_out/r2k_timeline.log 2>&1
