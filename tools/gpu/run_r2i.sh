python -m pytest tests/test_gpu_batch.py tests/test_gpu_parity_fullsize.py tests/test_gpu_eval_sweep_trainer.py -q -x -m gpu > gpurun_out/r2i_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2i_tests.log
python tools/batch_epoch_time.py 256 > gpurun_out/r2i_ab.log 2>&1
GLX_LIB=variants/lib_timing.so timeout 120 python tools/btc_timeline.py > gpurun_out/r2i_timeline.log 2>&1
bash tools/gpu/ab_variants.sh off0 p0 p1 >> gpurun_out/r2i_ab.log 2>&1
