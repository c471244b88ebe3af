for r in 1 2; do for v in base tred; do for h in 256 128; do
  echo -n "$v H=$h "; GLX_LIB=variants/lib_$v.so timeout 120 python tools/batch_epoch_time.py $h 2>&1 | tail -1 | cut -c1-200
done; done; done
GLX_LIB=variants/lib_tred.so timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_parity_fullsize.py -q -x -m gpu 2>&1 | tail -3
