for r in 1 2; do
for v in chk nochk; do
  for h in 256 33; do
  echo -n "$v H=$h "; GLX_LIB=variants/lib_$v.so timeout 120 python tools/batch_epoch_time.py $h 2>&1 | tail -1 | cut -c1-90
  done
done
done
timeout 600 python -m pytest tests/test_gpu_batch.py -q -x -m gpu -k "pipeline" 2>&1 | tail -3
