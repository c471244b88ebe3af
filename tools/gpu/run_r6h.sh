GLX_LIB=variants/lib_zb2acc.so timeout 900 python -m pytest tests/test_gpu_batch.py -q -x > gpurun_out/r6h_t.log 2>&1; echo "rc=$?" >> gpurun_out/r6h_t.log; tail -2 gpurun_out/r6h_t.log
grep -q "rc=0" gpurun_out/r6h_t.log || exit 1
for r in 1 2; do for v in base zb2 zb2acc; do for h in 256 128; do
  echo -n "$v H=$h "; GLX_LIB=variants/lib_$v.so timeout 120 python tools/batch_epoch_time.py $h 2>&1 | tail -1 | cut -c1-100
done; done; done > gpurun_out/r6h_ab.log 2>&1
cat gpurun_out/r6h_ab.log
