timeout 900 python -m pytest tests/test_gpu_batch.py -q -x > gpurun_out/r6f_t.log 2>&1; echo "rc=$?" >> gpurun_out/r6f_t.log; tail -2 gpurun_out/r6f_t.log
grep -q "rc=0" gpurun_out/r6f_t.log || exit 1
timeout 900 python -m pytest tests/test_gpu_parity_fullsize.py -q -x -s -k "33" > gpurun_out/r6f_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r6f_parity.log; grep -E "33-33|passed|rc=" gpurun_out/r6f_parity.log
for r in 1 2; do for v in n48 n34; do for h in 33 34; do
  echo -n "$v H=$h "; GLX_LIB=variants/lib_$v.so timeout 120 python tools/batch_epoch_time.py $h 2>&1 | tail -1 | cut -c1-100
done; done; done > gpurun_out/r6f_ab.log 2>&1
cat gpurun_out/r6f_ab.log
