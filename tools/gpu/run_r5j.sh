for r in 1 2; do for v in base rcp4 rs2 both; do for h in 256 128; do
  echo -n "$v H=$h "; GLX_LIB=variants/lib_$v.so timeout 120 python tools/batch_epoch_time.py $h 2>&1 | tail -1 | cut -c1-150
done; done; done > gpurun_out/r5j_ab.log 2>&1
cat gpurun_out/r5j_ab.log
