for r in 1 2 3; do for v in base s5 s4 dr16; do
  echo -n "$v "; GLX_LIB=variants/lib_$v.so timeout 120 python tools/batch_epoch_time.py 256 2>&1 | tail -1 | cut -c1-100
done; done > gpurun_out/r6s_ab.log 2>&1
cat gpurun_out/r6s_ab.log
