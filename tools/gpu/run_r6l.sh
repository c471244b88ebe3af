for r in 1 2; do for v in base dr16 dr32 poly1 notok; do
  echo -n "$v "; GLX_LIB=variants/lib_$v.so timeout 120 python tools/batch_epoch_time.py 256 2>&1 | tail -1 | cut -c1-100
done; done > gpurun_out/r6l_ab.log 2>&1
cat gpurun_out/r6l_ab.log
