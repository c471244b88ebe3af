for r in 1 2; do for v in base s38 s46 s74 nogate nohint; do
  echo -n "$v "; GLX_LIB=variants/lib_$v.so timeout 120 python tools/wide_time.py 4194304 2>&1 | tail -1
done; done > gpurun_out/r5h_ab.log 2>&1
cat gpurun_out/r5h_ab.log
