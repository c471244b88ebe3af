for r in 1 2; do for v in base stg2s3 s3; do
  echo -n "$v "; GLX_LIB=variants/lib_$v.so timeout 120 python tools/wide_time.py 4194304 2>&1 | tail -1
done; done > gpurun_out/r5l_ab.log 2>&1
cat gpurun_out/r5l_ab.log
