for r in 1 2; do for v in base mxr mxr2; do for h in 33 64 48; do
  echo -n "$v H=$h "; GLX_LIB=variants/lib_$v.so timeout 120 python tools/batch_epoch_time.py $h 2>&1 | tail -1 | cut -c1-120
done; done; done
