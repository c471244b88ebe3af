# A/B epoch timing of variant builds (tools/build_variants.py), 2 rounds each
for r in 1 2; do
for v in "$@"; do
  echo -n "$v "; GLX_LIB=variants/lib_$v.so python tools/batch_epoch_time.py 256 2>&1 | tail -1
done
done
