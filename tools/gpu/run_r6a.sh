for v in nb3rs2; do GLX_LIB=variants/lib_$v.so timeout 400 python -m pytest tests/test_gpu_batch.py -q -x -k "rows_on_lanes or pipeline_checker or full_size or any_width" > gpurun_out/r6a_t_$v.log 2>&1; echo "rc=$?" >> gpurun_out/r6a_t_$v.log; tail -2 gpurun_out/r6a_t_$v.log; done
for r in 1 2; do for v in base nb3rs2 nb2rs2; do for h in 33 48 64; do
  echo -n "$v H=$h "; GLX_LIB=variants/lib_$v.so timeout 120 python tools/batch_epoch_time.py $h 2>&1 | tail -1 | cut -c1-110
done; done; done > gpurun_out/r6a_ab.log 2>&1
cat gpurun_out/r6a_ab.log
