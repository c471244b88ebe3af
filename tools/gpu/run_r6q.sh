GLX_LIB=variants/lib_alt.so timeout 900 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/r6q_t.log 2>&1; echo "rc=$?" >> gpurun_out/r6q_t.log; tail -2 gpurun_out/r6q_t.log
grep -q "rc=0" gpurun_out/r6q_t.log || exit 1
for r in 1 2 3; do for v in noalt alt; do echo -n "$v "; GLX_LIB=variants/lib_$v.so timeout 200 python tools/wide_time.py 4194304; done; done > gpurun_out/r6q_ab.log 2>&1
cat gpurun_out/r6q_ab.log
GLX_LIB=variants/lib_alt.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 8 --csv --log-file gpurun_out/r6q_launches.csv python tools/wide_time.py 4194304 > gpurun_out/r6q_ncu.log 2>&1
