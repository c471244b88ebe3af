for r in 1 2 3; do for v in base rcp2; do echo -n "$v "; GLX_LIB=variants/lib_$v.so timeout 200 python tools/wide_time.py 4194304; done; done > gpurun_out/r5t_ab.log 2>&1
grep lib gpurun_out/r5t_ab.log
GLX_LIB=variants/lib_rcp2.so timeout 300 python -m pytest tests/test_gpu_tc.py -q -k "wide_config or fused_tail or sigmoid" > gpurun_out/r5t_t.log 2>&1; tail -1 gpurun_out/r5t_t.log
GLX_LIB=variants/lib_rcp2.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 8 --csv --log-file gpurun_out/r5t_launches.csv python tools/wide_time.py 4194304 > gpurun_out/r5t_ncu1.log 2>&1
