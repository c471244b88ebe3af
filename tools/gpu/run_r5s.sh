for r in 1 2 3; do for v in base direct; do echo -n "$v "; GLX_LIB=variants/lib_$v.so timeout 200 python tools/wide_time.py 4194304; done; done > gpurun_out/r5s_ab.log 2>&1
grep lib gpurun_out/r5s_ab.log
GLX_LIB=variants/lib_direct.so timeout 300 python -m pytest tests/test_gpu_tc.py -q -k "wide_config or fused_tail" > gpurun_out/r5s_t.log 2>&1; tail -1 gpurun_out/r5s_t.log
GLX_LIB=variants/lib_direct.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 8 --csv --log-file gpurun_out/r5s_direct_launches.csv python tools/wide_time.py 4194304 > gpurun_out/r5s_ncu1.log 2>&1
