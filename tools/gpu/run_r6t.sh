for r in 1 2; do for v in base bn128; do echo -n "$v "; GLX_LIB=variants/lib_$v.so timeout 200 python tools/wide_time.py 4194304; done; done > gpurun_out/r6t_ab.log 2>&1
cat gpurun_out/r6t_ab.log
GLX_LIB=variants/lib_bn128.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 8 --csv --log-file gpurun_out/r6t_launches.csv python tools/wide_time.py 4194304 > gpurun_out/r6t_ncu.log 2>&1
