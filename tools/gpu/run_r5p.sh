for v in sp36 sp72; do GLX_LIB=variants/lib_$v.so timeout 300 python -m pytest tests/test_gpu_tc.py -q -k "fused_tail and 1048704" -s 2>&1 | grep -E "N=.*dW1 vs" | sed "s/^/$v /"; done > gpurun_out/r5p_acc.log
cat gpurun_out/r5p_acc.log
for r in 1 2; do for v in sp9 sp18 sp36 sp72; do echo -n "$v "; GLX_LIB=variants/lib_$v.so timeout 200 python tools/wide_time.py 4194304; done; done > gpurun_out/r5p_time.log 2>&1
grep lib gpurun_out/r5p_time.log
GLX_LIB=variants/lib_sp9.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 30 --csv --log-file gpurun_out/r5p_sp9_launches.csv python tools/wide_time.py 4194304 > gpurun_out/r5p_ncu1.log 2>&1
