GLX_LIB=variants/lib_tmah.so timeout 900 python -m pytest tests/test_gpu_tc.py -q -x -k "tf32 or sigmoid or f32" > gpurun_out/r6o_t.log 2>&1; echo "rc=$?" >> gpurun_out/r6o_t.log; tail -2 gpurun_out/r6o_t.log
grep -q "rc=0" gpurun_out/r6o_t.log || exit 1
for r in 1 2; do for v in rowst tmah; do echo -n "$v tf32 "; GLX_LIB=variants/lib_$v.so timeout 200 python tools/wide_time_tf32.py 2097152; done; done > gpurun_out/r6o_ab.log 2>&1
cat gpurun_out/r6o_ab.log
GLX_LIB=variants/lib_tmah.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 9 --csv --log-file gpurun_out/r6o_launches.csv python tools/wide_time_tf32.py 2097152 > gpurun_out/r6o_ncu.log 2>&1
