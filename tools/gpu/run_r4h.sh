for v in tma direct tma direct; do
 echo -n "$v "; GLX_LIB=variants/lib_$v.so timeout 300 python tools/bench_configs.py --which 5 2>&1 | tail -1 | cut -c100-200
done
GLX_LIB=variants/lib_direct.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tc_gemm -s 10 -c 5 --csv --log-file gpurun_out/r4h_launches.csv python tools/bench_configs.py --which 5 > /dev/null 2>&1
