timeout 900 python bench.py --suite 5,5tf32,4,3,1 --out gpurun_out/r2q_suite.json > gpurun_out/r2q_suite.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_suite.log
GLX_BENCH_FORCE_DP=1 timeout 600 python bench.py > gpurun_out/r2q_bench_c4_dp1.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_bench_c4_dp1.log
timeout 600 python bench.py > gpurun_out/r2q_bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_bench_c4.log
