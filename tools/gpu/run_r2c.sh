set -x
python -m pytest tests/test_gpu_batch.py tests/test_gpu_tc.py tests/test_gpu_reference_suite.py -q -x -m gpu > gpurun_out/r2c_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2c_tests.log
timeout 600 python bench.py > gpurun_out/r2c_bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_bench_c4.log
timeout 600 python bench.py --workload c2 --steps 600 > gpurun_out/r2c_bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_bench_c2.log
GLX_BENCH_FORCE_DP=1 timeout 600 python bench.py > gpurun_out/r2c_bench_c4_dp1.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_bench_c4_dp1.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2c_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2c_launches.csv python bench.py --steps 5 --warmup 3 > gpurun_out/r2c_ncu_launch.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batchtc -s 4 -c 1 -o gpurun_out/r2c_batchtc_c4 python bench.py --steps 3 --warmup 3 > gpurun_out/r2c_ncu_full.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_ncu_full.log
