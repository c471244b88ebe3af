timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2x_gputests.log 2>&1; echo "gpu rc=$?" >> gpurun_out/r2x_gputests.log
timeout 600 python bench.py > gpurun_out/r2x_bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/r2x_bench_c4.log
timeout 600 python bench.py --workload c2 --steps 600 > gpurun_out/r2x_bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/r2x_bench_c2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batchtc_kernel -s 4 -c 1 -o gpurun_out/r2x_batchtc_c4 python bench.py --steps 3 --warmup 3 > gpurun_out/r2x_ncu_full.log 2>&1; echo "rc=$?" >> gpurun_out/r2x_ncu_full.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2x_launches.csv python bench.py --steps 5 --warmup 3 > gpurun_out/r2x_ncu_launch.log 2>&1; echo "rc=$?" >> gpurun_out/r2x_ncu_launch.log
