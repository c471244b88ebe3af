python -m pytest tests/test_gpu_batch.py tests/test_gpu_parity_fullsize.py tests/test_gpu_fullsize.py tests/test_gpu_eval_sweep_trainer.py -q -s -m gpu > gpurun_out/r2e_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2e_tests.log
timeout 600 python bench.py --workload c2 --steps 600 > gpurun_out/r2e_bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_bench_c2.log
timeout 600 python bench.py > gpurun_out/r2e_bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_bench_c4.log
