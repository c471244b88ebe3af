timeout 1500 python -m pytest tests/test_gpu_parity_fullsize.py tests/test_gpu_fullsize.py -q -x -s > gpurun_out/r6i_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r6i_parity.log; grep -E "err|passed|failed|rc=" gpurun_out/r6i_parity.log | tail -12
timeout 600 python bench.py --steps 60 --warmup 5 > gpurun_out/r6i_bench.log 2>&1; tail -c 300 gpurun_out/r6i_bench.log
