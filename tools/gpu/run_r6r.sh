set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r6r_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r6r_smoke.log
timeout 900 python bench.py > gpurun_out/r6r_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r6r_bench.log
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r6r_gputests.log 2>&1; echo "gpu rc=$?" >> gpurun_out/r6r_gputests.log
timeout 300 python tools/wide_time.py 16777216 > gpurun_out/r6r_wide.log 2>&1
timeout 600 python tools/wide_time_tf32.py 16777216 >> gpurun_out/r6r_wide.log 2>&1
tail -n 3 gpurun_out/r6r_gputests.log; tail -n 2 gpurun_out/r6r_smoke.log; cat gpurun_out/r6r_wide.log
