set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r4a_gputests.log 2>&1; echo "gpu rc=$?" >> gpurun_out/r4a_gputests.log
timeout 600 python bench.py > gpurun_out/r4a_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r4a_bench.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4a_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r4a_smoke.log
tail -5 gpurun_out/r4a_gputests.log gpurun_out/r4a_bench.log gpurun_out/r4a_smoke.log
