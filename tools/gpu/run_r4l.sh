set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r4l_gputests.log 2>&1; echo "gpu rc=$?" >> gpurun_out/r4l_gputests.log
timeout 900 python bench.py > gpurun_out/r4l_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r4l_bench.log
timeout 600 python bench.py --scaling 1 --steps 20 > gpurun_out/r4l_scaling.log 2>&1; echo "scaling rc=$?" >> gpurun_out/r4l_scaling.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4l_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r4l_smoke.log
tail -n 3 gpurun_out/r4l_gputests.log; tail -n 2 gpurun_out/r4l_smoke.log
