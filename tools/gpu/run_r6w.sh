timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r6w_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r6w_smoke.log
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r6w_gputests.log 2>&1; echo "gpu rc=$?" >> gpurun_out/r6w_gputests.log
tail -n 2 gpurun_out/r6w_gputests.log; tail -n 2 gpurun_out/r6w_smoke.log
