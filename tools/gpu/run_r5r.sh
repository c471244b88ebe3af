timeout 300 python tools/step_gap.py > gpurun_out/r5r_gap.log 2>&1; cat gpurun_out/r5r_gap.log | tail -3
