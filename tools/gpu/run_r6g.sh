timeout 300 python tools/sweep_probe.py > gpurun_out/r6g_probe.log 2>&1; tail -3 gpurun_out/r6g_probe.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:online_sgd_mt -s 1 -c 1 -o gpurun_out/r6g_sweep python tools/sweep_probe.py > gpurun_out/r6g_ncu.log 2>&1; tail -2 gpurun_out/r6g_ncu.log
