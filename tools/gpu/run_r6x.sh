timeout 600 python tools/sweep_split_probe.py 2>&1 | tail -2
