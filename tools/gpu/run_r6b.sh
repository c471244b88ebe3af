timeout 900 python -m pytest tests/test_gpu_batch.py -q -x > gpurun_out/r6b_batch.log 2>&1; echo "rc=$?" >> gpurun_out/r6b_batch.log; tail -2 gpurun_out/r6b_batch.log
timeout 900 python -m pytest tests/test_gpu_parity_fullsize.py -q -x -s -k "33 or rows_on" > gpurun_out/r6b_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r6b_parity.log; tail -4 gpurun_out/r6b_parity.log
for r in 1 2; do for h in 33 64 16; do echo -n "H=$h "; timeout 120 python tools/batch_epoch_time.py $h 2>&1 | tail -1 | cut -c1-100; done; done
