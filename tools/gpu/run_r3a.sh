timeout 600 python -m pytest tests/test_gpu_batch.py -q -x -m gpu > gpurun_out/r3a_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3a_tests.log
GLX_BATCH_KERNEL=tc timeout 200 python tools/batch_width_time.py 16 33 64 96 128 192 256 > gpurun_out/r3a_width.log 2>&1
GLX_BTC_PREC=fast GLX_BATCH_KERNEL=tc timeout 300 python - >> gpurun_out/r3a_width.log 2>&1 <<'PY'
import sys, numpy as np
sys.path.insert(0, '.')
import paper_1908_07847_b200 as g
from oracle import oracle as O
for H in (33, 128):
    x, l = g.synthetic_arrays(200_000, 33, 1, "planted-linear"); t = l.astype(np.float32)
    net0 = g.init_weights(g.NetworkConfig(input_dim=33, hidden_dim=H, seed=1))
    ref, net = net0.copy(), net0.copy()
    O.train_batch_par(ref.w_ih2d, ref.w_ho2d, x, t, 5, 0.1)
    g.run_train_segment_batch(net.w_ih2d, net.w_ho2d, x, t, 5, 0.1, g.cuda())
    e = max(np.max(np.abs(net.w_ih - ref.w_ih) / np.maximum(1, np.abs(ref.w_ih))), np.max(np.abs(net.w_ho - ref.w_ho) / np.maximum(1, np.abs(ref.w_ho))))
    print("fast H", H, "err", e)
PY
