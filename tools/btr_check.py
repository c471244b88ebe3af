"""Narrow-layer epoch kernel (rows on the TMEM lanes, kind 3) vs the f64 oracle (diagnostic).

    python tools/btr_check.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1908_07847_b200 as g  # noqa: E402
import paper_1908_07847_b200._lib as L  # noqa: E402
from oracle import oracle as O  # noqa: E402

lib = L.load()
for rows, H, epochs in ((200_000, 33, 4), (150_001, 64, 3), (131_072, 24, 3), (300_000, 48, 3), (1_000_000, 33, 5)):
    x, l = g.synthetic_arrays(rows, 33, 2, "planted-linear")
    t = l.astype(np.float32)
    net0 = g.init_weights(g.NetworkConfig(input_dim=33, hidden_dim=H, seed=3))
    ref, net = net0.copy(), net0.copy()
    O.train_batch_par(ref.w_ih2d, ref.w_ho2d, x, t, epochs, 0.1)
    stats = np.zeros((epochs, 5))
    g.run_train_segment_batch(net.w_ih2d, net.w_ho2d, x, t, epochs, 0.1, g.cuda(), stats)
    e1 = np.max(np.abs(net.w_ih - ref.w_ih) / np.maximum(1, np.abs(ref.w_ih)))
    e2 = np.max(np.abs(net.w_ho - ref.w_ho) / np.maximum(1, np.abs(ref.w_ho)))
    (tp, tn, fp, fn), loss = O.eval_counts(net0.w_ih2d, net0.w_ho2d, x, l)
    print(f"rows {rows} H {H} kind {lib.glx_batch_kernel_kind(rows, 33, H)}: w_ih {e1:.2e} w_ho {e2:.2e} "
          f"counts {stats[0, 1:].astype(int).tolist()} vs {[tp, tn, fp, fn]} loss {stats[0, 0]:.6g} vs {loss:.6g}",
          flush=True)
