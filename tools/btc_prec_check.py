"""tcgen05 epoch kernel vs the f64 oracle for each precision and row count (diagnostic).

    python tools/btc_prec_check.py
"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1908_07847_b200 as g  # noqa: E402
from oracle import oracle as O  # noqa: E402


def rel_err(a, b):
    return float(np.max(np.abs(a.astype(np.float64) - b) / np.maximum(1.0, np.abs(b.astype(np.float64)))))


for rows, epochs in ((4099, 2), (64 * 148 * 2, 2), (100_003, 2), (1_000_000, 2)):
    x, l = g.synthetic_arrays(rows, 33, 0, "planted-linear")
    t = l.astype(np.float32)
    net0 = g.init_weights(g.NetworkConfig(input_dim=33, hidden_dim=256, seed=0))
    ref = net0.copy()
    O.train_batch_par(ref.w_ih2d, ref.w_ho2d, x, t, epochs, 0.1)
    for prec in ("full", "fast"):
        os.environ["GLX_BTC_PREC"] = prec
        net = net0.copy()
        g.run_train_segment_batch(net.w_ih2d, net.w_ho2d, x, t, epochs, 0.1, g.cuda())
        print(f"rows {rows} {prec}: w_ih {rel_err(net.w_ih, ref.w_ih):.2e} w_ho {rel_err(net.w_ho, ref.w_ho):.2e}",
              flush=True)
