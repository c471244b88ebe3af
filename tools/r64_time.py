"""Time the exact (ref64) online engine on the paper shape (90 x 33-33-1):
sample-epochs/s over `epochs` epochs (GLX_LIB=variants/lib_X.so for a variant;
a GLX_R64_TIMING build also prints per-phase cycles per row)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1908_07847_b200 as g  # noqa: E402

epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
H = int(sys.argv[2]) if len(sys.argv) > 2 else 33
rng = np.random.default_rng(0)
x = rng.random((90, 33), dtype=np.float32)
t = (rng.random(90) < 0.5).astype(np.float32)
net = g.init_weights(g.NetworkConfig(input_dim=33, hidden_dim=H, seed=1))
g.run_train_segment(net.w_ih2d, net.w_ho2d, x, t, 10, 0.1, g.sequential())
for numerics in ("ref64", "fp32"):
    net = g.init_weights(g.NetworkConfig(input_dim=33, hidden_dim=H, seed=1))
    t0 = time.perf_counter()
    g.run_train_segment(net.w_ih2d, net.w_ho2d, x, t, epochs, 0.1, g.cuda(numerics=numerics))
    dt = time.perf_counter() - t0
    print(f"{numerics} H={H}: {90 * epochs / dt:.3e} sample-epochs/s ({dt / (90 * epochs) * 1e9:.0f} ns/row) "
          f"digest {net.w_ih.sum():.9e}", flush=True)
