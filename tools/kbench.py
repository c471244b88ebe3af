"""Kernel-only timing of the full-batch epoch kernel (tuning aid; bench.py is the contract)."""
import json, os, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
import paper_1908_07847_b200 as g
from paper_1908_07847_b200 import _lib, dp

L = _lib.load()
tfl = np.zeros(1); ms = np.zeros(1)
_lib.check(L.glx_fp32_peak(0, 50000, _lib.ptr(tfl), _lib.ptr(ms)))
res = {"lib": os.environ.get("GLX_LIB", "default"), "peak": float(tfl[0])}
for H in [int(h) for h in os.environ.get("KB_H", "256,33").split(",")]:
    N, D = 1_000_000, 33
    x, l = g.synthetic_arrays(N, D, 0, "planted-linear")
    net = g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=H, seed=0))
    eng = dp.DeviceEngine(x, l.astype(np.float32), net.w_ih, net.w_ho)
    st = torch.cuda.current_stream().cuda_stream
    def run(k):
        _lib.check(L.glx_train_batch(eng.w1.data_ptr(), eng.w2.data_ptr(), eng.Xp.data_ptr(), N, D, H, k, 0.1, None, None, st))
    run(3); torch.cuda.synchronize()
    L.glx_profile_enable(1); L.glx_profile_read(None, None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(50); e1.record(); torch.cuda.synchronize()
    kms = np.zeros(1); kn = np.zeros(1, np.int64); L.glx_profile_read(_lib.ptr(kms), _lib.ptr(kn)); L.glx_profile_enable(0)
    k = kms[0] / kn[0]
    flops = N * (4 * H * (D + 1) + 4 * (H + 1) + 2 * H)
    if hasattr(L, "glx3_timing_dump"):
        L.glx3_timing_dump()
    res[f"H{H}"] = {"kernel_ms": k, "step_ms": e0.elapsed_time(e1) / 50, "frac": flops / (k * 1e-3) / 1e12 / res["peak"]}
print(json.dumps(res))
