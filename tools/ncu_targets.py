"""Run each kernel family once at its benchmark shape, for an ncu launch list
(`ncu --metrics ... python tools/ncu_targets.py`); the numbers printed without
ncu are not benchmark values (bench.py is)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import paper_1908_07847_b200 as g
from conftest import load_case
from paper_1908_07847_b200 import _lib, dp
from paper_1908_07847_b200.sweep import pack_pool

L = _lib.load()
st = torch.cuda.current_stream().cuda_stream
dev = torch.device("cuda")

# min-max fit / apply and row packing at config 4's row count
rows, D = 1 << 24, 33
X = torch.rand((rows, D), device=dev) * 100.0
Y = torch.empty_like(X)
mn, mx = torch.empty(D, device=dev), torch.empty(D, device=dev)
_lib.check(L.glx_minmax_fit(X.data_ptr(), rows, D, mn.data_ptr(), mx.data_ptr(), st))
_lib.check(L.glx_minmax_apply(X.data_ptr(), rows, D, mn.data_ptr(), mx.data_ptr(), Y.data_ptr(), st))
ld = int(L.glx_packed_ld(D))
T = torch.rand(rows, device=dev)
Xp = torch.empty((rows, ld), device=dev)
_lib.check(L.glx_pack_rows(X.data_ptr(), T.data_ptr(), None, rows, D, Xp.data_ptr(), st))
del X, Y, Xp, T

# config 2 epoch kernel (1M rows, 33-256-1)
x, l = g.synthetic_arrays(1_000_000, 33, 0, "planted-linear")
net = g.init_weights(g.NetworkConfig(input_dim=33, hidden_dim=256, seed=0))
eng = dp.DeviceEngine(x, l.astype(np.float32), net.w_ih, net.w_ho)
_lib.check(L.glx_train_batch(eng.w1.data_ptr(), eng.w2.data_ptr(), eng.Xp.data_ptr(), eng.N, 33, 256, 2, 0.1, None,
                             None, st))

# exact eval (1M rows, 33-256-1)
Xd = torch.from_numpy(x).to(dev)
Yd = torch.from_numpy(l).to(dev)
cnt = torch.zeros(4, dtype=torch.int64, device=dev)
loss = torch.zeros(1, dtype=torch.float64, device=dev)
_lib.check(L.glx_eval(eng.w1.data_ptr(), eng.w2.data_ptr(), Xd.data_ptr(), Yd.data_ptr(), 1_000_000, 33, 256, 1,
                      cnt.data_ptr(), loss.data_ptr(), st))

# config 1 (one network, fp32 and ref64) and config 3 (sweep, 20 epochs)
c = load_case("paper_33_33_1")
xs, ts = c["train_x"], c["train_y"].astype(np.float32)
Xs, Ts = torch.from_numpy(np.ascontiguousarray(xs)).to(dev), torch.from_numpy(ts).to(dev)
one = g.init_weights(g.NetworkConfig(input_dim=33, hidden_dim=33, seed=7))
w1, w2 = torch.from_numpy(one.w_ih).to(dev), torch.from_numpy(one.w_ho).to(dev)
for numerics in (0, 1):
    _lib.check(L.glx_train_online(w1.data_ptr(), w2.data_ptr(), Xs.data_ptr(), Ts.data_ptr(), 90, 33, 33, 200, 0.1,
                                  numerics, st))
hs, ss = g.sweep_grid(range(8, 513, 8), range(64))
nets = [g.init_weights(g.NetworkConfig(input_dim=33, hidden_dim=h, seed=s)) for h, s in zip(hs, ss)]
pool, H, off = pack_pool(nets)
wp = torch.from_numpy(pool).to(dev)
_lib.check(L.glx_train_sweep(len(nets), _lib.ptr(H), _lib.ptr(off), wp.data_ptr(), Xs.data_ptr(), Ts.data_ptr(), 90,
                             33, 20, 0.1, 0, st))
torch.cuda.synchronize()
print("ok")
