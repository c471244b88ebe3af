"""Time glx_train_sweep on subsets of the config-3 grid (by hidden width) to see
where the sweep's time goes: python tools/sweep_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import json

import numpy as np
import torch

import paper_1908_07847_b200 as g
from conftest import load_case
from paper_1908_07847_b200 import _lib
from paper_1908_07847_b200.sweep import pack_pool

L = _lib.load()
c = load_case("paper_33_33_1")
x, t = c["train_x"], c["train_y"].astype(np.float32)
N, D = x.shape
X = torch.from_numpy(np.ascontiguousarray(x)).cuda()
T = torch.from_numpy(t).cuda()
st = torch.cuda.current_stream().cuda_stream
peak = 72.7
out = {}
for name, widths, seeds in (("all", range(8, 513, 8), range(64)), ("H<=64", range(8, 65, 8), range(64)),
                            ("H>=256", range(256, 513, 8), range(64)), ("H=512x64", [512], range(64)),
                            ("H=8x64", [8], range(64)), ("H=256x148", [256], range(148)),
                            ("H=512x148", [512], range(148)), ("H=128x296", [128], range(296))):
    hs, ss = g.sweep_grid(widths, seeds)
    nets = [g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=h, seed=s)) for h, s in zip(hs, ss)]
    pool, H, off = pack_pool(nets)
    wp = torch.from_numpy(pool).cuda()
    ep = 50
    run = lambda: _lib.check(L.glx_train_sweep(len(nets), _lib.ptr(H), _lib.ptr(off), wp.data_ptr(), X.data_ptr(),
                                               T.data_ptr(), N, D, ep, 0.1, 0, st))
    run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    fl = sum(4 * h * (D + 1) + 4 * (h + 1) + 2 * h for h in hs) * N * ep
    out[name] = {"nets": len(nets), "ms_per_epoch": ms / ep, "frac": fl / (ms * 1e-3) / 1e12 / peak,
                 "us_per_row_step": ms / ep / N * 1e3}
    print(name, json.dumps(out[name]), flush=True)
