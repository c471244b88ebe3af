"""Config-3 sweep: the whole grid in one launch vs its H >= 128 and H < 128 parts
launched separately (each with its automatic units-per-thread choice)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
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
EP = 50


def prep(widths):
    hs, ss = g.sweep_grid(widths, range(64))
    nets = [g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=h, seed=s)) for h, s in zip(hs, ss)]
    pool, H, off = pack_pool(nets)
    return len(nets), H, off, torch.from_numpy(pool).cuda()


s2 = torch.cuda.Stream()


def run(p, stream=None):
    n, H, off, wp = p
    _lib.check(L.glx_train_sweep(n, _lib.ptr(H), _lib.ptr(off), wp.data_ptr(), X.data_ptr(), T.data_ptr(), N, D, EP,
                                 0.1, _lib.NUMERICS["fp32"], stream or st))


def concurrent(a, b):
    ev = torch.cuda.Event()
    ev.record()
    s2.wait_event(ev)
    run(a)
    run(b, s2.cuda_stream)  # the small networks behind, on the second stream
    done = torch.cuda.Event()
    done.record(s2)
    torch.cuda.current_stream().wait_event(done)


def timed(f, reps=3):
    f()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best / EP


allp, big, small = prep(range(8, 513, 8)), prep(range(128, 513, 8)), prep(range(8, 128, 8))
out = {"all_one_launch": timed(lambda: run(allp)), "big_only": timed(lambda: run(big)),
       "small_only": timed(lambda: run(small)), "big_then_small": timed(lambda: (run(big), run(small))),
       "concurrent": timed(lambda: concurrent(big, small))}
print(json.dumps({k: round(v, 4) for k, v in out.items()}), "ms per epoch")
