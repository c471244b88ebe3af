"""ms per full-batch epoch (glx_train_batch, 1M rows x 33 -> H -> 1) for a list of widths,
with the kernel each one selects (diagnostic for the narrow-layer kernel choice).

    python tools/batch_width_time.py 33 36 64 128
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1908_07847_b200 as g  # noqa: E402
import paper_1908_07847_b200._lib as L  # noqa: E402

rows, D = 1_000_000, 33
lib = L.load()
st = torch.cuda.current_stream().cuda_stream
X, lab = g.synthetic_arrays_device(rows, D, 0, "planted-linear")
Xp = torch.empty((rows, int(lib.glx_packed_ld(D))), device="cuda")
L.check(lib.glx_pack_rows(X.data_ptr(), None, lab.data_ptr(), rows, D, Xp.data_ptr(), st))
for H in [int(a) for a in sys.argv[1:]]:
    net = g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=H, seed=0))
    w1, w2 = torch.from_numpy(net.w_ih).cuda(), torch.from_numpy(net.w_ho).cuda()
    run = lambda k: L.check(lib.glx_train_batch(w1.data_ptr(), w2.data_ptr(), Xp.data_ptr(), rows, D, H, k, 0.1, None,
                                                None, st))
    run(5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run(100)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"H": H, "kind": int(lib.glx_batch_kernel_kind(rows, D, H)), "ms": e0.elapsed_time(e1) / 100}))
