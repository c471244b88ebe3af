"""Where the per-epoch time of the headline loop goes beyond the epoch kernel:
glx_train_batch over K epochs (one call) timed with CUDA events, against the
per-launch kernel times (glx_profile, events around each epoch-kernel launch) of
the same call. Config 4 shape (64Mi rows x 33 -> 256 -> 1) unless argv[1] rows."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1908_07847_b200 as g  # noqa: E402
import paper_1908_07847_b200._lib as L  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
D, H = 33, 256
lib = L.load()
st = torch.cuda.current_stream().cuda_stream
X, lab = g.synthetic_arrays_device(rows, D, 0, "planted-linear")
ld = int(lib.glx_packed_ld(D))
Xp = torch.empty((rows, ld), device="cuda")
T = lab.float()
L.check(lib.glx_pack_rows(X.data_ptr(), T.data_ptr(), None, rows, D, Xp.data_ptr(), st))
del X
net = g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=H, seed=0))
w1 = torch.from_numpy(net.w_ih).cuda()
w2 = torch.from_numpy(net.w_ho).cuda()
flag = torch.zeros(1, dtype=torch.int32, device="cuda")


def run(k):
    L.check(lib.glx_train_batch(w1.data_ptr(), w2.data_ptr(), Xp.data_ptr(), rows, D, H, k, 0.1, None,
                                flag.data_ptr(), st))


run(3)
torch.cuda.synchronize()
out = {"rows": rows}
for k in (5, 20, 60):
    for prof in (0, 1):
        lib.glx_profile_enable(prof)
        lib.glx_profile_read(None, None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(k)
        e1.record()
        torch.cuda.synchronize()
        kms = np.zeros(1)
        kn = np.zeros(1, np.int64)
        lib.glx_profile_read(L.ptr(kms), L.ptr(kn))
        out[f"K{k}_prof{prof}"] = {"ms_per_epoch": e0.elapsed_time(e1) / k,
                                   "kernel_ms": float(kms[0]) / max(1, int(kn[0])) if prof else None}
lib.glx_profile_enable(0)
print(json.dumps(out))
