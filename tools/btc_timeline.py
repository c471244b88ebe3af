"""Per-phase clock64 timeline of the tcgen05 epoch kernel (CTA 0, tiles 8..23).

    python tools/build_variants.py timing="-DGLX_BTC_TIMING"
    GLX_LIB=variants/lib_timing.so python tools/btc_timeline.py [rows]
"""
import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1908_07847_b200 as g  # noqa: E402
import paper_1908_07847_b200._lib as L  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
D, H = 33, int(sys.argv[2]) if len(sys.argv) > 2 else 256
lib = L.load()
st = torch.cuda.current_stream().cuda_stream
X, lab = g.synthetic_arrays_device(rows, D, 0, "planted-linear")
Xp = torch.empty((rows, int(lib.glx_packed_ld(D))), device="cuda")
L.check(lib.glx_pack_rows(X.data_ptr(), None, lab.data_ptr(), rows, D, Xp.data_ptr(), st))
net = g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=H, seed=0))
w1, w2 = torch.from_numpy(net.w_ih).cuda(), torch.from_numpy(net.w_ho).cuda()
for _ in range(2):
    L.check(lib.glx_train_batch(w1.data_ptr(), w2.data_ptr(), Xp.data_ptr(), rows, D, H, 1, 0.1, None, None, st))
torch.cuda.synchronize()
fn = getattr(ctypes.CDLL(str(L.LIB_PATH)), sys.argv[3] if len(sys.argv) > 3 else "glx_btc_timing_dump"); fn()
