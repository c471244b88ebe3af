"""Time the full-batch epoch loop (glx_train_batch) on config 2's shape:
1Mi rows x 33 -> H -> 1, planted-linear synthetic rows packed on the device.

    python tools/batch_epoch_time.py [H]              # H = 256 (default) or 128
    GLX_BATCH_KERNEL=3 python tools/batch_epoch_time.py   # pin the FP32 three-role kernel
    GLX_LIB=variants/libX.so python tools/batch_epoch_time.py   # an alternative build

Prints ms per epoch (CUDA events around 20 epochs after warm-up) and the loss of
epochs 0, 1 and 19 (for A/B comparisons of numerics between builds).
"""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1908_07847_b200 as g  # noqa: E402
import paper_1908_07847_b200._lib as L  # noqa: E402


def main():
    H = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    rows, D = 1 << 20, 33
    lib = L.load()
    st = torch.cuda.current_stream().cuda_stream
    X, lab = g.synthetic_arrays_device(rows, D, 0, "planted-linear")
    ld = int(lib.glx_packed_ld(D))
    Xp = torch.empty((rows, ld), device="cuda")
    L.check(lib.glx_pack_rows(X.data_ptr(), None, lab.data_ptr(), rows, D, Xp.data_ptr(), st))
    net = g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=H, seed=0))
    w1, w2 = torch.from_numpy(net.w_ih).cuda(), torch.from_numpy(net.w_ho).cuda()
    stats = torch.zeros((20, 5), dtype=torch.float64, device="cuda")

    def run(k):
        L.check(lib.glx_train_batch(w1.data_ptr(), w2.data_ptr(), Xp.data_ptr(), rows, D, H, k, 0.1,
                                    stats.data_ptr(), None, st))

    run(3)
    torch.cuda.synchronize()
    w1.copy_(torch.from_numpy(net.w_ih))
    w2.copy_(torch.from_numpy(net.w_ho))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run(20)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"kernel_kind": int(lib.glx_batch_kernel_kind(rows, D, H)),
                      "GLX_BATCH_KERNEL": os.environ.get("GLX_BATCH_KERNEL"), "H": H,
                      "ms_per_epoch": e0.elapsed_time(e1) / 20,
                      "loss_epochs_0_1_19": stats[:, 0].cpu().numpy()[[0, 1, 19]].tolist()}))


if __name__ == "__main__":
    main()
