import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1908_07847_b200 import wide, _lib
N = int(sys.argv[1]) if len(sys.argv) > 1 else 4194304
L = _lib.load()
data = wide.WideData(N, seed=0)
w1, w2 = wide.init_wide_weights(0)
W1 = torch.from_numpy(w1).cuda(); W2 = torch.from_numpy(w2).cuda()
st = torch.cuda.current_stream().cuda_stream
run = lambda e: _lib.check(L.glx_wide_train(W1.data_ptr(), W2.data_ptr(), data.Xb.data_ptr(), data.XT.data_ptr(), data.labels.data_ptr(), N, e, 0.1, None, None, st))
run(1); torch.cuda.synchronize()
L.glx_profile_enable(1); L.glx_profile_read(None, None)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); run(2); e1.record(); torch.cuda.synchronize()
kms = np.zeros(1); kn = np.zeros(1, np.int64); L.glx_profile_read(_lib.ptr(kms), _lib.ptr(kn))
print(json.dumps({"lib": os.environ.get("GLX_LIB", "default").split("/")[-1], "N": N, "ms_per_epoch": e0.elapsed_time(e1) / 2, "tc_ms_per_epoch": kms[0] / 2}))
