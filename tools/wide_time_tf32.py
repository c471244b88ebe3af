"""Time the tf32 wide epoch (config 5 shape, f32 rows): ms per epoch over 2 epochs."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1908_07847_b200 import wide, _lib
N = int(sys.argv[1]) if len(sys.argv) > 1 else 2097152
L = _lib.load()
data = wide.WideData(N, seed=0, precision="tf32")
w1, w2 = wide.init_wide_weights(0)
W1 = torch.from_numpy(w1).cuda(); W2 = torch.from_numpy(w2).cuda()
st = torch.cuda.current_stream().cuda_stream
run = lambda e: _lib.check(L.glx_wide_train_tf32(W1.data_ptr(), W2.data_ptr(), data.Xb.data_ptr(), data.XT.data_ptr(), data.labels.data_ptr(), N, e, 0.1, None, None, st))
run(1); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); run(2); e1.record(); torch.cuda.synchronize()
print(json.dumps({"N": N, "ms_per_epoch": e0.elapsed_time(e1) / 2}))
