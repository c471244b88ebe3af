import sys, torch, time
sys.path.insert(0,'/root/repo')
import paper_1908_07847_b200 as g
from paper_1908_07847_b200 import _lib
L=_lib.load()
D=33
for rows in (1_000_000, 1<<20):
  for h in (33, 256):
    X, lab = g.synthetic_arrays_device(rows, D, 0, "planted-linear")
    Xp = torch.empty((rows, int(L.glx_packed_ld(D))), device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(L.glx_pack_rows(X.data_ptr(), None, lab.data_ptr(), rows, D, Xp.data_ptr(), st))
    net = g.init_weights(g.NetworkConfig(input_dim=D, hidden_dim=h, seed=0))
    w1, w2 = torch.from_numpy(net.w_ih).cuda(), torch.from_numpy(net.w_ho).cuda()
    run = lambda k: _lib.check(L.glx_train_batch(w1.data_ptr(), w2.data_ptr(), Xp.data_ptr(), rows, D, h, k, 0.1, None, None, st))
    run(5)
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(200); e1.record(); torch.cuda.synchronize()
        print(rows, h, L.glx_batch_kernel_kind(rows, D, h), e0.elapsed_time(e1)/200, flush=True)
