"""Time the tcgen05 GEMM alone through glx_tc_gemm_bf16 (CUDA events, L2-resident
weights, X streamed): python tools/tc_bench.py M N K [epi ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1908_07847_b200._lib as L

M, N, K = (int(a) for a in sys.argv[1:4])
epis = [int(e) for e in sys.argv[4:]] or [0, 1]
lib = L.load()
A = torch.rand(M, K, device="cuda").to(torch.bfloat16)
B = (torch.rand(N, K, device="cuda") - 0.5).mul(0.1).to(torch.bfloat16)
bias = torch.randn(N, device="cuda")
Df = torch.empty(M, N, device="cuda") if 0 in epis else None
Db = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
for epi in epis:
    run = lambda: L.check(lib.glx_tc_gemm_bf16(A.data_ptr(), B.data_ptr(), M, N, K, epi,
                                               Df.data_ptr() if epi == 0 else None,
                                               Db.data_ptr() if epi == 1 else None, bias.data_ptr(), N, st))
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"epi={epi} M={M} N={N} K={K}: {ms:.3f} ms  {2 * M * N * K / ms / 1e9:.1f} TFLOP/s")
