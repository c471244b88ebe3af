"""tcgen05 BF16 GEMM (csrc/glx_tc.cu) vs a plain fp32 torch reference of the same op."""

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K", [(256, 256, 1024), (128, 512, 64), (300, 256, 128), (128, 32, 64),
                                   (512, 128, 256), (1000, 64, 192)])
def test_tc_gemm_f32_epilogue(gpu, M, N, K):
    import torch

    import paper_1908_07847_b200._lib as L

    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
    D = torch.full((M, N), float("nan"), device="cuda")
    lib = L.load()
    L.check(lib.glx_tc_gemm_bf16(A.data_ptr(), B.data_ptr(), M, N, K, 0, D.data_ptr(), None, None, N,
                                 torch.cuda.current_stream().cuda_stream))
    ref = A.float() @ B.float().T
    torch.cuda.synchronize()
    err = ((D - ref).abs() / ref.abs().clamp_min(1.0)).max().item()
    assert err < 1e-4, err


def test_tc_gemm_sigmoid_epilogue(gpu):
    import torch

    import paper_1908_07847_b200._lib as L

    M, N, K = 384, 1024, 1024
    g = torch.Generator(device="cuda").manual_seed(3)
    A = (torch.rand(M, K, device="cuda", generator=g)).to(torch.bfloat16)
    B = (torch.rand(N, K, device="cuda", generator=g) - 0.5).mul(0.1).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda", generator=g)
    H = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    lib = L.load()
    L.check(lib.glx_tc_gemm_bf16(A.data_ptr(), B.data_ptr(), M, N, K, 1, None, H.data_ptr(), bias.data_ptr(), N,
                                 torch.cuda.current_stream().cuda_stream))
    ref = torch.sigmoid(A.float() @ B.float().T + bias)
    torch.cuda.synchronize()
    assert (H.float() - ref).abs().max().item() < 4e-3  # bf16 rounding of values in (0, 1)
