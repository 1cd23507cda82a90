"""tcgen05/TMEM/TMA building blocks on the GPU: the descriptor self-test GEMMs (K-major B as in
S = Q K^T, MN-major B as in O = P V) against a torch fp32 matmul of the same bf16 tiles."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_umma_descriptor_selftest():
    from paper_2505_22296_b200 import _lib as C

    g = torch.Generator(device="cuda").manual_seed(0)
    a, b, bmn = (torch.randn(128, 128, device="cuda", generator=g).bfloat16() for _ in range(3))
    d1 = torch.zeros(128, 128, device="cuda")
    d2 = torch.zeros(128, 128, device="cuda")
    d3 = torch.zeros(128, 128, device="cuda")
    C.check(C.lib().spattn_selftest_umma(torch.cuda.current_stream().cuda_stream, a.data_ptr(),
                                         b.data_ptr(), bmn.data_ptr(), d1.data_ptr(),
                                         d2.data_ptr(), d3.data_ptr()))
    torch.cuda.synchronize()
    want1 = a.float() @ b.float().T
    want2 = a.float() @ bmn.float()
    torch.testing.assert_close(d1, want1, rtol=1e-3, atol=1e-2)
    torch.testing.assert_close(d2, want2, rtol=1e-3, atol=1e-2)
    torch.testing.assert_close(d3, want2, rtol=1e-3, atol=1e-2)  # A operand from TMEM
