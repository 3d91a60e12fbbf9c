"""tcgen05 / TMEM / TMA building blocks: every operand layout of the tensor-core
ResidualAttention kernel, checked on small GEMMs against torch (fp32 math on
the same bf16 inputs)."""
import ctypes

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2604_06370_b200 import _lib as L  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("test,N,K", [(0, 64, 128), (0, 128, 64), (0, 256, 128), (1, 64, 128), (1, 128, 64),
                                      (2, 128, 16), (3, 64, 128), (4, 16, 128), (4, 64, 128), (6, 32, 16),
                                      (6, 128, 16)])
def test_umma_layouts(test, N, K):
    g = torch.Generator(device="cpu").manual_seed(test * 1000 + N + K)
    A = torch.randn(128, K, generator=g).to(torch.bfloat16).cuda()
    B = torch.randn(N, K, generator=g).to(torch.bfloat16).cuda()
    D = torch.full((128, N), float("nan"), dtype=torch.float32, device="cuda")
    lib = L.load()
    st = lib.fkv_selftest_umma(test, ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                               ctypes.c_void_p(D.data_ptr()), 128, N, K, None)
    assert st == 0
    torch.cuda.synchronize()
    ref = A.float() @ B.float().T
    assert torch.allclose(D, ref, atol=1e-3, rtol=1e-3), (D - ref).abs().max().item()


def test_tma_sw128_box_matches_layout_formula():
    A = torch.randn(256, 192).to(torch.bfloat16).cuda()
    D = torch.zeros(1, dtype=torch.float32, device="cuda")
    lib = L.load()
    st = lib.fkv_selftest_umma(5, ctypes.c_void_p(A.data_ptr()), None, ctypes.c_void_p(D.data_ptr()), 256, 0, 192,
                               None)
    assert st == 0
    torch.cuda.synchronize()
    assert D.item() == 0
