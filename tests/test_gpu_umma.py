"""tcgen05 descriptor self-test: one UMMA tile per operand layout used by the SSA kernels, compared
with a plain fp32 matmul of the same bf16 operands (exact products, fp32 sums -> tight tolerance)."""
import ctypes

import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(mode, n, k, a, b):
    from paper_2505_17412_b200 import ssa
    L = ssa.lib()
    f = L.ssa_selftest_umma
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                  ctypes.c_void_p]
    rows = 128
    cols = n if mode in (0, 5) else 64
    d = torch.zeros(rows, cols, dtype=torch.float32, device="cuda")
    st = f(mode, n, k, a.data_ptr(), b.data_ptr(), d.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert st == 0, L.ssa_last_error().decode()
    return d


@pytest.mark.parametrize("n", [16, 64, 96, 112, 128])
def test_kmajor_kmajor(n):
    g = torch.Generator(device="cuda").manual_seed(n)
    a = torch.randn(128, 64, device="cuda", generator=g).bfloat16()
    b = torch.randn(n, 64, device="cuda", generator=g).bfloat16()
    d = _run(0, n, 64, a, b)
    ref = a.float() @ b.float().T
    assert torch.allclose(d, ref, atol=1e-3, rtol=1e-4), (d - ref).abs().max()


def test_mnmajor_a_mnmajor_b():
    g = torch.Generator(device="cuda").manual_seed(1)
    at = torch.randn(128, 128, device="cuda", generator=g).bfloat16()   # [k][m]
    b = torch.randn(128, 64, device="cuda", generator=g).bfloat16()     # [k][n]
    d = _run(1, 64, 128, at, b)
    ref = at.float().T @ b.float()
    assert torch.allclose(d, ref, atol=1e-3, rtol=1e-4), (d - ref).abs().max()


@pytest.mark.parametrize("k", [64, 96, 128])
def test_kmajor_a_mnmajor_b(k):
    g = torch.Generator(device="cuda").manual_seed(k)
    a = torch.randn(128, k, device="cuda", generator=g).bfloat16()
    b = torch.randn(k, 64, device="cuda", generator=g).bfloat16()
    d = _run(2, 64, k, a, b)
    ref = a.float() @ b.float()
    assert torch.allclose(d, ref, atol=1e-3, rtol=1e-4), (d - ref).abs().max()



@pytest.mark.parametrize("k", [64, 96, 128])
def test_tmem_a_mnmajor_b(k):
    """A operand in TMEM (threads write rows with tcgen05.st), B MN-major from TMA: (P w)^T dO shape."""
    g = torch.Generator(device="cuda").manual_seed(40 + k)
    a = torch.randn(128, k, device="cuda", generator=g).bfloat16()
    b = torch.randn(k, 64, device="cuda", generator=g).bfloat16()
    d = _run(4, 64, k, a, b)
    ref = a.float() @ b.float()
    assert torch.allclose(d, ref, atol=1e-3, rtol=1e-4), (d - ref).abs().max()


@pytest.mark.parametrize("n", [64, 128])
def test_tmem_a_kmajor_b(n):
    """A operand in TMEM, B K-major [N][64] from TMA: S^T = K Q^T shape."""
    g = torch.Generator(device="cuda").manual_seed(50 + n)
    a = torch.randn(128, 64, device="cuda", generator=g).bfloat16()
    b = torch.randn(n, 64, device="cuda", generator=g).bfloat16()
    d = _run(5, n, 64, a, b)
    ref = a.float() @ b.float().T
    assert torch.allclose(d, ref, atol=1e-3, rtol=1e-4), (d - ref).abs().max()
