"""The trainer's fp32-accurate split-tf32 tcgen05 GEMM (csrc/train_gemm.cu)
against a PyTorch float64 product of the same fp32 operands: every operand
layout, ragged shapes, split K, beta accumulation."""

import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


def _gemm(a, b, ta, tb, m, n, k, beta=0.0, c=None, split=False):
    import torch
    from paper_2308_04669_b200 import _lib
    fn = _lib.load_library().nedf_diag_gemm
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int,
                   C.c_int, C.c_float, C.c_void_p, C.c_int64, C.c_void_p]
    if c is None:
        c = torch.zeros(m, n, device="cuda")
    ws = torch.empty(1 << 22, device="cuda") if split else None
    rc = fn(a.data_ptr(), a.shape[1], ta, b.data_ptr(), b.shape[1], tb, c.data_ptr(), n, m, n, k, beta,
            ws.data_ptr() if ws is not None else None, ws.numel() if ws is not None else 0, None)
    assert rc == 0
    torch.cuda.synchronize()
    return c


@pytest.mark.parametrize("m,n,k", [(128, 64, 32), (4096, 256, 256), (300, 65, 200), (1, 1, 1), (256, 1008, 4096),
                                   (77, 130, 1008)])
@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 1), (0, 1)])
@pytest.mark.parametrize("split", [False, True])
def test_gemm_matches_float64(m, n, k, ta, tb, split):
    import torch
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n * 3 + k + 10 * ta + tb)
    a = torch.randn((k, m) if ta else (m, k), device="cuda", generator=g)
    b = torch.randn((k, n) if tb else (n, k), device="cuda", generator=g)
    c = _gemm(a, b, ta, tb, m, n, k, split=split)
    A = (a.t() if ta else a).double()
    B = (b.t() if tb else b).double()
    ref = A @ B.t()
    # fp32-level: |err| <= 8 * 2^-24 * sum |a||b|  (the split keeps ~22 bits per product)
    bound = 8 * 2.0 ** -24 * (A.abs() @ B.abs().t()) + 1e-30
    assert ((c.double() - ref).abs() <= bound).all(), (c.double() - ref).abs().max().item()


def test_gemm_beta_accumulates():
    import torch
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(200, 96, device="cuda", generator=g)
    b = torch.randn(70, 96, device="cuda", generator=g)
    c0 = torch.randn(200, 70, device="cuda", generator=g)
    c = _gemm(a, b, 0, 0, 200, 70, 96, beta=1.0, c=c0.clone())
    ref = a.double() @ b.double().t() + c0.double()
    assert (c.double() - ref).abs().max().item() < 1e-4
