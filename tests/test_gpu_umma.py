"""Pins the tcgen05 operand layouts the network kernel relies on: SW128
K-major shared-memory descriptors and the TS form (A in tensor memory, packed
f16x2), against a plain PyTorch fp32 GEMM of the same fp16 operands."""

import ctypes

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2308_04669_b200 import _lib
    lib = _lib.load_library()
    lib.nedf_diag_umma.restype = ctypes.c_int
    lib.nedf_diag_umma.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 4 + [ctypes.c_void_p]
    return lib


@pytest.mark.parametrize("k", [64, 256])
@pytest.mark.parametrize("n", [64, 80, 256])
@pytest.mark.parametrize("ts", [0, 1])
def test_single_cta_umma(lib, k, n, ts):
    import torch
    g = torch.Generator(device="cuda").manual_seed(k * 1000 + n + ts)
    a = torch.randn(128, k, device="cuda", generator=g).half()
    b = torch.randn(n, k, device="cuda", generator=g).half()
    for dcol in ((0, 64) if n <= 192 else (0,)):
        d = torch.zeros(128, n, device="cuda")
        assert lib.nedf_diag_umma(a.data_ptr(), b.data_ptr(), d.data_ptr(), k, n, ts, dcol, None) == 0
        torch.cuda.synchronize()
        ref = a.float() @ b.float().t()
        assert (d - ref).abs().max().item() < 1e-2
