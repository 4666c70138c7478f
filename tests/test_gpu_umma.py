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


def _umma32(lib, a, b, bf16):
    import torch
    fn = lib.nedf_diag_umma32
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 4 + [ctypes.c_void_p]
    m, k = a.shape
    n = b.shape[0]
    d = torch.full((128, n), float("nan"), device="cuda")
    assert fn(a.data_ptr(), b.data_ptr(), d.data_ptr(), m, n, k, int(bf16), None) == 0
    torch.cuda.synchronize()
    return d


def _tf32_trunc(x):
    import torch
    return (x.view(torch.int32) & ~0x1FFF).view(torch.float32)


@pytest.mark.parametrize("m", [64, 128])
@pytest.mark.parametrize("n", [16, 32])
@pytest.mark.parametrize("bf16", [0, 1])
def test_kind_tf32_bf16_layouts(lib, m, n, bf16):
    """kind::tf32 and kind::f16(bf16) SS MMAs with SW128 K-major fp32 / bf16 tiles (the guard
    kernel's operands).  D rows of an M = 128 MMA sit in TMEM lanes 0-127; for M = 64, row r
    sits in lane 32 (r // 16) + r % 16 (lanes 16-31 of each warp quarter unused)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(m + n + 7 * bf16)
    k = 256
    a = torch.randn(m, k, device="cuda", generator=g)
    b = torch.randn(n, k, device="cuda", generator=g)
    d = _umma32(lib, a, b, bf16)
    if bf16:
        ref = a.bfloat16().double() @ b.bfloat16().double().t()
    else:
        ref = _tf32_trunc(a).double() @ _tf32_trunc(b).double().t()
    lanes = torch.arange(m) if m == 128 else (32 * (torch.arange(m) // 16) + torch.arange(m) % 16)
    got = d[lanes.cuda()].double()
    err = (got - ref).abs().max().item()
    assert err < 1e-3 * ref.abs().max().item(), (err, d[:, 0].tolist())


def test_tf32_operands_are_truncated(lib):
    """The guard's 3xTF32 split stores hi = x with the 13 low mantissa bits cleared, so it is
    exact whether the tensor core truncates or rounds; this pins which one it does (K = 8: a
    single MMA, fp32 accumulation of 8 products)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.randn(128, 32, device="cuda", generator=g)
    b = torch.randn(16, 32, device="cuda", generator=g)
    d = _umma32(lib, a, b, 0)[:, :16].double()
    rna = lambda x: ((x.view(torch.int32) + 0x1000) & ~0x1FFF).view(torch.float32)   # noqa: E731
    e_tr = (d - _tf32_trunc(a).double() @ _tf32_trunc(b).double().t()).abs().max().item()
    e_rn = (d - rna(a).double() @ rna(b).double().t()).abs().max().item()
    print("tf32 operand conversion: err vs truncation", e_tr, "vs round-to-nearest", e_rn)
    assert min(e_tr, e_rn) < 1e-4


def test_m64_accumulator_at_lane_16(lib):
    """An M = 64 accumulator addressed at TMEM lane 16 fills lanes 16-31 of each 32-lane
    quarter (row r -> lane 32 (r // 16) + 16 + r % 16): two M = 64 accumulators share
    columns, so one 32x32b load reads both (layout probe for the guard kernel)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(9)
    a = torch.randn(64, 32, device="cuda", generator=g)
    b = torch.randn(16, 32, device="cuda", generator=g)
    d = _umma32(lib, a, b, 16 << 8)
    ref = _tf32_trunc(a).double() @ _tf32_trunc(b).double().t()
    lanes = 32 * (torch.arange(64) // 16) + 16 + torch.arange(64) % 16
    got = d[lanes.cuda()].double()
    assert (got - ref).abs().max().item() < 1e-3 * ref.abs().max().item(), d[:, 0].tolist()
