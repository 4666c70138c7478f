import ctypes, sys, torch
sys.path.insert(0, '.')
from paper_2308_04669_b200 import _lib
lib = _lib.load_library()
f = lib.nedf_diag_umma
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p]*3 + [ctypes.c_int]*4 + [ctypes.c_void_p]
torch.manual_seed(0)
ok = True
for K in (64, 256):
    for N in (64, 256, 80):
        for ts in (0, 1):
            for dcol in (0, 64) if N <= 192 else (0,):
                A = torch.randn(128, K, device='cuda').half()
                B = torch.randn(N, K, device='cuda').half()
                D = torch.zeros(128, N, device='cuda')
                rc = f(A.data_ptr(), B.data_ptr(), D.data_ptr(), K, N, ts, dcol, None)
                torch.cuda.synchronize()
                ref = A.float() @ B.float().t()
                err = (D - ref).abs().max().item()
                print(f"K={K} N={N} ts={ts} dcol={dcol} rc={rc} maxerr={err:.3e}")
                ok &= rc == 0 and err < 1e-2
print("UMMA_OK" if ok else "UMMA_FAIL")
