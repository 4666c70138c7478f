import ctypes, sys, torch
sys.path.insert(0, '.')
from paper_2308_04669_b200 import _lib
lib = _lib.load_library()
f = lib.nedf_diag_umma2
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p]*3 + [ctypes.c_int]*3 + [ctypes.c_void_p]
torch.manual_seed(0)
ok = True
for K in (64, 256):
    for N in (64, 128, 256):
        for ts in (0, 1):
            A = torch.randn(256, K, device='cuda').half()
            B = torch.randn(N, K, device='cuda').half()
            D = torch.zeros(256, N, device='cuda')
            rc = f(A.data_ptr(), B.data_ptr(), D.data_ptr(), K, N, ts, None)
            torch.cuda.synchronize()
            ref = A.float() @ B.float().t()
            err = (D - ref).abs().max().item()
            print(f"pair K={K} N={N} ts={ts} rc={rc} maxerr={err:.3e}", flush=True)
            ok &= rc == 0 and err < 1e-2
print("UMMA2_OK" if ok else "UMMA2_FAIL")
