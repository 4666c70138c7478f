# tcgen05 rate with B cycling through distinct shared-memory slots (no operand reuse), single CTA vs CTA pair
import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_2308_04669_b200 import _lib
lib = _lib.load_library()
f = lib.nedf_diag_mma_rate
f.restype = C.c_int; f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
g = lib.nedf_diag_mma2_rate
g.restype = C.c_int; g.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p]
out = torch.zeros(2, dtype=torch.int64, device='cuda')
for ts in (1, 0):
    for N in (128, 256):
        for pc, name in ((-2, "same B"), (-7, "cycling B")) if N == 128 else ((-2, "same B"),):
            f(ts, N, 4096, pc, out.data_ptr()); torch.cuda.synchronize()
            f(ts, N, 4096, pc, out.data_ptr()); torch.cuda.synchronize()
            print(f"single {'TS' if ts else 'SS'} N={N}: {name:10s} {out[0].item() / 4096:7.1f} cycles/MMA")
        for cyc, name in ((0, "same B"), (2, "cycling B")) if N == 128 else ((0, "same B"),):
            g(ts | cyc, N, 4096, out.data_ptr()); torch.cuda.synchronize()
            g(ts | cyc, N, 4096, out.data_ptr()); torch.cuda.synchronize()
            print(f"pair   {'TS' if ts else 'SS'} N={N}: {name:10s} {out[0].item() / 4096:7.1f} cycles/MMA")
