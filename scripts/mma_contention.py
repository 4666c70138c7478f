import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_2308_04669_b200 import _lib
lib = _lib.load_library()
f = lib.nedf_diag_mma_rate
f.restype = C.c_int; f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
out = torch.zeros(2, dtype=torch.int64, device='cuda')
for ts in (1, 0):
    for N in (128, 256):
        for pc, name in ((-2, "alone"), (-3, "tmem ld/st contention"), (-4, "fma contention"), (-5, "bulk-copy contention"), (-6, "bulk copies, no MMA")):
            f(ts, N, 4096, pc, out.data_ptr()); torch.cuda.synchronize()
            f(ts, N, 4096, pc, out.data_ptr()); torch.cuda.synchronize()
            print(f"{'TS' if ts else 'SS'} N={N}: {name:24s} {out[0].item() / 4096:7.1f} cycles/MMA" + (f"  copies {out[1].item()} ({out[1].item() * 16384 / out[0].item():.1f} B/cycle)" if pc <= -5 else ""))
