import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_2308_04669_b200 import _lib
lib = _lib.load_library()
f = lib.nedf_diag_mma_rate
f.restype = C.c_int; f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
out = torch.zeros(1, dtype=torch.int64, device='cuda')
for ts in (0, 1):
    for N in (64, 128, 256):
        for pc in (-2, -1):
            f(ts, N, 4096, pc, out.data_ptr()); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); f(ts, N, 4096, pc, out.data_ptr()); e1.record(); torch.cuda.synchronize()
            cyc = out.item() / 4096
            print(f"{'TS' if ts else 'SS'} N={N:3d} variant={'warp-uniform-elect' if pc==-2 else 'single-thread-unrolled'}: {cyc:7.1f} cycles/MMA (ideal {128*N/256:.0f}); kernel {e0.elapsed_time(e1)*1e3:.1f} us")
