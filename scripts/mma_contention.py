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
for pc, name in ((-2, "plain 4-MMA groups"), (-8, "kernel issue pattern"), (-9, "+ slice alternation / restarts"),
                 (-10, "commit per group only"), (-11, "wait + fence per group only"),
                 (-12, "per 8 MMAs: 1 wait, 1 commit"), (-13, "per 8 MMAs: 2 waits, 2 commits"),
                 (-14, "per 16 MMAs: 1 wait, 1 commit"), (-17, "kernel pattern without the fence"),
                 (-19, "kernel pattern, test_wait spin"), (-20, "kernel pattern, generic commit")):
    f(1, 128, 4096, pc, out.data_ptr()); torch.cuda.synchronize()
    out.zero_(); f(1, 128, 4096, pc, out.data_ptr()); torch.cuda.synchronize()
    print(f"TS N=128: {name:34s} {out[0].item() / 4096:7.1f} cycles/MMA")
