import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_2308_04669_b200 import _lib
lib = _lib.load_library()
f = lib.nedf_diag_bulk_rate
f.restype = C.c_int; f.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_size_t, C.c_int, C.c_void_p]
span = 16 << 20
src = torch.zeros(span, dtype=torch.uint8, device='cuda')
out = torch.zeros(148, dtype=torch.int64, device='cuda')
for ctas in (1, 148):
    for stage, depth in ((16384, 8), (65536, 3), (98304, 2), (131072, 1), (16384, -8), (8192, -16), (32768, -4), (32768, -6)):
        total = 32 << 20
        f(src.data_ptr(), span, stage, depth, total, ctas, out.data_ptr()); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(src.data_ptr(), span, stage, depth, total, ctas, out.data_ptr()); e1.record(); torch.cuda.synchronize()
        cyc = out[:ctas].float().mean().item()
        ms = e0.elapsed_time(e1)
        print(f"ctas={ctas:3d} stage={stage//1024:2d}KB depth={depth:2d}: {total/cyc:6.1f} B/cycle/SM, "
              f"{total*ctas/ms/1e6:8.1f} GB/s total ({total/ms/1e6:6.1f} GB/s per SM)")
