# bulk-copy rate vs source footprint: is re-reading a small L2-resident region (as the
# network kernel does with its 2.4 MB weight image) slower than streaming a large one?
import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_2308_04669_b200 import _lib
lib = _lib.load_library()
f = lib.nedf_diag_bulk_rate
f.restype = C.c_int; f.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_size_t, C.c_int, C.c_void_p]
src = torch.zeros(64 << 20, dtype=torch.uint8, device='cuda')
out = torch.zeros(148, dtype=torch.int64, device='cuda')
for span in (128 << 10, 1 << 20, 2400 << 10, 16 << 20, 64 << 20):
    for ctas in (1, 148):
        for stage, depth in ((16384, -8), (8192, -16)):
            total = 16 << 20
            f(src.data_ptr(), span, stage, depth, total, ctas, out.data_ptr()); torch.cuda.synchronize()
            f(src.data_ptr(), span, stage, depth, total, ctas, out.data_ptr()); torch.cuda.synchronize()
            cyc = out[:ctas].float().mean().item()
            print(f"span={span >> 10:6d}KB ctas={ctas:3d} stage={stage >> 10:2d}KB lanes={-depth:2d}: {total / cyc:6.1f} B/cycle/SM")
