#!/usr/bin/env python3
"""Warm timing of the trainer's GEMM shapes (CUDA events, 20 repetitions)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import ctypes as C  # noqa: E402

from paper_2308_04669_b200 import _lib  # noqa: E402

fn = _lib.load_library().nedf_diag_gemm
fn.restype = C.c_int
fn.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int,
               C.c_int, C.c_float, C.c_void_p, C.c_int64, C.c_void_p]
ws = torch.empty(1 << 22, device="cuda")


def _gemm(a, b, ta, tb, m, n, k, c, split):
    assert fn(a.data_ptr(), a.shape[1], ta, b.data_ptr(), b.shape[1], tb, c.data_ptr(), n, m, n, k, 0.0,
              ws.data_ptr() if split else None, ws.numel() if split else 0, None) == 0

for (m, n, k, ta, tb, split) in [(4096, 256, 256, 0, 0, False), (4096, 256, 1008, 0, 0, False),
                                 (256, 256, 4096, 1, 1, True), (4096, 256, 256, 0, 1, False),
                                 (256, 1008, 4096, 1, 1, True)]:
    a = torch.randn((k, m) if ta else (m, k), device="cuda")
    b = torch.randn((k, n) if tb else (n, k), device="cuda")
    c = torch.zeros(m, n, device="cuda")
    for _ in range(3):
        _gemm(a, b, ta, tb, m, n, k, c=c, split=split)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        _gemm(a, b, ta, tb, m, n, k, c=c, split=split)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 20
    cf = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    A = (a.t() if ta else a).contiguous()
    B = (b.t() if tb else b).contiguous()
    for _ in range(3):
        A @ B.t()
    e0.record()
    for _ in range(20):
        A @ B.t()
    e1.record()
    torch.cuda.synchronize()
    us_ref = e0.elapsed_time(e1) * 1e3 / 20
    print(f"m {m} n {n} k {k} ta {ta} tb {tb}: {us:.1f} us ({3 * 2 * m * n * k / us / 1e6:.0f} TFLOP/s tf32 issued), "
          f"torch fp32 (cuBLAS) {us_ref:.1f} us")

tr = _lib.load_library().nedf_diag_gemm_trace
tr.restype = C.c_int
tr.argtypes = [C.c_int, C.c_void_p]
out = (C.c_ulonglong * 16)()
for (m, n, k, ta, tb, split) in [(4096, 256, 256, 0, 0, False), (256, 256, 4096, 1, 1, True)]:
    a = torch.randn((k, m) if ta else (m, k), device="cuda")
    b = torch.randn((k, n) if tb else (n, k), device="cuda")
    c = torch.zeros(m, n, device="cuda")
    _gemm(a, b, ta, tb, m, n, k, c, split)
    tr(1, None)
    _gemm(a, b, ta, tb, m, n, k, c, split)
    torch.cuda.synchronize()
    tr(0, out)
    t = list(out)
    print(m, n, k, "setup", t[1] - t[0], "chunks ready", [t[2 + i] - t[0] for i in range(8)], "done", t[10] - t[0],
          "tmem->smem", t[12] - t[0], "synced", t[13] - t[0], "stored", t[11] - t[0])
