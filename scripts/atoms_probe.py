"""Shared-atomic throughput by address pattern (trace build):
PGB_LIBRARY=build/trace.so PGB_LIB_LENIENT=1 python scripts/atoms_probe.py"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09664_b200 import _lib  # noqa: E402

lib = _lib.load(require_symbols=False)
lib.pgb_probe_atoms_dev.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
sink = torch.zeros(256, dtype=torch.int32, device="cuda")
blocks, iters = 148 * 8, 256
names = ["consecutive", "stride2", "one-bank", "hashed", "lane*37"]
for mode in range(5):
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        lib.pgb_probe_atoms_dev(blocks, iters, mode, sink.data_ptr(), None)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    warp_atoms = blocks * 8 * iters * 16
    per_sm_clk = best * 1e-3 * 1.965e9 * 148 / warp_atoms
    print(f"{names[mode]:12s} {best * 1e3:8.1f} us  {per_sm_clk:6.2f} SM-cycles per warp ATOMS", flush=True)
