"""Measure the practical HBM bandwidth for the expand kernel's read/write mix
(9 of 16 vectors read per 16 written) and a plain 1:1 copy with the same
streaming kernel shape (development aid)."""
import ctypes as C
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "_build", "mix.so")
if not os.path.exists(so):
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                    "-o", so, os.path.join(HERE, "mix_ceiling.cu")], check=True)
L = C.CDLL(so)
L.mix_time.restype = C.c_float
L.mix_time.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.c_int]
nout = 2038431744 // 16  # one OPT-66B layer's dense bytes
src = torch.empty(nout * 9 // 16 * 16 + 4096, dtype=torch.uint8, device="cuda")
dst = torch.empty(nout * 16, dtype=torch.uint8, device="cuda")
for blocks in (148 * 4, 148 * 8, 148 * 32):
    ms = L.mix_time(src.data_ptr(), dst.data_ptr(), nout, 10, 0, blocks)
    byts = nout * 16 + nout * 9
    print(f"mix  blocks {blocks}: {ms:.4f} ms  {byts / ms / 1e6:.1f} GB/s (read {nout * 9 * 16 / 1e9:.2f} GB, write {nout * 16 * 16 / 1e9 / 16:.2f} GB)")
    n2 = nout * 9 // 16
    ms = L.mix_time(src.data_ptr(), dst.data_ptr(), n2, 10, 1, blocks)
    print(f"copy blocks {blocks}: {ms:.4f} ms  {2 * n2 * 16 / ms / 1e6:.1f} GB/s")
