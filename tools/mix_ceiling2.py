"""Write-path variants for the 9:16 read:write streaming mix (development aid)."""
import ctypes as C
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
L = C.CDLL(os.path.join(HERE, "_build", "mix2.so"))
L.mix2_time.restype = C.c_float
L.mix2_time.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.c_int]
nblk = 2038431744 // 16384
src = torch.empty(nblk * 576 * 16 + 4096, dtype=torch.uint8, device="cuda")
dst = torch.empty(nblk * 16384, dtype=torch.uint8, device="cuda")
byts = nblk * (16384 + 576 * 16)
MODES = [int(m) for m in os.environ.get("MODES", "0,1,2,3,4,5,6,7").split(",")]
for mode in MODES:
    for blocks in (148 * 4, 148 * 8, 148 * 16):
        ms = L.mix2_time(src.data_ptr(), dst.data_ptr(), nblk, 10, mode, blocks)
        print(f"mode {mode} blocks {blocks}: {ms:.4f} ms {byts / ms / 1e6:.1f} GB/s", flush=True)
