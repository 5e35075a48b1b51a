import ctypes as C, time, sys
t=time.time()
L = C.CDLL("libcufile.so.0")
print("dlopen ok", time.time()-t, flush=True)
class Err(C.Structure):
    _fields_ = [("err", C.c_int), ("cu_err", C.c_int)]
L.cuFileDriverOpen.restype = Err
import torch
torch.zeros(1, device="cuda")
print("cuda ok", time.time()-t, flush=True)
e = L.cuFileDriverOpen()
print("cuFileDriverOpen", e.err, e.cu_err, time.time()-t, flush=True)
