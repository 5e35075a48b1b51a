"""Quick kernel timing (development aid): fc1 decompress via the C ABI."""
import ctypes as C, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_11674_b200 import codec as E, _lib
L = _lib.lib()
dev = torch.device("cuda", 0)
CFGS = [(9216, 36864, 0.5), (16384, 16384, 0.3), (16384, 16384, 0.9)]
if '--fc1' in sys.argv: CFGS = CFGS[:1]
for (rows, cols, s) in CFGS:
    w = E.synth_weight(rows, cols, 7, device=dev)
    E.magnitude_prune(w, s, inplace=True)
    t = E.compress(w)
    n = rows * cols
    out = E.DenseMatrix.empty(rows, cols, E.Dtype.F16, dev)
    ws = E.workspace(n, dev)
    v = t.view()
    st = torch.cuda.current_stream().cuda_stream
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    def run():
        E.check(L.endor_cuda_decompress(C.byref(v), out.data.data_ptr(), ws.data_ptr(), ws.numel(), st))
    for _ in range(3): run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); run(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    E.sync_status(ws, dev)
    assert torch.equal(out.data, w.data)
    ts.sort(); med = ts[len(ts)//2]
    alg = (n + 7)//8 + t.nnz()*2 + n*2
    print(f"{rows}x{cols} s={s}: median {med*1e3:.1f} us best {ts[0]*1e3:.1f} us  alg {alg/med/1e6:.0f} GB/s ({alg/med/1e6/6552.3:.3f} of peak)  dense {n*2/med/1e6:.0f} GB/s", flush=True)
    # gemv
    x = torch.randn(cols, dtype=torch.float16, device=dev)
    y = torch.empty(rows, dtype=torch.float32, device=dev)
    for _ in range(3): E.gemv(out, x, y)
    ts = []
    for _ in range(10):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); E.gemv(out, x, y); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); med = ts[len(ts)//2]
    print(f"   gemv median {med*1e3:.1f} us  {n*2/med/1e6:.0f} GB/s", flush=True)
    del w, t, out
    torch.cuda.empty_cache()
