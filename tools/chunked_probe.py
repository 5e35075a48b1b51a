"""decompress_chunked at the reference's chunk sizes (kDefaultChunkSize = 4096,
codec.hpp:19) and decompress_chunk_into over all chunks, on OPT-66B fc1
(development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import torch  # noqa: E402

from paper_2406_11674_b200 import _lib, catalog, codec as E  # noqa: E402

dev = torch.device("cuda", 0)
L = _lib.lib()
rows, cols = 9216, 36864
w = E.synth_weight(rows, cols, catalog.FC1_SEED, device=dev)
E.magnitude_prune(w, 0.5, inplace=True)
t = E.compress(w)
n = rows * cols
alg = catalog.algorithmic_bytes(n, t.nnz())
out = E.DenseMatrix.empty(rows, cols, E.Dtype.F16, dev)
ws = E.workspace(n, dev)
st = torch.cuda.current_stream().cuda_stream
v = t.view()
for cs in (1024, 2048, 4096, 8192, 65536):
    idx = E.build_rank_index(t.bitmap, cs)
    pre = idx.prefix.contiguous()

    def run():
        E.check(L.endor_cuda_decompress_chunked(C.byref(v), cs, pre.data_ptr(), pre.numel(), out.data.data_ptr(),
                                                ws.data_ptr(), ws.numel(), st))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        run()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    E.sync_status(ws, dev)
    assert torch.equal(out.data, w.data)
    print(f"decompress_chunked cs={cs:6d}: {ms:.4f} ms  {alg / ms / 1e6 / 6549.8:.3f} of peak", flush=True)
