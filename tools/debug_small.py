import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
from paper_2406_11674_b200 import codec as E
for (rows, cols, eb) in [(2, 2, 2), (1, 3, 2), (37, 200, 2), (16, 100, 1), (300, 1000, 2)]:
    w = O.random_dense(rows, cols, eb, 5, 0.5)
    bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
    bitmap = E.Bitmap.from_bytes(bm.tobytes(), rows * cols, device="cuda")
    values = torch.from_numpy(vals.copy()).cuda() if len(vals) else torch.zeros(0, dtype=torch.uint8, device="cuda")
    t = E.EndorTensor(rows, cols, E.Dtype.F16 if eb == 2 else E.Dtype.I8, bitmap, values)
    out = E.decompress(t)
    print(rows, cols, eb, out.bytes() == w.tobytes(), flush=True)
