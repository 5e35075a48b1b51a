"""Development timing of the coded-values decoder (csrc/vcode.cu) on one
OPT-66B layer's packed values (reference synth_weight + magnitude_prune 0.5):
blob sizes, host encode time, and the device decode against the HBM copy peak
(algorithmic bytes = blob read + 2 B per value written), L2 flushed between reps."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import torch  # noqa: E402

from paper_2406_11674_b200 import _lib, catalog  # noqa: E402
from paper_2406_11674_b200 import codec as E  # noqa: E402

dev = torch.device("cuda", 0)
PEAK = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json"))).get("hbm_gbs", 6550.0)
L = _lib.lib()
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
rows = []
for i, o in enumerate(catalog.model_catalog("opt-66b").ops):
    w = E.synth_weight(o.rows, o.cols, 1000 + i, device=dev)
    E.magnitude_prune(w, 0.5, inplace=True)
    t = E.compress(w)
    t0 = time.perf_counter()
    blob = E.encode_values(t.values)
    enc = time.perf_counter() - t0
    info = E.vcode_info(blob)
    hb = blob[:256].clone()
    bd = torch.empty(blob.numel() + 16, dtype=torch.uint8, device=dev)[: blob.numel()]
    bd.copy_(blob)
    out = torch.empty(t.nnz() * 2 + 16, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    ms = []
    for r in range(8):
        flush.fill_(r)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        E.check(L.endor_cuda_values_decode(hb.data_ptr(), bd.data_ptr(), out.data_ptr(), st))
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    ok = torch.equal(out[: t.nnz() * 2].cpu(), t.values.cpu())
    m = sorted(ms)[len(ms) // 2]
    alg = blob.numel() + t.nnz() * 2
    rows.append({"op": o.name, "nnz": t.nnz(), "mode": info["mode"], "k": info["k"], "n_exc": info["n_exc"],
                 "ratio": round(blob.numel() / (2 * t.nnz()), 4), "encode_s": round(enc, 3),
                 "decode_ms": round(m, 4), "decode_gbs": round(alg / (m * 1e-3) / 1e9, 1),
                 "frac_of_peak": round(alg / (m * 1e-3) / 1e9 / PEAK, 3), "bit_exact": ok})
    print(json.dumps(rows[-1]), flush=True)
print(json.dumps({"layer_values_ratio": round(sum(r["ratio"] * r["nnz"] for r in rows) / sum(r["nnz"] for r in rows), 4),
                  "layer_decode_ms": round(sum(r["decode_ms"] for r in rows), 4)}))
