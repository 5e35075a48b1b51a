"""Fused decompress -> GEMM (csrc/gemm_fused.cu) timings on the OPT-66B layer
shapes across token counts, next to the materialised alternatives:
decompress (our expand) + torch.matmul (cuBLAS) and cuBLAS on a resident
dense W.  Measurement aid.  CUDA events on the current stream, L2 flushed
(512 MiB write) before every repetition.

Reported per (shape, tokens): ms, TFLOP/s (2 * rows * cols * tokens), and
the HBM roofline of the fused kernel: algorithmic bytes = compressed W
(bitmap + values) + X + Y(fp32) per launch (W read once per n-tile column is
L2-shared).

Usage: python tools/gemm_bench.py [--tokens 1,16,...] [--reps N] [--out FILE]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2406_11674_b200 import codec as E  # noqa: E402

PK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6550.0, "bf16_tflops": 1687.9}
DEV = torch.device("cuda", 0)


def timed(fn, reps, flush):
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", default="1,16,64,128,256,512,2048")
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--shapes", default="fc1,fc2,qkv")
    ap.add_argument("--out", default="gpurun_out/gemm_bench.json")
    args = ap.parse_args()
    shapes = {"qkv": (9216, 9216), "fc1": (9216, 36864), "fc2": (36864, 9216)}  # catalog rows x cols
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=DEV)
    res = {"peak_hbm_gbs": PK["hbm_gbs"], "peak_tflops": PK.get("bf16_tflops"), "rows": []}
    for name in args.shapes.split(","):
        rows, cols = shapes[name]
        w = E.synth_weight(rows, cols, rows + cols, device=DEV)
        E.magnitude_prune(w, 0.5, inplace=True)
        t = E.compress(w)
        idx = E.build_rank_index(t.bitmap, 1024)
        Wd = w.data.view(torch.float16).reshape(rows, cols)
        comp = t.bitmap.data.numel() + t.values.numel()
        for T in [int(x) for x in args.tokens.split(",")]:
            X = ((torch.rand(T, cols, device=DEV) * 2 - 1)).half()
            flops = 2.0 * rows * cols * T
            fused = timed(lambda: E.gemm_compressed(t, X, index=idx), args.reps, flush)
            fused16 = timed(lambda: E.gemm_compressed(t, X, index=idx, out_dtype=torch.float16), args.reps, flush)
            cub = timed(lambda: torch.matmul(X, Wd.T), args.reps, flush)
            dec = timed(lambda: torch.matmul(X, E.decompress_chunked(t, idx).data.view(torch.float16)
                                             .reshape(rows, cols).T), args.reps, flush)
            alg = comp + T * cols * 2 + T * rows * 4
            row = {"shape": name, "rows": rows, "cols": cols, "tokens": T,
                   "fused_ms": round(fused, 4), "fused_f16out_ms": round(fused16, 4),
                   "fused_tflops": round(flops / fused / 1e9, 1),
                   "fused_hbm_gbs": round(alg / fused / 1e6, 1),
                   "fused_hbm_frac": round(alg / fused / 1e6 / PK["hbm_gbs"], 3),
                   "fused_tensor_frac": round(flops / fused / 1e9 / PK.get("bf16_tflops", 1687.9), 3),
                   "cublas_dense_resident_ms": round(cub, 4),
                   "decompress_plus_cublas_ms": round(dec, 4)}
            print(json.dumps(row), flush=True)
            res["rows"].append(row)
        del w, t, Wd
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
