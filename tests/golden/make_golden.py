"""Generate the golden fixtures under tests/golden/ FROM THE REFERENCE ITSELF.

Runs in the build container only (needs oracle/_ref/libendor_ref.so, compiled
from /root/reference by oracle/Makefile).  Every expected value written here is
produced by the reference's own code: synth_weight / magnitude_prune
(weight_gen.hpp:40-113), compress (codec.hpp:97-126), decompress
(codec.hpp:157-166), build_rank_index (bitmap.hpp:117-132), encode_endor
(file_io.hpp:187-210) and the reference tests' generators (test_helpers.hpp,
acceptance.cpp:53-157 -- std::mt19937_64 via the reference's own headers).

Outputs (small, committed):
  kats.json            literal known-answer cases with full expected bytes
  seeded_cases.json    test_codec.cpp-style seeded round trips (CRC32s)
  acceptance_1000.json acceptance.cpp criterion-3 suite (CRC32s per case)
  large.json           BASELINE.json configs at full size (CRC32s + nnz)

Usage:  python tests/golden/make_golden.py [--skip-large]
"""
from __future__ import annotations

import ctypes as C
import json
import multiprocessing as mp
import os
import sys
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

sys.path.insert(0, os.path.join(ROOT))
from paper_2406_11674_b200 import catalog  # noqa: E402


def crc(b) -> int:
    return zlib.crc32(np.ascontiguousarray(b).view(np.uint8).tobytes()) & 0xFFFFFFFF


def R():
    r = O.ref()
    if r is None:
        raise SystemExit("oracle/_ref/libendor_ref.so missing: run make -C oracle")
    return r


def ref_compress(dense, rows, cols, eb):
    n = rows * cols
    bm = np.zeros(max((n + 7) // 8, 1), np.uint8)
    vals = np.zeros(max(n * eb, 1), np.uint8)
    nnz, nz = C.c_uint64(0), C.c_int(0)
    st = R().ref_compress(rows, cols, eb, np.ascontiguousarray(dense.view(np.uint8)) if n else np.zeros(1, np.uint8),
                          bm, vals, C.byref(nnz), C.byref(nz))
    assert st == 0
    return bm[: (n + 7) // 8], vals[: nnz.value * eb], nnz.value, bool(nz.value)


def ref_decompress(rows, cols, eb, bm, vals, nnz):
    n = rows * cols
    out = np.zeros(max(n * eb, 1), np.uint8)
    st = R().ref_decompress(rows, cols, eb, bm if len(bm) else np.zeros(1, np.uint8),
                            vals if len(vals) else np.zeros(1, np.uint8), nnz, out)
    return st, out[: n * eb]


def ref_rank_index(bm, n, cs):
    chunks = 0 if (n == 0 or cs == 0) else (n + cs - 1) // cs
    out = np.zeros(max(chunks, 1), np.uint64)
    st = R().ref_rank_index(bm if len(bm) else np.zeros(1, np.uint8), n, cs, out)
    return st, out[:chunks]


def ref_random_dense(rows, cols, eb, seed, zf):
    out = np.zeros(max(rows * cols * eb, 1), np.uint8)
    R().ref_random_dense(rows, cols, eb, seed, zf, out)
    return out[: rows * cols * eb]


def hexs(a) -> str:
    return np.ascontiguousarray(a).view(np.uint8).tobytes().hex()


# ---------------------------------------------------------------------------

def make_kats():
    k = {}
    # test_codec.cpp:15-24,138-145: 2x2 bitmap 1010, values {0x3C00, 0x4200}
    bm = np.array([0b0101], np.uint8)
    vals = np.array([0x3C00, 0x4200], np.uint16).view(np.uint8)
    st, out = ref_decompress(2, 2, 2, bm, vals, 2)
    k["hand_2x2"] = dict(rows=2, cols=2, eb=2, bitmap=hexs(bm), values=hexs(vals), nnz=2,
                         dense=hexs(out), status=st)
    # test_codec.cpp:132-136: empty tensor 3x3 decompresses to zeros
    st, out = ref_decompress(3, 3, 2, np.zeros(2, np.uint8), np.zeros(0, np.uint8), 0)
    k["empty_3x3"] = dict(rows=3, cols=3, eb=2, bitmap="0000", values="", nnz=0, dense=hexs(out),
                          status=st)
    # test_codec.cpp:123-130: NaN payload / -inf survive
    w = np.array([0x7E01, 0x0000, 0xFC00], np.uint16)
    bm, vals, nnz, nz = ref_compress(w, 1, 3, 2)
    st, out = ref_decompress(1, 3, 2, bm, vals, nnz)
    k["nan_inf"] = dict(rows=1, cols=3, eb=2, bitmap=hexs(bm), values=hexs(vals), nnz=nnz,
                        dense=hexs(out), status=st, negzero=nz)
    # test_codec.cpp:110-121: negative zero dropped and flagged
    w = np.array([0x8000, 0xBC00, 0, 0], np.uint16)
    bm, vals, nnz, nz = ref_compress(w, 2, 2, 2)
    st, out = ref_decompress(2, 2, 2, bm, vals, nnz)
    k["negzero"] = dict(rows=2, cols=2, eb=2, bitmap=hexs(bm), values=hexs(vals), nnz=nnz,
                        dense=hexs(out), status=st, negzero=nz)
    # test_codec.cpp:147-153: values/popcount mismatch -> CorruptionError (2)
    bm = np.array([0b0001], np.uint8)
    st, _ = ref_decompress(2, 2, 2, bm, np.zeros(4, np.uint8), 2)
    k["popcount_mismatch"] = dict(rows=2, cols=2, eb=2, bitmap=hexs(bm), values="00000000", nnz=2,
                                  status=st)
    # test_codec.cpp:64-82: checkerboard 8x16 ratio 0.5625
    w = np.zeros(128, np.uint16)
    w[::2] = 0x3C00
    bm, vals, nnz, nz = ref_compress(w, 8, 16, 2)
    k["checkerboard"] = dict(rows=8, cols=16, eb=2, bitmap=hexs(bm), values=hexs(vals), nnz=nnz,
                             compressed_bytes=len(bm) + len(vals), dense_bytes=256)
    # test_bitmap.cpp:30-42: bits {0,3,8} of 16 -> bytes 0x09, 0x01
    k["lsb_first"] = dict(n=16, bits=[0, 3, 8], bytes="0901")
    # test_bitmap.cpp:77-88: alternating 256 @64 -> [0,32,64,96]; all-zero 300 @128 -> [0,0,0]
    alt = np.full(32, 0x55, np.uint8)
    st, p = ref_rank_index(alt, 256, 64)
    k["alt_prefix"] = dict(n=256, cs=64, bitmap=hexs(alt), prefix=[int(x) for x in p])
    st, p = ref_rank_index(np.zeros(38, np.uint8), 300, 128)
    k["zero_prefix"] = dict(n=300, cs=128, prefix=[int(x) for x in p])
    # test_bitmap.cpp:99-105: bad chunk sizes -> invalid_argument (4)
    k["bad_chunk"] = {str(cs): ref_rank_index(np.zeros(16, np.uint8), 128, cs)[0] for cs in (0, 32, 96, 64)}
    # test_weight_gen.cpp:21-30: synth_weight 4x4 seed 0
    out = np.zeros(32, np.uint8)
    R().ref_synth_prune(4, 4, 2, 0, 0.0, out)
    k["synth_4x4_seed0"] = [int(x) for x in out.view(np.uint16)]
    # test_weight_gen.cpp: 1x4 [4,1,3,2] @0.5 prunes the smallest two
    w = np.array([O.lib().or_f32_to_f16(v) for v in (4.0, 1.0, 3.0, 2.0)], np.uint16)
    st, p = O.magnitude_prune(w.view(np.uint8), 4, 2, 0.5)
    k["prune_1x4"] = dict(input=[int(x) for x in w], output=[int(x) for x in p.view(np.uint16)])
    # test_io.cpp:30-57: .endor golden layout (41 bytes) and all-zero 4x4 (38 bytes)
    bm = np.array([0b0101], np.uint8)
    vals = np.array([0x3C00, 0x4200], np.uint16).view(np.uint8)
    buf = np.zeros(256, np.uint8)
    ln = R().ref_encode_endor(2, 2, 2, bm, vals, 2, 0, buf, 256)
    k["endor_file_2x2"] = dict(bytes=hexs(buf[:ln]))
    ln = R().ref_encode_endor(4, 4, 2, np.zeros(2, np.uint8), np.zeros(1, np.uint8), 0, 0, buf, 256)
    k["endor_file_zero_4x4"] = dict(bytes=hexs(buf[:ln]))
    # f32->f16 on a grid of awkward inputs (float16.hpp:35-73), incl. subnormals/ties
    probes = np.array([0.0, -0.0, 1.0, -1.0, 65504.0, 65520.0, 1e-8, 5.960464477539063e-08,
                       2.9802322387695312e-08, 2.98023224e-08 * 1.5, 6.1035156e-05, 6.0e-05,
                       np.inf, -np.inf, 1.0 / 3.0, 0.1, -2.5e-6, 3.0517578125e-05], np.float32)
    k["f32_to_f16"] = [[float(v), int(R().ref_f32_to_f16(float(v)))] for v in probes]
    return k


def make_seeded():
    cases = []
    add = []
    # test_codec.cpp:38-49 (8x8 seed 42 @0.5), :155-166 (37x200 seed 3 @0.6),
    # :168-179 (16x100 i8 seed 21), :181-200 (8x64 seed 5 @0.4), :202-213
    add += [(8, 8, 2, 42, 0.5), (37, 200, 2, 3, 0.6), (16, 100, 1, 21, 0.5), (8, 64, 2, 5, 0.4),
            (10, 10, 2, 9, 0.5), (10, 10, 2, 10, 0.2)]
    # test_codec.cpp:51-62: 60 iterations of mt19937_64(7)
    g = O.MT64(7)
    for _ in range(60):
        rows = 1 + g() % 33
        cols = 1 + g() % 33
        eb = 2 if g() % 2 else 1
        zeros = (g() % 101) / 100.0
        seed = g()
        add.append((rows, cols, eb, seed, zeros))
    for rows, cols, eb, seed, zf in add:
        w = ref_random_dense(rows, cols, eb, seed, zf)
        bm, vals, nnz, nz = ref_compress(w, rows, cols, eb)
        st, out = ref_decompress(rows, cols, eb, bm, vals, nnz)
        assert st == 0 and (out == w).all()
        idx = {}
        for cs in (64, 128, 256, 4096, 8192):
            _, p = ref_rank_index(bm, rows * cols, cs)
            idx[str(cs)] = [int(x) for x in p]
        cases.append(dict(rows=rows, cols=cols, eb=eb, seed=int(seed), zero_fraction=zf, nnz=nnz,
                          crc_dense=crc(w), crc_bitmap=crc(bm), crc_values=crc(vals),
                          prefix=idx))
    return cases


def make_acceptance():
    out = []
    for it, rows, cols, eb, zeros, w, chunk, rsel, csel in O.acceptance_cases(1000):
        bm, vals, nnz, nz = ref_compress(w, rows, cols, eb)
        st, dense = ref_decompress(rows, cols, eb, bm, vals, nnz)
        assert st == 0
        _, p = ref_rank_index(bm, rows * cols, chunk)
        out.append(dict(iter=it, rows=rows, cols=cols, eb=eb, zeros=zeros, chunk=chunk, nnz=nnz,
                        crc_input=crc(w), crc_dense=crc(dense), crc_bitmap=crc(bm),
                        crc_values=crc(vals), crc_prefix=crc(p.astype("<u8"))))
    return out


def make_quant():
    """quantize_values + decompress(dequantize_values(t)) (codec.hpp:306-349),
    produced by the reference on seeded f16 tensors."""
    out = []
    g = O.MT64(99)
    for it in range(40):
        rows, cols = 1 + g() % 70, 1 + g() % 70
        zeros = (g() % 101) / 100.0
        seed = g()
        w = ref_random_dense(rows, cols, 2, seed, zeros)
        bm, vals, nnz, _ = ref_compress(w, rows, cols, 2)
        q = np.zeros(max(nnz, 1), np.uint8)
        scale = R().ref_quantize_values(rows, cols, bm if len(bm) else np.zeros(1, np.uint8),
                                        vals if nnz else np.zeros(1, np.uint8), nnz, q)
        dense = np.zeros(max(rows * cols * 2, 1), np.uint8)
        assert R().ref_decompress_dequant(rows, cols, bm if len(bm) else np.zeros(1, np.uint8), q, nnz,
                                          scale, dense) == 0
        out.append(dict(rows=rows, cols=cols, seed=int(seed), zero_fraction=zeros, nnz=nnz,
                        scale_bits=int(np.float32(scale).view(np.uint32)), crc_q=crc(q[:nnz]),
                        crc_dense=crc(dense[: rows * cols * 2])))
    return out


def _large_one(args):
    name, rows, cols, seed, s = args
    n = rows * cols
    w = np.zeros(n * 2, np.uint8)
    assert R().ref_synth_prune(rows, cols, 2, seed, s, w) == 0
    bm, vals, nnz, nz = ref_compress(w, rows, cols, 2)
    crc_in = crc(w)
    del w
    st, dense = ref_decompress(rows, cols, 2, bm, vals, nnz)
    assert st == 0
    _, p = ref_rank_index(bm, n, 4096)
    rec = dict(name=name, rows=rows, cols=cols, eb=2, seed=seed, sparsity=s, nnz=nnz,
               crc_dense=crc(dense), crc_bitmap=crc(bm), crc_values=crc(vals),
               crc_prefix_4096=crc(p.astype("<u8")), dense_equals_pruned=crc(dense) == crc_in)
    print(rec, flush=True)
    return rec


def make_large():
    jobs = [("opt-66b.fc1.seed7", 9216, 36864, 7, 0.5)]
    for li, lname in ((0, "opt-66b"), (1, "llama2-70b")):
        spec = catalog.model_catalog(lname)
        for oi, op in enumerate(spec.ops):
            jobs.append((f"{lname}.L0.{op.name}", op.rows, op.cols, catalog.op_seed(0, oi), 0.5))
    for s in catalog.SWEEP_SPARSITIES:
        jobs.append((f"sweep16384.s{int(round(s * 100))}", 16384, 16384, catalog.sweep_seed(s), s))
    with mp.get_context("fork").Pool(min(6, os.cpu_count() or 1)) as pool:
        return pool.map(_large_one, jobs, chunksize=1)


def main():
    skip_large = "--skip-large" in sys.argv
    with open(os.path.join(HERE, "kats.json"), "w") as f:
        json.dump(make_kats(), f, indent=1)
    with open(os.path.join(HERE, "seeded_cases.json"), "w") as f:
        json.dump(make_seeded(), f)
    with open(os.path.join(HERE, "acceptance_1000.json"), "w") as f:
        json.dump(make_acceptance(), f)
    with open(os.path.join(HERE, "quant.json"), "w") as f:
        json.dump(make_quant(), f)
    if not skip_large:
        with open(os.path.join(HERE, "large.json"), "w") as f:
            json.dump(make_large(), f, indent=1)


if __name__ == "__main__":
    main()
