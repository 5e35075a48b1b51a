"""The CPU oracle pinned against the reference's own golden vectors (no GPU).

tests/golden/*.json were produced by the reference itself (make_golden.py via
oracle/_ref/libendor_ref.so); the literal KATs restate the reference's
test_codec.cpp / test_bitmap.cpp / test_weight_gen.cpp / test_io.cpp.  When
oracle/_ref is present (this container) the oracle is also compared with the
reference directly on fresh random cases.
"""
import ctypes as C
import json
import os
import zlib

import numpy as np
import pytest

from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))


def crc(b) -> int:
    return zlib.crc32(np.ascontiguousarray(b).view(np.uint8).tobytes()) & 0xFFFFFFFF


def h(s):
    return np.frombuffer(bytes.fromhex(s), np.uint8).copy()


# ---- literal KATs ----------------------------------------------------------------

def test_hand_built_2x2(kats):
    k = kats["hand_2x2"]
    st, out = O.decompress(2, 2, 2, h(k["bitmap"]), h(k["values"]), 2)
    assert st == 0 and out.tobytes().hex() == k["dense"] == "003c000000420000"


def test_empty_and_special_values(kats):
    st, out = O.decompress(3, 3, 2, np.zeros(2, np.uint8), np.zeros(0, np.uint8), 0)
    assert st == 0 and out.tobytes().hex() == kats["empty_3x3"]["dense"]
    for name in ("nan_inf", "negzero"):
        k = kats[name]
        st, out = O.decompress(k["rows"], k["cols"], 2, h(k["bitmap"]), h(k["values"]), k["nnz"])
        assert out.tobytes().hex() == k["dense"]
    w = np.array([0x7E01, 0x0000, 0xFC00], np.uint16)
    bm, vals, nnz, nz = O.compress(w, 1, 3, 2)
    assert O.decompress(1, 3, 2, bm, vals, nnz)[1].tobytes() == w.tobytes()
    w = np.array([0x8000, 0xBC00, 0, 0], np.uint16)
    bm, vals, nnz, nz = O.compress(w, 2, 2, 2)
    assert nz and nnz == 1 and bm.tobytes().hex() == kats["negzero"]["bitmap"]


def test_popcount_mismatch_is_corruption(kats):
    k = kats["popcount_mismatch"]
    st, _ = O.decompress(2, 2, 2, h(k["bitmap"]), h(k["values"]), 2)
    assert st == O.CORRUPTION == k["status"]


def test_size_law_checkerboard(kats):
    k = kats["checkerboard"]
    w = np.zeros(128, np.uint16)
    w[::2] = 0x3C00
    bm, vals, nnz, _ = O.compress(w, 8, 16, 2)
    assert bm.tobytes().hex() == k["bitmap"] and (len(bm) + len(vals)) / 256 == 0.5625


def test_bitmap_and_rank_index_kats(kats):
    bm = np.zeros(2, np.uint8)
    for b in kats["lsb_first"]["bits"]:
        bm[b >> 3] |= 1 << (b & 7)
    assert bm.tobytes().hex() == kats["lsb_first"]["bytes"]
    a = kats["alt_prefix"]
    assert O.rank_index(h(a["bitmap"]), 256, 64)[1].tolist() == a["prefix"] == [0, 32, 64, 96]
    assert O.rank_index(np.zeros(38, np.uint8), 300, 128)[1].tolist() == kats["zero_prefix"]["prefix"]
    for cs, st in kats["bad_chunk"].items():
        assert O.rank_index(np.zeros(16, np.uint8), 128, int(cs))[0] == st


def test_synth_prune_f16_kats(kats):
    assert O.synth_weight(4, 4, 2, 0).view(np.uint16).tolist() == kats["synth_4x4_seed0"]
    k = kats["prune_1x4"]
    st, p = O.magnitude_prune(np.array(k["input"], np.uint16).view(np.uint8), 4, 2, 0.5)
    assert p.view(np.uint16).tolist() == k["output"]
    for v, want in kats["f32_to_f16"]:
        assert O.lib().or_f32_to_f16(v) == want, v


def test_prune_exact_counts():
    # test_weight_gen.cpp:60-69: exactly floor(s*n) zeros
    w = O.synth_weight(31, 17, 2, 11)
    for s in (0.1, 0.25, 0.5, 0.77, 0.999):
        _, p = O.magnitude_prune(w, 31 * 17, 2, s)
        zeros = int(((p.view(np.uint16) & 0x7FFF) == 0).sum())
        assert zeros == int(s * 31 * 17)


# ---- seeded / acceptance suites ------------------------------------------------------

def test_seeded_cases(seeded_cases):
    for c in seeded_cases:
        rows, cols, eb = c["rows"], c["cols"], c["eb"]
        w = O.random_dense(rows, cols, eb, c["seed"], c["zero_fraction"])
        assert crc(w) == c["crc_dense"]
        bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
        assert (nnz, crc(bm), crc(vals)) == (c["nnz"], c["crc_bitmap"], c["crc_values"])
        st, out = O.decompress(rows, cols, eb, bm, vals, nnz)
        assert st == 0 and crc(out) == c["crc_dense"]
        for cs, pref in c["prefix"].items():
            st, p = O.rank_index(bm, rows * cols, int(cs))
            assert p.tolist() == pref
            dst = np.zeros(rows * cols * eb, np.uint8)
            assert O.lib().or_decompress_chunked(rows, cols, eb, bm, vals, nnz, int(cs),
                                                 np.ascontiguousarray(p, np.uint64), len(p), dst) == 0
            assert crc(dst) == c["crc_dense"]


def test_chunk_into_order_and_isolation():
    w = O.random_dense(8, 64, 2, 5, 0.4)
    bm, vals, nnz, _ = O.compress(w, 8, 64, 2)
    _, p = O.rank_index(bm, 512, 128)
    for k in range(len(p)):
        buf = np.full(1024, 0xAB, np.uint8)
        assert O.lib().or_decompress_chunk_into(8, 64, 2, bm, vals, nnz, 128, p, len(p), k, buf, 1024) == 0
        b, e = k * 256, (k + 1) * 256
        assert (buf[b:e] == w[b:e]).all() and (buf[:b] == 0xAB).all() and (buf[e:] == 0xAB).all()
    buf = np.zeros(1024, np.uint8)
    assert O.lib().or_decompress_chunk_into(8, 64, 2, bm, vals, nnz, 128, p, len(p), len(p), buf, 1024) == O.BOUNDS
    assert O.lib().or_decompress_chunk_into(8, 64, 2, bm, vals, nnz, 128, p, len(p), 0, buf, 1022) == O.INVALID


def test_acceptance_1000(acceptance_cases):
    gold = {c["iter"]: c for c in acceptance_cases}
    for it, rows, cols, eb, zeros, w, chunk, _r, _c in O.acceptance_cases(1000):
        g = gold[it]
        assert (rows, cols, eb, chunk) == (g["rows"], g["cols"], g["eb"], g["chunk"])
        assert crc(w) == g["crc_input"]
        bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
        assert (nnz, crc(bm), crc(vals)) == (g["nnz"], g["crc_bitmap"], g["crc_values"])
        assert crc(O.decompress(rows, cols, eb, bm, vals, nnz)[1]) == g["crc_dense"]
        assert crc(O.rank_index(bm, rows * cols, chunk)[1].astype("<u8")) == g["crc_prefix"]


def test_quantize_dequant_oracle_matches_golden(quant_cases):
    """quantize_values / dequantize_values + decompress (codec.hpp:306-349)."""
    for c in quant_cases:
        w = O.random_dense(c["rows"], c["cols"], 2, c["seed"], c["zero_fraction"])
        bm, vals, nnz, _ = O.compress(w, c["rows"], c["cols"], 2)
        q, scale = O.quantize_values(vals, nnz)
        assert np.float32(scale).view(np.uint32) == c["scale_bits"] and crc(q) == c["crc_q"]
        st, dense = O.decompress_dequant(c["rows"], c["cols"], bm, q, nnz, scale)
        assert st == 0 and crc(dense) == c["crc_dense"]


def test_multithreaded_op_generator_matches_golden(large_cases):
    L = O.lib()
    L.or_make_op_mt.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_int, O._u8p, O._u8p]
    L.or_make_op_mt.restype = C.c_uint64
    g = {c["name"]: c for c in large_cases}["llama2-70b.L0.attn.k_proj"]
    n = g["rows"] * g["cols"]
    bm, vals = np.zeros((n + 7) // 8, np.uint8), np.zeros(n * 2, np.uint8)
    nnz = L.or_make_op_mt(g["rows"], g["cols"], g["seed"], g["sparsity"], 4, bm, vals)
    assert (nnz, crc(bm), crc(vals[: nnz * 2])) == (g["nnz"], g["crc_bitmap"], g["crc_values"])


# ---- oracle vs the reference itself (only where oracle/_ref was built) ----------------

@pytest.fixture(scope="module")
def R():
    r = O.ref()
    if r is None:
        pytest.skip("oracle/_ref/libendor_ref.so not built (needs /root/reference)")
    return r


def test_oracle_equals_reference_random(R):
    rng = np.random.default_rng(1)
    for it in range(200):
        rows, cols = int(rng.integers(1, 70)), int(rng.integers(1, 70))
        eb = 2 if it % 2 else 1
        w = O.random_dense(rows, cols, eb, int(rng.integers(1 << 40)), float(rng.random()))
        n = rows * cols
        bm, vals, nnz, nz = O.compress(w, rows, cols, eb)
        rb, rv = np.zeros((n + 7) // 8, np.uint8), np.zeros(n * eb, np.uint8)
        rn, rz = C.c_uint64(), C.c_int()
        assert R.ref_compress(rows, cols, eb, w, rb, rv, C.byref(rn), C.byref(rz)) == 0
        assert rb.tobytes() == bm.tobytes() and rn.value == nnz and rv[: nnz * eb].tobytes() == vals.tobytes()
        out = np.zeros(n * eb, np.uint8)
        assert R.ref_decompress(rows, cols, eb, bm, vals if len(vals) else np.zeros(1, np.uint8), nnz, out) == 0
        assert out.tobytes() == O.decompress(rows, cols, eb, bm, vals, nnz)[1].tobytes()
        cs = 64 << int(rng.integers(0, 7))
        rp = np.zeros((n + cs - 1) // cs, np.uint64)
        R.ref_rank_index(bm, n, cs, rp)
        assert rp.tolist() == O.rank_index(bm, n, cs)[1].tolist()


def test_oracle_error_codes_equal_reference(R):
    w = O.random_dense(10, 10, 2, 9, 0.5)
    bm, vals, nnz, _ = O.compress(w, 10, 10, 2)
    out = np.zeros(200, np.uint8)
    # popcount mismatch: one value short
    assert R.ref_decompress(10, 10, 2, bm, vals, nnz - 1, out) == O.CORRUPTION
    assert O.decompress(10, 10, 2, bm, vals[:-2], nnz - 1)[0] == O.CORRUPTION
    _, p = O.rank_index(bm, 100, 64)
    bad = p.copy()
    bad[-1] += 1
    assert R.ref_decompress_chunked(10, 10, 2, bm, vals, nnz, 64, bad, len(bad), out) == O.CORRUPTION
    assert O.lib().or_decompress_chunked(10, 10, 2, bm, vals, nnz, 64, bad, len(bad), out) == O.CORRUPTION
    assert R.ref_decompress_chunk_into(10, 10, 2, bm, vals, nnz, 64, p, len(p), 5, out, 200) == O.BOUNDS
    assert R.ref_decompress_chunk_into(10, 10, 2, bm, vals, nnz, 64, p, len(p), 0, out, 198) == O.INVALID


def test_nm_prune_equals_reference(R):
    w = O.synth_weight(9, 37, 2, 3)
    for n, m in ((2, 4), (1, 3), (3, 8)):
        a = np.zeros(9 * 37 * 2, np.uint8)
        b = np.zeros(9 * 37 * 2, np.uint8)
        assert R.ref_nm_prune(9, 37, 2, w, n, m, a) == 0
        assert O.lib().or_nm_prune(9, 37, 2, n, m, w, b) == 0
        assert a.tobytes() == b.tobytes()
