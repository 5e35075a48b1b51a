"""§8(f) row 3: fused INT8 dequant + decompress on the GPU, bit-exact against
decompress(dequantize_values(t)) (codec.hpp:334-349 then :157)."""
import zlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E(cuda_lib):
    from paper_2406_11674_b200 import codec
    return codec


def _dev(a, offset=0):
    a = np.ascontiguousarray(np.asarray(a).view(np.uint8).reshape(-1))
    buf = torch.zeros(a.size + offset + 32, dtype=torch.uint8, device="cuda")
    v = buf[offset: offset + a.size]
    if a.size:
        v.copy_(torch.from_numpy(a.copy()))
    return v


def _i8_tensor(E, rows, cols, bm, q, nnz, scale, values_offset=0, bitmap_offset=0):
    n = rows * cols
    bitmap = E.Bitmap(n, data=_dev(bm, bitmap_offset) if n else None)
    return E.EndorTensor(rows, cols, E.Dtype.I8, bitmap, _dev(q, values_offset), quant_scale=scale,
                         validate=False, nnz=nnz)


def test_quantized_round_trip_matches_reference_chain(E, quant_cases):
    for c in quant_cases:
        rows, cols = c["rows"], c["cols"]
        w = O.random_dense(rows, cols, 2, c["seed"], c["zero_fraction"])
        bm, vals, nnz, _ = O.compress(w, rows, cols, 2)
        q, scale = O.quantize_values(vals, nnz)
        assert np.float32(scale).view(np.uint32) == c["scale_bits"]
        assert zlib.crc32(q.tobytes()) == c["crc_q"]
        for voff, boff in ((0, 0), (3, 0), (1, 4)):
            t = _i8_tensor(E, rows, cols, bm, q, nnz, scale, voff, boff)
            out = E.decompress_dequant(t)
            assert zlib.crc32(out.bytes()) == c["crc_dense"], (c, voff, boff)


SCALES = [1.0, 0.00311, 1e-6, 1e-8, 3.0517578125e-05, 600.0, 65504.0 / 127, -0.5, 0.0, -0.0,
          float("inf"), float("-inf"), float("nan")]


@pytest.mark.parametrize("scale", SCALES)
def test_every_int8_value_every_edge_scale(E, scale):
    """All 256 i8 values (incl. -128, which quantize_values never emits) at
    scales hitting subnormals, overflow to inf, -0, NaN; alternate bitmap
    slots unset (must stay +0 even for negative / NaN scales)."""
    rows, cols = 4, 256
    n = rows * cols
    bits = np.zeros(n, bool)
    bits[::2] = True
    bits[1::7] = True
    bm = np.packbits(bits, bitorder="little")
    nnz = int(bits.sum())
    q = (np.arange(nnz) * 37 % 256).astype(np.uint8)
    want_st, want = O.decompress_dequant(rows, cols, bm, q, nnz, np.float32(scale))
    assert want_st == 0
    t = _i8_tensor(E, rows, cols, bm, q, nnz, float(np.float32(scale)))
    got = E.decompress_dequant(t).bytes()
    assert got == want.tobytes()


@pytest.mark.parametrize("scale", SCALES)
def test_dequantize_values_every_int8_value(E, scale):
    """dequantize_values (codec.hpp:334-349) of the packed values alone: all
    256 i8 values at every edge scale == the oracle's f32_to_f16 restatement,
    and decompress(dequantize_values(t)) == the fused dequant expand."""
    nnz = 256 * 3
    q = (np.arange(nnz) * 101 % 256).astype(np.uint8)
    want = np.zeros(nnz, np.uint16)
    O.lib().or_dequantize_values(q, nnz, np.float32(scale), want)
    bits = np.ones(nnz, bool)
    bm = np.packbits(bits, bitorder="little")
    t = _i8_tensor(E, 3, 256, bm, q, nnz, float(np.float32(scale)), values_offset=1)
    d = E.dequantize_values(t)
    assert d.dtype == E.Dtype.F16 and d.values.cpu().numpy().tobytes() == want.tobytes()
    assert E.decompress(d).bytes() == E.decompress_dequant(t).bytes()


def test_dequant_large_layer_shape(E):
    """fc1-sized: 9216 x 36864 @ 50%, GPU-generated, quantized on the host
    oracle, fused dequant+decompress == oracle chain (CRC)."""
    rows, cols = 2304, 36864  # a quarter of fc1 keeps host-side quantization fast
    w = E.synth_weight(rows, cols, 7, device="cuda")
    E.magnitude_prune(w, 0.5, inplace=True)
    t = E.compress(w)
    bm = t.bitmap.data.cpu().numpy()
    vals = t.values.cpu().numpy()
    q, scale = O.quantize_values(vals, t.nnz())
    st, want = O.decompress_dequant(rows, cols, bm, q, t.nnz(), scale)
    assert st == 0
    ti = _i8_tensor(E, rows, cols, bm, q, t.nnz(), scale)
    got = E.decompress_dequant(ti)
    assert zlib.crc32(got.bytes()) == zlib.crc32(want.tobytes())


def test_gpu_quantize_values_matches_reference(E, quant_cases):
    for c in quant_cases:
        w = O.random_dense(c["rows"], c["cols"], 2, c["seed"], c["zero_fraction"])
        bm, vals, nnz, _ = O.compress(w, c["rows"], c["cols"], 2)
        t = E.EndorTensor(c["rows"], c["cols"], E.Dtype.F16, E.Bitmap(c["rows"] * c["cols"], data=_dev(bm)),
                          _dev(vals), validate=False, nnz=nnz)
        q = E.quantize_values(t)
        assert np.float32(q.quant_scale).view(np.uint32) == c["scale_bits"]
        assert zlib.crc32(q.values.cpu().numpy().tobytes()) == c["crc_q"]
        assert zlib.crc32(E.decompress_dequant(q).bytes()) == c["crc_dense"]
    # special values: inf / NaN among the values (x86 lround semantics)
    vals = np.array([0x3C00, 0x7C00, 0xFC00, 0x7E01, 0x0001, 0x8001, 0x4000], np.uint16)
    q_ref, s_ref = O.quantize_values(vals.view(np.uint8), len(vals))
    t = E.EndorTensor(1, 7, E.Dtype.F16, E.Bitmap(7, data=_dev(np.array([0x7F], np.uint8))),
                      _dev(vals.view(np.uint8)), validate=False, nnz=7)
    q = E.quantize_values(t)
    assert np.float32(q.quant_scale) == np.float32(s_ref) or (np.isnan(q.quant_scale) and np.isnan(s_ref))
    assert q.values.cpu().numpy().tobytes() == q_ref.tobytes()


def test_dequant_errors(E):
    w = O.random_dense(10, 10, 2, 9, 0.5)
    bm, vals, nnz, _ = O.compress(w, 10, 10, 2)
    t = E.EndorTensor(10, 10, E.Dtype.F16, E.Bitmap(100, data=_dev(bm)), _dev(vals))
    with pytest.raises(E.InvalidArgument):  # f16 tensor: codec.hpp:335-337
        E.decompress_dequant(t)
    with pytest.raises(E.InvalidArgument):
        E.dequantize_values(t)
    q, scale = O.quantize_values(vals, nnz)
    bad = _i8_tensor(E, 10, 10, bm, q[:-1], nnz - 1, scale)
    with pytest.raises(E.CorruptionError):  # popcount != nnz
        E.decompress_dequant(bad)
