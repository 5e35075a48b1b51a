""".endor containers straight to the GPU.

CPU: the encoder is byte-identical to the reference's (test_io.cpp:30-57
golden bytes; reference encoder on seeded cases) and endor_file_probe rejects
each header/layout corruption with decode_endor's FormatError kind
(test_io.cpp:106-176).  GPU: the reader (cuFile or POSIX) reproduces the
tensor bit-exactly; verify catches BadCrc / CountMismatch / Malformed padding
on the device copy; every single-byte flip of a valid file is rejected
(test_io.cpp:178-186)."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import oracle as O

KIND = {"Truncated": 0, "BadMagic": 1, "BadVersion": 2, "BadCrc": 3, "CountMismatch": 4, "Malformed": 5}


@pytest.fixture(scope="module")
def L():
    from paper_2406_11674_b200 import _lib
    return _lib.lib()


def encode(L, rows, cols, dtype, bm, vals, nnz, flags=0, scale=0.0):
    n = L.endor_file_encode(rows, cols, dtype, flags, scale, bm.ctypes.data if bm.size else None,
                            vals.ctypes.data if vals.size else None, nnz, None, 0)
    buf = C.create_string_buffer(n)
    assert L.endor_file_encode(rows, cols, dtype, flags, scale, bm.ctypes.data if bm.size else None,
                               vals.ctypes.data if vals.size else None, nnz, buf, n) == n
    return buf.raw


def tiny(L):
    # test_io.cpp tiny_tensor: the 2x2 hand-built tensor (bitmap 1010, values 0x3C00 0x4200)
    bm = np.array([0x05], np.uint8)
    vals = np.array([0x00, 0x3C, 0x00, 0x42], np.uint8)
    return encode(L, 2, 2, 0, bm, vals, 2)


def test_encoder_matches_reference_golden_bytes(L, kats):
    assert tiny(L).hex() == kats["endor_file_2x2"]["bytes"]
    z = encode(L, 4, 4, 0, np.zeros(2, np.uint8), np.zeros(0, np.uint8), 0)
    assert z.hex() == kats["endor_file_zero_4x4"]["bytes"] and len(z) == 38


def test_encoder_matches_reference_encoder_on_random_cases(L):
    R = O.ref()
    if R is None:
        pytest.skip("reference library not built")
    for seed, (rows, cols, eb) in enumerate([(7, 9, 2), (16, 16, 2), (3, 64, 1), (1, 1, 2)]):
        w = O.random_dense(rows, cols, eb, seed, 0.5)
        bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
        mine = encode(L, rows, cols, 0 if eb == 2 else 1, bm, vals, nnz)
        out = np.zeros(len(mine) + 64, np.uint8)
        n = R.ref_encode_endor(rows, cols, eb, bm, vals, nnz, 0, out, out.size)
        assert bytes(out[:n]) == mine


def probe_kind(L, tmp_path, data):
    from paper_2406_11674_b200 import _lib
    p = tmp_path / "t.endor"
    p.write_bytes(bytes(data))
    info = _lib.FileInfo()
    st = L.endor_file_probe(os.fsencode(str(p)), C.byref(info))
    return st, (L.endor_cuda_last_format_kind() if st == 7 else None), info


def test_probe_accepts_and_describes_a_valid_file(L, tmp_path):
    st, _, info = probe_kind(L, tmp_path, tiny(L))
    assert st == 0
    assert (info.rows, info.cols, info.nnz, info.dtype) == (2, 2, 2, 0)
    assert (info.bitmap_offset, info.bitmap_bytes, info.values_offset, info.values_bytes) == (32, 1, 33, 4)
    assert info.file_bytes == 41


@pytest.mark.parametrize("mutate,kind", [
    (lambda b: b.__setitem__(0, ord("X")), "BadMagic"),       # test_io.cpp:109-118
    (lambda b: b.__setitem__(4, 9), "BadVersion"),            # :119-128
    (lambda b: b.pop(), "Truncated"),                         # :155-164
    (lambda b: b.append(0), "Malformed"),                     # :165-174 trailing bytes
    (lambda b: b.__setitem__(6, 7), "Malformed"),             # unknown dtype code
    (lambda b: b.__setitem__(7, 0x80), "Malformed"),          # unknown flag bits
    (lambda b: b.__setitem__(24, 9), "Malformed"),            # nnz > rows*cols
    (lambda b: b.__setitem__(8, 20), "Truncated"),            # rows 20: layout longer than the file
    (lambda b: b.__delitem__(slice(20, None)), "Truncated"),  # ends mid-field
])
def test_probe_rejects_each_header_corruption(L, tmp_path, mutate, kind):
    b = bytearray(tiny(L))
    mutate(b)
    st, k, _ = probe_kind(L, tmp_path, b)
    assert st == 7 and k == KIND[kind]


def test_probe_rejects_layout_sizes_that_wrap(L, tmp_path):
    """rows=2^31, cols=2^32, nnz=2^63-2^59 (quantized f16) makes
    header + bitmap + values + crc wrap to 40 bytes; the reference's cursor
    runs off the end (Truncated).  The probe must not report ~2^60-byte
    sections for a 40-byte file."""
    import struct
    rows, cols, nnz = 1 << 31, 1 << 32, (1 << 63) - (1 << 59)
    hdr = b"ENDR" + struct.pack("<HBB", 1, 0, 1) + struct.pack("<QQQ", rows, cols, nnz) + struct.pack("<f", 1.0)
    for tail in (b"\0\0\0\0", b"\0" * 8):
        st, k, info = probe_kind(L, tmp_path, hdr + tail)
        assert st == 7 and k == KIND["Truncated"]


def encode_v2(L, rows, cols, dtype, bm, vals, nnz, flags=0, scale=0.0):
    args = (rows, cols, dtype, flags, scale, bm.ctypes.data if bm.size else None,
            vals.ctypes.data if vals.size else None, nnz)
    n = L.endor_file_encode_v2(*args, None, 0)
    buf = C.create_string_buffer(n)
    assert L.endor_file_encode_v2(*args, buf, n) == n
    return buf.raw


@pytest.mark.parametrize("rows,cols,eb,flags", [(2, 2, 2, 0), (300, 1000, 2, 0), (77, 333, 1, 1), (128, 256, 2, 2),
                                                (4, 4, 2, 0)])
def test_v2_container_layout(L, tmp_path, rows, cols, eb, flags):
    """Version 2: the v1 fields with the bitmap at byte 4096 and the values at
    the next 4 KiB boundary (GDS-ready offsets), zero fill, CRC-32 over every
    preceding byte; the v1 encoder is unchanged (golden test above)."""
    import zlib
    w = O.random_dense(rows, cols, eb, rows * cols, 0.5)
    bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
    v1 = encode(L, rows, cols, 0 if eb == 2 else 1, bm, vals, nnz, flags, 0.25)
    v2 = encode_v2(L, rows, cols, 0 if eb == 2 else 1, bm, vals, nnz, flags, 0.25)
    hdr = 36 if flags & 1 else 32
    assert v2[:4] == b"ENDR" and v2[4:6] == b"\x02\x00" and v2[6:hdr] == v1[6:hdr]
    voff = 4096 + (bm.size + 4095) // 4096 * 4096
    assert len(v2) == voff + vals.size + 4
    assert v2[4096:4096 + bm.size] == bm.tobytes() and v2[voff:voff + vals.size] == vals.tobytes()
    assert not any(v2[hdr:4096]) and not any(v2[4096 + bm.size:voff])
    assert int.from_bytes(v2[-4:], "little") == zlib.crc32(v2[:-4]) & 0xFFFFFFFF
    st, _, info = probe_kind(L, tmp_path, v2)
    assert st == 0
    assert (info.bitmap_offset, info.bitmap_bytes, info.values_offset, info.values_bytes, info.file_bytes) == \
        (4096, bm.size, voff, vals.size, len(v2))
    assert info.gap_bytes == voff - 4096 - bm.size
    assert info.values_out_bytes == info.values_bytes
    assert info.header_crc == zlib.crc32(v2[:4096]) & 0xFFFFFFFF
    # a dirty fill byte (header page or the gap) is Malformed even with a fixed-up CRC
    for at in ([100] + ([4096 + bm.size] if voff > 4096 + bm.size else [])):
        bad = bytearray(v2)
        bad[at] = 1
        bad[-4:] = (zlib.crc32(bytes(bad[:-4])) & 0xFFFFFFFF).to_bytes(4, "little")
        st, k, _ = probe_kind(L, tmp_path, bad)
        assert st == 7 and k == KIND["Malformed"]
    # truncated / trailing as v1
    st, k, _ = probe_kind(L, tmp_path, v2[:-1])
    assert st == 7 and k == KIND["Truncated"]
    st, k, _ = probe_kind(L, tmp_path, v2 + b"\0")
    assert st == 7 and k == KIND["Malformed"]


def encode_v3(L, rows, cols, bm, vals, nnz, flags=0, k_max=0):
    """v3 container: v2 with the values as a coded-values blob (csrc/vcode.cu)."""
    need = C.c_size_t(0)
    vp = vals.ctypes.data if vals.size else None
    assert L.endor_values_encode(vp, nnz, k_max, None, 0, C.byref(need)) == 0
    blob = np.zeros(need.value, np.uint8)
    assert L.endor_values_encode(vp, nnz, k_max, blob.ctypes.data, blob.size, C.byref(need)) == 0
    bmp = bm.ctypes.data if bm.size else None
    n = L.endor_file_encode_v3(rows, cols, flags, bmp, blob.ctypes.data, nnz, None, 0)
    buf = C.create_string_buffer(n)
    assert n and L.endor_file_encode_v3(rows, cols, flags, bmp, blob.ctypes.data, nnz, buf, n) == n
    return buf.raw, blob


@pytest.mark.parametrize("rows,cols,flags,k_max", [(2, 2, 0, 0), (300, 1000, 0, 0), (128, 256, 2, 4), (64, 4096, 0, 0)])
def test_v3_container_layout(L, tmp_path, rows, cols, flags, k_max):
    """Version 3 (no reference counterpart): the v2 layout, flags bit 2, and the
    values section holding the coded-values blob, whose header gives its
    length; the CRC covers it like any section."""
    import zlib
    w = O.synth_weight(rows, cols, 2, rows + cols)
    _, w = O.magnitude_prune(w, rows * cols, 2, 0.5)
    bm, vals, nnz, _ = O.compress(w, rows, cols, 2)
    v3, blob = encode_v3(L, rows, cols, bm, vals, nnz, flags, k_max)
    assert v3[:4] == b"ENDR" and v3[4:6] == b"\x03\x00" and v3[7] == (flags | 4)
    voff = 4096 + (bm.size + 4095) // 4096 * 4096
    assert len(v3) == voff + blob.size + 4 and v3[voff:voff + blob.size] == blob.tobytes()
    assert int.from_bytes(v3[-4:], "little") == zlib.crc32(v3[:-4]) & 0xFFFFFFFF
    st, _, info = probe_kind(L, tmp_path, v3)
    assert st == 0 and info.flags == flags | 4
    assert (info.values_offset, info.values_bytes, info.file_bytes) == (voff, blob.size, len(v3))
    assert info.values_out_bytes == 2 * nnz  # what the reader writes: the decoded values
    # a blob header that disagrees with the container, bit 2 missing, or a quantized v3: Malformed
    for at, x in ((voff + 8, 1), (voff, 0x10), (7, 4), (7, 1)):
        bad = bytearray(v3)
        bad[at] ^= x
        bad[-4:] = (zlib.crc32(bytes(bad[:-4])) & 0xFFFFFFFF).to_bytes(4, "little")
        st, k, _ = probe_kind(L, tmp_path, bad)
        assert st == 7 and k == KIND["Malformed"], (at, x)
    st, k, _ = probe_kind(L, tmp_path, v3[:voff + 100])
    assert st == 7 and k == KIND["Truncated"]
    # v1 / v2 readers of other tools: version 3 is its own version number
    assert L.endor_file_encode_v3(rows, cols, 1, None, blob.ctypes.data, nnz, None, 0) == 0  # quantized
    assert L.endor_file_encode_v3(rows, cols, 0, None, blob.ctypes.data, nnz + 1, None, 0) == 0  # nnz mismatch



# ---------------------------------------------------------------------------- GPU

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def S(cuda_lib):
    from paper_2406_11674_b200 import storage
    return storage


@pytest.fixture(scope="module")
def E(cuda_lib):
    from paper_2406_11674_b200 import codec
    return codec


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 3])  # auto = GDS when nvidia-fs is loaded, else POSIX
@pytest.mark.parametrize("rows,cols,s,dtype", [(2, 2, 0.5, 0), (300, 1000, 0.5, 0), (1024, 9216, 0.7, 0),
                                               (77, 333, 0.4, 1), (5, 5, 1.0, 0)])
def test_reader_round_trip_bit_exact(S, E, tmp_path, mode, rows, cols, s, dtype):
    eb = 2 if dtype == 0 else 1
    w = O.random_dense(rows, cols, eb, rows + cols, s)
    bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
    t = E.EndorTensor(rows, cols, E.Dtype(dtype), E.Bitmap.from_bytes(bm.tobytes(), rows * cols, device="cuda"),
                      torch.from_numpy(vals.copy()).cuda())
    p = str(tmp_path / "w.endor")
    n = S.write_endor_file(t, p)
    assert n == os.path.getsize(p) == 32 + bm.size + vals.size + 4
    r = S.Reader("cuda", mode=mode, bounce_bytes=1 << 16)  # small bounce: many chunks
    got = r.read(p, verify=True)
    assert r.mode in ("gds", "cufile-compat", "posix-odirect")
    assert got.bitmap.to_bytes() == bm.tobytes()
    assert got.values.cpu().numpy().tobytes() == vals.tobytes()
    assert E.decompress(got).bytes() == w.tobytes()
    r.close()


@pytest.mark.gpu
def test_reader_verify_detects_payload_corruption(S, E, L, tmp_path):
    w = O.random_dense(64, 100, 2, 5, 0.5)
    bm, vals, nnz, _ = O.compress(w, 64, 100, 2)
    good = bytearray(encode(L, 64, 100, 0, bm, vals, nnz))
    p = str(tmp_path / "c.endor")

    def kind_of(data):
        open(p, "wb").write(bytes(data))
        with pytest.raises(E.FormatError) as ei:
            S.read_endor_file(p, "cuda", verify=True)
        return ei.value.kind.name

    bad = bytearray(good)
    bad[-1] ^= 0xFF
    assert kind_of(bad) == "BadCrc"
    bad = bytearray(good)
    bad[40] ^= 0x10  # a value byte: CRC catches it on the GPU
    assert kind_of(bad) == "BadCrc"

    def refix_crc(b):
        import zlib
        b[-4:] = (zlib.crc32(bytes(b[:-4])) & 0xFFFFFFFF).to_bytes(4, "little")
        return b

    bad = bytearray(good)
    bad[32] ^= 0x01  # one set bit more or fewer; CRC fixed up
    b2 = refix_crc(bad)
    assert kind_of(b2) == "CountMismatch"  # test_io.cpp:139-154


@pytest.mark.gpu
def test_reader_rejects_every_single_byte_flip(S, E, L, tmp_path):
    # test_io.cpp:178-186
    w = O.random_dense(4, 6, 2, 2, 0.5)
    bm, vals, nnz, _ = O.compress(w, 4, 6, 2)
    good = encode(L, 4, 6, 0, bm, vals, nnz)
    p = str(tmp_path / "f.endor")
    r = S.Reader("cuda")
    for i in range(len(good)):
        bad = bytearray(good)
        bad[i] ^= 0x5B
        open(p, "wb").write(bytes(bad))
        with pytest.raises(E.FormatError):
            r.read(p, verify=True)
    r.close()


@pytest.mark.gpu
def test_pipeline_file_sourced_ops_match_host_sourced(S, E, tmp_path):
    """EndorDirect through the offload pipeline: ops read from .endor files give
    the same y as the same ops streamed from pinned host memory."""
    from paper_2406_11674_b200.pipeline import HostOp, OffloadPipeline, pinned_copy
    shapes = [(64, 2048), (33, 1000), (128, 4096)]
    ys = {}
    for src in ("host", "file"):
        ops = []
        for i, (r, c) in enumerate(shapes):
            w = E.synth_weight(r, c, 50 + i, device="cuda")
            E.magnitude_prune(w, 0.5, inplace=True)
            t = E.compress(w)
            x = ((torch.rand(c, generator=torch.Generator().manual_seed(i)) * 2 - 1).half()).cuda()
            kw = dict(x=x, y=torch.empty(r, dtype=torch.float32, device="cuda"),
                      y_host=torch.empty(r, dtype=torch.float32, pin_memory=True))
            if src == "file":
                p = str(tmp_path / f"op{i}.endor")
                S.write_endor_file(t, p)
                e = torch.empty(0, dtype=torch.uint8)
                ops.append(HostOp(r, c, 0, e, e, t.nnz(), path=p, **kw))
            else:
                ops.append(HostOp(r, c, 0, pinned_copy(t.bitmap.data), pinned_copy(t.values), t.nnz(), **kw))
        pipe = OffloadPipeline(0, max(r * c for r, c in shapes))
        pipe.run(ops, sync=True)
        st = pipe.stats()
        pipe.close()
        assert st["h2d_bytes"] == sum(o.compressed_bytes for o in ops)
        ys[src] = [o.y_host.clone() for o in ops]
    for a, b in zip(ys["host"], ys["file"]):
        assert torch.equal(a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,s,dtype", [(2, 2, 0.5, 0), (300, 1000, 0.5, 0), (1024, 9216, 0.7, 0),
                                               (77, 333, 0.4, 1)])
def test_reader_v2_round_trip_and_crc(S, E, L, tmp_path, rows, cols, s, dtype):
    """v2 containers through the GPU reader: the sections land at their 4 KiB
    offsets, the device CRC check folds in the zero fill, corruption is caught."""
    eb = 2 if dtype == 0 else 1
    w = O.random_dense(rows, cols, eb, rows + cols, s)
    bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
    t = E.EndorTensor(rows, cols, E.Dtype(dtype), E.Bitmap.from_bytes(bm.tobytes(), rows * cols, device="cuda"),
                      torch.from_numpy(vals.copy()).cuda())
    p = str(tmp_path / "w2.endor")
    n = S.write_endor_file(t, p, version=2)
    assert n == os.path.getsize(p) and S.probe(p).bitmap_offset == 4096
    r = S.Reader("cuda", mode=3, bounce_bytes=1 << 16)
    got = r.read(p, verify=True)
    assert got.bitmap.to_bytes() == bm.tobytes()
    assert got.values.cpu().numpy().tobytes() == vals.tobytes()
    assert E.decompress(got).bytes() == w.tobytes()
    data = bytearray(open(p, "rb").read())
    if vals.size:
        data[S.probe(p).values_offset] ^= 0x20
        open(p, "wb").write(bytes(data))
        with pytest.raises(E.FormatError) as ei:
            r.read(p, verify=True)
        assert ei.value.kind.name == "BadCrc"
    r.close()


@pytest.mark.gpu
def test_cufile_compat_mode_never_hangs(tmp_path):
    """ENDOR_IO_CUFILE_COMPAT runs cuFileDriverOpen under a watchdog: on a box
    without nvidia-fs (where the open blocks) the reader reports an IO error
    within the timeout instead of hanging; where it opens, reads are exact.
    Run in a child process -- a parked driver thread must not outlive the test."""
    import subprocess
    import sys
    code = (
        "import sys, torch; sys.path.insert(0, %r)\n"
        "from oracle import oracle as O\n"
        "from paper_2406_11674_b200 import codec as E, storage as S\n"
        "w = O.random_dense(64, 128, 2, 1, 0.5); bm, vals, nnz, _ = O.compress(w, 64, 128, 2)\n"
        "t = E.EndorTensor(64, 128, E.Dtype.F16, E.Bitmap.from_bytes(bm.tobytes(), 8192, device='cuda'),"
        " torch.from_numpy(vals.copy()).cuda())\n"
        "p = %r; S.write_endor_file(t, p, version=2)\n"
        "try:\n"
        "    r = S.Reader('cuda', mode=2)\n"
        "except E.Error as e:\n"
        "    print('IOERR', e); sys.stdout.flush(); import os; os._exit(0)\n"
        "got = r.read(p, verify=True); assert E.decompress(got).bytes() == w.tobytes(); print('OK', r.mode)\n"
        "sys.stdout.flush(); import os; os._exit(0)\n"
    ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), str(tmp_path / "c.endor"))
    env = dict(os.environ, ENDOR_CUFILE_OPEN_TIMEOUT_S="5")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.startswith("OK") or "cuFileDriverOpen" in out.stdout, out.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,s,synth", [(2, 2, 0.5, True), (300, 1000, 0.5, True), (1024, 9216, 0.5, True),
                                               (1024, 9216, 0.7, False), (5, 5, 1.0, True)])
def test_reader_v3_decodes_coded_values(S, E, L, tmp_path, rows, cols, s, synth):
    """v3 containers: the reader moves the coded section, checks the CRC over it,
    and decodes it on the GPU into the exact packed values."""
    if synth:
        w = O.synth_weight(rows, cols, 2, rows + cols)
        _, w = O.magnitude_prune(w, rows * cols, 2, s)
    else:
        w = O.random_dense(rows, cols, 2, rows + cols, s)
    bm, vals, nnz, _ = O.compress(w, rows, cols, 2)
    t = E.EndorTensor(rows, cols, E.Dtype.F16, E.Bitmap.from_bytes(bm.tobytes(), rows * cols, device="cuda"),
                      torch.from_numpy(vals.copy()).cuda())
    p = str(tmp_path / "w3.endor")
    n = S.write_endor_file(t, p, version=3)
    info = S.probe(p)
    assert n == os.path.getsize(p) and info.flags & 4 and info.bitmap_offset == 4096
    r = S.Reader("cuda", mode=3, bounce_bytes=1 << 16)
    got = r.read(p, verify=True)
    assert got.bitmap.to_bytes() == bm.tobytes()
    assert got.values.cpu().numpy().tobytes() == vals.tobytes()
    assert E.decompress(got).bytes() == w.tobytes()
    assert r.read(p, verify=False).values.cpu().numpy().tobytes() == vals.tobytes()
    if nnz:
        data = bytearray(open(p, "rb").read())
        data[info.values_offset + info.values_bytes // 2] ^= 0x20  # inside the coded section
        open(p, "wb").write(bytes(data))
        with pytest.raises(E.FormatError) as ei:
            r.read(p, verify=True)
        assert ei.value.kind.name == "BadCrc"
    r.close()


@pytest.mark.gpu
def test_pipeline_v3_file_ops_match_host_sourced(S, E, tmp_path):
    """EndorDirect from v3 files through the offload pipeline: fewer bytes read,
    the same y as the raw host-sourced ops."""
    from paper_2406_11674_b200.pipeline import HostOp, OffloadPipeline, pinned_copy
    shapes = [(64, 2048), (33, 1000), (128, 4096)]
    ys, nbytes = {}, {}
    for src in ("host", "file"):
        ops = []
        for i, (r, c) in enumerate(shapes):
            w = E.synth_weight(r, c, 70 + i, device="cuda")
            E.magnitude_prune(w, 0.5, inplace=True)
            t = E.compress(w)
            x = ((torch.rand(c, generator=torch.Generator().manual_seed(i)) * 2 - 1).half()).cuda()
            kw = dict(x=x, y=torch.empty(r, dtype=torch.float32, device="cuda"),
                      y_host=torch.empty(r, dtype=torch.float32, pin_memory=True))
            if src == "file":
                p = str(tmp_path / f"v3op{i}.endor")
                S.write_endor_file(t, p, version=3)
                e = torch.empty(0, dtype=torch.uint8)
                ops.append(HostOp(r, c, 0, e, e, t.nnz(), path=p, **kw))
            else:
                ops.append(HostOp(r, c, 0, pinned_copy(t.bitmap.data), pinned_copy(t.values), t.nnz(), **kw))
        pipe = OffloadPipeline(0, max(r * c for r, c in shapes))
        pipe.run(ops, sync=True)
        nbytes[src] = pipe.stats()["h2d_bytes"]
        pipe.close()
        ys[src] = [o.y_host.clone() for o in ops]
    assert nbytes["file"] < nbytes["host"]
    for a, b in zip(ys["host"], ys["file"]):
        assert torch.equal(a, b)
