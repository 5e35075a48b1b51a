"""Full-size parity at every BASELINE.json shape (GPU).

Inputs are regenerated on the device by the bit-exact synth_weight +
magnitude_prune + compress kernels and pinned to CRC-32s the REFERENCE
produced on the same seeds (tests/golden/large.json, make_golden.py).  The
decompressed dense matrix is then checked three ways: its CRC against the
reference's decompress output, a device-side round trip (decompress(compress(w))
== w, the size-independent property), and the rank index CRC at chunk 4096.
"""
import zlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def crc(t: "torch.Tensor") -> int:
    # stream the CRC in 256 MiB slices to bound host memory
    c = 0
    flat = t.reshape(-1)
    step = 256 << 20
    for i in range(0, flat.numel(), step):
        c = zlib.crc32(flat[i: i + step].cpu().numpy().tobytes(), c)
    return c & 0xFFFFFFFF


def test_large_shapes(cuda_lib, large_cases):
    from paper_2406_11674_b200 import codec as E
    for c in large_cases:
        rows, cols, s = c["rows"], c["cols"], c["sparsity"]
        w = E.synth_weight(rows, cols, c["seed"], device="cuda")
        E.magnitude_prune(w, s, inplace=True)
        t = E.compress(w)
        assert t.nnz() == c["nnz"], c["name"]
        assert crc(t.bitmap.data) == c["crc_bitmap"], c["name"]
        assert crc(t.values) == c["crc_values"], c["name"]
        out = E.decompress(t)
        assert torch.equal(out.data, w.data), c["name"]      # round trip on device
        assert crc(out.data) == c["crc_dense"], c["name"]     # == reference decompress
        idx = E.build_rank_index(t.bitmap, 4096)
        assert crc(idx.prefix.view(torch.uint8)) == c["crc_prefix_4096"], c["name"]
        # the reference's default chunk: one launch, sub-tile starts derived on chip
        assert torch.equal(E.decompress_chunked(t, idx).data, w.data), c["name"]
        idx1k = E.build_rank_index(t.bitmap, 1024)  # load-time index: single-launch path
        assert torch.equal(E.decompress_chunked(t, idx1k).data, w.data), c["name"]
        del w, t, out, idx
        torch.cuda.empty_cache()
