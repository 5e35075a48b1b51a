"""Row-block sharded deployment on the GPU (north star (c)).

One compressed tensor is SLICED into G row shards with shard.shard_tensor --
bitmap bits [r0 C, r1 C), values [rank(r0 C), rank(r1 C)) (bitmap.hpp:41,
codec.hpp:21-23); nothing is recompressed.  Every shard is decompressed by the
CUDA kernels and the shards, joined in row order, must reproduce the
reference's whole-matrix output:

  * catalog shapes at full size, G in {2, 4, 8}: per-shard CRC-32s joined with
    crc32_combine == the reference's decompress CRC (tests/golden/large.json);
  * ragged / unaligned shapes (checked against the oracle): a bitmap slice that
    is 4- but not 16-byte aligned (the plain fallback expand), one that is not
    4-byte aligned (copied), and cols % 8 != 0 (bit-shifted re-pack);
  * the fused GEMV of every shard == the rows of the whole matrix's GEMV;
  * a world-size-2 gloo job on the GPU box: each rank slices and decompresses
    its shard on cuda:0 and all_gather_dense / all_gather_y rebuild the whole W
    and y.
"""
import os
import socket
import zlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def crc(t) -> int:
    c, flat, step = 0, t.reshape(-1), 256 << 20
    for i in range(0, flat.numel(), step):
        c = zlib.crc32(flat[i: i + step].cpu().numpy().tobytes(), c)
    return c & 0xFFFFFFFF


CATALOG = ["opt-66b.L0.attn.q_proj", "llama2-70b.L0.attn.k_proj", "llama2-70b.L0.mlp.down_proj"]


@pytest.mark.parametrize("name", CATALOG)
def test_catalog_shards_join_to_reference_crc(cuda_lib, large_cases, name):
    from paper_2406_11674_b200 import codec as E, shard as S
    c = next(x for x in large_cases if x["name"] == name)
    w = E.synth_weight(c["rows"], c["cols"], c["seed"], device="cuda")
    E.magnitude_prune(w, c["sparsity"], inplace=True)
    t = E.compress(w)
    del w
    for G in (2, 4, 8):
        joined, nnz = 0, 0
        for sh in S.row_shards(c["rows"], c["cols"], G):
            for copy in (False, True):
                p = S.shard_tensor(t, sh, copy=copy)
                if copy:  # the per-GPU path: own buffers, load-time 1024 index, one launch
                    out = E.decompress_chunked(p, E.build_rank_index(p.bitmap, 1024))
                else:     # views into the whole tensor's buffers
                    out = E.decompress(p)
                if copy:
                    joined = S.crc32_combine(joined, crc(out.data), out.data.numel())
                    nnz += p.nnz()
                else:
                    ref_view = out
            assert torch.equal(ref_view.data, out.data), (name, G, sh.rank)
        assert nnz == c["nnz"], (name, G)
        assert joined == c["crc_dense"], (name, G)
    torch.cuda.empty_cache()


# (rows, cols, G): 1056 cols -> 132 bitmap bytes per row (views 4- but not
# 16-byte aligned: fallback expand); 1000 -> 125 B per row (not 4-aligned:
# copied); 1001 -> shard bit ranges not byte aligned (re-packed)
RAGGED = [(99, 1056, 4), (95, 1000, 3), (67, 1001, 2), (64, 2048, 8), (5, 40, 8)]


@pytest.mark.parametrize("rows,cols,G", RAGGED)
def test_ragged_unaligned_shards(cuda_lib, rows, cols, G):
    from oracle import oracle as O
    from paper_2406_11674_b200 import codec as E, shard as S
    w = O.random_dense(rows, cols, 2, 1000 + rows + cols, 0.5)
    bm, vals, nnz, _ = O.compress(w, rows, cols, 2)
    st, ref = O.decompress(rows, cols, 2, bm, vals, nnz)
    assert st == 0
    t = E.EndorTensor(rows, cols, E.Dtype.F16, E.Bitmap.from_bytes(bm.tobytes(), rows * cols, device="cuda"),
                      torch.from_numpy(vals.copy()).cuda())
    for copy in (False, True):
        parts, total = [], 0
        for sh in S.row_shards(rows, cols, G):
            p = S.shard_tensor(t, sh, copy=copy)
            assert p.bitmap.size() == sh.rows * cols
            total += p.nnz()
            parts.append(E.decompress(p).bytes() if sh.rows else b"")
            # the shard's own bitmap must be a valid Endor bitmap (zero padding bits)
            E.Bitmap.from_bytes(p.bitmap.to_bytes(), sh.rows * cols)
        assert total == nnz
        assert b"".join(parts) == ref.tobytes(), (rows, cols, G, copy)


@pytest.mark.parametrize("rows,cols,G", [(96, 2048, 4), (1000, 3072, 8)])
def test_sharded_fused_gemv_rows(cuda_lib, rows, cols, G):
    """y of every shard (fused decompress -> GEMV on its slice) == the matching
    rows of the whole matrix's y, element-wise within 1e-3 of sum |W_ij x_j|."""
    from oracle import oracle as O
    from paper_2406_11674_b200 import codec as E, shard as S
    w = O.random_dense(rows, cols, 2, 31 + G, 0.5)
    bm, vals, nnz, _ = O.compress(w, rows, cols, 2)
    t = E.EndorTensor(rows, cols, E.Dtype.F16, E.Bitmap.from_bytes(bm.tobytes(), rows * cols, device="cuda"),
                      torch.from_numpy(vals.copy()).cuda())
    x = torch.randn(cols, dtype=torch.float16, device="cuda")
    W = torch.from_numpy(w.view(np.float16).astype(np.float32).reshape(rows, cols))
    yref = W @ x.cpu().float()
    mag = W.abs() @ x.cpu().float().abs()
    ys = [E.gemv_compressed(S.shard_tensor(t, sh, copy=True), x).cpu() for sh in S.row_shards(rows, cols, G)]
    y = torch.cat(ys)
    assert ((y - yref).abs() <= 1e-3 * mag + 1e-6).all()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, rows, cols, q):
    import sys
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2406_11674_b200 import codec as E, shard as S
        torch.cuda.set_device(0)
        w = O.random_dense(rows, cols, 2, 4242, 0.5)  # the same tensor on every rank
        bm, vals, nnz, _ = O.compress(w, rows, cols, 2)
        t = E.EndorTensor(rows, cols, E.Dtype.F16,
                          E.Bitmap.from_bytes(bm.tobytes(), rows * cols, device="cuda"),
                          torch.from_numpy(vals.copy()).cuda())
        sh = S.row_shard(rows, cols, rank, world)
        p = S.shard_tensor(t, sh, copy=True)
        part = E.decompress(p)
        full = S.all_gather_dense(part, rows)
        ok_w = full.cpu().numpy().tobytes() == w.tobytes()
        x = torch.from_numpy(np.random.default_rng(9).standard_normal(cols).astype(np.float16)).cuda()
        y = S.all_gather_y(E.gemv_compressed(p, x), rows)
        W = torch.from_numpy(w.view(np.float16).astype(np.float32).reshape(rows, cols))
        yref = W @ x.cpu().float()
        ok_y = bool(((y.cpu() - yref).abs() <= 1e-3 * (W.abs() @ x.cpu().float().abs()) + 1e-6).all())
        q.put((rank, ok_w and ok_y and y.device.type == "cuda"))
    finally:
        dist.destroy_process_group()


def test_all_gather_on_gpu_gloo_world2(cuda_lib):
    import torch.multiprocessing as mp
    world, rows, cols = 2, 128, 2048
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, rows, cols, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    assert dict(q.get(timeout=10) for _ in range(world)) == {0: True, 1: True}
