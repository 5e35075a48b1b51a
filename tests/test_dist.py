"""Multi-process (world_size 2, gloo, CPU) coverage of the row-sharded path:
each rank takes its row shard of a compressed tensor (bitmap/values slices at
host-computed rank boundaries), decompresses it with the oracle (the checker,
standing in for the GPU kernel here), and an all-gather reassembles the full
dense matrix, which must equal the reference-format round trip bit-exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, rows, cols, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import oracle as O
        from paper_2406_11674_b200 import shard as S
        w = O.random_dense(rows, cols, 2, 2024, 0.5)      # same inputs on every rank
        bm, vals, nnz, _ = O.compress(w, rows, cols, 2)
        sh = S.row_shard(rows, cols, rank, world)
        sb, sv, snnz = S.host_shard_slices(bm, vals, 2, sh)
        st, part = O.decompress(sh.rows, cols, 2, sb, sv, snnz)
        assert st == 0
        # nnz of all shards sums to the tensor's nnz
        t = torch.tensor([snnz], dtype=torch.int64)
        dist.all_reduce(t)
        assert int(t.item()) == nnz
        # all-gather of equal row shards = the full dense matrix
        mine = torch.from_numpy(part.copy())
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)
        full = torch.cat(parts).numpy()
        q.put((rank, full.tobytes() == w.tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rows,cols", [(64, 96), (128, 256)])
def test_row_sharded_decompress_gloo_world2(rows, cols):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, rows, cols, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = dict(q.get(timeout=10) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert results == {0: True, 1: True}


def _gemv_worker(rank, world, port, rows, cols, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import oracle as O
        from paper_2406_11674_b200 import shard as S
        w = O.random_dense(rows, cols, 2, 77, 0.5)
        bm, vals, nnz, _ = O.compress(w, rows, cols, 2)
        x = np.random.default_rng(5).standard_normal(cols).astype(np.float32)
        sh = S.row_shard(rows, cols, rank, world)
        sb, sv, snnz = S.host_shard_slices(bm, vals, 2, sh)
        st, part = O.decompress(sh.rows, cols, 2, sb, sv, snnz)
        assert st == 0
        wpart = part.view(np.float16).reshape(sh.rows, cols).astype(np.float32)
        y = S.all_gather_y(torch.from_numpy(wpart @ x), rows)
        yfull = w.view(np.float16).reshape(rows, cols).astype(np.float32) @ x
        q.put((rank, bool(np.allclose(y.numpy(), yfull, rtol=0, atol=1e-4 * np.abs(yfull).max()))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rows", [64, 67])  # 67: ragged shards
def test_row_sharded_gemv_all_gather_y_gloo_world2(rows):
    world, cols = 2, 128
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gemv_worker, args=(r, world, port, rows, cols, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = dict(q.get(timeout=10) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert results == {0: True, 1: True}
