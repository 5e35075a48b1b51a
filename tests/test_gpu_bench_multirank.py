"""`bench.py --gpus N` launches N ranks itself (GPU).

The driver runs `python bench.py --gpus N ...` (and the torchrun form); both
must run one process per rank and print ONE JSON line with n_gpus == N and a
bit-exact N>1 parity check (every rank CRCs the row shards it SLICED out of
the whole compressed matrices; rank 0 joins them with crc32_combine against
the reference's whole-matrix CRC-32s).  This box has one GPU, so the ranks
share it (ENDOR_BENCH_SHARE_GPU=1, gloo plumbing): a code-path check, not a
scaling measurement."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n,extra", [(2, []), (4, ["--no-e2e"])])
def test_bench_self_launches_n_ranks(cuda_lib, n, extra):
    env = dict(os.environ, ENDOR_BENCH_SHARE_GPU="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "3",
                        "--warmup", "3", "--no-extras", "--no-cpu-baseline", *extra],
                       cwd=ROOT, capture_output=True, text=True, timeout=1500, env=env)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == n
    assert d["config"]["sharding"] == f"row-block x{n}"
    assert d["parity"] is not None and d["parity"]["bit_exact"] is True, d["parity"]
    assert d["parity"]["tensors"] == 6
    assert d["value"] > 0


def test_reference_arm_self_launch_prints_once(cuda_lib):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=1500, env=env)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    import bench
    assert d["config"]["workload"] == bench.WORKLOAD  # same config string as our arm
