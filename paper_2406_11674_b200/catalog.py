"""Model catalog and synthetic-weight seeding (host side, no GPU needed).

Shapes restate ``model_catalog`` (reference model_catalog.hpp:55-86):
OPT-66B has 64 layers of q/k/v/out 9216x9216, fc1 9216x36864 and fc2
36864x9216; Llama2-70B has 80 layers of q/o 8192x8192, k/v 1024x8192,
gate/up 8192x28672 and down 28672x8192.  All f16.

Orientation: the catalog gives sizes only.  The GEMV consumer treats every
op as ``y = W @ x`` with W's rows as outputs, which keeps row-block sharding
free of partial-sum reductions ("GEMV orientation").

Seeds (stated so every run regenerates identical weights):
  layer l, op index o  ->  seed = 1000*l + o
  sparsity sweep       ->  seed = 100 + round(100*s)
  standalone fc1 (BASELINE config 1) -> seed 7
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

F16, I8 = 0, 1  # Dtype codes, dense_matrix.hpp:18-21


def elem_bytes(dtype: int) -> int:
    """dense_matrix.hpp:23."""
    return 2 if dtype == F16 else 1


@dataclass(frozen=True)
class OpShape:
    """model_catalog.hpp:14-26."""
    name: str
    rows: int
    cols: int
    dtype: int = F16

    @property
    def element_count(self) -> int:
        return self.rows * self.cols

    @property
    def dense_bytes(self) -> int:
        return self.element_count * elem_bytes(self.dtype)


@dataclass(frozen=True)
class ModelSpec:
    """model_catalog.hpp:29-36."""
    model_name: str
    num_layers: int
    ops: List[OpShape]

    @property
    def bytes_per_layer(self) -> int:
        return sum(o.dense_bytes for o in self.ops)

    def total_bytes(self) -> int:
        return self.bytes_per_layer * self.num_layers


def model_catalog(name: str) -> ModelSpec:
    """model_catalog.hpp:55-86; unknown names raise ValueError (ConfigError there)."""
    if name == "opt-66b":
        return ModelSpec(name, 64, [
            OpShape("attn.q_proj", 9216, 9216), OpShape("attn.k_proj", 9216, 9216),
            OpShape("attn.v_proj", 9216, 9216), OpShape("attn.out_proj", 9216, 9216),
            OpShape("fc1", 9216, 36864), OpShape("fc2", 36864, 9216)])
    if name == "llama2-70b":
        return ModelSpec(name, 80, [
            OpShape("attn.q_proj", 8192, 8192), OpShape("attn.k_proj", 1024, 8192),
            OpShape("attn.v_proj", 1024, 8192), OpShape("attn.o_proj", 8192, 8192),
            OpShape("mlp.gate_proj", 8192, 28672), OpShape("mlp.up_proj", 8192, 28672),
            OpShape("mlp.down_proj", 28672, 8192)])
    raise ValueError(f"unknown model: {name} (expected opt-66b or llama2-70b)")


def find_op(spec: ModelSpec, op_name: str) -> OpShape:
    """model_catalog.hpp:89-94."""
    for op in spec.ops:
        if op.name == op_name:
            return op
    raise ValueError(f"model {spec.model_name} has no op named {op_name}")


def op_seed(layer: int, op_index: int) -> int:
    return 1000 * layer + op_index


SWEEP_SPARSITIES = (0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9)


def sweep_seed(s: float) -> int:
    return 100 + int(round(100 * s))


FC1_SEED = 7


def pruned_nnz(n: int, sparsity: float) -> int:
    """nnz after magnitude_prune: n - floor(s*n) computed in double like
    weight_gen.hpp:102 (for inputs without pre-existing zeros)."""
    return n - int(sparsity * float(n))


def algorithmic_bytes(n: int, nnz: int, eb: int = 2) -> int:
    """Decompress roofline traffic: bitmap ceil(n/8) + values nnz*eb read,
    dense n*eb written."""
    return (n + 7) // 8 + nnz * eb + n * eb
