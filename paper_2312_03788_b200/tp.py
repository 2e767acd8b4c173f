"""Tensor-parallel sharding of the Code Llama linear stack.

Column-parallel layers (qkv, gate|up) split output channels N; row-parallel layers
(o_proj, down_proj) split input channels K **along group boundaries** (g = 128), so
every rank's quantization is a bit-identical slice of the 1-GPU quantization
(P14) and a group never straddles two ranks.  Row-parallel partial outputs are
summed with an all-reduce (NCCL over NVLink on the GPU box; gloo in CPU tests).

Architecture constants are public Code Llama model-card facts (not in PAPER.md):
  7B : hidden 4096, MLP 11008, 32 layers, 32 heads (MHA), head_dim 128
  34B: hidden 8192, MLP 22016, 48 layers, 64 q heads / 8 kv heads, head_dim 128
"""

from __future__ import annotations

from dataclasses import dataclass

GROUP = 128


@dataclass(frozen=True)
class ModelShape:
    name: str
    hidden: int
    mlp: int
    layers: int
    q_heads: int
    kv_heads: int
    head_dim: int = 128

    @property
    def qkv_out(self) -> int:
        return (self.q_heads + 2 * self.kv_heads) * self.head_dim


CODELLAMA_7B = ModelShape("codellama-7b", 4096, 11008, 32, 32, 32)
CODELLAMA_34B = ModelShape("codellama-34b", 8192, 22016, 48, 64, 8)


def group_split(n_groups: int, parts: int) -> list[tuple[int, int]]:
    """Balanced contiguous split of n_groups groups into `parts` ranges
    (the first n_groups % parts ranges get one extra group)."""
    if parts <= 0 or n_groups < parts:
        raise ValueError(f"cannot split {n_groups} groups over {parts} ranks")
    base, extra = divmod(n_groups, parts)
    out, g = [], 0
    for r in range(parts):
        n = base + (1 if r < extra else 0)
        out.append((g, g + n))
        g += n
    return out


def channel_split(channels: int, parts: int, group: int = GROUP) -> list[tuple[int, int]]:
    """Group-aligned split of `channels` (a multiple of `group`) into channel ranges."""
    if channels % group:
        raise ValueError(f"{channels} is not a multiple of {group}")
    return [(a * group, b * group) for a, b in group_split(channels // group, parts)]


@dataclass(frozen=True)
class LinearShard:
    """One rank's slice of a linear layer W[N][K]: rows (output channels) listed as
    ranges into the full N, columns as one range into the full K."""
    name: str
    kind: str                       # "col" or "row"
    n_ranges: tuple                 # ((n0, n1), ...) into the full N
    k_range: tuple                  # (k0, k1) into the full K
    allreduce: bool

    @property
    def N(self) -> int:
        return sum(b - a for a, b in self.n_ranges)

    @property
    def K(self) -> int:
        return self.k_range[1] - self.k_range[0]


def layer_shards(m: ModelShape, rank: int, world: int) -> list[LinearShard]:
    """The four W4A16 linears of one decoder layer for `rank` of `world`
    (Fig. 6: all 7 linears of the LlamaDecoderLayer are INT4;
    q|k|v and gate|up are fused as vLLM does)."""
    if m.q_heads % world or m.kv_heads % world:
        raise ValueError(f"{world} ranks do not divide the heads of {m.name}")
    H, I, D = m.hidden, m.mlp, m.head_dim
    qh, kvh = m.q_heads // world, m.kv_heads // world
    q0 = rank * qh * D
    k0 = m.q_heads * D + rank * kvh * D
    v0 = (m.q_heads + m.kv_heads) * D + rank * kvh * D
    qkv = LinearShard("qkv", "col", ((q0, q0 + qh * D), (k0, k0 + kvh * D), (v0, v0 + kvh * D)),
                      (0, H), False)
    o_k = channel_split(m.q_heads * D, world)[rank]
    o = LinearShard("o_proj", "row", ((0, H),), o_k, world > 1)
    mlp_r = channel_split(I, world)[rank]
    gate_up = LinearShard("gate_up", "col", (mlp_r, (I + mlp_r[0], I + mlp_r[1])), (0, H), False)
    down = LinearShard("down_proj", "row", ((0, H),), mlp_r, world > 1)
    return [qkv, o, gate_up, down]


def full_shapes(m: ModelShape) -> list[tuple[str, int, int]]:
    """(name, K, N) of the unsharded fused linears."""
    return [("qkv", m.hidden, m.qkv_out), ("o_proj", m.q_heads * m.head_dim, m.hidden),
            ("gate_up", m.hidden, 2 * m.mlp), ("down_proj", m.mlp, m.hidden)]


def w4_bytes(K: int, N: int, group: int = GROUP, zeros_u4: bool = False) -> int:
    """Bytes of the W4 layout: codes + fp16 Δ + fp16 Z (or packed u4 Z, SQ_ZEROS_U4)."""
    return K * N // 2 + 2 * N * (K // group) + (N * (K // group) // 2 if zeros_u4 else 2 * N * (K // group))


def decode_bytes(M: int, K: int, N: int, group: int = GROUP, zeros_u4: bool = False) -> int:
    """Algorithmic HBM bytes of one W4A16 GEMM:
    K·N/2 + 4·N·K/g + 2·M·K + 2·M·N (u4 zeros: 2.5·N·K/g for Δ and Z)."""
    return w4_bytes(K, N, group, zeros_u4) + 2 * M * K + 2 * M * N


def gemm_flops(M: int, K: int, N: int) -> int:
    return 2 * M * N * K
