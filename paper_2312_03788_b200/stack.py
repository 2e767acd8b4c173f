"""The Code Llama W4A16 linear stack on one rank: synthetic weights quantized on the
device (PAPER.md:176 load-time quantization), and decode / prefill passes through
sq_w4a16_gemm with an all-reduce after the row-parallel layers.

Attention, RMSNorm, SiLU and the residual stream are not part of the hot path
(SURVEY.md §3 (5)): each linear reads a fixed, pre-filled activation buffer of the
right shape, so a pass streams exactly the W4 weights of every layer once.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import sq
from .tp import CODELLAMA_34B, LinearShard, ModelShape, decode_bytes, gemm_flops, layer_shards


@dataclass
class Linear:
    shard: LinearShard
    q: sq.QuantizedLinear


@dataclass
class LinearStack:
    model: ModelShape
    rank: int
    world: int
    layers: list = field(default_factory=list)   # list[list[Linear]]
    group: object = None                          # torch.distributed process group (None: no AR)
    dtype: torch.dtype = torch.float16
    peer_ar: object = None                        # peer.PeerAllReduce (None: NCCL all_reduce)

    @property
    def shards(self) -> list[LinearShard]:
        return [l.shard for l in self.layers[0]]


def synth_weight(N: int, K: int, seed: int, device, dtype=torch.float16) -> torch.Tensor:
    """W ~ N(0, 0.02^2) drawn on the device with a seeded generator (synthetic
    stand-in for a Code Llama checkpoint)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return (torch.randn((N, K), generator=g, device=device, dtype=torch.float32) * 0.02).to(dtype)


def synth_act_max(K: int, seed: int, device) -> torch.Tensor:
    """Per-channel calibration maxima with 8 x100 outlier channels."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    a = 3.0 + torch.rand(K, generator=g, device=device)
    idx = torch.randperm(K, generator=g, device=device)[:8]
    a[idx] *= 100.0
    return a.float().contiguous()


def build_stack(model: ModelShape = CODELLAMA_34B, layers: int | None = None, rank: int = 0,
                world: int = 1, device="cuda", seed: int = 1234, smooth: bool = True,
                group=None, zeros_u4: bool = False) -> LinearStack:
    """Quantize `layers` decoder layers' linears for this rank (setup, not timed).  Each
    rank draws only its own shard.  Eq. 6's weight maxima are those of the FULL weight: a
    column-parallel shard holds some output rows of every input channel, so the ranks
    all-reduce their shard's column maxima with MAX before computing s (every rank folds
    the same s, as a real tensor-parallel deployment of Eq. 5/6 would); a row-parallel
    shard holds whole input channels, so its maxima are already complete.  The returned
    weights are resident and final, so their GEMMs run with SQ_GEMM_WEIGHTS_STATIC.
    zeros_u4: the zero points in the packed u4 layout (SQ_ZEROS_U4)."""
    import torch.distributed as dist

    L = model.layers if layers is None else layers
    st = LinearStack(model, rank, world, group=group)
    shards = layer_shards(model, rank, world)
    for li in range(L):
        row = []
        for si, sh in enumerate(shards):
            W = synth_weight(sh.N, sh.K, seed + 1000 * li + 10 * si + 100000 * rank, device)
            s = None
            if smooth:
                am = synth_act_max(sh.K, seed + 7 * si, device)
                w_max = sq.weight_absmax(W)
                if group is not None and world > 1 and sh.kind == "col":
                    dist.all_reduce(w_max, op=dist.ReduceOp.MAX, group=group)
                s = sq.smooth_scales_wmax(w_max, am, 0.5)
            row.append(Linear(sh, sq.quantize_pack_groupwise(W, s, zeros_u4=zeros_u4)))
            del W
        st.layers.append(row)
    torch.cuda.synchronize(device)  # the quantize kernels are done: the weights are final
    for row in st.layers:
        for lin in row:
            lin.q.mark_static()
    return st


@dataclass
class PassBuffers:
    M: int
    x: dict      # shard name -> input [M][K_r]
    y: dict      # shard name -> output [M][N_r]


def make_buffers(st: LinearStack, M: int, device="cuda", seed: int = 7) -> PassBuffers:
    g = torch.Generator(device=device)
    g.manual_seed(seed + M)
    xs, ys = {}, {}
    for sh in st.shards:
        xs[sh.name] = torch.randn((M, sh.K), generator=g, device=device).to(st.dtype)
        ys[sh.name] = torch.empty((M, sh.N), device=device, dtype=st.dtype)
    return PassBuffers(M, xs, ys)


def run_pass(st: LinearStack, buf: PassBuffers, path: int = sq.SQ_PATH_AUTO, workspace=None) -> int:
    """One pass of every layer's linears at buf.M tokens; returns #kernel launches."""
    import torch.distributed as dist

    n = 0
    for row in st.layers:
        for lin in row:
            y = buf.y[lin.shard.name]
            fused = (lin.shard.allreduce and st.group is not None and st.peer_ar is not None
                     and y.numel() <= st.peer_ar.n_max and path == sq.SQ_PATH_AUTO)
            if fused:
                # row-parallel linear + all-reduce over peer memory: one kernel at decode
                # sizes (sq_w4a16_gemm_allreduce), GEMM + one-shot exchange kernel above
                st.peer_ar.gemm(buf.x[lin.shard.name], lin.q, out=y, workspace=workspace)
                n += 1 if buf.M <= sq.decode_max_m() else 2
                continue
            sq.w4a16_gemm(buf.x[lin.shard.name], lin.q, out=y, path=path, workspace=workspace)
            n += 1
            if lin.shard.allreduce and st.group is not None:
                if y.dtype == torch.bfloat16:
                    # reduce bf16 partials in fp32, round once
                    y32 = y.float()
                    dist.all_reduce(y32, group=st.group)
                    y.copy_(y32)
                else:
                    dist.all_reduce(y, group=st.group)
    return n


def pass_bytes(st: LinearStack, M: int) -> int:
    """Algorithmic HBM bytes of one pass on this rank."""
    return len(st.layers) * sum(decode_bytes(M, sh.K, sh.N) for sh in st.shards)


def pass_flops(st: LinearStack, M: int) -> int:
    return len(st.layers) * sum(gemm_flops(M, sh.K, sh.N) for sh in st.shards)


def attach_peer_allreduce(st: LinearStack, n_max: int, device="cuda") -> str:
    """Use the one-shot peer-memory all-reduce for the row-parallel
    layers of messages up to n_max outputs (decode sizes), NCCL above.  Collective.  The
    path is validated once with known data; if the IPC mapping or the exchange fails the
    stack keeps NCCL and the reason is returned (plumbing choice, reported by bench.py)."""
    import torch.distributed as dist

    from . import peer

    def agree(flag: bool) -> bool:
        t = torch.tensor([1 if flag else 0], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=st.group)
        return int(t.item()) == 1

    ar, why = None, ""
    try:
        ar = peer.PeerAllReduce(n_max, device, group=st.group)
    except Exception as e:  # IPC not permitted etc.
        why = f"{type(e).__name__}: {e}"
    if not agree(ar is not None):
        return f"nccl (peer setup failed: {why or 'on another rank'})"[:200]
    y = torch.full((4096,), float(st.rank + 1), dtype=st.dtype, device=device)
    ar(y)
    torch.cuda.synchronize()
    want = float(st.world * (st.world + 1) // 2)
    if not agree((not ar.failed()) and bool((y.float() == want).all())):
        return "nccl (peer all-reduce validation failed)"
    st.peer_ar = ar
    return "peer: fused GEMM+all-reduce kernel (decode sizes) over NVLink peer memory"
