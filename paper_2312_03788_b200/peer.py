"""Symmetric peer buffers and the one-shot row-parallel all-reduce.

Plumbing only: torch allocates each rank's buffer and torch.distributed exchanges the
CUDA IPC handles (libsq's sq_ipc_*); the exchange of the partial outputs is one kernel,
sq_allreduce_oneshot (csrc/k_allreduce.cu), over NVLink/NVSwitch peer memory.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import sq


class PeerAllReduce:
    """Row-parallel all-reduce of up to n_max fp16/bf16 outputs per call, one instance per
    process group.  Collective construction (every rank of `group` must build it); a rank
    whose mapping fails raises after the exchange, so callers agree on success with one
    more collective (stack.attach_peer_allreduce) before the first call."""

    def __init__(self, n_max: int, device, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.n_max = (int(n_max) + 7) // 8 * 8
        nb = sq.allreduce_buffer_bytes(self.n_max, self.world)
        self.buf = torch.zeros(nb, dtype=torch.uint8, device=device)  # flags must start at 0
        self.err = torch.zeros(1, dtype=torch.int32, device=device)
        torch.cuda.synchronize(device)
        try:
            mine = sq.ipc_get_handle(self.buf)
        except Exception:
            mine = None  # still join the exchange, so no rank is left waiting in it
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        if any(h is None for h in allh):
            raise RuntimeError("PeerAllReduce: a rank could not export its buffer")
        self._opened = []
        addrs = []
        for q, (h, o) in enumerate(allh):
            if q == self.rank:
                addrs.append(self.buf.data_ptr())
            else:
                base = sq.ipc_open_handle(h)
                self._opened.append(base)
                addrs.append(base + o)
        self.peers = torch.tensor(addrs, dtype=torch.int64, device=device)

    def __call__(self, y: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """In place by default: y (this rank's partial) becomes the sum over ranks.  The epoch
        is device-managed (epoch 0), so the call may be captured in a CUDA graph."""
        if y.numel() > self.n_max:
            raise ValueError(f"PeerAllReduce: {y.numel()} outputs > n_max {self.n_max}")
        return sq.allreduce_oneshot(y, self.peers, self.rank, self.world, 0, self.n_max, self.err,
                                    out=out, stream=stream)

    def failed(self) -> bool:
        """True if any call timed out waiting for a peer (host sync)."""
        return bool(self.err.item())

    def close(self):
        torch.cuda.synchronize()
        for base in self._opened:
            sq.ipc_close(base)
        self._opened = []

    def gemm(self, X: torch.Tensor, q: sq.QuantizedLinear, out: torch.Tensor | None = None,
             workspace: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """Row-parallel linear + all-reduce in one call (sq_w4a16_gemm_allreduce): X is this
        rank's input shard, q its weight shard; returns the summed Y on every rank."""
        if X.shape[0] * q.N > self.n_max:
            raise ValueError(f"PeerAllReduce.gemm: {X.shape[0] * q.N} outputs > n_max {self.n_max}")
        return sq.w4a16_gemm_allreduce(X, q, self.peers, self.rank, self.world, self.n_max, self.err,
                                       out=out, workspace=workspace, stream=stream)

