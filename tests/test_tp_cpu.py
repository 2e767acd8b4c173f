"""Tensor-parallel host logic on CPU (world size 2, gloo): group-aligned shard
arithmetic and the row-parallel all-reduce / column-parallel
concatenation reproduce the unsharded layer (P14).  The per-rank GEMM here is the
oracle; on the GPU box the same shards run through sq_w4a16_gemm + NCCL."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2312_03788_b200 import synth, tp

TINY = tp.ModelShape("tiny", hidden=256, mlp=384, layers=1, q_heads=4, kv_heads=2, head_dim=64)


def test_group_split_balanced_and_aligned():
    for G, P in ((172, 8), (64, 8), (86, 4), (86, 8), (3, 2), (21, 1)):
        parts = tp.group_split(G, P)
        assert parts[0][0] == 0 and parts[-1][1] == G
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
        sizes = [b - a for a, b in parts]
        assert max(sizes) - min(sizes) <= 1
    assert [b - a for a, b in tp.group_split(172, 8)] == [22, 22, 22, 22, 21, 21, 21, 21]
    with pytest.raises(ValueError):
        tp.group_split(3, 4)
    with pytest.raises(ValueError):
        tp.channel_split(200, 2)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_34b_shards_cover_layer(P):
    m = tp.CODELLAMA_34B
    full = {n: (K, N) for n, K, N in tp.full_shapes(m)}
    per = [tp.layer_shards(m, r, P) for r in range(P)]
    for i, name in enumerate(["qkv", "o_proj", "gate_up", "down_proj"]):
        shards = [p[i] for p in per]
        K, N = full[name]
        if shards[0].kind == "col":
            rows = sorted(x for s in shards for rg in s.n_ranges for x in range(*rg))
            assert rows == list(range(N))
            assert all(s.k_range == (0, K) for s in shards)
        else:
            ks = [s.k_range for s in shards]
            assert ks[0][0] == 0 and ks[-1][1] == K
            assert all(k0 % 128 == 0 for k0, _ in ks)
            assert all(s.allreduce == (P > 1) for s in shards)
    # gate|up shard rows match down_proj's K range (the MLP intermediate stays local)
    for r in range(P):
        gu, dn = per[r][2], per[r][3]
        assert gu.n_ranges[0] == dn.k_range
    # per-rank W4 bytes sum to the full layer's
    tot = sum(tp.w4_bytes(s.K, s.N) for p in per for s in p)
    assert tot == sum(tp.w4_bytes(K, N) for _, K, N in tp.full_shapes(m))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        M = 3
        X = synth.activations(M, TINY.hidden, seed=5).astype(np.float16)
        ok = []
        for i, (name, K, N) in enumerate(tp.full_shapes(TINY)):
            W = synth.weights(N, K, seed=10 + i)
            Xk = synth.activations(M, K, seed=20 + i).astype(np.float16) if K != TINY.hidden else X
            full = oracle.quantize_pack(W, None, 128)
            Y_full = oracle.gemm(Xk, full["Wq"], full["scales"], full["zeros"])
            sh = tp.layer_shards(TINY, rank, world)[i]
            rows = np.concatenate([np.arange(a, b) for a, b in sh.n_ranges])
            k0, k1 = sh.k_range
            part = oracle.quantize_pack(W[rows][:, k0:k1], None, 128)
            # P14: the shard's quantization is a bit-identical slice of the full one
            ok.append(bool((part["Wq"] == full["Wq"][rows][:, k0 // 2:k1 // 2]).all()))
            ok.append(bool((part["scales"] == full["scales"][k0 // 128:k1 // 128][:, rows]).all()))
            Y = oracle.gemm(Xk[:, k0:k1], part["Wq"], part["scales"], part["zeros"])
            t = torch.from_numpy(Y)
            if sh.kind == "row":
                dist.all_reduce(t)
                ok.append(bool(np.allclose(t.numpy(), Y_full, rtol=1e-12, atol=1e-12)))
            else:
                # gloo's all_gather needs equal sizes: pad every shard to the widest
                widths = [tp.layer_shards(TINY, r, world)[i].N for r in range(world)]
                padded = torch.zeros(M, max(widths), dtype=t.dtype)
                padded[:, :t.shape[1]] = t
                outs = [torch.zeros_like(padded) for _ in range(world)]
                dist.all_gather(outs, padded)
                Y_cat = np.zeros_like(Y_full)
                for r in range(world):
                    rs = np.concatenate([np.arange(a, b) for a, b in
                                         tp.layer_shards(TINY, r, world)[i].n_ranges])
                    Y_cat[:, rs] = outs[r].numpy()[:, :widths[r]]
                ok.append(bool(np.array_equal(Y_cat, Y_full)))
        result_q.put((rank, all(ok)))
    except Exception as e:  # report instead of hanging the parent
        result_q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_tp_world2_gloo_matches_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
