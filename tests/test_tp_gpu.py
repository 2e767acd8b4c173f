"""Tensor-parallel path on the GPU (world size 2 on one device, gloo for the
collective): each rank quantizes its group-aligned shards of one Code-Llama-shaped
layer with the CUDA kernels, runs sq_w4a16_gemm on them, and the row-parallel
all-reduce / column-parallel concatenation must reproduce the unsharded GPU GEMM
and the fp64 oracle.  The NCCL transport is not exercised
here (one GPU); the shard arithmetic and the kernels on shard shapes are."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SMALL = None  # filled in the worker (import inside the spawned process)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        import oracle
        from paper_2312_03788_b200 import sq, synth, tp
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        torch.cuda.set_device(0)
        model = tp.ModelShape("tiny-34b-like", hidden=1024, mlp=2816, layers=1, q_heads=8, kv_heads=2,
                              head_dim=128)
        ok = []
        for M in (1, 5, 16, 40):
            for i, (name, K, N) in enumerate(tp.full_shapes(model)):
                W = synth.weights(N, K, seed=20 + i)
                X = synth.activations(M, K, seed=30 + i).astype(np.float16)
                sh = tp.layer_shards(model, rank, world)[i]
                rows = np.concatenate([np.arange(a, b) for a, b in sh.n_ranges])
                k0, k1 = sh.k_range
                Wsh = np.ascontiguousarray(W[rows][:, k0:k1])
                qsh = sq.quantize_pack_groupwise(torch.from_numpy(Wsh).cuda())
                y = sq.w4a16_gemm(torch.from_numpy(np.ascontiguousarray(X[:, k0:k1])).cuda(), qsh)
                t = y.float().cpu()
                full = oracle.quantize_pack(W, None)
                y_ref = oracle.gemm(X, full["Wq"], full["scales"], full["zeros"])
                if sh.kind == "row":
                    dist.all_reduce(t)  # fp32 reduction of the fp16 partials
                    got = t.double().numpy()
                else:
                    widths = [tp.layer_shards(model, r, world)[i].N for r in range(world)]
                    pad = torch.zeros(M, max(widths))
                    pad[:, :t.shape[1]] = t
                    outs = [torch.zeros_like(pad) for _ in range(world)]
                    dist.all_gather(outs, pad)
                    got = np.zeros_like(y_ref)
                    for r in range(world):
                        rs = np.concatenate([np.arange(a, b) for a, b in
                                             tp.layer_shards(model, r, world)[i].n_ranges])
                        got[:, rs] = outs[r].numpy()[:, :widths[r]]
                err = np.linalg.norm(got - y_ref) / np.linalg.norm(y_ref)
                ok.append(bool(err <= 2e-3))
        q.put((rank, all(ok)))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_tp_world2_one_gpu():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


def _nccl_worker(port, q):
    """One rank, NCCL process group (init_process_group("nccl", device_id=...)) as bench.py
    does for N > 1: the row-parallel layers of a 1-rank stack reduced through the NCCL
    fallback (fp16 in place, bf16 through an fp32 copy) and through the peer-memory path
    (attach_peer_allreduce: IPC setup, validation, fused GEMM + all-reduce kernel) must
    equal the plain GEMM of the same shard -- a 1-rank sum is the partial itself."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
        from paper_2312_03788_b200 import sq, stack, tp
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        dist.init_process_group("nccl", device_id=dev)
        pg = dist.group.WORLD
        model = tp.ModelShape("tiny-34b-like", hidden=1024, mlp=2816, layers=2, q_heads=8, kv_heads=2,
                              head_dim=128)
        st = stack.build_stack(model, 2, 0, 1, dev, group=pg)
        ok = []
        for dt in (torch.float16, torch.bfloat16):
            st.dtype = dt
            for M in (1, 16, 40):
                b = stack.make_buffers(st, M, dev)
                stack.run_pass(st, b)               # NCCL all_reduce after row-parallel layers
                torch.cuda.synchronize()
                for lin in st.layers[-1]:
                    want = sq.w4a16_gemm(b.x[lin.shard.name], lin.q)
                    ok.append(bool(torch.equal(b.y[lin.shard.name], want)))
        impl = stack.attach_peer_allreduce(st, 16 * model.hidden, dev)
        ok.append(impl.startswith("peer"))
        st.dtype = torch.float16
        for M in (1, 16):
            b = stack.make_buffers(st, M, dev)
            stack.run_pass(st, b)                   # fused GEMM + peer all-reduce (1 rank)
            torch.cuda.synchronize()
            for lin in st.layers[-1]:
                want = sq.w4a16_gemm(b.x[lin.shard.name], lin.q).float()
                got = b.y[lin.shard.name].float()
                ok.append(bool(((got - want).abs() <= 2e-3 * want.abs() + 1e-3).all()))
        ok.append(not st.peer_ar.failed())
        q.put(all(ok) or f"failed: {ok} ({impl})")
    except Exception as e:
        q.put(repr(e))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_nccl_process_group_one_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    res = q.get(timeout=600)
    p.join(timeout=60)
    assert res is True, res
