"""One-shot row-parallel all-reduce over peer memory on one
GPU.  The expected value is fixed by the definition, not by the kernel: every rank gets
RN( ((0 + p_0) + p_1) + ... ) in fp32, rank order -- bit-exact, identical on all ranks.

  * single process, one stream per "rank": the kernel's protocol (push, per-chunk flags,
    wait, ordered reduce, epoch parity double buffering) with world 2 and 3, ragged sizes
    and back-to-back calls;
  * two processes (gloo for the handle exchange), CUDA IPC mapping of the symmetric
    buffers (PeerAllReduce), several epochs, and the row-parallel layer of the TP stack
    reduced with it against the unsharded oracle.
The NVLink transport itself is not exercised (one GPU); the peer mapping and protocol are.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_03788_b200 import sq

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _expected(parts):
    acc = torch.zeros_like(parts[0], dtype=torch.float32)
    for p in parts:
        acc = acc + p.float()
    return acc.to(parts[0].dtype)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("n", [8, 2048, 8192 * 16 + 5, 8192 * 64])
@pytest.mark.parametrize("mode", ["explicit", "device"])
def test_oneshot_protocol_streams(world, n, dtype, mode):
    n_max = (n + 7) // 8 * 8 + 64
    nb = sq.allreduce_buffer_bytes(n_max, world)
    bufs = [torch.zeros(nb, dtype=torch.uint8, device=DEV) for _ in range(world)]
    peers = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=DEV)
    errs = [torch.zeros(1, dtype=torch.int32, device=DEV) for _ in range(world)]
    streams = [torch.cuda.Stream() for _ in range(world)]
    g = torch.Generator(device=DEV).manual_seed(n + world)
    torch.cuda.synchronize()
    for epoch in range(1, 6):  # back-to-back calls: both parities, reuse
        parts = [torch.randn(n, generator=g, device=DEV).to(dtype) for _ in range(world)]
        outs = [torch.empty_like(parts[0]) for _ in range(world)]
        torch.cuda.synchronize()
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                sq.allreduce_oneshot(parts[r], peers, r, world, epoch if mode == "explicit" else 0, n_max,
                                     errs[r], out=outs[r], stream=streams[r])
        torch.cuda.synchronize()
        assert all(int(e.item()) == 0 for e in errs)
        want = _expected(parts)
        for r in range(world):
            assert torch.equal(outs[r].view(torch.int16), want.view(torch.int16)), (epoch, r)


def test_oneshot_in_place_and_timeout():
    world, n = 2, 4096
    n_max = n
    nb = sq.allreduce_buffer_bytes(n_max, world)
    bufs = [torch.zeros(nb, dtype=torch.uint8, device=DEV) for _ in range(world)]
    peers = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=DEV)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    # rank 1 never arrives: the bounded wait must give up and flag it, not hang
    y = torch.randn(n, device=DEV).half()
    sq.allreduce_oneshot(y, peers, 0, world, 7, n_max, err)
    torch.cuda.synchronize()
    assert int(err.item()) == 1


@pytest.mark.parametrize("zeros_u4", [False, True])
@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("M", [1, 5, 16])
@pytest.mark.parametrize("N,K", [(1024, 1024), (2048, 2048), (1024, 3072)])
def test_fused_gemm_allreduce_streams(M, N, K, dtype, zeros_u4):
    """sq_w4a16_gemm_allreduce (decode: one kernel) for two ranks on two streams of one GPU
    (grids of <= 148 CTAs, so both kernels are resident together), over back-to-back calls
    (both epoch parities, device-managed epoch).  Every rank gets the bit-identical Y, equal
    to the unsharded fp64 oracle within the dtype bound and the element-wise bound (the
    fused call cuts N from N alone, so its fp32 partials may be summed in another order
    than a plain sq_w4a16_gemm of the same shard; fp16 partials travel as fp16, bf16 ones as
    fp32)."""
    import oracle
    from paper_2312_03788_b200 import synth, tp
    from tests.gemm_bounds import elementwise_ratio

    world = 2
    W_np = synth.weights(N, K, seed=N + K)
    W = torch.from_numpy(W_np).to(DEV)
    ranges = tp.channel_split(K, world)
    qs = [sq.quantize_pack_groupwise(W[:, a:b].contiguous(), zeros_u4=zeros_u4) for a, b in ranges]
    full = oracle.quantize_pack(W_np, None)
    W_hat = oracle.dequant(full["Wq"], full["scales"], full["zeros"])
    n_max = M * N
    nb = sq.allreduce_buffer_bytes(n_max, world)
    bufs = [torch.zeros(nb, dtype=torch.uint8, device=DEV) for _ in range(world)]
    peers = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=DEV)
    errs = [torch.zeros(1, dtype=torch.int32, device=DEV) for _ in range(world)]
    wss = [torch.zeros(sq.w4a16_gemm_workspace_bytes(M, N, K), dtype=torch.uint8, device=DEV) for _ in range(world)]
    streams = [torch.cuda.Stream() for _ in range(world)]
    g = torch.Generator(device=DEV).manual_seed(M * 7 + N)
    for it in range(4):
        X = (torch.randn(M, K, generator=g, device=DEV) * 2).to(dtype)
        xs = [X[:, a:b].contiguous() for a, b in ranges]
        outs = [torch.empty(M, N, dtype=dtype, device=DEV) for _ in range(world)]
        torch.cuda.synchronize()
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                sq.w4a16_gemm_allreduce(xs[r], qs[r], peers, r, world, n_max, errs[r], out=outs[r],
                                        workspace=wss[r], stream=streams[r])
        torch.cuda.synchronize()
        assert all(int(e.item()) == 0 for e in errs)
        assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16)), it
        xd = "f16" if dtype == torch.float16 else "bf16"
        x64 = X.float().cpu().double().numpy()
        y_ref = x64 @ W_hat.T
        y = outs[0].float().cpu().double().numpy()
        assert np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref) <= (1e-3 if xd == "f16" else 4e-3)
        assert elementwise_ratio(y, y_ref, x64, W_hat, xd) <= 1.0


@pytest.fixture
def grid_limit():
    """Cap decode grids so that P simulated ranks' fused kernels are co-resident on one GPU."""
    def set_limit(v):
        sq.set_option(sq.SQ_OPT_DECODE_GRID_LIMIT, v)
    yield set_limit
    sq.set_option(sq.SQ_OPT_DECODE_GRID_LIMIT, 0)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("layer", ["o_proj", "down"])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_fused_allreduce_34b_tp_shards(P, layer, dtype, grid_limit):
    """The fused row-parallel GEMM + all-reduce at the Code Llama-34B tensor-parallel shard
    shapes: o_proj K_r = 8192 / P, down_proj K_r from the group-aligned
    split of 172 groups (P = 8: 22,22,22,22,21,21,21,21 -> K_r = 2816 / 2688, a rank-dependent
    ragged final stage).  All P ranks run as concurrent kernels on P streams (grids capped
    so they are co-resident), M in {1, 16}, device-managed epochs, against the unsharded
    fp64 oracle on sampled output rows; every rank holds the bit-identical Y."""
    import oracle
    from paper_2312_03788_b200 import stack, tp
    from tests.gemm_bounds import elementwise_ratio

    K, N = (8192, 8192) if layer == "o_proj" else (22016, 8192)
    W = stack.synth_weight(N, K, 41 + P, DEV)
    ranges = tp.channel_split(K, P)
    qs = [sq.quantize_pack_groupwise(W[:, a:b].contiguous()).mark_static() for a, b in ranges]
    rows = np.sort(np.random.default_rng(P).choice(N, 48, replace=False))
    ref = oracle.quantize_pack(W[rows].cpu().numpy(), None)      # rows quantize independently (P14)
    W_hat = oracle.dequant(ref["Wq"], ref["scales"], ref["zeros"])
    torch.cuda.synchronize()
    n_max = 16 * N
    nb = sq.allreduce_buffer_bytes(n_max, P)
    bufs = [torch.zeros(nb, dtype=torch.uint8, device=DEV) for _ in range(P)]
    peers = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=DEV)
    errs = [torch.zeros(1, dtype=torch.int32, device=DEV) for _ in range(P)]
    wss = [torch.zeros(sq.w4a16_gemm_workspace_bytes(16, N, b - a), dtype=torch.uint8, device=DEV)
           for a, b in ranges]
    streams = [torch.cuda.Stream() for _ in range(P)]
    grid_limit(max(1, 2 * torch.cuda.get_device_properties(0).multi_processor_count // P - 2))
    g = torch.Generator(device=DEV).manual_seed(P * 3 + K)
    for M in (1, 16, 1):
        X = torch.randn(M, K, generator=g, device=DEV).to(dtype)
        xs = [X[:, a:b].contiguous() for a, b in ranges]
        outs = [torch.empty(M, N, dtype=dtype, device=DEV) for _ in range(P)]
        torch.cuda.synchronize()
        for r in range(P):
            with torch.cuda.stream(streams[r]):
                sq.w4a16_gemm_allreduce(xs[r], qs[r], peers, r, P, n_max, errs[r], out=outs[r],
                                        workspace=wss[r], stream=streams[r])
        torch.cuda.synchronize()
        assert all(int(e.item()) == 0 for e in errs), [int(e.item()) for e in errs]
        for r in range(1, P):
            assert torch.equal(outs[0].view(torch.int16), outs[r].view(torch.int16)), (M, r)
        x64 = X.float().cpu().double().numpy()
        y_ref = x64 @ W_hat.T
        y = outs[0].float().cpu().double().numpy()[:, rows]
        xd = "f16" if dtype == torch.float16 else "bf16"
        assert np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref) <= (1e-3 if xd == "f16" else 4e-3), M
        assert elementwise_ratio(y, y_ref, x64, W_hat, xd) <= 1.0, M


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_fused_allreduce_back_to_back_pdl(dtype):
    """Back-to-back fused calls on one stream with NO host synchronization, programmatic
    dependent launch on, device-managed epochs (epoch 0), interleaved with plain GEMMs
    (a call must read the epoch only after the previous call's grid completed,
    or two calls share an epoch).  One rank, so no cross-rank scheduling is involved (two
    simulated ranks on one GPU can starve each other's streams, which separate GPUs
    cannot): the buffer's epoch must advance by exactly one per call, no error may be
    raised, and every result must equal the same call made in isolation (deterministic)."""
    from paper_2312_03788_b200 import synth

    M, N, K = 4, 1024, 2048
    q = sq.quantize_pack_groupwise(torch.from_numpy(synth.weights(N, K, seed=5)).to(DEV)).mark_static()
    qp = sq.quantize_pack_groupwise(torch.from_numpy(synth.weights(N, 1024, seed=6)).to(DEV)).mark_static()
    n_max = M * N
    buf = torch.zeros(sq.allreduce_buffer_bytes(n_max, 1), dtype=torch.uint8, device=DEV)
    peers = torch.tensor([buf.data_ptr()], dtype=torch.int64, device=DEV)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    ws = torch.zeros(sq.w4a16_gemm_workspace_bytes(M, N, K), dtype=torch.uint8, device=DEV)
    g = torch.Generator(device=DEV).manual_seed(11)
    calls = 12
    Xs = [torch.randn(M, K, generator=g, device=DEV).to(dtype) for _ in range(calls)]
    outs = [torch.empty(M, N, dtype=dtype, device=DEV) for _ in range(calls)]
    plain = [None] * calls
    old = sq.get_option(sq.SQ_OPT_PDL)
    sq.set_option(sq.SQ_OPT_PDL, 1)
    try:
        torch.cuda.synchronize()
        for c in range(calls):
            sq.w4a16_gemm_allreduce(Xs[c], q, peers, 0, 1, n_max, err, out=outs[c], workspace=ws)
            if c % 3 == 1:  # a plain decode GEMM between two fused calls, same workspace
                plain[c] = sq.w4a16_gemm(Xs[c][:, :1024].contiguous(), qp, workspace=ws)
        torch.cuda.synchronize()
    finally:
        sq.set_option(sq.SQ_OPT_PDL, old)
    assert int(err.item()) == 0
    assert int(buf[:4].view(torch.int32).item()) == calls   # one epoch per call
    for c in range(calls):
        ref = sq.w4a16_gemm_allreduce(Xs[c], q, peers, 0, 1, n_max, err, workspace=ws)
        torch.cuda.synchronize()
        assert torch.equal(outs[c].view(torch.int16), ref.view(torch.int16)), c
        if plain[c] is not None:
            assert torch.equal(plain[c], sq.w4a16_gemm(Xs[c][:, :1024].contiguous(), qp)), c
    assert int(err.item()) == 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        import oracle
        from paper_2312_03788_b200 import peer, synth, tp

        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        ar = peer.PeerAllReduce(1 << 20, DEV)
        ok = []
        g = torch.Generator(device="cpu").manual_seed(1)
        for it in range(4):
            parts = [torch.randn(5000 + 8 * it, generator=g).half() for _ in range(world)]
            y = parts[rank].to(DEV)
            ar(y)
            torch.cuda.synchronize()
            ok.append(torch.equal(y.cpu().view(torch.int16), _expected(parts).view(torch.int16)))
        # captured in a CUDA graph: the device-managed epoch advances on every replay
        yg = torch.zeros(4096, dtype=torch.float16, device=DEV)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            ar(yg)  # warm-up on a side stream before capture
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            ar(yg)
        for it in range(3):
            parts = [torch.randn(4096, generator=g).half() for _ in range(world)]
            yg.copy_(parts[rank].to(DEV))
            torch.cuda.synchronize()
            dist.barrier()
            graph.replay()
            torch.cuda.synchronize()
            ok.append(torch.equal(yg.cpu().view(torch.int16), _expected(parts).view(torch.int16)))
        # row-parallel layer of the TP stack reduced through the peer buffers
        model = tp.ModelShape("tiny-34b-like", hidden=1024, mlp=2816, layers=1, q_heads=8, kv_heads=2,
                              head_dim=128)
        for i, (name, K, N) in enumerate(tp.full_shapes(model)):
            sh = tp.layer_shards(model, rank, world)[i]
            if sh.kind != "row":
                continue
            W = synth.weights(N, K, seed=20 + i)
            X = synth.activations(4, K, seed=30 + i).astype(np.float16)
            k0, k1 = sh.k_range
            qsh = sq.quantize_pack_groupwise(torch.from_numpy(np.ascontiguousarray(W[:, k0:k1])).to(DEV))
            y = sq.w4a16_gemm(torch.from_numpy(np.ascontiguousarray(X[:, k0:k1])).to(DEV), qsh)
            ar(y)
            full = oracle.quantize_pack(W, None)
            y_ref = oracle.gemm(X, full["Wq"], full["scales"], full["zeros"])
            err = np.linalg.norm(y.float().cpu().double().numpy() - y_ref) / np.linalg.norm(y_ref)
            ok.append(bool(err <= 2e-3))
        # the fused row-parallel linear (one kernel at decode sizes) on the same buffers
        for i, (name, K, N) in enumerate(tp.full_shapes(model)):
            sh = tp.layer_shards(model, rank, world)[i]
            if sh.kind != "row":
                continue
            W = synth.weights(N, K, seed=20 + i)
            k0, k1 = sh.k_range
            qsh = sq.quantize_pack_groupwise(torch.from_numpy(np.ascontiguousarray(W[:, k0:k1])).to(DEV))
            full = oracle.quantize_pack(W, None)
            for M in (1, 16, 40):  # 40: prefill GEMM + exchange kernel
                X = synth.activations(M, K, seed=50 + i + M).astype(np.float16)
                y = ar.gemm(torch.from_numpy(np.ascontiguousarray(X[:, k0:k1])).to(DEV), qsh)
                torch.cuda.synchronize()
                y_ref = oracle.gemm(X, full["Wq"], full["scales"], full["zeros"])
                err = np.linalg.norm(y.float().cpu().double().numpy() - y_ref) / np.linalg.norm(y_ref)
                ok.append(bool(err <= 2e-3))
        ok.append(not ar.failed())
        ar.close()
        q.put((rank, all(ok)))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_peer_allreduce_two_processes_ipc():
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
