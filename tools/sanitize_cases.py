"""Small launches of every hot-path kernel for compute-sanitizer (SURVEY.md §4 layer 3, §5):

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_cases.py

C1 (BASELINE.json configs[0]: K = N = 512, M = 1) end to end, plus one ragged / tail shape per
kernel: decode at M = 1 and 16 under both schedules (stream-K fixups, row blocks), prefill with
stream-K and a ragged token tile, quantize with edge groups, the packed u4 zero-point layout
(SQ_ZEROS_U4: quantizer, decode at M = 1 / 16, prefill, g = 128 and 32), the one-shot all-reduce
and the fused GEMM + all-reduce (one rank).  Results are checked against
the plain relations (no oracle needed here; the parity tests do that), so a sanitizer run also
fails loudly on wrong output.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03788_b200 import sq, synth, tp  # noqa: E402

DEV = "cuda"


def main():
    torch.manual_seed(0)
    # C1 pipeline
    W = torch.from_numpy(synth.weights(512, 512, seed=0)).to(DEV)
    Xc = torch.from_numpy(synth.activations(164 * 16, 512, seed=1).astype(np.float16)).to(DEV)
    am = sq.act_absmax(Xc)
    s = sq.smooth_scales(W, am, 0.5)
    q = sq.quantize_pack_groupwise(W, s)
    x = sq.smooth_activations(torch.randn(1, 512, device=DEV).half(), s)
    y = sq.w4a16_gemm(x, q)
    sq.sq_diff_sum(y, torch.zeros_like(y))
    # quantize edge groups (constant, one-sided, ties, extremes, subnormal)
    E = synth.edge_groups(128, seed=5)
    pad = (-E.shape[0]) % 8
    We = np.concatenate([E, synth.weights(pad, 128, seed=6)]).astype(np.float16)
    nf = torch.zeros(1, dtype=torch.int32, device=DEV)
    sq.quantize_pack_groupwise(torch.from_numpy(We).to(DEV), nonfinite=nf)
    # decode: ragged row block (N = 264), ragged stage (K = 1152 = 9 groups), both schedules
    Wd = torch.from_numpy(synth.weights(264, 1152, seed=7)).to(DEV)
    qd = sq.quantize_pack_groupwise(Wd)
    for sched in (sq.SQ_SCHED_STREAMK, sq.SQ_SCHED_ROWBLOCK, sq.SQ_SCHED_AUTO):
        sq.set_option(sq.SQ_OPT_DECODE_SCHEDULE, sched)
        for M in (1, 16):
            xd = torch.randn(M, 1152, device=DEV).half()
            a = sq.w4a16_gemm(xd, qd, path=sq.SQ_PATH_DECODE)
            b = sq.w4a16_gemm(xd, qd, path=sq.SQ_PATH_PREFILL)
            torch.cuda.synchronize()
            assert ((a.float() - b.float()).abs() <= 5e-3 * b.float().abs() + 5e-3).all(), (sched, M)
    sq.set_option(sq.SQ_OPT_DECODE_SCHEDULE, sq.SQ_SCHED_AUTO)
    # decode stream-K with many units per CTA (fixups) and bf16
    Wk = torch.from_numpy(synth.weights(2048, 4096, seed=8)).to(DEV)
    qk = sq.quantize_pack_groupwise(Wk)
    for dt in (torch.float16, torch.bfloat16):
        sq.w4a16_gemm(torch.randn(5, 4096, device=DEV).to(dt), qk)
    # prefill: stream-K over (tile x group) units and a ragged token tile
    Wp = torch.from_numpy(synth.weights(1024, 2048, seed=9)).to(DEV)
    qp = sq.quantize_pack_groupwise(Wp)
    for M in (17, 300):
        sq.w4a16_gemm(torch.randn(M, 2048, device=DEV).half(), qp, path=sq.SQ_PATH_PREFILL)
    # packed u4 zero points (N3): quantizer output, decode (both schedules' tails: N = 288 is a
    # ragged 64-row block) and prefill, g = 128 and 32; results equal the fp16-Z GEMM bit for bit
    Wu = torch.from_numpy(synth.weights(288, 1152, seed=11)).to(DEV)
    for g in (128, 32):
        qz = sq.quantize_pack_groupwise(Wu, group=g, zeros_u4=True)
        qf = sq.quantize_pack_groupwise(Wu, group=g)
        for M, path in ((1, sq.SQ_PATH_DECODE), (16, sq.SQ_PATH_DECODE), (40, sq.SQ_PATH_PREFILL)):
            xu = torch.randn(M, 1152, device=DEV).half()
            a = sq.w4a16_gemm(xu, qz, path=path)
            b = sq.w4a16_gemm(xu, qf, path=path)
            torch.cuda.synchronize()
            assert torch.equal(a, b), (g, M)
    # one-shot all-reduce and fused GEMM + all-reduce.  One rank (the sanitizer may serialize
    # concurrent kernels, and two simulated ranks must be co-resident); push, flag, wait and
    # reduce all run with world = 1 too.
    world, M, N, K = 1, 4, 1024, 1024
    ranges = tp.channel_split(K, world)
    Wa = torch.from_numpy(synth.weights(N, K, seed=10)).to(DEV)
    qs = [sq.quantize_pack_groupwise(Wa[:, a:b].contiguous()) for a, b in ranges]
    n_max = M * N
    nb = sq.allreduce_buffer_bytes(n_max, world)
    bufs = [torch.zeros(nb, dtype=torch.uint8, device=DEV) for _ in range(world)]
    peers = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=DEV)
    errs = [torch.zeros(1, dtype=torch.int32, device=DEV) for _ in range(world)]
    streams = [torch.cuda.Stream() for _ in range(world)]
    wss = [torch.zeros(sq.w4a16_gemm_workspace_bytes(M, N, K), dtype=torch.uint8, device=DEV) for _ in range(world)]
    X = torch.randn(M, K, device=DEV).half()
    torch.cuda.synchronize()
    for r in range(world):
        with torch.cuda.stream(streams[r]):
            a, b = ranges[r]
            sq.w4a16_gemm_allreduce(X[:, a:b].contiguous(), qs[r], peers, r, world, n_max, errs[r],
                                    workspace=wss[r], stream=streams[r])
    torch.cuda.synchronize()
    parts = [torch.randn(n_max, device=DEV).half() for _ in range(world)]
    for r in range(world):
        with torch.cuda.stream(streams[r]):
            sq.allreduce_oneshot(parts[r], peers, r, world, 0, n_max, errs[r], out=torch.empty_like(parts[r]),
                                 stream=streams[r])
    torch.cuda.synchronize()
    assert all(int(e.item()) == 0 for e in errs)
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
