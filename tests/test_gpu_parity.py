"""GPU parity: the CUDA path (through the C ABI) against the fp64 CPU oracle on the
same seeded inputs.

  * act_absmax, smooth_scales (α in {0, 0.5, 1}), quantize/pack: BIT-EXACT.
  * smooth_scales for general α: <= 1 ulp fp32 (reading S12: pow is not correctly
    rounded on either side).
  * GEMM: relative Frobenius error <= 5e-3 (BASELINE.json north_star), fp32
    accumulate; the expected error from rounding Ŵ/Y is ~3e-4 (fp16) / ~2.4e-3
    (bf16), so the test also checks a tighter dtype-specific bound.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_2312_03788_b200 import sq, synth

pytestmark = pytest.mark.gpu

DEV = "cuda"
TOL_FROB = 5e-3
TIGHT = {torch.float16: 1e-3, torch.bfloat16: 4e-3}


def _t(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(DEV)


def _bits16(t: torch.Tensor) -> np.ndarray:
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


def _rel_frob(y_gpu: torch.Tensor, y_ref: np.ndarray) -> float:
    y = y_gpu.float().cpu().double().numpy()
    return float(np.linalg.norm(y - y_ref) / max(np.linalg.norm(y_ref), 1e-300))


def _x_np_for(x: torch.Tensor):
    """Host copy of a device activation tensor in the oracle's input format."""
    if x.dtype == torch.float16:
        return x.cpu().numpy(), "f16"
    return x.cpu().view(torch.int16).numpy().view(np.uint16), "bf16"


# ------------------------------------------------------------------ a1/a2
@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_act_absmax_bitexact(dtype):
    Xc = synth.activations(333, 1024, seed=1)
    x = _t(Xc, dtype)
    got = sq.act_absmax(x).cpu().numpy()
    xn, xd = _x_np_for(x)
    ref = oracle.act_absmax(xn, xd)
    assert (got.view(np.uint32) == ref.view(np.uint32)).all()
    # running max over two batches
    x2 = _t(synth.activations(17, 1024, seed=2), dtype)
    got2 = sq.act_absmax(x2, out=sq.act_absmax(x), accumulate=True).cpu().numpy()
    xn2, _ = _x_np_for(x2)
    ref2 = np.maximum(ref, oracle.act_absmax(xn2, xd))
    assert (got2 == ref2).all()


@pytest.mark.parametrize("alpha", [0.5, 0.0, 1.0, 0.35, 0.85])
@pytest.mark.parametrize("N,K", [(256, 512), (1000, 1536), (24, 128)])
def test_smooth_scales(alpha, N, K):
    W = synth.weights(N, K, seed=N + K, heavy=True)
    W[:, 5] = 0  # a dead weight channel -> ε floor
    am = oracle.act_absmax(synth.activations(512, K, seed=K).astype(np.float16))
    am[7] = 0.0  # dead activation channel
    s_gpu = sq.smooth_scales(_t(W), _t(am), alpha).cpu().numpy()
    s_ref = oracle.smooth_scales(oracle.weight_absmax(W), am, alpha)
    if alpha in (0.0, 0.5, 1.0):
        assert (s_gpu.view(np.uint32) == s_ref.view(np.uint32)).all()
    else:
        ulp = np.abs(s_gpu.view(np.int32).astype(np.int64) - s_ref.view(np.int32).astype(np.int64))
        assert ulp.max() <= 1


# ------------------------------------------------------------------ a3/a4
def _check_quant(W_np, s_np, q: sq.QuantizedLinear, w_dtype="f16", nonfinite=None):
    ref = oracle.quantize_pack(W_np, s_np, 128, w_dtype)
    assert (q.Wq.cpu().numpy() == ref["Wq"]).all()
    assert (_bits16(q.scales) == ref["scales"]).all()
    assert (_bits16(q.zeros) == ref["zeros"]).all()
    if nonfinite is not None:
        assert int(nonfinite.item()) == ref["nonfinite"]


@pytest.mark.parametrize("smooth", [False, True])
@pytest.mark.parametrize("N,K", [(512, 512), (24, 1024), (264, 384), (4096, 128)])
def test_quantize_bitexact(N, K, smooth):
    W = synth.weights(N, K, seed=3 * N + K, heavy=True)
    s = None
    if smooth:  # both sides consume the oracle's s (s-parity is tested on its own)
        am = oracle.act_absmax(synth.activations(1024, K, seed=K).astype(np.float16))
        s = oracle.smooth_scales(oracle.weight_absmax(W), am, 0.5)
    nf = torch.zeros(1, dtype=torch.int32, device=DEV)
    q = sq.quantize_pack_groupwise(_t(W), None if s is None else _t(s), nonfinite=nf)
    _check_quant(W, s, q, nonfinite=nf)


def test_quantize_edge_groups_bitexact():
    E = synth.edge_groups(128, seed=5)                      # [R][128]
    R = E.shape[0]
    pad = (-R) % 8
    W = np.concatenate([E, synth.weights(pad, 128, seed=6)]).astype(np.float16)
    W = np.concatenate([W, W[:, ::-1]], axis=1)            # two groups per row
    nf = torch.zeros(1, dtype=torch.int32, device=DEV)
    q = sq.quantize_pack_groupwise(_t(W), None, nonfinite=nf)
    _check_quant(W, None, q, nonfinite=nf)
    # the same rows folded with wild (but finite) smoothing factors
    s = np.float32(np.exp(synth.rng(7).uniform(-8, 8, size=256))).astype(np.float32)
    nf.zero_()
    q2 = sq.quantize_pack_groupwise(_t(W), _t(s), nonfinite=nf)
    _check_quant(W, s, q2, nonfinite=nf)


def test_quantize_nonfinite_groups():
    bad = synth.nonfinite_groups(128)
    W = np.concatenate([bad, synth.weights(5, 128, seed=8)]).astype(np.float16)
    nf = torch.zeros(1, dtype=torch.int32, device=DEV)
    q = sq.quantize_pack_groupwise(_t(W), None, nonfinite=nf)
    _check_quant(W, None, q, nonfinite=nf)
    assert int(nf.item()) == 3


def test_quantize_bf16_weights_bitexact():
    Wf = synth.weights(256, 512, seed=9, heavy=True).astype(np.float32)
    Wb = torch.from_numpy(Wf).to(torch.bfloat16)
    Wbits = Wb.view(torch.int16).numpy().view(np.uint16)
    s = np.float32(np.exp(synth.rng(10).uniform(-3, 3, size=512))).astype(np.float32)
    nf = torch.zeros(1, dtype=torch.int32, device=DEV)
    q = sq.quantize_pack_groupwise(Wb.to(DEV), _t(s), nonfinite=nf)
    _check_quant(Wbits, s, q, w_dtype="bf16", nonfinite=nf)


# ------------------------------------------------------------------ a6/a7 GEMM
def _gemm_case(M, N, K, dtype, path, seed=0, smooth=True):
    W = synth.weights(N, K, seed=seed + 100, heavy=True)
    s = None
    if smooth:
        am = oracle.act_absmax(synth.activations(2048, K, seed=seed + 200).astype(np.float16))
        s = oracle.smooth_scales(oracle.weight_absmax(W), am, 0.5)
    ref_q = oracle.quantize_pack(W, s, 128)
    q = sq.quantize_pack_groupwise(_t(W), None if s is None else _t(s))
    X = synth.activations(M, K, seed=seed + 300, outlier_seed=seed + 200)
    if s is not None:  # a5: X̂ = X diag(s)^-1, rounded once to the activation dtype
        X = X.astype(np.float64) / s.astype(np.float64)[None, :]
    x = torch.from_numpy(np.ascontiguousarray(X)).to(dtype).to(DEV)
    ws = None
    nbytes = sq.w4a16_gemm_workspace_bytes(M, N, K)
    if nbytes:
        ws = torch.zeros(nbytes, dtype=torch.uint8, device=DEV)
    y = sq.w4a16_gemm(x, q, workspace=ws, path=path)
    torch.cuda.synchronize()
    xn, xd = _x_np_for(x)
    y_ref = oracle.gemm(xn, ref_q["Wq"], ref_q["scales"], ref_q["zeros"], 128, xd)
    return y, y_ref


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("M", [1, 2, 3, 4, 7, 8, 9, 13, 16])
@pytest.mark.parametrize("N,K", [(512, 512), (264, 1152), (2048, 4096)])
def test_gemm_decode_parity(M, N, K, dtype):
    y, y_ref = _gemm_case(M, N, K, dtype, sq.SQ_PATH_DECODE, seed=M)
    err = _rel_frob(y, y_ref)
    assert err <= TOL_FROB and err <= TIGHT[dtype], err


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("M", [17, 64, 256, 300, 520])
@pytest.mark.parametrize("N,K", [(256, 512), (392, 1152), (1024, 2048)])
def test_gemm_prefill_parity(M, N, K, dtype):
    y, y_ref = _gemm_case(M, N, K, dtype, sq.SQ_PATH_PREFILL, seed=M)
    err = _rel_frob(y, y_ref)
    assert err <= TOL_FROB and err <= TIGHT[dtype], err


@pytest.mark.parametrize("M", [1, 16, 32])
def test_gemm_prefill_small_m(M):
    """The prefill path is legal for any M (the M sweep maps both paths)."""
    y, y_ref = _gemm_case(M, 384, 1024, torch.float16, sq.SQ_PATH_PREFILL, seed=7)
    assert _rel_frob(y, y_ref) <= TIGHT[torch.float16]


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("path,M", [(sq.SQ_PATH_DECODE, 16), (sq.SQ_PATH_PREFILL, 256)])
def test_p13_one_hot_rows_bitwise(path, M, dtype):
    """P13: a one-hot X row picks out one Ŵ column exactly: Y = RN_dtype((q-Z)Δ)."""
    N, K = 256, 512
    W = synth.weights(N, K, seed=11, heavy=True)
    q = sq.quantize_pack_groupwise(_t(W))
    ref = oracle.quantize_pack(W, None)
    What = oracle.dequant(ref["Wq"], ref["scales"], ref["zeros"])
    ks = synth.rng(12).integers(0, K, size=M)
    X = np.zeros((M, K), np.float32)
    X[np.arange(M), ks] = 1.0
    x = torch.from_numpy(X).to(dtype).to(DEV)
    y = sq.w4a16_gemm(x, q, path=path)
    exp = torch.from_numpy(What[:, ks].T.copy()).to(dtype)   # one rounding of the exact value
    assert torch.equal(y.cpu(), exp)


@pytest.mark.parametrize("path,M", [(sq.SQ_PATH_DECODE, 5), (sq.SQ_PATH_PREFILL, 40)])
def test_p13_zero_input(path, M):
    q = sq.quantize_pack_groupwise(_t(synth.weights(128, 256, seed=13)))
    x = torch.zeros((M, 256), dtype=torch.float16, device=DEV)
    y = sq.w4a16_gemm(x, q, path=path)
    assert (y == 0).all()


def test_gemm_auto_threshold():
    """SQ_PATH_AUTO: M <= M_dec runs decode, larger M prefill -- both correct."""
    assert sq.decode_max_m() == 16
    for M in (16, 17):
        y, y_ref = _gemm_case(M, 256, 512, torch.float16, sq.SQ_PATH_AUTO, seed=M)
        assert _rel_frob(y, y_ref) <= TIGHT[torch.float16]


def test_gemm_m_zero_noop():
    q = sq.quantize_pack_groupwise(_t(synth.weights(128, 256, seed=13)))
    x = torch.zeros((0, 256), dtype=torch.float16, device=DEV)
    y = sq.w4a16_gemm(x, q)
    assert y.shape == (0, 128)


@pytest.mark.parametrize("pdl,static", [(0, 0), (1, 0), (1, 1)])
@pytest.mark.parametrize("M", [1, 16])
def test_gemm_chain_launch_options(pdl, static, M):
    """A dependent chain y_{i+1} = y_i · Ŵ_i^T (each GEMM reads the previous one's
    output) under programmatic dependent launch and early weight streaming: the
    kernels must still wait for their inputs (include/libsq.h SQ_OPT_*)."""
    D = 512
    Ws = [synth.weights(D, D, seed=300 + i) for i in range(4)]
    refs = [oracle.quantize_pack(W, None) for W in Ws]
    qs = [sq.quantize_pack_groupwise(_t(W)) for W in Ws]
    torch.cuda.synchronize()  # weights static before the chain (SQ_OPT_WEIGHTS_STATIC contract)
    X = (synth.activations(M, D, seed=9) * 0.05).astype(np.float16)
    old = (sq.get_option(sq.SQ_OPT_PDL), sq.get_option(sq.SQ_OPT_WEIGHTS_STATIC))
    try:
        sq.set_option(sq.SQ_OPT_PDL, pdl)
        sq.set_option(sq.SQ_OPT_WEIGHTS_STATIC, static)
        y = torch.from_numpy(X).to(DEV)
        for _ in range(3):
            for q in qs:
                y = sq.w4a16_gemm(y, q, path=sq.SQ_PATH_DECODE)
        torch.cuda.synchronize()
    finally:
        sq.set_option(sq.SQ_OPT_PDL, old[0])
        sq.set_option(sq.SQ_OPT_WEIGHTS_STATIC, old[1])
    yr = X.copy()
    for _ in range(3):
        for r in refs:
            yr = oracle.gemm(yr, r["Wq"], r["scales"], r["zeros"]).astype(np.float16)
    yr = yr.astype(np.float64)
    assert _rel_frob(y, yr) <= 1e-2


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("M,N,K", [(64, 2048, 4096), (300, 1024, 4096), (520, 8192, 512), (17, 4096, 2048),
                                   (128, 2816, 1024)])
def test_gemm_prefill_streamk(M, N, K, dtype):
    """Prefill shapes whose tiles leave the last wave mostly idle, so the (tile x group)
    units are split between CTAs (stream-K) and finished by the fixup: ragged token
    tiles, whole tiles in the middle of a CTA's range, several CTAs per tile.  Bit-identical
    on every launch (fixed summation order)."""
    y, y_ref = _gemm_case(M, N, K, dtype, sq.SQ_PATH_PREFILL, seed=M + N)
    err = _rel_frob(y, y_ref)
    assert err <= TOL_FROB and err <= TIGHT[dtype], err
    x = torch.randn(M, K, device=DEV).to(dtype)
    q = sq.quantize_pack_groupwise(torch.randn(N, K, device=DEV).half() * 0.02)
    ys = [sq.w4a16_gemm(x, q, path=sq.SQ_PATH_PREFILL) for _ in range(3)]
    torch.cuda.synchronize()
    assert all(torch.equal(ys[0], yy) for yy in ys[1:])


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("M", [1, 3, 8, 9, 16])
@pytest.mark.parametrize("N,K", [(512, 512), (264, 1152), (2048, 4096), (8192, 8192)])
def test_gemm_decode_tcgen05_parity(M, N, K, dtype):
    """The tcgen05 decode kernel (SQ_OPT_DECODE_KERNEL = SQ_DECK_TCGEN05): ragged row
    blocks (N = 264), ragged 4-group stages (K = 1152 = 9 groups), stream-K fixups and a
    wrapping stage ring (8192 x 8192), against the oracle; deterministic."""
    sq.set_option(sq.SQ_OPT_DECODE_KERNEL, sq.SQ_DECK_TCGEN05)
    try:
        y, y_ref = _gemm_case(M, N, K, dtype, sq.SQ_PATH_DECODE, seed=M + 7, smooth=N <= 2048)
        err = _rel_frob(y, y_ref)
        assert err <= TOL_FROB and err <= TIGHT[dtype], err
        if N == 8192:
            x = torch.randn(M, K, device=DEV).to(dtype)
            q = sq.quantize_pack_groupwise(torch.randn(N, K, device=DEV).half() * 0.02)
            ys = [sq.w4a16_gemm(x, q, path=sq.SQ_PATH_DECODE) for _ in range(3)]
            torch.cuda.synchronize()
            assert all(torch.equal(ys[0], yy) for yy in ys[1:])
    finally:
        sq.set_option(sq.SQ_OPT_DECODE_KERNEL, sq.SQ_DECK_MMA_SYNC)


@pytest.mark.parametrize("sched", ["streamk", "rowblock"])
def test_gemm_decode_schedules_shared_workspace(sched):
    """Both decode schedules (SQ_OPT_DECODE_SCHEDULE) against the oracle, on one shared
    default workspace: a small-N GEMM first, then shapes whose CTAs wrap the stage ring
    after a row-block segment end (8192 x 8192: 7 stream-K units per CTA > 4 stages),
    then the small one again; every result deterministic across launches."""
    code = {"streamk": sq.SQ_SCHED_STREAMK, "rowblock": sq.SQ_SCHED_ROWBLOCK}[sched]
    sq.set_option(sq.SQ_OPT_DECODE_SCHEDULE, code)
    try:
        for i, (N, K) in enumerate([(1024, 1024), (8192, 8192), (1536, 2048), (1024, 1024)]):
            W = synth.weights(N, K, seed=90 + i)
            ref = oracle.quantize_pack(W, None)
            q = sq.quantize_pack_groupwise(_t(W))
            for M in (1, 16):
                X = synth.activations(M, K, seed=95 + i).astype(np.float16)
                x = torch.from_numpy(X).to(DEV)
                y_ref = oracle.gemm(X, ref["Wq"], ref["scales"], ref["zeros"], 128, "f16")
                ys = [sq.w4a16_gemm(x, q, path=sq.SQ_PATH_DECODE) for _ in range(2)]
                torch.cuda.synchronize()
                assert _rel_frob(ys[0], y_ref) <= TIGHT[torch.float16], (N, K, M)
                assert torch.equal(ys[0], ys[1]), (N, K, M)
    finally:
        sq.set_option(sq.SQ_OPT_DECODE_SCHEDULE, sq.SQ_SCHED_AUTO)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("M", [1, 5, 16])
def test_gemm_decode_streamk_fixup(M, dtype):
    """A shape with several stream-K units per CTA, so row blocks are split between
    CTAs and finished by the fixup; repeated launches check that the workspace
    counters are left reset and that the result is bit-identical (deterministic)."""
    N, K = 8192, 4096
    W = synth.weights(N, K, seed=77)
    ref = oracle.quantize_pack(W, None)
    q = sq.quantize_pack_groupwise(_t(W))
    X = synth.activations(M, K, seed=78).astype(np.float16)
    x = torch.from_numpy(X).to(dtype).to(DEV)
    xn, xd = _x_np_for(x)
    y_ref = oracle.gemm(xn, ref["Wq"], ref["scales"], ref["zeros"], 128, xd)
    ys = [sq.w4a16_gemm(x, q, path=sq.SQ_PATH_DECODE) for _ in range(3)]
    torch.cuda.synchronize()
    for y in ys:
        assert _rel_frob(y, y_ref) <= TIGHT[dtype]
    # deterministic: identical bits on every launch
    assert all(torch.equal(ys[0], y) for y in ys[1:])
