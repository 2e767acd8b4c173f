"""GPU parity: the CUDA path (through the C ABI) against the fp64 CPU oracle on the
same seeded inputs.

  * act_absmax, smooth_scales (α in {0, 0.5, 1}), quantize/pack: BIT-EXACT.
  * smooth_scales for general α: <= 1 ulp fp32 (reading S12: pow is not correctly
    rounded on either side).
  * GEMM: relative Frobenius error <= 5e-3 (BASELINE.json north_star), fp32
    accumulate; the expected error from rounding Ŵ/Y is ~3e-4 (fp16) / ~2.4e-3
    (bf16), so the test also checks a tighter dtype-specific bound, AND every output
    element against the floating-point bound of tests/gemm_bounds.py (a wrong row block
    or tail tile cannot hide under the norm).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_2312_03788_b200 import sq, synth
from tests.gemm_bounds import elementwise_ratio

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
def _check_quant(W_np, s_np, q: sq.QuantizedLinear, w_dtype="f16", nonfinite=None, group=128):
    ref = oracle.quantize_pack(W_np, s_np, group, w_dtype)
    assert (q.Wq.cpu().numpy() == ref["Wq"]).all()
    assert (_bits16(q.scales) == ref["scales"]).all()
    if q.zeros_u4:
        assert (q.zeros.cpu().numpy() == oracle.pack_zeros_u4(ref["zeros"])).all()
    else:
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


def test_quantize_fold_ties_and_signs_bitexact():
    """Eq. 5 fold RN(W * s) (reading S13) on products that land exactly on fp16 midpoints or
    one fp32 ulp beside them, through both kernel paths in one launch: CTAs whose 512-k slice
    of s has only clear sign bits take the |w|-based fold, the others (a negative s, -0.0)
    the signed one."""
    N, K = 64, 4096
    W = synth.weights(N, K, seed=21, heavy=True)
    r = synth.rng(22)
    base = np.array([1 + 2.0 ** -11, 1 - 2.0 ** -12, 1 + 3 * 2.0 ** -12, 0.75 * (1 + 2.0 ** -10),
                     1 + 2.0 ** -11 + 2.0 ** -23, 1 + 2.0 ** -11 - 2.0 ** -23, 2.0 ** -14, 3.0],
                    dtype=np.float64)
    sv = base[r.integers(0, len(base), size=K)] * np.exp2(r.integers(-3, 4, size=K))
    sv[K // 2:] *= np.where(r.random(K - K // 2) < 0.1, -1.0, 1.0)   # second half: some negative
    sv[3 * K // 4 + 5] = -0.0
    s = sv.astype(np.float32)
    nf = torch.zeros(1, dtype=torch.int32, device=DEV)
    q = sq.quantize_pack_groupwise(_t(W), _t(s), nonfinite=nf)
    _check_quant(W, s, q, nonfinite=nf)


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



def test_quantize_bf16_ties_and_near_ties_bitexact():
    """Eq. 1 codes RHA(v / Δ) (reading S2) for bf16 weights at exact ties and one bf16 ulp
    beside them: groups with lo = 0, hi = 15/16 (Δ = 1/16, Z = 0), their negatives
    (Z = 15), scaled by powers of two, and random bf16 groups; RTN and an exact
    power-of-two fold."""
    r = synth.rng(31)
    rows = []
    for e in range(-12, 13, 3):
        for sign in (1.0, -1.0):
            base = np.concatenate([[0.0, 15 / 16], (np.arange(15) + 0.5) / 16, np.arange(16) / 16])
            g = np.resize(base, 128)
            near = (np.arange(15) + 0.5) / 16 * (1 + 2.0 ** -7)    # one bf16 ulp above a tie
            g[40:55] = near
            g[60:75] = (np.arange(15) + 0.5) / 16 * (1 - 2.0 ** -8)  # one ulp below
            rows.append(sign * g * 2.0 ** e)
    rows.append(r.normal(0, 1, size=128) * 2.0 ** -20)
    rows.append(r.normal(0, 1, size=128) * 1e3)
    W = np.stack(rows)
    W = np.concatenate([W, W[:, ::-1]], axis=1)                   # [R][256]
    pad = (-W.shape[0]) % 8
    W = np.concatenate([W, np.resize(W[:1], (pad, W.shape[1]))]).astype(np.float32)
    Wb = torch.from_numpy(W).to(torch.bfloat16)
    Wbits = Wb.view(torch.int16).numpy().view(np.uint16)
    for s in (None, np.float32(2.0) ** synth.rng(32).integers(-3, 4, size=256).astype(np.float32)):
        nf = torch.zeros(1, dtype=torch.int32, device=DEV)
        q = sq.quantize_pack_groupwise(Wb.to(DEV), None if s is None else _t(s), nonfinite=nf)
        _check_quant(Wbits, s, q, w_dtype="bf16", nonfinite=nf)

# ------------------------------------------------------------------ a6/a7 GEMM
class GemmCase:
    """GPU output and the oracle's exact result of one GEMM, plus what the element-wise
    bound needs (the activations as fed, the exact dequantized weights)."""

    def __init__(self, y, y_ref, x64, W_hat, xd):
        self.y, self.y_ref, self.x64, self.W_hat, self.xd = y, y_ref, x64, W_hat, xd

    def check(self, dtype, frob=None):
        err = _rel_frob(self.y, self.y_ref)
        assert err <= TOL_FROB and err <= (TIGHT[dtype] if frob is None else frob), err
        ratio = elementwise_ratio(self.y.float().cpu().double().numpy(), self.y_ref, self.x64, self.W_hat,
                                  self.xd)
        assert ratio <= 1.0, ratio
        return err


def _gemm_case(M, N, K, dtype, path, seed=0, smooth=True, W=None, x_scale=1.0, group=128, zeros_u4=False):
    if W is None:
        W = synth.weights(N, K, seed=seed + 100, heavy=True)
    s = None
    if smooth:
        am = oracle.act_absmax(synth.activations(2048, K, seed=seed + 200).astype(np.float16))
        s = oracle.smooth_scales(oracle.weight_absmax(W), am, 0.5)
    ref_q = oracle.quantize_pack(W, s, group)
    q = sq.quantize_pack_groupwise(_t(W), None if s is None else _t(s), group=group, zeros_u4=zeros_u4)
    X = synth.activations(M, K, seed=seed + 300, outlier_seed=seed + 200) * x_scale
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
    zref = oracle.pack_zeros_u4(ref_q["zeros"]) if zeros_u4 else ref_q["zeros"]
    y_ref = oracle.gemm(xn, ref_q["Wq"], ref_q["scales"], zref, group, xd, zeros_u4=zeros_u4)
    W_hat = oracle.dequant(ref_q["Wq"], ref_q["scales"], zref, group, zeros_u4=zeros_u4)
    x64 = x.float().cpu().double().numpy()
    c = GemmCase(y, y_ref, x64, W_hat, xd)
    c.q, c.x, c.ws = q, x, ws
    return c


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("M", [1, 2, 3, 4, 7, 8, 9, 13, 16])
@pytest.mark.parametrize("N,K", [(512, 512), (264, 1152), (2048, 4096)])
def test_gemm_decode_parity(M, N, K, dtype):
    _gemm_case(M, N, K, dtype, sq.SQ_PATH_DECODE, seed=M).check(dtype)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("M", [17, 64, 65, 100, 128, 129, 256, 300, 520])
@pytest.mark.parametrize("N,K", [(256, 512), (392, 1152), (1024, 2048)])
def test_gemm_prefill_parity(M, N, K, dtype):
    _gemm_case(M, N, K, dtype, sq.SQ_PATH_PREFILL, seed=M).check(dtype)


@pytest.mark.parametrize("M", [1, 16, 32])
def test_gemm_prefill_small_m(M):
    """The prefill path is legal for any M (the M sweep maps both paths)."""
    _gemm_case(M, 384, 1024, torch.float16, sq.SQ_PATH_PREFILL, seed=7).check(torch.float16)


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
        _gemm_case(M, 256, 512, torch.float16, sq.SQ_PATH_AUTO, seed=M).check(torch.float16)


def test_gemm_m_zero_noop():
    q = sq.quantize_pack_groupwise(_t(synth.weights(128, 256, seed=13)))
    x = torch.zeros((0, 256), dtype=torch.float16, device=DEV)
    y = sq.w4a16_gemm(x, q)
    assert y.shape == (0, 128)


@pytest.mark.parametrize("pdl,static", [(0, 0), (1, 0), (1, 1)])
@pytest.mark.parametrize("M", [1, 16, 40])
def test_gemm_chain_launch_options(pdl, static, M):
    """A dependent chain y_{i+1} = y_i · Ŵ_i^T (each GEMM reads the previous one's output,
    no host sync in between) under programmatic dependent launch and early weight
    streaming (SQ_GEMM_WEIGHTS_STATIC on the handle): every kernel must still wait for its
    input.  Each link is checked against the oracle applied to the GPU's own input of that
    link, so a GEMM that read a stale X cannot pass; all links obey the 5e-3 contract and
    the element-wise bound."""
    D = 512
    Ws = [synth.weights(D, D, seed=300 + i) for i in range(4)]
    refs = [oracle.quantize_pack(W, None) for W in Ws]
    qs = [sq.quantize_pack_groupwise(_t(W)) for W in Ws]
    torch.cuda.synchronize()  # the quantize kernels finished: the weights are static now
    for q in qs:
        q.mark_static(bool(static))
    X = (synth.activations(M, D, seed=9) * 0.05).astype(np.float16)
    old = sq.get_option(sq.SQ_OPT_PDL)
    ys = [torch.from_numpy(X).to(DEV)]
    try:
        sq.set_option(sq.SQ_OPT_PDL, pdl)
        for _ in range(3):
            for q in qs:
                ys.append(sq.w4a16_gemm(ys[-1], q))
        torch.cuda.synchronize()
    finally:
        sq.set_option(sq.SQ_OPT_PDL, old)
    for i in range(1, len(ys)):
        r = refs[(i - 1) % len(refs)]
        xin = ys[i - 1].cpu().numpy()
        y_ref = oracle.gemm(xin, r["Wq"], r["scales"], r["zeros"])
        W_hat = oracle.dequant(r["Wq"], r["scales"], r["zeros"])
        GemmCase(ys[i], y_ref, xin.astype(np.float64), W_hat, "f16").check(torch.float16)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("M,N,K", [(64, 2048, 4096), (300, 1024, 4096), (520, 8192, 512), (17, 4096, 2048),
                                   (128, 2816, 1024)])
def test_gemm_prefill_streamk(M, N, K, dtype):
    """Prefill shapes whose tiles leave the last wave mostly idle, so the (tile x group)
    units are split between CTAs (stream-K) and finished by the fixup: ragged token
    tiles, whole tiles in the middle of a CTA's range, several CTAs per tile.  Bit-identical
    on every launch (fixed summation order)."""
    _gemm_case(M, N, K, dtype, sq.SQ_PATH_PREFILL, seed=M + N).check(dtype)
    x = torch.randn(M, K, device=DEV).to(dtype)
    q = sq.quantize_pack_groupwise(torch.randn(N, K, device=DEV).half() * 0.02)
    ys = [sq.w4a16_gemm(x, q, path=sq.SQ_PATH_PREFILL) for _ in range(3)]
    torch.cuda.synchronize()
    assert all(torch.equal(ys[0], yy) for yy in ys[1:])


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
                W_hat = oracle.dequant(ref["Wq"], ref["scales"], ref["zeros"])
                GemmCase(ys[0], y_ref, X.astype(np.float64), W_hat, "f16").check(torch.float16)
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
    W_hat = oracle.dequant(ref["Wq"], ref["scales"], ref["zeros"])
    for y in ys:
        GemmCase(y, y_ref, x.float().cpu().double().numpy(), W_hat, xd).check(dtype)
    # deterministic: identical bits on every launch
    assert all(torch.equal(ys[0], y) for y in ys[1:])


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("path,M", [(sq.SQ_PATH_DECODE, 1), (sq.SQ_PATH_DECODE, 16), (sq.SQ_PATH_PREFILL, 40),
                                    (sq.SQ_PATH_PREFILL, 300)])
def test_gemm_edge_groups(path, M, dtype):
    """The quantizer's edge-group suite (constant, one-sided, tie, subnormal, ±65504 and
    −0.0 groups) as GEMM weights, through both paths.  Decode applies Δ
    to the fp32 sum, so every output obeys the element-wise bound.  Prefill feeds
    Ŵ = RN((q − Z)·Δ) to the tensor cores in the activation dtype: for fp16 a group whose
    |(q − Z)·Δ| exceeds 65504 saturates to ±65504 (include/libsq.h), so those rows are
    checked to be finite and the others against the bound."""
    E = synth.edge_groups(128, seed=5)
    R = E.shape[0]
    N = (R + 63) // 64 * 64
    W = np.concatenate([E, synth.weights(N - R, 128, seed=6)]).astype(np.float16)
    W = np.concatenate([W, W[:, ::-1], synth.weights(N, 128, seed=7)], axis=1)   # K = 384
    c = _gemm_case(M, N, 384, dtype, path, seed=3, smooth=False, W=W, x_scale=1e-3)
    y = c.y.float().cpu().double().numpy()
    assert np.isfinite(y).all()
    ok_rows = np.ones(N, bool)
    if path == sq.SQ_PATH_PREFILL and dtype == torch.float16:
        ok_rows = np.abs(c.W_hat).max(axis=1) <= 65504.0
    ratio = elementwise_ratio(y[:, ok_rows], c.y_ref[:, ok_rows], c.x64, c.W_hat[ok_rows], c.xd)
    assert ratio <= 1.0, ratio


# ------------------------------------------------------------------ N3: group sizes 64 / 32
@pytest.mark.parametrize("group", [32, 64])
@pytest.mark.parametrize("N,K", [(264, 384), (512, 1024)])
def test_quantize_group_sizes_bitexact(group, N, K):
    """PAPER.md:185 "different group sizes": codes, Δ and Z bit-exact with the oracle at
    g = 32 / 64, with the smoothing fold, on edge groups and on bf16 weights."""
    W = synth.weights(N, K, seed=group + N, heavy=True)
    am = oracle.act_absmax(synth.activations(512, K, seed=K).astype(np.float16))
    s = oracle.smooth_scales(oracle.weight_absmax(W), am, 0.5)
    nf = torch.zeros(1, dtype=torch.int32, device=DEV)
    q = sq.quantize_pack_groupwise(_t(W), _t(s), group=group, nonfinite=nf)
    assert q.scales.shape == (K // group, N)
    _check_quant(W, s, q, nonfinite=nf, group=group)
    E = synth.edge_groups(group, seed=group)
    pad = (-E.shape[0]) % 8
    We = np.concatenate([E, synth.weights(pad, group, seed=6)]).astype(np.float16)
    We = np.tile(We, (1, 128 // group))                       # K = 128: 128 / group groups per row
    nf.zero_()
    qe = sq.quantize_pack_groupwise(_t(We), group=group, nonfinite=nf)
    _check_quant(We, None, qe, nonfinite=nf, group=group)
    Wb = torch.from_numpy(W.astype(np.float32)).to(torch.bfloat16)
    qb = sq.quantize_pack_groupwise(Wb.to(DEV), _t(s), group=group)
    _check_quant(Wb.view(torch.int16).numpy().view(np.uint16), s, qb, w_dtype="bf16", group=group)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("group", [32, 64])
@pytest.mark.parametrize("path,M", [(sq.SQ_PATH_DECODE, 1), (sq.SQ_PATH_DECODE, 5), (sq.SQ_PATH_DECODE, 16),
                                    (sq.SQ_PATH_PREFILL, 17), (sq.SQ_PATH_PREFILL, 300)])
@pytest.mark.parametrize("N,K", [(264, 1152), (2048, 4096)])
def test_gemm_group_sizes_parity(path, M, N, K, group, dtype):
    """W4A16 GEMM at g = 32 / 64 through both paths (decode feeds RN((q - Z)Δ) operands to
    mma.sync, prefill to tcgen05), ragged row blocks and 128-k stages, stream-K fixups,
    against the oracle element by element."""
    _gemm_case(M, N, K, dtype, path, seed=M + group, group=group).check(dtype)


# ------------------------------------------------------------------ N3: packed u4 zero points
@pytest.mark.parametrize("group", [128, 64, 32])
def test_quantize_zeros_u4_bitexact(group):
    """SQ_ZEROS_U4: the quantizer writes Z packed two
    per byte along n, equal to oracle.pack_zeros_u4 of the oracle's fp16 Z, codes and Δ
    unchanged -- on smoothed weights, the edge-group suite and a non-finite group (Z = 0)."""
    N, K = 288, 512
    W = synth.weights(N, K, seed=group + 11, heavy=True)
    am = oracle.act_absmax(synth.activations(512, K, seed=K).astype(np.float16))
    s = oracle.smooth_scales(oracle.weight_absmax(W), am, 0.5)
    nf = torch.zeros(1, dtype=torch.int32, device=DEV)
    q = sq.quantize_pack_groupwise(_t(W), _t(s), group=group, nonfinite=nf, zeros_u4=True)
    assert q.zeros.shape == (K // group, N // 2) and q.zeros.dtype == torch.uint8
    _check_quant(W, s, q, nonfinite=nf, group=group)
    E = synth.edge_groups(group, seed=group)
    pad = (-E.shape[0]) % 32
    We = np.concatenate([E, synth.weights(pad, group, seed=6)]).astype(np.float16)
    We = np.tile(We, (1, 128 // group))
    We[3, 0] = np.inf                                            # a non-finite group: Z = 0
    nf.zero_()
    qe = sq.quantize_pack_groupwise(_t(We), group=group, nonfinite=nf, zeros_u4=True)
    _check_quant(We, None, qe, nonfinite=nf, group=group)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("group", [128, 32])
@pytest.mark.parametrize("path,M", [(sq.SQ_PATH_DECODE, 1), (sq.SQ_PATH_DECODE, 4), (sq.SQ_PATH_DECODE, 16),
                                    (sq.SQ_PATH_PREFILL, 17), (sq.SQ_PATH_PREFILL, 64), (sq.SQ_PATH_PREFILL, 300)])
@pytest.mark.parametrize("N,K", [(288, 1152), (2048, 4096)])
def test_gemm_zeros_u4_parity(path, M, N, K, group, dtype):
    """W4A16 GEMM with packed u4 zero points through both paths (ragged 32/64/128-row blocks,
    ragged stages, stream-K) against the oracle element by element, and BIT-identical to the
    same GEMM with fp16 zero points (Z is the same integer either way)."""
    c = _gemm_case(M, N, K, dtype, path, seed=M + group, group=group, zeros_u4=True)
    c.check(dtype)
    c16 = _gemm_case(M, N, K, dtype, path, seed=M + group, group=group, zeros_u4=False)
    assert torch.equal(c.y, c16.y)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("M", [48, 49, 57, 64, 96, 97, 113, 128])
@pytest.mark.parametrize("N,K", [(392, 1152), (1024, 2048)])
def test_gemm_prefill_warp_set_boundary(M, N, K, dtype):
    """Prefill at the 48 | 49 and 96 | 97 boundaries between the three- and four-warp-set
    configurations of the 64- and 128-token tiles (ragged N, ragged stream-K), against the
    oracle element by element."""
    _gemm_case(M, N, K, dtype, sq.SQ_PATH_PREFILL, seed=M + 7).check(dtype)
