"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(weights static + PDL, launches captured in a CUDA graph), on sampled outputs the oracle
computes one by one (configs[1]-[2]: Code Llama-34B layers).

Per 34B linear (qkv 8192->10240, o_proj 8192->8192, gate|up 8192->44032, down 22016->8192):
  * smoothing factors of the full weight (α = 0.5, exact sqrt form): BIT-EXACT;
  * packed codes, Δ and Z of 24 sampled output channels: BIT-EXACT (quantization is per
    output channel, so the oracle quantizes just those rows of W' = RN(W·s));
  * Y at M = 1, 4, 16 (decode kernel) and M = 2048 (prefill kernel, 16 sampled tokens) on
    those 24 output channels: relative Frobenius error <= 5e-3 (north_star) and <= 1e-3
    (the fp16 bound of DESIGN.md §3) against the exact fp64 products.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_2312_03788_b200 import sq, stack
from tests.gemm_bounds import elementwise_ratio

pytestmark = pytest.mark.gpu
DEV = "cuda"
# (K, N) of the Code Llama-34B linears (BASELINE.json configs[2]/[3]) and the Code Llama-7B
# ones (configs[1]: hidden 4096, MLP 11008; K = 11008 is 86 groups, a ragged 2-group final
# stage of the 4-group decode units plus stream-K)
SHAPES = {"qkv": (8192, 10240), "o_proj": (8192, 8192), "gate_up": (8192, 44032), "down": (22016, 8192),
          "7b_qkv": (4096, 12288), "7b_o_proj": (4096, 4096), "7b_gate_up": (4096, 22016),
          "7b_down": (11008, 4096)}


@pytest.fixture(autouse=True)
def _bench_launch_config():
    old = sq.get_option(sq.SQ_OPT_PDL)
    sq.set_option(sq.SQ_OPT_PDL, 1)
    yield
    sq.set_option(sq.SQ_OPT_PDL, old)


@pytest.mark.parametrize("name", list(SHAPES))
def test_fullsize_sampled_parity(name):
    K, N = SHAPES[name]
    seed = 10 + list(SHAPES).index(name)
    W = stack.synth_weight(N, K, seed, DEV)
    am = stack.synth_act_max(K, seed + 1, DEV)
    s = sq.smooth_scales(W, am, 0.5)
    q = sq.quantize_pack_groupwise(W, s)
    torch.cuda.synchronize()

    # Eq. 6 over the full weight: bit-exact
    W_h = W.cpu().numpy()
    s_ref = oracle.smooth_scales(oracle.weight_absmax(W_h), am.cpu().numpy(), 0.5)
    assert np.array_equal(s.cpu().numpy().view(np.uint32), s_ref.view(np.uint32))

    # Eq. 5 + Eq. 1 on sampled output channels: bit-exact codes / Δ / Z
    rows = np.sort(np.random.default_rng(seed).choice(N, 24, replace=False))
    ref = oracle.quantize_pack(W_h[rows], s_ref)
    Wq_h = q.Wq.cpu().numpy()[rows]
    sc_h = q.scales.cpu().numpy().view(np.uint16)[:, rows]
    z_h = q.zeros.cpu().numpy().view(np.uint16)[:, rows]
    assert np.array_equal(Wq_h, ref["Wq"])
    assert np.array_equal(sc_h, ref["scales"])
    assert np.array_equal(z_h, ref["zeros"])
    W_hat = oracle.dequant(ref["Wq"], ref["scales"], ref["zeros"])  # [24][K], exact
    q.mark_static()  # the bench's launch configuration: resident weights, early weight streaming

    ws = sq.default_workspace(DEV, max(sq.w4a16_gemm_workspace_bytes(m, N, K) for m in (1, 4, 16, 2048)))
    g = torch.Generator(device=DEV).manual_seed(seed + 2)
    for M in (1, 4, 16, 2048):
        X = (torch.randn(M, K, generator=g, device=DEV) * 2.0).half()
        Y = torch.empty(M, N, dtype=torch.float16, device=DEV)
        sq.w4a16_gemm(X, q, out=Y, workspace=ws)  # warm-up outside the capture
        Y.zero_()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            sq.w4a16_gemm(X, q, out=Y, workspace=ws)
        graph.replay()
        torch.cuda.synchronize()
        toks = np.arange(M) if M <= 16 else np.sort(np.random.default_rng(M).choice(M, 16, replace=False))
        x_h = X.cpu().numpy()[toks].astype(np.float64)
        y_ref = x_h @ W_hat.T
        y = Y.cpu().numpy()[np.ix_(toks, rows)].astype(np.float64)
        err = np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref)
        assert err <= 1e-3, (name, M, err)
        assert elementwise_ratio(y, y_ref, x_h, W_hat, "f16") <= 1.0, (name, M)


def test_fullsize_bf16_activations_and_large_m():
    """bf16 activations at a full 34B shape (down_proj, K = 22016: 172 groups, the longest K),
    decode and prefill, plus the largest M the sweep uses (4096) on a gate-shaped layer,
    sampled against the exact products (bf16 bound 4e-3)."""
    K, N = 22016, 8192
    W = stack.synth_weight(N, K, 77, DEV)
    q = sq.quantize_pack_groupwise(W)
    rows = np.sort(np.random.default_rng(5).choice(N, 16, replace=False))
    ref = oracle.quantize_pack(W.cpu().numpy()[rows], None)
    W_hat = oracle.dequant(ref["Wq"], ref["scales"], ref["zeros"])
    g = torch.Generator(device=DEV).manual_seed(78)
    for M in (1, 16, 512):
        X = torch.randn(M, K, generator=g, device=DEV).to(torch.bfloat16)
        Y = sq.w4a16_gemm(X, q)
        torch.cuda.synchronize()
        toks = np.arange(min(M, 16))
        x_h = X[: len(toks)].float().cpu().double().numpy()
        y_ref = x_h @ W_hat.T
        y = Y[: len(toks)].float().cpu().double().numpy()[:, rows]
        err = np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref)
        assert err <= 4e-3, (M, err)
    # M = 4096 (prefill, several token tiles) on 8192 -> 22016
    K2, N2 = 8192, 22016
    W2 = stack.synth_weight(N2, K2, 79, DEV)
    q2 = sq.quantize_pack_groupwise(W2)
    rows2 = np.sort(np.random.default_rng(6).choice(N2, 16, replace=False))
    ref2 = oracle.quantize_pack(W2.cpu().numpy()[rows2], None)
    W_hat2 = oracle.dequant(ref2["Wq"], ref2["scales"], ref2["zeros"])
    X2 = torch.randn(4096, K2, generator=g, device=DEV).half()
    Y2 = sq.w4a16_gemm(X2, q2)
    torch.cuda.synchronize()
    toks = np.sort(np.random.default_rng(7).choice(4096, 24, replace=False))
    y_ref = X2.cpu().numpy()[toks].astype(np.float64) @ W_hat2.T
    y = Y2.cpu().numpy()[np.ix_(toks, rows2)].astype(np.float64)
    assert np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref) <= 1e-3


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("name", ["qkv", "o_proj", "gate_up", "down", "7b_gate_up", "7b_o_proj"])
def test_fullsize_decode_vs_prefill_all_rows(name, dtype):
    """EVERY output of the decode kernel at M = 1, 3 and 16 (the 128-row-block, four-row and
    sixteen-row configurations of the full-size shapes) against the independently written
    prefill kernel on the same weights: the two paths round differently (exact (q - Z) with
    fp32 Δ vs Ŵ = RN((q - Z) Δ)), so they agree to the fp16 bound, and a wrong
    row block, stage or fixup -- which sampled rows could miss -- is an O(1) difference."""
    K, N = SHAPES[name]
    W = stack.synth_weight(N, K, 200 + list(SHAPES).index(name), DEV)
    q = sq.quantize_pack_groupwise(W).mark_static()
    g = torch.Generator(device=DEV).manual_seed(201)
    tol = 2e-3 if dtype == torch.float16 else 1e-2  # bf16: 8-bit operands and outputs
    for M in (1, 3, 9, 16):
        X = torch.randn(M, K, generator=g, device=DEV).to(dtype)
        yd = sq.w4a16_gemm(X, q, path=sq.SQ_PATH_DECODE).float()
        yp = sq.w4a16_gemm(X, q, path=sq.SQ_PATH_PREFILL).float()
        torch.cuda.synchronize()
        rel = ((yd - yp).norm() / yp.norm()).item()
        assert rel <= tol, (name, M, rel)
        worst = ((yd - yp).abs() / (yp.abs() + 1e-2 * yp.abs().max())).max().item()
        assert worst <= 25 * tol, (name, M, worst)


@pytest.mark.parametrize("name", ["qkv", "o_proj", "gate_up", "down", "7b_gate_up", "7b_down"])
def test_fullsize_zeros_u4_every_configuration(name):
    """Packed u4 zero points (SQ_ZEROS_U4) through every decode configuration the full-size
    shapes dispatch to (M = 1, 3, 9, 16: 32/48/64/96/128-row blocks, four/eight/sixteen staged
    rows) and the prefill kernel (M = 40, 300): the launch must succeed (every TMA box of the
    packed zero rows a multiple of 16 bytes) and agree with the fp16-Z result to fp32
    summation order."""
    K, N = SHAPES[name]
    W = stack.synth_weight(N, K, 300 + list(SHAPES).index(name), DEV)
    q16 = sq.quantize_pack_groupwise(W).mark_static()
    q4 = sq.quantize_pack_groupwise(W, zeros_u4=True).mark_static()
    g = torch.Generator(device=DEV).manual_seed(301)
    for M in (1, 3, 9, 16, 40, 300):
        X = torch.randn(M, K, generator=g, device=DEV).half()
        y16 = sq.w4a16_gemm(X, q16).float()
        y4 = sq.w4a16_gemm(X, q4).float()
        torch.cuda.synchronize()
        rel = ((y4 - y16).norm() / y16.norm()).item()
        assert rel <= 1e-3, (name, M, rel)
