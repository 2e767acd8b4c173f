"""GPU parity of the N2 calibration steps and the N3 smoothing folds
against the fp64 oracle.

  * sq_smooth_activations: BIT-EXACT with oracle.smooth_activations (fp16 and bf16).
  * sq_sq_diff_sum: fp64 sum of squared differences; equal to numpy's fp64 sum within
    1e-12 relative (summation order only) and bit-reproducible run to run.
  * calib.alpha_search: per-α Eq. 4 losses within 3 % of the oracle's exact losses (the
    GPU compares fp16-rounded outputs: the rounding noise is ~(5e-4 / 1e-2)^2 of the
    loss), and the chosen α is the oracle's or has a loss within 3 % of the oracle's
    minimum (a near-tie), tie rule included.
  * sq_fold_rows (s^-1 folded into the producer's output rows, Fig. 5): BIT-EXACT.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_2312_03788_b200 import calib, sq, synth

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _bits(t: torch.Tensor) -> np.ndarray:
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("M,K", [(1, 8), (7, 512), (333, 1024), (2048, 4096)])
def test_smooth_activations_bitexact(dtype, M, K):
    X = torch.from_numpy(synth.activations(M, K, seed=M + K)).to(dtype).to(DEV)
    s = torch.from_numpy(np.random.default_rng(K).uniform(1e-3, 1e3, K).astype(np.float32)).to(DEV)
    got = sq.smooth_activations(X, s)
    if dtype == torch.float16:
        want = oracle.smooth_activations(X.cpu().numpy(), s.cpu().numpy(), "f16").view(np.uint16)
    else:
        want = oracle.smooth_activations(_bits(X), s.cpu().numpy(), "bf16")
    assert np.array_equal(_bits(got), want)
    # in place
    Xc = X.clone()
    sq.smooth_activations(Xc, s, out=Xc)
    assert torch.equal(Xc, got)


def test_smooth_activations_edges():
    K = 64
    x = np.zeros((2, K), dtype=np.float16)
    x[0, :8] = [0.0, -0.0, 65504.0, -65504.0, 6e-8, -6e-8, np.inf, -np.inf]
    x[1, :] = np.random.default_rng(0).standard_normal(K).astype(np.float16)
    s = np.full(K, 0.5, np.float32)  # overflow to Inf for ±65504 / 0.5
    s[1::2] = 3.0
    got = sq.smooth_activations(torch.from_numpy(x).to(DEV), torch.from_numpy(s).to(DEV))
    want = oracle.smooth_activations(x, s, "f16").view(np.uint16)
    assert np.array_equal(_bits(got), want)
    assert sq.smooth_activations(torch.empty(0, K, dtype=torch.float16, device=DEV),
                                 torch.from_numpy(s).to(DEV)).numel() == 0


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("n", [0, 1, 1000, 3 * 1024 * 1024 + 7])
def test_sq_diff_sum(dtype, n):
    g = torch.Generator(device="cpu").manual_seed(n)
    A = torch.randn(n, generator=g).to(dtype).to(DEV)
    B = (torch.randn(n, generator=g) * 0.5).to(dtype).to(DEV)
    r1 = sq.sq_diff_sum(A, B)
    r2 = sq.sq_diff_sum(A, B)
    a = A.float().cpu().double().numpy()
    b = B.float().cpu().double().numpy()
    want = float(((a - b) ** 2).sum())
    got = float(r1.cpu())
    assert got == float(r2.cpu())  # fixed reduction order
    assert abs(got - want) <= 1e-12 * max(want, 1e-300)


@pytest.mark.parametrize("T,N,K,seed", [(64, 256, 512, 1), (16, 384, 768, 2), (200, 512, 1024, 3)])
def test_alpha_search_parity(T, N, K, seed):
    Xn = synth.activations(T, K, seed=seed).astype(np.float16)
    Wn = synth.weights(N, K, seed=seed + 100)
    best_o, loss_o = oracle.alpha_search(Xn, Wn)
    best_g, loss_g = calib.alpha_search(torch.from_numpy(Xn).to(DEV), torch.from_numpy(Wn).to(DEV))
    loss_g = loss_g.numpy()
    np.testing.assert_allclose(loss_g, loss_o, rtol=3e-2)
    i_g = calib.ALPHA_GRID.index(best_g)
    assert best_g == best_o or loss_o[i_g] <= loss_o.min() * 1.03


def test_alpha_search_zero_loss_tie_rule():
    """The oracle pin's exact layer (s = 1, W on the Eq. 1 grid) with X = 0: every loss is
    exactly 0 on the GPU too, and the search returns α = 0."""
    from tests.test_oracle_pins import _exact_layer

    X, W = _exact_layer()
    best, losses = calib.alpha_search(torch.zeros(X.shape, dtype=torch.float16, device=DEV),
                                      torch.from_numpy(W).to(DEV))
    assert best == 0.0 and bool((losses == 0).all())


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("N,K", [(1, 8), (256, 128), (1024, 4096)])
def test_fold_rows_bitexact(N, K, dtype):
    """Fig. 5 fusion: W'[n][k] = RN(W[n][k] / d[n]) bit-exact with the
    oracle, in place too; and the RMSNorm-gain fold is sq_smooth_activations on g[1][K]."""
    W = torch.from_numpy(synth.weights(N, K, seed=N)).to(dtype).to(DEV)
    d = torch.from_numpy(np.random.default_rng(N).uniform(1e-2, 1e2, N).astype(np.float32)).to(DEV)
    got = sq.fold_rows(W, d)
    if dtype == torch.float16:
        want = oracle.fold_rows(W.cpu().numpy(), d.cpu().numpy(), "f16").view(np.uint16)
    else:
        want = oracle.fold_rows(_bits(W), d.cpu().numpy(), "bf16")
    assert np.array_equal(_bits(got), want)
    Wc = W.clone()
    sq.fold_rows(Wc, d, out=Wc)
    assert torch.equal(Wc, got)
    if N == 1:
        g = W  # a gain vector g[K] as [1][K]: divide by the consumer's s (per column)
        s = torch.from_numpy(np.random.default_rng(3).uniform(0.1, 10, K).astype(np.float32)).to(DEV)
        gs = sq.smooth_activations(g, s)
        ref = oracle.smooth_activations(g.cpu().numpy() if dtype == torch.float16 else _bits(g), s.cpu().numpy(),
                                        "f16" if dtype == torch.float16 else "bf16")
        assert np.array_equal(_bits(gs), ref.view(np.uint16) if dtype == torch.float16 else ref)
