"""Single-layer smoothing-strength search on the GPU.

PAPER.md:166 / :213: "We use grid search with an interval of 0.05 between 0 and 1 to
search for the smoothing strength that minimizes the quantization loss", with the loss of
Eq. 4.  Per α of the grid (21 values):

    s_α  = sq_smooth_scales(W, act_max, α)            Eq. 6       (k_smooth.cu)
    Ŵ_α  = sq_quantize_pack_groupwise(W, s_α)         Eq. 5 + 1   (k_quant.cu)
    X̂_α  = sq_smooth_activations(X, s_α)              Eq. 5       (k_calib.cu)
    Y_α  = sq_w4a16_gemm(X̂_α, Ŵ_α)                    Eq. 3       (k_decode.cu / k_prefill.cu)
    E(α) = sq_sq_diff_sum(Y_ref, Y_α)                 Eq. 4       (k_calib.cu)

with act_max = sq_act_absmax(X) and Y_ref = X·Wᵀ, the unquantized layer, computed once by
a plain library GEMM (torch.matmul / cuBLAS, fp32 accumulate) -- the reference the loss
compares against, not a step of the quantized path.  The best α is the first minimum in
grid order (ties go to the smallest α), read back with one host synchronization.

The paper minimizes the loss of the entire model; per layer is this repo's reading
(DESIGN.md §3): the whole-model search needs the checkpoints.
"""

from __future__ import annotations

import torch

from . import sq

#: the searched smoothing strengths: i / 20 for i = 0..20
ALPHA_GRID = tuple(i / 20.0 for i in range(21))


def alpha_search(X: torch.Tensor, W: torch.Tensor, alphas=ALPHA_GRID, group: int = sq.GROUP,
                 stream=None):
    """X[T][K] calibration activations, W[N][K] the layer (or stacked q|k|v, gate|up)
    weight, both fp16 or both bf16, on the GPU.  Returns (best_alpha, losses) with losses
    a host float64 tensor aligned with `alphas`."""
    if X.dtype != W.dtype:
        raise TypeError("alpha_search: X and W need the same dtype")
    T, K = X.shape
    N, K2 = W.shape
    if K != K2:
        raise ValueError("alpha_search: X and W disagree on K")
    dev = X.device
    act_max = sq.act_absmax(X, stream=stream)
    y_ref = torch.matmul(X, W.t())                 # unquantized reference X·Wᵀ
    xh = torch.empty_like(X)
    y = torch.empty(T, N, dtype=X.dtype, device=dev)
    s = torch.empty(K, dtype=torch.float32, device=dev)
    ws = sq.default_workspace(dev, sq.w4a16_gemm_workspace_bytes(T, N, K, group))
    red_ws = torch.empty(sq.lib().sq_sq_diff_sum_workspace_bytes(), dtype=torch.uint8, device=dev)
    losses = torch.empty(len(alphas), dtype=torch.float64, device=dev)
    for i, a in enumerate(alphas):
        sq.smooth_scales(W, act_max, float(a), out=s, stream=stream)
        q = sq.quantize_pack_groupwise(W, s, group=group, stream=stream)
        sq.smooth_activations(X, s, out=xh, stream=stream)
        sq.w4a16_gemm(xh, q, out=y, workspace=ws, stream=stream)
        sq.sq_diff_sum(y_ref, y, out=losses[i], workspace=red_ws, stream=stream)
    host = losses.cpu()
    best = int(torch.argmin(host))  # first minimum: ties go to the smallest α
    return float(alphas[best]), host
