"""Element-wise error bound for GEMM parity (used next to the relative Frobenius norm).

For Y = X̂·Ŵᵀ (Eq. 3) computed with
  * Ŵ either exact (decode: (q − Z) exact in fp16/bf16, Δ applied to the fp32 sum) or
    rounded once to the activation dtype (prefill: RN((q − Z)·Δ), the P13 value),
  * exact products and an fp32 accumulation over K terms,
  * one final rounding of Y to the activation dtype,
the standard floating-point bound gives, per output element,

    |y − y_ref| <= u_out·|y_ref| + (u_w + K·2^-24)·S,   S = Σ_k |x_k·Ŵ_nk|,

with u_out = u_w = 2^-11 (fp16) or 2^-8 (bf16).  The K·2^-24 term is the worst case of a
sequential fp32 sum (any order, S15).  A wrong row block, a dropped or duplicated group or a
swapped row shows up as an error of order |y_ref| ~ S/√K, which is far above this bound for
the shapes tested; the Frobenius norm alone could hide it among 10^5 correct outputs.
"""

from __future__ import annotations

import numpy as np

UNIT = {"f16": 2.0 ** -11, "bf16": 2.0 ** -8}


def elementwise_ratio(y: np.ndarray, y_ref: np.ndarray, x: np.ndarray, W_hat: np.ndarray,
                      x_dtype: str) -> float:
    """max over elements of |y − y_ref| / bound (<= 1 passes).  y, y_ref: [M][N];
    x: fp64 [M][K] (the activations as fed); W_hat: fp64 [N][K] exact dequantized weights."""
    u = UNIT[x_dtype]
    K = x.shape[1]
    S = np.abs(x) @ np.abs(W_hat).T
    bound = u * np.abs(y_ref) + (u + K * 2.0 ** -24) * S + 2.0 ** -24
    return float((np.abs(np.asarray(y, dtype=np.float64) - y_ref) / bound).max())
