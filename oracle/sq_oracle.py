"""fp64 CPU oracle: smoothing (Eq. 5-6), group-wise INT4 quantization (Eq. 1),
dequantization and the W4A16 linear layer (Eq. 2-3) of SmoothQuant+.

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.  Never imported by the
product package.

Conventions (SURVEY.md §8 notation):
  M = tokens (T of Eq. 2), K = input channels (C_i), N = output channels (C_o),
  g = group size (128), G = K / g.
  Weights are stored nn.Linear-style, ``W[N][K]`` = the transpose of Eq. 2's
  ``W ∈ R^{C_i×C_o}``, so Eq. 2's W_eq2[k][n] == W[n][k].
  RN = round to nearest even, RZ = round toward zero,
  RHA = round half away from zero.

Readings of silent/ambiguous points:
  S1  round() of Eq. 1 is RHA                       ("round(z) rounds z to the nearest integer")
  S2  Z = clamp(RHA(-min/Δ), 0, 15)                 ("Z is zero point")
  S3  Δ stored fp16, rounded toward zero from the exact (W_max-W_min)/15
  S4  constant group c: Δ = 1 if c == 0 else |c|; Δ that underflows to 0 -> 2^-24
  S5  Z stored as fp16 holding an integer 0..15
  S6  groups are g consecutive input channels (k) of one output channel
  S8  literal min/max, no clipping search
  S10 ε = 1e-5 floor on both maxima of Eq. 6
  S12 Eq. 6 evaluated in fp64, RN to fp32; sqrt/div forms for α ∈ {0, 0.5, 1}
  S13 fold rounding: one rounding RN16(exact w·s)
  S14 GEMM accumulates exactly (fp64 here); the GPU uses fp32 accumulate
  S17 bf16 source weights: W' = RN_bf16(exact w·s); Δ still fp16; a group whose
      r/15 exceeds the fp16 range is treated as non-finite
"""

from __future__ import annotations

import numpy as np

#: ε of Eq. 6's floors (reading S10).
EPS = 1e-5

#: Encoding of a group that contains NaN/Inf after the fold:
#: scale = fp16 quiet NaN, zero = 0, codes = 0.
NONFINITE_SCALE_BITS = 0x7E00

_F16_MAX = 65504.0
_F16_MIN_SUBNORMAL = 2.0 ** -24


# --------------------------------------------------------------------------
# number-format helpers (plain definitions, no method arithmetic)
# --------------------------------------------------------------------------

def _as_f64(a, dtype: str) -> np.ndarray:
    """Exact conversion of fp16 (numpy float16) or bf16 (uint16 bit pattern) to fp64."""
    a = np.asarray(a)
    if dtype == "f16":
        return a.astype(np.float16).astype(np.float64)
    if dtype == "bf16":
        bits = a.astype(np.uint16).astype(np.uint32) << np.uint32(16)
        return bits.view(np.float32).astype(np.float64)
    if dtype in ("f32", "f64"):
        return a.astype(np.float64)
    raise ValueError(f"unknown dtype {dtype!r}")


def rn_bf16_bits(x: np.ndarray) -> np.ndarray:
    """RN-even of fp64 values to bfloat16 (8-bit significand, fp32 exponent range);
    returns the uint16 bit patterns.  Done directly from fp64 (single rounding)."""
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros(x.shape, dtype=np.uint16)
    flat = x.reshape(-1)
    o = out.reshape(-1)
    for i, v in enumerate(flat):
        if np.isnan(v):
            o[i] = 0x7FC0
            continue
        sign = 0x8000 if np.signbit(v) else 0
        a = abs(float(v))
        if a == 0.0:
            o[i] = sign
            continue
        if np.isinf(a):
            o[i] = sign | 0x7F80
            continue
        m, e = np.frexp(a)              # a = m * 2^e, m in [0.5, 1)
        exp_unbiased = e - 1            # a = (2m) * 2^(e-1), 2m in [1, 2)
        if exp_unbiased < -126:         # subnormal: quantum 2^-133
            quantum_exp = -133
        else:
            quantum_exp = exp_unbiased - 7
        scaled = a / 2.0 ** quantum_exp  # exact (power-of-two scaling)
        r = np.rint(scaled)              # half-even
        val = r * 2.0 ** quantum_exp
        if val > (2.0 - 2.0 ** -7) * 2.0 ** 127:
            o[i] = sign | 0x7F80
            continue
        f32 = np.float32(val)            # exactly representable
        o[i] = sign | ((int(np.array(f32).view(np.uint32)) >> 16) & 0x7FFF)
    return out


def rz_fp16(x: np.ndarray) -> np.ndarray:
    """RZ of fp64 values to fp16 (reading S3): the fp16 value of largest magnitude
    not exceeding |x| in magnitude.  numpy's float64->float16 cast is RN; step one
    ulp toward zero when it rounded away."""
    x = np.asarray(x, dtype=np.float64)
    with np.errstate(over="ignore"):
        h = x.astype(np.float16)
    away = np.abs(h.astype(np.float64)) > np.abs(x)
    h = np.where(away, np.nextafter(h, np.float16(0)), h)
    return h.astype(np.float16)


def rha(x: np.ndarray) -> np.ndarray:
    """Round half away from zero (reading S1; C ``round``).  Exact: the fractional
    part x - trunc(x) is exact in fp64."""
    x = np.asarray(x, dtype=np.float64)
    t = np.trunc(x)
    frac = np.abs(x - t)
    return t + np.where(frac >= 0.5, np.sign(x), 0.0)


# --------------------------------------------------------------------------
# a1/a2: Eq. 6 smoothing factors
# --------------------------------------------------------------------------

def act_absmax(X_cal: np.ndarray, x_dtype: str = "f16") -> np.ndarray:
    """Calibration statistic max(|X_j|) of Eq. 6 over the calibration rows
    (Eq. 6; PAPER.md:166 calibration set).  X_cal[T][K] -> fp32[K]."""
    x = _as_f64(X_cal, x_dtype)
    return np.abs(x).max(axis=0).astype(np.float32)


def weight_absmax(W: np.ndarray, w_dtype: str = "f16") -> np.ndarray:
    """max(|W_j|) of Eq. 6 for input channel j.  W is stored
    [N][K], so channel j = column k.  Exact (max is a selection).  -> fp64[K]."""
    w = _as_f64(W, w_dtype)
    return np.abs(w).max(axis=0)


def smooth_scales(w_max: np.ndarray, act_max: np.ndarray, alpha: float,
                  eps: float = EPS) -> np.ndarray:
    """Eq. 6: s_j = max(|X_j|)^α / max(|W_j|)^(1-α), with the ε
    floor of reading S10, evaluated in fp64 and RN to fp32 (reading S12).
    α = 1 gives s_j = max|X_j| and α = 0 gives 1/max|W_j|."""
    a = np.maximum(np.asarray(act_max, dtype=np.float64), float(eps))
    w = np.maximum(np.asarray(w_max, dtype=np.float64), float(eps))
    alpha = float(alpha)
    if alpha == 0.5:
        s = np.sqrt(a) / np.sqrt(w)
    elif alpha == 1.0:
        s = a
    elif alpha == 0.0:
        s = 1.0 / w
    else:
        s = np.power(a, alpha) / np.power(w, 1.0 - alpha)
    return s.astype(np.float32)


# --------------------------------------------------------------------------
# a3: Eq. 5 weight-side fold
# --------------------------------------------------------------------------

def smooth_weight_exact(W: np.ndarray, s: np.ndarray, w_dtype: str = "f16") -> np.ndarray:
    """diag(s)·W of Eq. 5 in the [N][K] storage layout: channel
    k of every output row is multiplied by s[k].  Exact in fp64 (11+24 bits)."""
    w = _as_f64(W, w_dtype)
    return w * np.asarray(s, dtype=np.float32).astype(np.float64)[None, :]


def fold(W: np.ndarray, s, w_dtype: str = "f16"):
    """W' = RN(W·s) to the weight's own format (reading S13).  s=None means RTN
    (s = 1).  Returns W' as fp64 values (exactly the rounded ones)."""
    if s is None:
        return _as_f64(W, w_dtype)
    exact = smooth_weight_exact(W, s, w_dtype)
    if w_dtype == "f16":
        with np.errstate(over="ignore"):
            return exact.astype(np.float16).astype(np.float64)
    if w_dtype == "bf16":
        return _as_f64(rn_bf16_bits(exact), "bf16")
    raise ValueError(w_dtype)


# --------------------------------------------------------------------------
# a4: Eq. 1 group-wise asymmetric INT4 quantization
# --------------------------------------------------------------------------

def _quantize_groups(v: np.ndarray, n_bits: int = 4):
    """Eq. 1 applied to each row of v[R][g] (fp64 values of W').
    Returns (q int64[R][g], delta fp64[R], Z fp64[R], nonfinite bool[R]).

    Steps, in the paper's order:
      Δ = (W_max - W_min) / (2^N - 1)                 -- Eq. 1 line 3, stored RZ16 (S3)
      W̄ = clamp(round(W/Δ) + Z, 0, 2^N - 1)          -- Eq. 1 line 1, round = RHA (S1)
      Z = clamp(RHA(-W_min/Δ), 0, 2^N - 1)            -- reading S2
    """
    qmax = float(2 ** n_bits - 1)
    v = np.asarray(v, dtype=np.float64)
    R = v.shape[0]
    nonfinite = ~np.isfinite(v).all(axis=1)
    vv = np.where(np.isfinite(v), v, 0.0)
    lo = vv.min(axis=1)
    hi = vv.max(axis=1)
    r = hi - lo                                   # exact: <= 41 significant bits

    delta = np.empty(R, dtype=np.float64)
    pos = r > 0
    d = rz_fp16(r[pos] / qmax).astype(np.float64)  # RZ16 of the fp64 quotient (S3)
    d = np.where(d == 0.0, _F16_MIN_SUBNORMAL, d)  # underflow floor (S4)
    # a range too wide for fp16 (only possible for bf16 weights, S17) is non-finite
    overflow = (r[pos] / qmax) > _F16_MAX
    nonfinite[np.flatnonzero(pos)[overflow]] = True
    delta[pos] = d
    c = lo[~pos]                                   # constant group (S4)
    delta[~pos] = np.where(c == 0.0, 1.0, np.abs(c))
    delta = np.where(nonfinite, 1.0, delta)

    Z = np.clip(rha(-lo / delta), 0.0, qmax)
    q = np.clip(rha(vv / delta[:, None]) + Z[:, None], 0.0, qmax)

    q = np.where(nonfinite[:, None], 0.0, q).astype(np.int64)
    Z = np.where(nonfinite, 0.0, Z)
    delta = np.where(nonfinite, np.nan, delta)
    return q, delta, Z, nonfinite


def quantize_group(values, n_bits: int = 4):
    """One group of Eq. 1.  values: sequence of fp16-representable
    numbers.  Returns (codes list[int], delta float (an fp16 value), Z int)."""
    v = np.asarray(values, dtype=np.float64)[None, :]
    q, d, z, nf = _quantize_groups(v, n_bits)
    if nf[0]:
        raise ValueError("non-finite input")    # SPEC.md:115 "errors: ... non-finite input"
    return [int(x) for x in q[0]], float(d[0]), int(z[0])


def pack_nibbles(q: np.ndarray) -> np.ndarray:
    """Two 4-bit codes per byte along k: element 2i in the low nibble, 2i+1 in
    the high nibble.  q[..., K] (K even) -> uint8[..., K/2]."""
    q = np.asarray(q, dtype=np.int64)
    if q.shape[-1] % 2:
        raise ValueError("pack_nibbles needs an even count")
    if (q < 0).any() or (q > 15).any():
        raise ValueError("code out of range")
    return (q[..., 0::2] | (q[..., 1::2] << 4)).astype(np.uint8)


def unpack_nibbles(b: np.ndarray) -> np.ndarray:
    """Inverse of pack_nibbles: uint8[..., K/2] -> int64[..., K]."""
    b = np.asarray(b, dtype=np.uint8).astype(np.int64)
    out = np.empty(b.shape[:-1] + (2 * b.shape[-1],), dtype=np.int64)
    out[..., 0::2] = b & 0xF
    out[..., 1::2] = b >> 4
    return out


def pack_zeros_u4(zeros: np.ndarray) -> np.ndarray:
    """Packed 4-bit zero points, the u4 variant of N3 (SURVEY.md §8(f) "a packed u4
    zero-point variant"; SPEC.md:185-186 stores Z as u4).  Every Z is an integer 0..15
    (Eq. 1 clamps it, reading S2), so it fits a nibble exactly.  Two per byte along the
    output-channel axis: channel 2i in the low nibble, 2i+1 in the high nibble -- the
    nibble order pack_nibbles uses along k.
    zeros fp16 bits uint16[G][N] (N even) -> uint8[G][N/2]."""
    z = np.asarray(zeros, dtype=np.uint16).view(np.float16).astype(np.float64)
    if not np.all(np.isfinite(z)) or (z != np.round(z)).any() or (z < 0).any() or (z > 15).any():
        raise ValueError("zero points must be integers 0..15")
    return pack_nibbles(z.astype(np.int64))


def unpack_zeros_u4(zeros_u4: np.ndarray) -> np.ndarray:
    """Inverse of pack_zeros_u4: uint8[G][N/2] -> fp16 bits uint16[G][N]."""
    return unpack_nibbles(zeros_u4).astype(np.float16).view(np.uint16)


def quantize_pack(W: np.ndarray, s=None, group: int = 128, w_dtype: str = "f16"):
    """sq_quantize_pack_groupwise semantics: Eq. 5 fold (W' = RN(W·s)) then Eq. 1 per
    (output channel n, group of g consecutive input channels) (PAPER.md:160
    "Group-size is usually set to be 128"; PAPER.md:176 load-time quantization).

    W[N][K] (fp16 array, or uint16 bf16 bits with w_dtype='bf16'); s fp32[K] or None.
    Returns dict(Wq=uint8[N][K/2], scales=uint16[G][N] (fp16 bits),
                 zeros=uint16[G][N] (fp16 bits), nonfinite=int, codes=int64[N][K],
                 delta=fp64[G][N], Z=fp64[G][N], w_folded=fp64[N][K]).
    Non-finite groups are encoded as scale NaN (0x7E00), zero 0, codes 0 and counted.
    """
    Wf = fold(W, s, w_dtype)
    N, K = Wf.shape
    if K % group:
        raise ValueError("K must be a multiple of group")
    G = K // group
    v = Wf.reshape(N * G, group)
    q, d, z, nf = _quantize_groups(v)
    codes = q.reshape(N, K)
    delta = d.reshape(N, G).T.copy()
    Z = z.reshape(N, G).T.copy()
    scale_bits = np.where(np.isnan(delta), NONFINITE_SCALE_BITS,
                          np.nan_to_num(delta).astype(np.float16).view(np.uint16))
    zero_bits = Z.astype(np.float16).view(np.uint16)
    return dict(
        Wq=pack_nibbles(codes),
        scales=scale_bits.astype(np.uint16),
        zeros=zero_bits.astype(np.uint16),
        nonfinite=int(nf.sum()),
        codes=codes,
        delta=delta,
        Z=Z,
        w_folded=Wf,
    )


# --------------------------------------------------------------------------
# a6/a7: Eq. 1 line 2 dequantization and Eq. 3 linear layer
# --------------------------------------------------------------------------

def dequant(Wq: np.ndarray, scales: np.ndarray, zeros: np.ndarray, group: int = 128,
            zeros_u4: bool = False) -> np.ndarray:
    """Ŵ = (W̄ - Z)·Δ (Eq. 1 line 2), exact in fp64.
    Wq uint8[N][K/2], scales/zeros fp16 bits [G][N] (zeros_u4: zeros packed by
    pack_zeros_u4, uint8[G][N/2]) -> fp64[N][K]."""
    if zeros_u4:
        zeros = unpack_zeros_u4(zeros)
    q = unpack_nibbles(Wq)
    N, K = q.shape
    G = K // group
    d = np.asarray(scales, dtype=np.uint16).view(np.float16).astype(np.float64)   # [G][N]
    z = np.asarray(zeros, dtype=np.uint16).view(np.float16).astype(np.float64)
    d_full = np.repeat(d.T, group, axis=1)    # [N][K]: group gi covers k in [gi*g, (gi+1)*g)
    z_full = np.repeat(z.T, group, axis=1)
    return (q.astype(np.float64) - z_full) * d_full


def gemm(X: np.ndarray, Wq: np.ndarray, scales: np.ndarray, zeros: np.ndarray,
         group: int = 128, x_dtype: str = "f16", zeros_u4: bool = False) -> np.ndarray:
    """Eq. 3: Y = X̂·Ŵ, with Eq. 2's W_eq2 = Ŵ[N][K]^T
    (PAPER.md:95-100).  X[M][K] fp16 (or bf16 bits) -> Y fp64[M][N]."""
    x = _as_f64(X, x_dtype)
    return x @ dequant(Wq, scales, zeros, group, zeros_u4).T


def quant_loss(X: np.ndarray, W: np.ndarray, W_hat: np.ndarray) -> float:
    """Eq. 4: E = ||X·W - X·Ŵ||_2^2 (sum of squared element
    differences), W and Ŵ in [N][K] storage, fp64."""
    x = np.asarray(X, dtype=np.float64)
    D = x @ np.asarray(W, dtype=np.float64).T - x @ np.asarray(W_hat, dtype=np.float64).T
    return float((D * D).sum())


# --------------------------------------------------------------------------
# N2: single-layer smoothing-strength grid search
# --------------------------------------------------------------------------

def smooth_activations(X: np.ndarray, s: np.ndarray, x_dtype: str = "f16") -> np.ndarray:
    """Activation side of Eq. 5: X̂ = X·diag(s)^-1, per input
    channel k, as stored activations: RN(fp64(X) / fp64(s)) to x_dtype (fp16 array,
    or uint16 bf16 bits).  fp64 division is correctly rounded, then rounded once."""
    q = _as_f64(X, x_dtype) / np.asarray(s, dtype=np.float32).astype(np.float64)[None, :]
    if x_dtype == "f16":
        with np.errstate(over="ignore"):
            return q.astype(np.float16)
    if x_dtype == "bf16":
        return rn_bf16_bits(q)
    raise ValueError(x_dtype)


def fold_rows(W: np.ndarray, d: np.ndarray, w_dtype: str = "f16") -> np.ndarray:
    """Model-level smoothing fusion (Fig. 5): the division of the next
    layer's input by its smoothing factors folded into the OUTPUT rows of the producing
    linear, W'[n][k] = RN(fp64(W[n][k]) / fp64(d[n])) to w_dtype (one rounding)."""
    q = _as_f64(W, w_dtype) / np.asarray(d, dtype=np.float32).astype(np.float64)[:, None]
    if w_dtype == "f16":
        with np.errstate(over="ignore"):
            return q.astype(np.float16)
    if w_dtype == "bf16":
        return rn_bf16_bits(q)
    raise ValueError(w_dtype)


def alpha_grid() -> np.ndarray:
    """The smoothing strengths searched: 0 to 1 at an interval of 0.05 (PAPER.md:166
    "grid search with an interval of 0.05 between 0 and 1"), 21 values,
    each the double nearest to i/20."""
    return np.array([i / 20.0 for i in range(21)], dtype=np.float64)


def layer_loss(X: np.ndarray, W: np.ndarray, alpha: float, group: int = 128,
               x_dtype: str = "f16", act_max=None) -> float:
    """Eq. 4 of one smoothed, quantized layer:
        E(α) = || X·W - X̂_α·Ŵ_α ||²,  X̂_α = RN(X/s_α) (Eq. 5 activation side),
        Ŵ_α = dequant(Q(RN(W·s_α))) (Eq. 5 weight side + Eq. 1), s_α from Eq. 6
    with act_max taken over the same X unless given.  Everything after the two stored
    roundings (X̂, the codes/Δ/Z) is exact fp64."""
    x = _as_f64(X, x_dtype)
    if act_max is None:
        act_max = act_absmax(X, x_dtype)
    s = smooth_scales(weight_absmax(W), act_max, alpha)
    q = quantize_pack(W, s, group)
    x_hat = _as_f64(smooth_activations(X, s, x_dtype), x_dtype)
    D = x @ _as_f64(W, "f16").T - x_hat @ dequant(q["Wq"], q["scales"], q["zeros"], group).T
    return float((D * D).sum())


def alpha_search(X: np.ndarray, W: np.ndarray, group: int = 128, x_dtype: str = "f16",
                 alphas=None):
    """Grid search of the smoothing strength for ONE layer: the α of
    the grid with the smallest Eq. 4 loss; ties go to the smallest α (the first minimum
    in grid order).  The paper minimizes the loss of the entire model;
    the per-layer objective is this repo's reading.
    Returns (best_alpha, losses fp64[len(alphas)])."""
    alphas = alpha_grid() if alphas is None else np.asarray(alphas, dtype=np.float64)
    am = act_absmax(X, x_dtype)
    losses = np.array([layer_loss(X, W, float(a), group, x_dtype, am) for a in alphas])
    best = int(np.argmin(losses))  # numpy argmin returns the first minimum
    return float(alphas[best]), losses


def footprint_ratio(N: int, K: int, group: int = 128, zeros_u4: bool = False) -> float:
    """Bytes of the W4 layout (codes + fp16 Δ + fp16 or u4 Z per group) over fp16 bytes
    ("reducing the memory footprint by approximately 75%")."""
    packed = N * K / 2 + 2 * N * (K // group) + (0.5 if zeros_u4 else 2) * N * (K // group)
    return packed / (2.0 * N * K)
