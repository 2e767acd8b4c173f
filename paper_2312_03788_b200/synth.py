"""Seeded synthetic inputs shaped like the paper's workloads.

This module holds ONLY random draws -- none of the method's arithmetic -- so that
both the CUDA path and the CPU oracle (tests) can consume identical bits.

Recipe:
  * W ~ N(0, 0.02^2) -> fp16 [N][K]  (SPEC.md:243 fixture recipe; PAPER.md:120
    Fig. 1: weight "mean ... below 0.3, and the maximum value is below 2.5").
    The "heavy" variant sets 0.01 % of entries to ±U(0.5, 2.5).
  * calibration activations X ~ N(0, 1), T_cal = 164 x 128 rows (PAPER.md:166:
    164 HumanEval prompts; 128 tokens/prompt is our choice), with 8 fixed
    seeded outlier channels scaled x100 ("100 times").
  * GEMM activations: a fresh draw of the same distribution.
  * edge groups for the quantizer: constants, one-sided, exact ties,
    subnormals, ±65504, -0.0, NaN/Inf.
"""

from __future__ import annotations

import numpy as np

N_OUTLIER_CHANNELS = 8
OUTLIER_GAIN = 100.0
T_CAL = 164 * 128


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def weights(N: int, K: int, seed: int, heavy: bool = False) -> np.ndarray:
    """fp16 W[N][K] ~ N(0, 0.02^2)."""
    g = rng(seed)
    w = g.normal(0.0, 0.02, size=(N, K))
    if heavy:
        n_heavy = max(1, int(round(N * K * 1e-4)))
        idx = g.choice(N * K, size=n_heavy, replace=False)
        w.reshape(-1)[idx] = g.uniform(0.5, 2.5, size=n_heavy) * g.choice([-1.0, 1.0], size=n_heavy)
    return w.astype(np.float16)


def outlier_channels(K: int, seed: int) -> np.ndarray:
    g = rng(seed + 7919)
    return np.sort(g.choice(K, size=min(N_OUTLIER_CHANNELS, K), replace=False))


def activations(T: int, K: int, seed: int, outlier_seed: int | None = None) -> np.ndarray:
    """fp32 X[T][K] ~ N(0, 1) with N_OUTLIER_CHANNELS fixed channels x100.
    The outlier channels depend only on (K, outlier_seed), so calibration and
    GEMM draws share them ("outliers always appear in a small number
    of fixed channels")."""
    g = rng(seed)
    x = g.normal(0.0, 1.0, size=(T, K))
    ch = outlier_channels(K, seed if outlier_seed is None else outlier_seed)
    x[:, ch] *= OUTLIER_GAIN
    return x.astype(np.float32)


def edge_groups(group: int, seed: int) -> np.ndarray:
    """fp16 [R][group] rows exercising the degenerate / rounding corners of Eq. 1.
    All finite (the NaN/Inf path has its own helper)."""
    g = rng(seed)
    rows = []
    f16 = np.float16
    rows.append(np.zeros(group))                                   # constant 0
    rows.append(np.full(group, 0.25))                              # constant +c
    rows.append(np.full(group, -0.25))                             # constant -c
    rows.append(np.full(group, -0.0))                              # all -0.0
    z = np.zeros(group); z[::2] = -0.0; rows.append(z)             # mixed ±0
    rows.append(np.full(group, 6.0e-8))                            # subnormal constant
    rows.append(g.uniform(1.0, 2.0, size=group))                   # one-sided positive
    rows.append(g.uniform(-3.0, -0.5, size=group))                 # one-sided negative
    t = np.resize([-0.8125, 1.0625, 0.3125], group); rows.append(t)  # exact RHA ties (P2)
    rows.append(np.resize([-65504.0, 65504.0, 0.0, 1.0], group))   # fp16 extremes
    rows.append(np.resize([65504.0, 65504.0, 65504.0, 65280.0], group))  # huge one-sided
    sub = g.integers(-1023, 1024, size=group) * 2.0 ** -24; rows.append(sub)  # subnormal range
    tiny = np.zeros(group); tiny[0] = 2.0 ** -24; rows.append(tiny)  # r/15 underflows
    rows.append(np.resize([0.0, 2.0 ** -24, 3 * 2.0 ** -24], group))
    grid = g.integers(0, 16, size=group) * 0.125 - 0.875; rows.append(grid)  # on-grid values
    rows.append(g.normal(0.0, 0.02, size=group))                   # typical
    rows.append(g.normal(0.0, 0.02, size=group) * 100.0)           # wide
    rand_bits = g.integers(0, 0x7C00, size=group).astype(np.uint16)  # random finite fp16
    rand_bits |= (g.integers(0, 2, size=group).astype(np.uint16) << 15)
    rows.append(rand_bits.view(np.float16).astype(np.float64))
    for _ in range(8):                                             # near-tie constructions
        d = f16(g.uniform(0.001, 0.1))
        k = g.integers(-7, 8, size=group)
        v = ((k + 0.5) * float(d)).astype(np.float16)
        v[0] = f16(-7.5 * float(d)); v[1] = f16(7.5 * float(d))
        rows.append(v.astype(np.float64))
    return np.stack([np.asarray(r, dtype=np.float64) for r in rows]).astype(np.float16)


def nonfinite_groups(group: int) -> np.ndarray:
    rows = []
    for bad in (np.nan, np.inf, -np.inf):
        r = np.linspace(-1, 1, group)
        r[group // 3] = bad
        rows.append(r)
    return np.stack(rows).astype(np.float16)
