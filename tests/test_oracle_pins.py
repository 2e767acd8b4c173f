"""Pins of the CPU oracle against what the paper and the mathematics fix
(SURVEY.md §8(c) P1-P14).  No GPU, no CUDA library: these run with -m "not gpu".

Each test names the pin and the passage it follows.  None of them re-types the
oracle's own formula; they check worked examples, closed forms, invariants,
brute force and a third exact-rational implementation (tests/exact_rational.py).
"""

from __future__ import annotations

import itertools
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_2312_03788_b200 import synth
from tests import exact_rational as ex

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "eq1_worked_examples.json")


def _golden():
    with open(GOLDEN) as f:
        return json.load(f)


def _bits(x: float) -> int:
    return int(np.float16(x).view(np.uint16))


# ---------------------------------------------------------------- P1-P4
@pytest.mark.parametrize("case", _golden()["cases"], ids=lambda c: c["name"])
def test_p1_p4_eq1_worked_examples(case):
    """P1-P4: Eq. 1 worked examples."""
    vals = np.array(case["values"], dtype=np.float16).astype(np.float64)
    codes, delta, Z = oracle.quantize_group(vals)
    assert codes == case["codes"]
    assert _bits(delta) == int(case["delta_bits"], 16)
    assert Z == case["Z"]
    if "dequant" in case:
        deq = [(c - Z) * delta for c in codes]
        assert deq == case["dequant"]


# ---------------------------------------------------------------- P5
def test_p5_packing_example_and_exhaustive():
    """P5: nibble packing."""
    g = _golden()["packing"]
    assert oracle.pack_nibbles(np.array(g["codes"])).tolist() == g["bytes"]
    pairs = np.array(list(itertools.product(range(16), repeat=2)))
    packed = oracle.pack_nibbles(pairs.reshape(-1))
    assert packed.size == 256 and len(set(packed.tolist())) == 256
    assert (oracle.unpack_nibbles(packed) == pairs.reshape(-1)).all()
    # element 2i is the LOW nibble: a lone code at an even position stays < 16
    assert oracle.pack_nibbles(np.array([7, 0])).tolist() == [0x07]
    assert oracle.pack_nibbles(np.array([0, 7])).tolist() == [0x70]
    with pytest.raises(ValueError):
        oracle.pack_nibbles(np.array([16, 0]))


# ---------------------------------------------------------------- P6
@pytest.mark.parametrize("case", _golden()["eq6"]["cases"])
def test_p6_eq6_values(case):
    """P6: Eq. 6 values and endpoints."""
    s = oracle.smooth_scales(np.array([case["w_max"]]), np.array([case["act_max"]], np.float32),
                             case["alpha"])
    assert s.dtype == np.float32
    assert float(s[0]) == case["s"]


def test_p6_eq6_general_alpha_closed_form():
    """Eq. 6 for general α against the independent form exp(α ln a - (1-α) ln w)
    (2 ulp of fp32), and the α=1 / α=0 endpoints of PAPER.md:160."""
    g = synth.rng(3)
    a = np.float32(g.uniform(1e-3, 2e3, size=2000)).astype(np.float32)
    w = g.uniform(1e-3, 2.5, size=2000)
    for alpha in (0.05, 0.35, 0.8, 0.95):
        s = oracle.smooth_scales(w, a, alpha).astype(np.float64)
        ref = np.exp(alpha * np.log(a.astype(np.float64)) - (1 - alpha) * np.log(w))
        ulp = np.spacing(ref.astype(np.float32)).astype(np.float64)
        assert (np.abs(s - ref) <= 2 * ulp).all()
    assert (oracle.smooth_scales(w, a, 1.0) == a).all()
    assert (oracle.smooth_scales(w, a, 0.0) == (1.0 / w).astype(np.float32)).all()
    # α = 1: every smoothed activation channel has maximum 1 (PAPER.md:160
    # "all activation channels have the same maximum value of 1")
    s1 = oracle.smooth_scales(w, a, 1.0).astype(np.float64)
    assert np.allclose(a / s1, 1.0, rtol=0, atol=0)


def test_eq6_eps_floor():
    """Reading S10: dead channels are floored at ε = 1e-5 on both maxima."""
    s = oracle.smooth_scales(np.array([0.0, 1.0]), np.array([1.0, 0.0], np.float32), 0.5)
    assert float(s[0]) == np.float32(math.sqrt(1.0) / math.sqrt(1e-5))
    assert float(s[1]) == np.float32(math.sqrt(1e-5) / math.sqrt(1.0))


def test_absmax_brute_force():
    """O2 / calibration statistic: per-channel max |.| by explicit loops."""
    W = synth.weights(7, 256, seed=1)
    wm = oracle.weight_absmax(W)
    for k in range(256):
        assert wm[k] == max(abs(float(W[n, k])) for n in range(7))
    X = synth.activations(9, 64, seed=2)
    am = oracle.act_absmax(X.astype(np.float16))
    for k in range(64):
        assert am[k] == np.float32(max(abs(float(np.float16(X[t, k]))) for t in range(9)))


# ---------------------------------------------------------------- P7
@pytest.mark.parametrize("N,K", [(48, 64), (64, 64)])
def test_p7_eq5_equivalence(N, K):
    """P7: Y = (X diag(s)^-1)(diag(s) W) with the oracle's fold
    axis.  N == K catches a fold along the wrong (output) axis."""
    g = synth.rng(11)
    X = g.normal(size=(5, K))
    W = synth.weights(N, K, seed=4)
    s = np.float32(np.exp(g.uniform(np.log(1e-3), np.log(1e3), size=K))).astype(np.float32)
    lhs = X @ W.astype(np.float64).T
    rhs = (X / s.astype(np.float64)) @ oracle.smooth_weight_exact(W, s).T
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(lhs)


def test_fold_is_single_rounding_of_exact_product():
    """Reading S13: W' = RN16(w·s) computed from the exact rational product."""
    g = synth.rng(5)
    W = synth.weights(4, 128, seed=9, heavy=True)
    s = g.uniform(0.01, 50.0, size=128).astype(np.float32)
    Wf = oracle.fold(W, s)
    for n in range(4):
        for k in range(0, 128, 3):
            exact = Fraction(float(W[n, k])) * Fraction(float(s[k]))
            r = ex.rn_f16(exact)
            assert r is not None and Fraction(Wf[n, k]) == r


def test_rz_fp16_against_exact():
    g = synth.rng(6)
    xs = np.concatenate([g.uniform(0, 1, 500) * 10.0 ** g.integers(-9, 5, 500),
                         [2.0 ** -25, 2.0 ** -24, 65504.0, 65519.0, 1e-9]])
    h = oracle.rz_fp16(xs)
    for x, y in zip(xs, h):
        assert Fraction(float(y)) == ex.rz_f16(Fraction(float(x)))


def test_rha_ties():
    assert oracle.rha(np.array([0.5, 1.5, 2.5, -0.5, -2.5, 0.49999999999999994, -0.0])).tolist() == \
        [1.0, 2.0, 3.0, -1.0, -3.0, 0.0, 0.0]


# ---------------------------------------------------------------- P8-P10
def _groups_for_invariants():
    g = synth.rng(21)
    gauss = synth.weights(2000, 128, seed=22).astype(np.float64)
    edge = synth.edge_groups(128, seed=23).astype(np.float64)
    return np.concatenate([gauss, edge])


def _straddles_or_constant(v):
    return (v.min() <= 0 <= v.max()) or (v.min() == v.max())


def test_p8_idempotence():
    """P8: Q(D(Q(W))) == Q(W) with D exact (BASELINE.json north_star
    'quantize->dequantize idempotence'), for zero-straddling / constant groups."""
    V = _groups_for_invariants()
    for v in V:
        if not _straddles_or_constant(v):
            continue
        c1, d1, z1 = oracle.quantize_group(v)
        # D is exact in fp64 ((c-Z)·Δ has <= 15 significant bits); re-quantize
        # those exact values (an fp16-rounded D is not idempotent)
        deq = np.array([(c - z1) * d1 for c in c1])
        c2, d2, z2 = oracle.quantize_group(deq)
        assert (c1, _bits(d1), z1) == (c2, _bits(d2), z2)


def test_p9_ranges():
    """P9: codes and Z in [0, 15]; Δ > 0 finite (PAPER.md:89 clamp to [0, 2^N-1])."""
    V = _groups_for_invariants()
    for v in V:
        c, d, z = oracle.quantize_group(v)
        assert all(0 <= x <= 15 for x in c) and 0 <= z <= 15
        assert d > 0 and math.isfinite(d)


def test_p10_brute_force_min_error():
    """P10: each element's reconstruction is the nearest grid point (ties allowed),
    and zero-straddling groups obey |v - Ŵ| <= Δ/2 + max(0, r - 15Δ)."""
    V = _groups_for_invariants()
    for v in V:
        c, d, z = oracle.quantize_group(v)
        grid = np.array([(k - z) * d for k in range(16)])
        rec = np.array([(k - z) * d for k in c])
        err = np.abs(v - rec)
        best = np.abs(v[:, None] - grid[None, :]).min(axis=1)
        assert (err <= best).all()
        if v.min() < 0 < v.max():
            r = v.max() - v.min()
            assert (err <= d / 2 + max(0.0, r - 15 * d)).all()


# ---------------------------------------------------------------- P11
def test_p11_exact_rational_tiny_groups():
    """P11: the fp64 oracle equals an exact Fraction quantizer on tiny groups
    (random fp16 bit patterns, near ties, subnormals, ±65504)."""
    g = synth.rng(31)
    cases = []
    for size in (1, 2, 3, 4, 8):
        for _ in range(300):
            bits = g.integers(0, 0x7C00, size=size).astype(np.uint16)
            bits |= (g.integers(0, 2, size=size).astype(np.uint16) << 15)
            cases.append(bits.view(np.float16).astype(np.float64))
    for _ in range(300):  # constructed near-ties: v = (k + 1/2)·Δ rounded to fp16
        d = float(np.float16(g.uniform(1e-4, 1.0)))
        k = g.integers(-8, 8, size=4)
        v = ((k + 0.5) * d).astype(np.float16).astype(np.float64)
        cases.append(np.concatenate([v, [-7.5 * d, 7.5 * d]]).astype(np.float16).astype(np.float64))
    for _ in range(100):  # subnormal ranges
        cases.append((g.integers(-1023, 1024, size=4) * 2.0 ** -24))
    cases.append(np.array([-65504.0, 65504.0]))
    cases.append(np.array([65504.0, 65504.0, 1.0]))
    for v in cases:
        c1, d1, z1 = oracle.quantize_group(v)
        c2, d2, z2 = ex.quantize_group([float(x) for x in v])
        assert c1 == c2 and z1 == z2 and Fraction(d1) == d2, v


# ---------------------------------------------------------------- P12
def test_p12_footprint():
    """P12: fp16 Δ + fp16 Z at g=128 -> 0.265625 of fp16 bytes (PAPER.md:74 ~75% saved)."""
    f = _golden()["footprint"]
    assert oracle.footprint_ratio(f["N"], f["K"], f["group"]) == f["ratio"]
    # and the layout really has that many bytes
    q = oracle.quantize_pack(synth.weights(16, 256, seed=1), None, 128)
    nbytes = q["Wq"].nbytes + q["scales"].nbytes + q["zeros"].nbytes
    assert nbytes / (16 * 256 * 2) == f["ratio"]


# ---------------------------------------------------------------- P13
def test_p13_gemm_special_cases_and_brute_force():
    """P13 + Eq. 2/3 orientation: Y[m][n] = sum_k X[m][k] Ŵ[n][k]
    (PAPER.md:95-106), checked with explicit loops."""
    N, K = 24, 256
    W = synth.weights(N, K, seed=41)
    q = oracle.quantize_pack(W, None, 128)
    What = oracle.dequant(q["Wq"], q["scales"], q["zeros"], 128)
    # dequant brute force from the stored bits
    codes = oracle.unpack_nibbles(q["Wq"])
    for n in range(0, N, 5):
        for k in range(0, K, 7):
            gi = k // 128
            d = float(np.uint16(q["scales"][gi, n]).view(np.float16))
            z = float(np.uint16(q["zeros"][gi, n]).view(np.float16))
            assert What[n, k] == (codes[n, k] - z) * d
    # identity: Y = Ŵ^T
    Xi = np.eye(K, dtype=np.float16)
    assert (oracle.gemm(Xi, q["Wq"], q["scales"], q["zeros"]) == What.T).all()
    # zero
    assert (oracle.gemm(np.zeros((3, K), np.float16), q["Wq"], q["scales"], q["zeros"]) == 0).all()
    # brute force
    X = synth.activations(3, K, seed=42).astype(np.float16)
    Y = oracle.gemm(X, q["Wq"], q["scales"], q["zeros"])
    for m in range(3):
        for n in range(0, N, 3):
            acc = math.fsum(float(X[m, k]) * What[n, k] for k in range(K))
            assert abs(Y[m, n] - acc) <= 1e-12 * max(1.0, abs(acc))


def test_quantize_pack_matches_groupwise_loop():
    """quantize_pack == quantize_group applied per (n, group of 128 consecutive k)
    (reading S6), including the smoothing fold."""
    g = synth.rng(51)
    N, K = 6, 384
    W = synth.weights(N, K, seed=52, heavy=True)
    s = g.uniform(0.1, 10, size=K).astype(np.float32)
    q = oracle.quantize_pack(W, s, 128)
    for n in range(N):
        for gi in range(K // 128):
            v = [float(np.float16(float(W[n, k]) * float(s[k])))
                 for k in range(gi * 128, (gi + 1) * 128)]
            c, d, z = ex.quantize_group(v)
            assert q["codes"][n, gi * 128:(gi + 1) * 128].tolist() == c
            assert Fraction(float(np.uint16(q["scales"][gi, n]).view(np.float16))) == d
            assert float(np.uint16(q["zeros"][gi, n]).view(np.float16)) == z


def test_nonfinite_groups_encoding():
    """a group with NaN/Inf after the fold gets scale NaN (0x7E00),
    zero 0, codes 0 and is counted; the others are unaffected."""
    bad = synth.nonfinite_groups(128)
    good = synth.weights(1, 128, seed=3)
    W = np.concatenate([bad, good]).astype(np.float16)
    q = oracle.quantize_pack(W, None, 128)
    assert q["nonfinite"] == 3
    assert q["scales"][0, :3].tolist() == [0x7E00] * 3
    assert (q["zeros"][0, :3] == 0).all() and (q["codes"][:3] == 0).all()
    ref = oracle.quantize_pack(good, None, 128)
    assert q["scales"][0, 3] == ref["scales"][0, 0]
    # overflow of the fold is non-finite too (O5)
    q2 = oracle.quantize_pack(np.full((1, 128), 60000, np.float16), np.full(128, 2.0, np.float32))
    assert q2["nonfinite"] == 1
    with pytest.raises(ValueError):
        oracle.quantize_group([1.0, float("nan")])


# ---------------------------------------------------------------- Eq. 4
def test_eq4_loss_properties():
    """Eq. 4: ≥0; zero on exactly representable W; X×10 -> ×100."""
    K, N = 128, 8
    g = synth.rng(61)
    grid = (g.integers(0, 16, size=(N, K)) - 7) * 0.125
    grid[:, 0] = -0.875
    grid[:, 1] = 1.0
    W = grid.astype(np.float16)
    q = oracle.quantize_pack(W, None, 128)
    What = oracle.dequant(q["Wq"], q["scales"], q["zeros"])
    X = g.normal(size=(4, K))
    assert oracle.quant_loss(X, W.astype(np.float64), What) == 0.0
    W2 = synth.weights(N, K, seed=62)
    q2 = oracle.quantize_pack(W2, None, 128)
    W2h = oracle.dequant(q2["Wq"], q2["scales"], q2["zeros"])
    l1 = oracle.quant_loss(X, W2.astype(np.float64), W2h)
    l10 = oracle.quant_loss(10 * X, W2.astype(np.float64), W2h)
    assert l1 > 0 and abs(l10 - 100 * l1) <= 1e-9 * l10


def test_smoothing_reduces_loss_under_outliers():
    """smoothing before quantization lowers Eq. 4's loss
    when activations carry ×100 outlier channels (the paper's core claim, on
    synthetic data)."""
    K, N = 512, 256
    Xc = synth.activations(2048, K, seed=71)
    W = synth.weights(N, K, seed=72)
    am = oracle.act_absmax(Xc.astype(np.float16))
    wm = oracle.weight_absmax(W)
    X = synth.activations(64, K, seed=73, outlier_seed=71).astype(np.float64)
    q0 = oracle.quantize_pack(W, None, 128)
    l_rtn = oracle.quant_loss(X, W.astype(np.float64), oracle.dequant(q0["Wq"], q0["scales"], q0["zeros"]))
    s = oracle.smooth_scales(wm, am, 0.5)
    q1 = oracle.quantize_pack(W, s, 128)
    What_s = oracle.dequant(q1["Wq"], q1["scales"], q1["zeros"]) / s.astype(np.float64)[None, :]
    l_sq = oracle.quant_loss(X, W.astype(np.float64), What_s)
    assert l_sq < l_rtn


# ---------------------------------------------------------------- P14
def test_p14_tp_shards():
    """P14: column shards quantize bit-identically to their rows; group-aligned
    row shards too; the sum of row-shard partial GEMMs equals the full GEMM."""
    N, K = 64, 768
    W = synth.weights(N, K, seed=81)
    s = synth.rng(82).uniform(0.5, 2, size=K).astype(np.float32)
    full = oracle.quantize_pack(W, s, 128)
    col = oracle.quantize_pack(W[16:48], s, 128)
    assert (col["Wq"] == full["Wq"][16:48]).all()
    assert (col["scales"] == full["scales"][:, 16:48]).all()
    row = oracle.quantize_pack(W[:, 256:640], s[256:640], 128)
    assert (row["Wq"] == full["Wq"][:, 128:320]).all()
    assert (row["scales"] == full["scales"][2:5]).all()
    X = synth.activations(4, K, seed=83).astype(np.float16)
    Y = oracle.gemm(X, full["Wq"], full["scales"], full["zeros"])
    parts = 0
    for k0, k1 in ((0, 256), (256, 640), (640, 768)):
        p = oracle.quantize_pack(W[:, k0:k1], s[k0:k1], 128)
        parts = parts + oracle.gemm(X[:, k0:k1], p["Wq"], p["scales"], p["zeros"])
    assert np.allclose(parts, Y, rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- N2: α grid search
def test_n2_alpha_grid():
    """PAPER.md:166 / :213: grid over [0, 1] at an interval of 0.05 -> 21 points."""
    g = oracle.alpha_grid()
    assert len(g) == 21 and g[0] == 0.0 and g[-1] == 1.0
    assert np.allclose(np.diff(g), 0.05, atol=1e-15, rtol=0)
    assert [Fraction(x).limit_denominator(20) for x in g] == [Fraction(i, 20) for i in range(21)]


def test_n2_smooth_activations_exact_rational():
    """X̂ = X·diag(s)^-1 (Eq. 5), stored once-rounded: the oracle's
    fp64 route equals the exact-rational RN16 of x / s (third implementation), including
    power-of-two s (exact scaling), s = 1 (identity) and random fp32 s."""
    r = np.random.default_rng(11)
    x = r.standard_normal((6, 64)).astype(np.float16)
    x[0, :8] = np.array([0.0, -0.0, 65504.0, -65504.0, 6e-8, -6e-8, 1.0, 2049.0], dtype=np.float16)
    for s in (np.full(64, 1.0, np.float32), np.full(64, 0.25, np.float32),
              r.uniform(1e-3, 1e3, 64).astype(np.float32), r.uniform(0.9, 1.1, 64).astype(np.float32)):
        got = oracle.smooth_activations(x, s)
        for (i, k), xv in np.ndenumerate(x):
            want = ex.rn_f16(Fraction(float(xv)) / Fraction(float(s[k])))
            g = float(got[i, k])
            if want is None:
                assert np.isinf(g)
            else:
                assert Fraction(g) == want, (i, k, float(xv), float(s[k]))
    assert np.array_equal(oracle.smooth_activations(x, np.ones(64, np.float32)).view(np.uint16), x.view(np.uint16))


def _exact_layer(N=16, K=256, T=8, seed=3):
    """A layer the pipeline reproduces exactly: every column max |W_k| = 1 and max |X_k| = 1
    (so s = 1 for every α by Eq. 6), every group on the grid (q - 8)·0.125 with both q = 0
    and q = 15 present (so Δ = 0.125, Z = 8 and Ŵ = W by Eq. 1)."""
    r = np.random.default_rng(seed)
    q = r.integers(0, 16, size=(N, K))
    q[0, 0::2], q[0, 1::2] = 0, 15
    q[1, 0::2], q[1, 1::2] = 15, 0
    W = ((q - 8) * 0.125).astype(np.float16)
    X = r.uniform(-1, 1, size=(T, K))
    X[0, :] = 1.0
    return X.astype(np.float16), W


def test_n2_zero_loss_layer_and_tie_rule():
    """Eq. 4 special case: when smoothing is the identity (s = 1) and W lies on the Eq. 1
    grid, X̂ = X and Ŵ = W exactly, so E(α) = 0 for every α; all 21 tie and the search
    returns the smallest α (the tie rule).  X = 0 likewise gives E = 0 everywhere."""
    X, W = _exact_layer()
    best, losses = oracle.alpha_search(X, W)
    assert best == 0.0 and np.all(losses == 0.0)
    best0, losses0 = oracle.alpha_search(np.zeros_like(X), W)
    assert best0 == 0.0 and np.all(losses0 == 0.0)


def test_n2_loss_invariant_under_channel_permutations():
    """Eq. 4-6 are per input channel and per output channel: permuting whole groups of
    input channels (X and W columns together) or output channels (W rows) permutes s
    and the quantization groups but leaves every E(α) unchanged.  A fold or smoothing
    along the wrong axis breaks this (N == K here)."""
    X = synth.activations(32, 384, seed=5).astype(np.float16)
    W = synth.weights(384, 384, seed=6)
    a = [0.0, 0.35, 0.5, 1.0]
    _, base = oracle.alpha_search(X, W, alphas=a)
    pg = np.array([2, 0, 1])
    cols = np.concatenate([np.arange(g * 128, (g + 1) * 128) for g in pg])
    _, pk = oracle.alpha_search(X[:, cols], W[:, cols], alphas=a)
    rows = np.random.default_rng(0).permutation(384)
    _, pn = oracle.alpha_search(X, W[rows], alphas=a)
    np.testing.assert_allclose(pk, base, rtol=1e-12)
    np.testing.assert_allclose(pn, base, rtol=1e-12)
    assert not np.allclose(base[0], base[2])  # α matters on this data


def test_n2_search_under_outliers():
    """×100 outlier channels amplify the weight quantization error; the
    search picks an interior α whose loss is below both endpoints and below RTN (s = 1,
    PAPER.md:206), and it is the argmin of the grid."""
    X = synth.activations(64, 512, seed=7).astype(np.float16)
    W = synth.weights(256, 512, seed=8)
    best, losses = oracle.alpha_search(X, W)
    assert 0.0 < best < 1.0
    assert losses[int(round(best * 20))] == losses.min()
    assert losses.min() < losses[0] and losses.min() < losses[-1]
    q = oracle.quantize_pack(W, None)
    x = X.astype(np.float64)
    rtn = float(((x @ W.astype(np.float64).T - x @ oracle.dequant(q["Wq"], q["scales"], q["zeros"]).T) ** 2).sum())
    assert losses.min() < rtn


# ---------------------------------------------------------------- N3: model-level fusion
def test_n3_fold_rows_exact_rational_and_mlp_equivalence():
    """Fig. 5: dividing down_proj's input by s is fused into up_proj's
    output rows, and down_proj's weights take s on their input channels.  (1) fold_rows is
    the once-rounded exact quotient (exact-rational third implementation); (2) the fused
    pair computes the same function: in fp64 with unrounded weights the results agree to
    1e-12 relative, and with the stored fp16 weights within the two roundings' bound."""
    r = np.random.default_rng(21)
    Wup = (r.standard_normal((256, 128)) * 0.02).astype(np.float16)      # [N=256][K=128]
    Wdn = (r.standard_normal((64, 256)) * 0.02).astype(np.float16)       # consumer, K = 256
    s = r.uniform(0.05, 20.0, 256).astype(np.float32)
    got = oracle.fold_rows(Wup, s)
    for (n, k), wv in np.ndenumerate(Wup[:16]):
        want = ex.rn_f16(Fraction(float(wv)) / Fraction(float(s[n])))
        assert Fraction(float(got[n, k])) == want
    x = r.standard_normal((8, 128))
    ref = (x @ Wup.astype(np.float64).T) @ Wdn.astype(np.float64).T
    exact = (x @ (Wup.astype(np.float64) / s.astype(np.float64)[:, None]).T) @ \
        (Wdn.astype(np.float64) * s.astype(np.float64)[None, :]).T
    assert np.linalg.norm(exact - ref) <= 1e-12 * np.linalg.norm(ref)
    stored = (x @ got.astype(np.float64).T) @ oracle.fold(Wdn, s).T
    assert np.linalg.norm(stored - ref) <= 2e-3 * np.linalg.norm(ref)


def _bf16_bits_to_fraction(b: int):
    v = float(np.array([int(b) << 16], dtype=np.uint32).view(np.float32)[0])
    return v, (Fraction(v) if np.isfinite(v) else None)


def test_rn_bf16_bits_against_exact():
    """oracle.rn_bf16_bits decides every bf16 bit-exact test (S17 fold, bf16 X/s, bf16
    fold_rows).  Pinned here against an exact-rational RN-even to bf16 (third
    implementation, tests/exact_rational.py) on random fp64 values over the whole bf16
    exponent range, exact midpoints (ties to even), subnormal values and ties,
    the overflow threshold, signed zeros and non-finite inputs."""
    r = np.random.default_rng(2024)
    xs = list(r.standard_normal(600) * 2.0 ** r.integers(-140, 128, 600))
    # exact midpoints between consecutive bf16 values (normal and subnormal binades),
    # and values one fp64 ulp either side of them
    for _ in range(300):
        e = int(r.integers(-133, 127))
        m = int(r.integers(0, 256))
        q = 2.0 ** (max(e, -126) - 7) if e >= -126 else 2.0 ** -133
        base = (m + (128 if e >= -126 else 0)) * q
        mid = base + q / 2
        for v in (mid, np.nextafter(mid, 0.0), np.nextafter(mid, np.inf)):
            xs.append(float(v) * (1 if r.integers(0, 2) else -1))
    big = float((2 - 2.0 ** -7) * 2.0 ** 127)
    thr = float((2 - 2.0 ** -8) * 2.0 ** 127)            # midpoint BF16_MAX .. 2^128
    xs += [big, -big, thr, -thr, float(np.nextafter(thr, 0.0)), 2.0 ** -133, 2.0 ** -134,
           float(np.nextafter(2.0 ** -134, 1.0)), 3 * 2.0 ** -134, 1e-45, 1.0, -1.0]
    got = oracle.rn_bf16_bits(np.array(xs, dtype=np.float64))
    for x, b in zip(xs, got):
        want = ex.rn_bf16(Fraction(x))
        v, fv = _bf16_bits_to_fraction(b)
        if want is None:
            assert np.isinf(v) and np.signbit(v) == (x < 0), x
        else:
            assert fv == want, (x, hex(int(b)))
            if want == 0:
                assert np.signbit(v) == np.signbit(x), x   # sign of zero kept
    # special values
    sp = oracle.rn_bf16_bits(np.array([0.0, -0.0, np.inf, -np.inf, np.nan]))
    assert [int(v) for v in sp[:4]] == [0x0000, 0x8000, 0x7F80, 0xFF80]
    assert (int(sp[4]) & 0x7F80) == 0x7F80 and (int(sp[4]) & 0x007F) != 0


@pytest.mark.parametrize("group", [32, 64])
def test_n3_group_sizes_match_groupwise_loop(group):
    """N3 ("Support group-wise quantization for different group sizes"):
    quantize_pack with g = 32 / 64 equals the exact-rational Eq. 1 quantizer applied to every
    (n, group of g consecutive k) (readings S1-S4, S6), including the smoothing fold; codes,
    Δ bits and Z are identical, and dequant reconstructs (q - Z)·Δ per group."""
    g = synth.rng(70 + group)
    N, K = 5, 256
    W = synth.weights(N, K, seed=71, heavy=True)
    s = g.uniform(0.1, 10, size=K).astype(np.float32)
    q = oracle.quantize_pack(W, s, group)
    assert q["scales"].shape == (K // group, N)
    for n in range(N):
        for gi in range(K // group):
            v = [float(np.float16(float(W[n, k]) * float(s[k]))) for k in range(gi * group, (gi + 1) * group)]
            c, d, z = ex.quantize_group(v)
            assert q["codes"][n, gi * group:(gi + 1) * group].tolist() == c
            assert Fraction(float(np.uint16(q["scales"][gi, n]).view(np.float16))) == d
            assert float(np.uint16(q["zeros"][gi, n]).view(np.float16)) == z
    What = oracle.dequant(q["Wq"], q["scales"], q["zeros"], group)
    codes = oracle.unpack_nibbles(q["Wq"])
    for n in range(N):
        for k in (0, group - 1, group, K - 1):
            gi = k // group
            d = float(np.uint16(q["scales"][gi, n]).view(np.float16))
            z = float(np.uint16(q["zeros"][gi, n]).view(np.float16))
            assert What[n, k] == (codes[n, k] - z) * d


@pytest.mark.parametrize("group", [32, 64])
def test_n3_group_sizes_idempotence_and_bound(group):
    """P8 and P10 at g = 32 / 64: Q(D(Q(W))) == Q(W) for zero-straddling groups and every
    element within Δ/2 (+ the 2^-24 floor excess) of its reconstruction."""
    W = synth.weights(64, 512, seed=72)
    q = oracle.quantize_pack(W, None, group)
    What = oracle.dequant(q["Wq"], q["scales"], q["zeros"], group)
    codes = q["codes"].reshape(-1, group)
    for i, grp in enumerate(What.reshape(-1, group)[::7]):   # every 7th group: D exact in fp64
        c2, _, _ = oracle.quantize_group(grp)
        assert c2 == codes[7 * i].tolist()
    v = W.astype(np.float64).reshape(-1, group)
    r = v.max(axis=1) - v.min(axis=1)
    d = q["delta"].T.reshape(-1)
    err = np.abs(v - What.reshape(-1, group)).max(axis=1)
    assert (err <= d / 2 + np.maximum(0.0, r - 15 * d) + 1e-12).all()


def test_n3_footprint_by_group_size():
    """P12 generalised: bytes / fp16 bytes = (0.5 + 4/g) / 2: 0.265625 (g = 128),
    0.28125 (64), 0.3125 (32), measured on the layout the quantizer writes."""
    for group, want in ((128, 0.265625), (64, 0.28125), (32, 0.3125)):
        assert oracle.footprint_ratio(64, 512, group) == want
        q = oracle.quantize_pack(synth.weights(64, 512, seed=73), None, group)
        nbytes = q["Wq"].nbytes + q["scales"].nbytes + q["zeros"].nbytes
        assert nbytes / (2.0 * 64 * 512) == want


# ---------------------------------------------------------------- N3: packed u4 zero points

def test_n3_zeros_u4_worked_example():
    """Hand-packed example (tests/golden/zeros_u4_example.json): channel 2i in the low
    nibble, 2i+1 in the high nibble, one byte row per group row."""
    f = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "zeros_u4_example.json")))
    z = np.array(f["zeros_f16_bits"], dtype=np.uint16)
    assert z.view(np.float16).astype(float).tolist() == [[1, 2, 15, 0], [3, 3, 0, 7]]
    assert oracle.pack_zeros_u4(z).tolist() == f["zeros_u4"]
    assert oracle.unpack_zeros_u4(np.array(f["zeros_u4"], dtype=np.uint8)).tolist() == z.tolist()


def test_n3_zeros_u4_roundtrip_and_same_layer():
    """Packing loses nothing: every Z the quantizer emits (integers 0..15, incl. edge and
    non-finite groups) survives pack/unpack bit for bit, so the dequantized layer and the
    GEMM are identical with either zero-point layout; the u4 layout is 3/4 smaller."""
    W = np.concatenate([synth.weights(56, 256, seed=81), synth.edge_groups(256, seed=82)[:8]])
    W[3, 5] = np.float16(np.inf)
    q = oracle.quantize_pack(W.astype(np.float16))
    assert q["nonfinite"] >= 1
    zu4 = oracle.pack_zeros_u4(q["zeros"])
    assert zu4.shape == (q["zeros"].shape[0], q["zeros"].shape[1] // 2) and zu4.dtype == np.uint8
    assert np.array_equal(oracle.unpack_zeros_u4(zu4), q["zeros"])
    X = synth.activations(3, 256, seed=83).astype(np.float16)
    ok = ~np.isnan(q["delta"]).any(axis=0)  # channels without a non-finite group
    y16 = oracle.gemm(X, q["Wq"], q["scales"], q["zeros"])
    y4 = oracle.gemm(X, q["Wq"], q["scales"], zu4, zeros_u4=True)
    assert np.array_equal(y16[:, ok], y4[:, ok])
    for group, want in ((128, 0.259765625), (32, 0.2890625)):   # (0.5 + 2.5/g) / 2
        assert oracle.footprint_ratio(64, 512, group, zeros_u4=True) == want


def test_n3_zeros_u4_rejects_non_codes():
    with pytest.raises(ValueError):
        oracle.pack_zeros_u4(np.array([[0x3C00, 0x3800]], dtype=np.uint16))   # 1, 0.5
    with pytest.raises(ValueError):
        oracle.pack_zeros_u4(np.array([[0x4C00, 0]], dtype=np.uint16))        # 16
    with pytest.raises(ValueError):
        oracle.pack_zeros_u4(np.array([[0, 0, 0]], dtype=np.uint16))          # odd N
