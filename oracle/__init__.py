"""CPU oracle for the SmoothQuant+ W4A16 hot path (arxiv 2312.03788).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import anything
under ``oracle/``.  The product path (``paper_2312_03788_b200``) never imports it
and shares no code, header, table or constant generator with it.

Everything here is plain, slow and written to be checked by eye against the
paper (``/root/reference/PAPER.md``, cited as PAPER.md:<line>):

* fp64 throughout, except where a step explicitly rounds to fp16/fp32;
* no blocking, fusion or reordering beyond what Eq. 1-6 state;
* each function cites the passage it follows.

Readings of points where the paper is silent (tie rule, Δ precision, zero point,
degenerate groups, ...) are listed in DESIGN.md §3 and SURVEY.md §8(c) S1-S17.

Pinning status (see DESIGN.md §3 and tests/test_oracle_pins.py):
  weight_absmax, act_absmax, smooth_scales, fold, quantize_group,
  quantize_pack, pack/unpack, dequant, gemm  -- pinned.
  smooth_activations, alpha_grid, layer_loss,
  alpha_search (N2)                          -- pinned (exact-rational X̂, zero-loss
                                               layer + tie rule, permutation invariance).
  gemm summation order                      -- parity unpinned beyond tolerance
                                               (any order is a correct result).
"""

from .sq_oracle import (  # noqa: F401
    EPS,
    act_absmax,
    weight_absmax,
    smooth_scales,
    smooth_weight_exact,
    fold,
    rz_fp16,
    rn_bf16_bits,
    rha,
    quantize_group,
    quantize_pack,
    pack_nibbles,
    unpack_nibbles,
    pack_zeros_u4,
    unpack_zeros_u4,
    dequant,
    gemm,
    quant_loss,
    smooth_activations,
    fold_rows,
    alpha_grid,
    layer_loss,
    alpha_search,
    footprint_ratio,
    NONFINITE_SCALE_BITS,
)
