/*
 * libsq.h -- C ABI of the B200-native SmoothQuant+ W4A16 hot path.
 *
 * The operations follow the paper's statement of the problem
 * (/root/reference/PAPER.md, "SmoothQuant+", arxiv 2312.03788):
 *   Eq. 6  smoothing factors   s_j = max|X_j|^a / max|W_j|^(1-a)
 *   Eq. 5  weight-side fold    W' = diag(s) W
 *   Eq. 1    group-wise asymmetric INT4 quantization, g = 128
 *                             ("Group-size is usually set to be 128")
 *   Eq. 3  W4A16 linear layer  Y = X^ W^
 * Readings of points the paper leaves open are in DESIGN.md §3.
 *
 * Conventions (all calls):
 *  - Every tensor pointer is a CUDA DEVICE pointer owned by the caller.  The
 *    library never allocates device memory, never frees, and never synchronizes
 *    the host.  Every call is asynchronous on `stream` (a cudaStream_t passed as
 *    void*; NULL = legacy default stream).
 *  - Row-major throughout.  Shapes (SURVEY.md §8 notation): M = tokens, K = input
 *    channels (C_i), N = output channels (C_o), G = K / group.
 *  - Weights are stored nn.Linear-style W[N][K] (the transpose of Eq. 2's
 *    W in R^{C_i x C_o}).
 *  - Packed codes Wq[N][K/2] (uint8): element k of row n is the LOW nibble of byte
 *    Wq[n][k/2] when k is even, the HIGH nibble when k is odd.
 *  - scales[G][N] and zeros[G][N] are fp16 bit patterns (uint16), group-major:
 *    scales[gi][n] is Delta of the group (n, k in [gi*group, (gi+1)*group)).
 *    zeros hold integers 0..15 stored as fp16.  With SQ_ZEROS_U4 (SURVEY.md §8(f) N3,
 *    SPEC.md:185 "Z stored as unsigned 4-bit") zeros are instead PACKED uint8[G][N/2]: Z of channel n is
 *    the LOW nibble of byte zeros[gi][n/2] when n is even, the HIGH nibble when n is
 *    odd (the nibble order of the codes, along n; oracle/sq_oracle.py pack_zeros_u4).
 *    The packed layout needs N % 32 == 0 (16-byte rows for TMA), else SQ_ERR_ALIGN.
 *  - dtype codes: SQ_F16 (IEEE binary16) or SQ_BF16 (bfloat16).
 *
 * Errors:
 *  - Argument errors are detected on the host, return a status and launch
 *    nothing: NULL pointer -> SQ_ERR_NULL; negative/zero dims -> SQ_ERR_SHAPE
 *    (M == 0 is a valid no-op); group not in {32, 64, 128}, K % 128 != 0 or an unknown dtype
 *    -> SQ_ERR_UNSUPPORTED; a pointer not 16-byte aligned or N % 8 != 0 ->
 *    SQ_ERR_ALIGN; a workspace that is too small -> SQ_ERR_WORKSPACE.
 *  - Launch failures return SQ_ERR_CUDA; sq_last_error() then holds the CUDA
 *    error string (thread-local).
 *  - Data-dependent problems (NaN/Inf) are never reported by host sync: see
 *    nonfinite_count of sq_quantize_pack_groupwise.
 */
#ifndef LIBSQ_H
#define LIBSQ_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SQ_API __attribute__((visibility("default")))
#else
#define SQ_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef int sq_status;
enum {
  SQ_OK = 0,
  SQ_ERR_NULL = 1,
  SQ_ERR_SHAPE = 2,
  SQ_ERR_UNSUPPORTED = 3,
  SQ_ERR_ALIGN = 4,
  SQ_ERR_CUDA = 5,
  SQ_ERR_WORKSPACE = 6
};
enum { SQ_F16 = 0, SQ_BF16 = 1 };
/* GEMM paths: AUTO picks by M (sq_w4a16_gemm); DECODE = the mma.sync kernel (M <= 16),
 * PREFILL = the tcgen05 kernel with Ŵ in TMEM (any M). */
enum { SQ_PATH_AUTO = 0, SQ_PATH_DECODE = 1, SQ_PATH_PREFILL = 2 };
/* Process-wide launch options (sq_set_option):
 *  SQ_OPT_PDL (default 1): launch the GEMM kernels with programmatic dependent
 *    launch, so a kernel's prologue overlaps the previous kernel's tail; every
 *    read of X and every global write still waits for the previous kernel
 *    (griddepcontrol.wait), so results are unchanged.
 *  SQ_OPT_DECODE_SCHEDULE (default SQ_SCHED_AUTO): how the decode kernel splits
 *    the weight matrix over its persistent CTAs.  SQ_SCHED_STREAMK: equal
 *    contiguous ranges of (row block x 4 groups) units, row blocks cut between
 *    CTAs finished by a deterministic fixup through the workspace.
 *    SQ_SCHED_ROWBLOCK: whole row blocks (32 or 64 rows) per CTA, no fixup.
 *    AUTO picks per shape.  Results agree to fp32 rounding either way.
 *  SQ_OPT_DECODE_GRID_LIMIT (default 0 = none): at most this many CTAs per decode
 *    launch.  For tests that run several simulated tensor-parallel ranks of
 *    sq_w4a16_gemm_allreduce as concurrent kernels on ONE GPU (their grids must be
 *    co-resident); results do not depend on it.
 * Option 2 (a process-wide "weights static" switch in version 1) is now the per-call
 * flag SQ_GEMM_WEIGHTS_STATIC; sq_set_option(2, ...) returns SQ_ERR_UNSUPPORTED. */
enum { SQ_OPT_PDL = 1, SQ_OPT_DECODE_SCHEDULE = 3, SQ_OPT_DECODE_GRID_LIMIT = 5 };
enum { SQ_SCHED_AUTO = 0, SQ_SCHED_STREAMK = 1, SQ_SCHED_ROWBLOCK = 2 };
/* Per-call GEMM flags (sq_w4a16_gemm_ex, sq_w4a16_gemm_allreduce):
 *  SQ_GEMM_WEIGHTS_STATIC: the caller promises that Wq/scales/zeros of THIS call are
 *    not written by the kernels that precede it on its stream (true for inference with
 *    resident weights; false right after sq_quantize_pack_groupwise wrote them).  With
 *    PDL the kernel then streams its first weight stages BEFORE waiting on the previous
 *    kernel; X and every global write still wait.  Without the flag the weights are
 *    read only after the previous kernel has completed. */
enum { SQ_GEMM_WEIGHTS_STATIC = 1u };
/* SQ_ZEROS_U4 (GEMM and quantize flags): the zeros argument is the packed u4 layout
 *    uint8[G][N/2] described above instead of fp16 bits uint16[G][N]; it is passed
 *    through the same `zeros` pointer (cast).  Results are identical either way (Z is an
 *    integer 0..15); the packed layout moves 0.5 instead of 2 bytes per group row. */
enum { SQ_ZEROS_U4 = 2u };

/* Library version (major*10000 + minor*100 + patch). */
SQ_API int sq_version(void);
/* Static description of a status code. */
SQ_API const char* sq_status_string(sq_status st);
/* Detail of the last failure on the calling host thread ("" if none). */
SQ_API const char* sq_last_error(void);
/* Largest M served by the decode path under SQ_PATH_AUTO (M_dec). */
SQ_API int sq_decode_max_m(void);
/* Set / read a launch option (SQ_OPT_*); returns SQ_ERR_UNSUPPORTED for an
 * unknown option.  sq_get_option returns -1 for an unknown option. */
SQ_API sq_status sq_set_option(int option, int value);
SQ_API int sq_get_option(int option);

/*
 * Calibration statistic of Eq. 6: act_max[k] = max_t |X[t][k]| over the T rows
 * of a calibration batch X[T][K] (x_dtype).  If `accumulate` is non-zero the
 * result is max(act_max[k], ...) (running maximum over several batches);
 * otherwise act_max is overwritten.  NaN in X propagates to act_max.
 * act_max: fp32[K], device, written.
 */
SQ_API sq_status sq_act_absmax(const void* X, int x_dtype, int64_t T, int64_t K,
                        float* act_max, int accumulate, void* stream);

/*
 * Eq. 6.  W[N][K] (w_dtype) is the consumer weight; when
 * several linears share one input (q|k|v, gate|up) the caller passes the
 * stacked weight, so w_max is the max over all consumers (S11).
 *   w_max[k] = max_n |W[n][k]|                  (exact)
 *   s[k] = RN_fp32( max(act_max[k], eps)^alpha / max(w_max[k], eps)^(1-alpha) )
 * evaluated in fp64; alpha in {0, 0.5, 1} use the exactly rounded forms
 * 1/w, sqrt(a)/sqrt(w), a; other alpha use fp64 pow (<= 1 ulp fp32 from the
 * oracle).  alpha must lie in [0, 1] (else SQ_ERR_UNSUPPORTED); eps > 0.
 * act_max: fp32[K] (>= 0), read.  s_out: fp32[K], written (also used as the
 * kernel's scratch for w_max, so it must not alias act_max).
 */
SQ_API sq_status sq_smooth_scales(const void* W, int w_dtype, int64_t N, int64_t K,
                           const float* act_max, double alpha, double eps,
                           float* s_out, void* stream);

/*
 * Eq. 6 from precomputed maxima: s[k] = RN_fp32(max(act_max[k],eps)^alpha /
 * max(w_max[k],eps)^(1-alpha)), the same evaluation as sq_smooth_scales.  For weights
 * sharded over ranks (tensor parallel), w_max is the column abs-max of the FULL weight:
 * each rank takes sq_act_absmax of its shard (a [N_r][K] matrix's column maxima) and the
 * ranks all-reduce it with MAX before this call, so every rank folds the same s.
 * w_max, act_max: fp32[K] device, read; s_out: fp32[K] device, written (may alias w_max,
 * must not alias act_max).  16-byte aligned pointers.
 */
SQ_API sq_status sq_smooth_scales_wmax(const float* w_max, const float* act_max, int64_t K,
                                double alpha, double eps, float* s_out, void* stream);

/*
 * Eq. 5 + Eq. 1 (load-time quantization).  For every output
 * channel n and group gi of `group` consecutive input channels:
 *   W'[n][k] = RN(W[n][k] * s[k]) to w_dtype, one rounding    (s == NULL: RTN, s = 1)
 *   lo, hi   = min/max of the group of W';  r = hi - lo (fp64)
 *   Delta    = RZ_fp16(r / 15); 2^-24 if that underflows to 0;
 *              constant group c: Delta = 1 if c == 0 else |c|
 *   Z        = clamp(RHA(-lo / Delta), 0, 15)                  (RHA: half away from 0)
 *   q        = clamp(RHA(W' / Delta) + Z, 0, 15)
 * Outputs (device, written): Wq uint8[N][K/2], scales uint16[G][N] (fp16 bits
 * of Delta), zeros uint16[G][N] (fp16 bits of Z).  Bit-exact with the oracle.
 * nonfinite_count (device int*, nullable): incremented once per group that holds
 * NaN/Inf after the fold (or whose r/15 exceeds the fp16 range); such a group is
 * stored as scale = 0x7E00 (NaN), zero = 0, codes = 0.
 * s: fp32[K] device or NULL.  Requires group in {32, 64, 128},
 * K % 128 == 0, N % 8 == 0, 16-byte aligned W/Wq/scales/zeros.
 */
SQ_API sq_status sq_quantize_pack_groupwise(const void* W, int w_dtype, const float* s,
                                     int64_t N, int64_t K, int group,
                                     uint8_t* Wq, uint16_t* scales, uint16_t* zeros,
                                     int* nonfinite_count, void* stream);
/* Same with flags: 0 (== sq_quantize_pack_groupwise) or SQ_ZEROS_U4 -- zeros is then
 * written as packed uint8[G][N/2] (N % 32 == 0), a non-finite group's Z as 0.  Other
 * bits -> SQ_ERR_UNSUPPORTED. */
SQ_API sq_status sq_quantize_pack_groupwise_ex(const void* W, int w_dtype, const float* s,
                                        int64_t N, int64_t K, int group,
                                        uint8_t* Wq, uint16_t* scales, void* zeros,
                                        int* nonfinite_count, unsigned flags, void* stream);

/*
 * Bytes of caller-allocated device workspace sq_w4a16_gemm needs for this shape
 * (the decode path's stream-K fixup: fp32 partial tiles, then per-row-block
 * counters).  The workspace must be 16-byte aligned and zero-filled once before
 * its first use (sq_workspace_reset); every completed call leaves the counters zero
 * again, so one workspace can serve any sequence of shapes on one stream.  Calls
 * that may run concurrently (different streams) need different workspaces.  After a
 * launch that did not complete (an error, a killed context) reset the workspace before
 * reusing it: stale counters would mis-identify the last stream-K contributor.
 */
SQ_API size_t sq_w4a16_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, int group);
/* Zero-fill a GEMM workspace (or an all-reduce symmetric buffer) on `stream`
 * (cudaMemsetAsync).  workspace_bytes == 0 is a no-op. */
SQ_API sq_status sq_workspace_reset(void* workspace, size_t workspace_bytes, void* stream);

/*
 * Eq. 3, W4A16 linear layer:
 *   Y[m][n] = sum_k X[m][k] * (q[n][k] - Z[gi][n]) * Delta[gi][n],  gi = k / group
 * fp32 accumulation; Y is written in x_dtype (fp16 or bf16)
 * "the input and output of all linear layers ... are FP16".
 * X[M][K], Y[M][N]: device, x_dtype.  Wq/scales/zeros as produced by
 * sq_quantize_pack_groupwise.  M <= sq_decode_max_m() runs the decode kernel
 * (TMA-fed mma.sync, persistent stream-K over K), larger M the prefill kernel
 * (TMA + tcgen05.mma with TMEM operands/accumulators).  One rule, no other
 * backends.  Y must not alias X.
 */
SQ_API sq_status sq_w4a16_gemm(const void* X, int x_dtype,
                        const uint8_t* Wq, const uint16_t* scales, const uint16_t* zeros,
                        void* Y, int64_t M, int64_t N, int64_t K, int group,
                        void* workspace, size_t workspace_bytes, void* stream);

/* Same as sq_w4a16_gemm with an explicit path (SQ_PATH_*: AUTO, DECODE for M <= 16,
 * PREFILL) and per-call flags (SQ_GEMM_WEIGHTS_STATIC | SQ_ZEROS_U4 or 0; other bits ->
 * SQ_ERR_UNSUPPORTED; with SQ_ZEROS_U4 `zeros` points to the packed uint8[G][N/2]).  sq_w4a16_gemm == sq_w4a16_gemm_ex(..., SQ_PATH_AUTO, 0, stream). */
SQ_API sq_status sq_w4a16_gemm_ex(const void* X, int x_dtype,
                           const uint8_t* Wq, const uint16_t* scales, const uint16_t* zeros,
                           void* Y, int64_t M, int64_t N, int64_t K, int group,
                           void* workspace, size_t workspace_bytes, int path, unsigned flags,
                           void* stream);
/* sq_w4a16_gemm_ex with flags = 0 (kept for the M sweep and the parity tests). */
SQ_API sq_status sq_w4a16_gemm_path(const void* X, int x_dtype,
                             const uint8_t* Wq, const uint16_t* scales, const uint16_t* zeros,
                             void* Y, int64_t M, int64_t N, int64_t K, int group,
                             void* workspace, size_t workspace_bytes, int path, void* stream);

/*
 * ---- Calibration: single-layer smoothing-strength search ----
 * The grid search over alpha in {0, 0.05, ..., 1} that minimizes
 * the Eq. 4 loss  E(alpha) = || X W^T - Xhat_alpha What_alpha^T ||^2  of one layer
 * is host logic (paper_2312_03788_b200/calib.py) over the calls above
 * plus these two device steps.
 */

/*
 * Activation side of Eq. 5: Xs[m][k] = RN_dtype(X[m][k] / s[k]),
 * the quotient correctly rounded in fp64 and rounded once to x_dtype (bit-identical to
 * the oracle's RN(fp64(X) / fp64(s))).  X, Xs: device [M][K] in x_dtype (may alias:
 * in-place is allowed); s: device fp32[K] (> 0, e.g. from sq_smooth_scales).
 * K % 8 == 0 and 16-byte aligned X/Xs (else SQ_ERR_ALIGN).  M == 0 is a no-op that
 * returns SQ_OK without looking at the pointers (argument order: shape, dtype, null, align).
 */
SQ_API sq_status sq_smooth_activations(const void* X, int x_dtype, const float* s,
                                int64_t M, int64_t K, void* Xs, void* stream);

/*
 * Model-level smoothing fusion (Fig. 5): the
 * activation division X diag(s)^-1 is folded into the layer that produces X.  For an
 * RMSNorm producer the gain g[K] becomes RN(g / s), which is sq_smooth_activations on
 * g as a [1][K] matrix.  For a linear producer (down_proj's input comes from up_proj)
 * the producer's OUTPUT rows are divided:
 *   W_out[n][k] = RN_dtype(W[n][k] / d[n])     (fp64 quotient, one rounding)
 * with d = the consumer's s.  W, W_out: device [N][K] in w_dtype (may alias); d: device
 * fp32[N] (> 0).  K % 8 == 0, 16-byte aligned W/W_out.  N == 0 is a no-op.
 */
SQ_API sq_status sq_fold_rows(const void* W, int w_dtype, const float* d, int64_t N, int64_t K,
                       void* W_out, void* stream);

/*
 * Squared Frobenius distance of Eq. 4: *out = sum_i (A[i] - B[i])^2 over n elements of
 * two device arrays in `dtype` (fp16/bf16), accumulated in fp64 with a fixed reduction
 * order (bit-reproducible run to run).  out: device double, written.  workspace: device,
 * at least sq_sq_diff_sum_workspace_bytes() bytes (per-CTA partials), caller-owned.
 * n == 0 writes 0 (A and B may then be null).
 */
SQ_API size_t sq_sq_diff_sum_workspace_bytes(void);
SQ_API sq_status sq_sq_diff_sum(const void* A, const void* B, int dtype, int64_t n,
                         double* out, void* workspace, size_t workspace_bytes, void* stream);

/*
 * ---- Row-parallel all-reduce over peer memory ----
 * After a row-parallel linear (o_proj, down_proj) every rank holds a partial Y[M][N]; the
 * layer output is their sum (BASELINE.json north_star: "an all-reduce over NVLink after
 * row-parallel layers").  Instead of a separate NCCL call this is a one-shot exchange in
 * ONE kernel over NVLink/NVSwitch peer memory: each CTA pushes its chunk of the local
 * partial into every rank's symmetric buffer, raises a per-chunk flag there, waits for
 * the same chunk from every rank and sums the world partials in rank order (fp32, so all
 * ranks get bit-identical Y).  Launched with PDL, so its prologue overlaps the GEMM tail.
 *
 * Symmetric buffer: each rank allocates sq_allreduce_buffer_bytes(n_max, world) bytes of
 * device memory, ZERO-FILLED once, and shares it with its peers (sq_ipc_* below, or any
 * peer mapping); peer_bufs is a DEVICE array of `world` device pointers, entry q = rank q's
 * buffer as mapped in this process (entry `rank` = its own).  epoch: 0 = device-managed
 * (the kernel takes the rank's buffer counter + 1 and advances it when done: safe under
 * CUDA graph replay, since every rank makes the same sequence of calls); or an explicit
 * 1, 2, 3, ... per call, the same on every rank (after 2^32 - 1 continue at 2).  Use one
 * mode per buffer.
 * n <= n_max elements of dtype (fp16/bf16) in y_local and y_out (may alias).  error_flag:
 * device int, set to 1 if a peer did not arrive within the bounded wait (~seconds); the
 * kernel then leaves y_out partially written instead of hanging (the buffer header stays
 * consistent; to restart a broken collective, zero every rank's buffer with
 * sq_workspace_reset and restart the epochs).  Stream-ordered; every rank must make the
 * matching call (a collective).
 */
SQ_API size_t sq_allreduce_buffer_bytes(int64_t n_max, int world);
SQ_API sq_status sq_allreduce_oneshot(const void* y_local, int dtype, void* y_out, int64_t n, int64_t n_max,
                               void* const* peer_bufs, int rank, int world, uint32_t epoch,
                               int* error_flag, void* stream);

/*
 * Row-parallel W4A16 linear + all-reduce in ONE kernel (decode, M <= sq_decode_max_m()):
 * the decode GEMM's epilogue pushes every row block it finalizes straight into slot
 * [rank] of every rank's symmetric buffer (the sq_allreduce_oneshot layout, one flag per
 * row block), and after a CTA has pushed all of its row blocks it waits for the other
 * ranks' copies of them and writes the rank-ordered fp32 sum to Y -- so Y (local) ends up
 * bit-identical on every rank, and no partial is written to or re-read from local HBM.
 * For M > sq_decode_max_m() (prefill) this is sq_w4a16_gemm followed by
 * sq_allreduce_oneshot on Y.  Arguments: those of sq_w4a16_gemm (X is this rank's input
 * shard [M][K_r], Wq/scales/zeros its row-parallel weight shard) plus those of
 * sq_allreduce_oneshot with n_max >= M*N, and the per-call flags of sq_w4a16_gemm_ex.
 * fp16 partials are exchanged in fp16, bf16 partials in fp32; the sum
 * is always taken in fp32.  Every rank must cut N into the same row blocks, so the decode
 * schedule here depends on N and M only, never on the rank's K.  A buffer serves either
 * this call or sq_allreduce_oneshot calls, in the same epoch mode, in one stream order on
 * every rank.
 */
SQ_API sq_status sq_w4a16_gemm_allreduce(const void* X, int x_dtype,
                                  const uint8_t* Wq, const uint16_t* scales, const uint16_t* zeros,
                                  void* Y, int64_t M, int64_t N, int64_t K, int group,
                                  void* workspace, size_t workspace_bytes,
                                  void* const* peer_bufs, int rank, int world, int64_t n_max,
                                  uint32_t epoch, int* error_flag, unsigned flags, void* stream);

/*
 * CUDA IPC plumbing for the symmetric buffers (host calls, no stream work).
 * sq_ipc_get_handle: export the cudaMalloc block containing dev_ptr into handle_out
 * (sq_ipc_handle_bytes() bytes) and report dev_ptr's byte offset inside that block (a
 * caching allocator may sub-allocate); the importer adds the offset to the mapped base.
 * sq_ipc_open_handle: map a peer's handle in this process (enables peer access lazily)
 * and return the block base; sq_ipc_close: unmap it.  A handle cannot be opened by the
 * process that exported it.  The symmetric buffer needs n_max % 8 == 0 (16-B slots).
 */
SQ_API size_t sq_ipc_handle_bytes(void);
SQ_API sq_status sq_ipc_get_handle(void* dev_ptr, void* handle_out, size_t* offset_out);
SQ_API sq_status sq_ipc_open_handle(const void* handle, void** dev_ptr_out);
SQ_API sq_status sq_ipc_close(void* dev_ptr);

#ifdef __cplusplus
}
#endif

#endif /* LIBSQ_H */
