// libsq C ABI: argument validation and dispatch (include/libsq.h).
// Host-only code; every kernel launch is asynchronous on the caller's stream.
#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <string>

#include <cuda.h>

#include "sq_internal.cuh"

namespace sq {

static thread_local std::string g_last_error;

static sq_status fail(sq_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

static sq_status cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return SQ_OK;
  return fail(SQ_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
static bool valid_dtype(int d) { return d == SQ_F16 || d == SQ_BF16; }
// PAPER.md:160 "Group-size is usually set to be 128"; "different group sizes"
static bool valid_group(int g) { return g == 128 || g == 64 || g == 32; }

int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  static int cached[64] = {0};
  if (dev < 0 || dev >= 64) dev = 0;
  if (cached[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cached[dev] = n;
  }
  return cached[dev];
}

constexpr int kDecodeMaxM = 16;

size_t ws_partials_bytes() { return std::max(decode_partials_bytes(), prefill_partials_bytes()); }

static int g_opt_pdl = 1;
static int g_opt_decode_schedule = SQ_SCHED_AUTO;
static int g_opt_decode_grid_limit = 0;

int option(int opt) {
  switch (opt) {
    case SQ_OPT_PDL: return g_opt_pdl;
    case SQ_OPT_DECODE_SCHEDULE: return g_opt_decode_schedule;
    case SQ_OPT_DECODE_GRID_LIMIT: return g_opt_decode_grid_limit;
    default: return -1;
  }
}

}  // namespace sq

using namespace sq;

extern "C" {

int sq_version(void) { return 200; }

const char* sq_status_string(sq_status st) {
  switch (st) {
    case SQ_OK: return "SQ_OK";
    case SQ_ERR_NULL: return "SQ_ERR_NULL: null pointer argument";
    case SQ_ERR_SHAPE: return "SQ_ERR_SHAPE: invalid dimension";
    case SQ_ERR_UNSUPPORTED: return "SQ_ERR_UNSUPPORTED: unsupported group/dtype/shape";
    case SQ_ERR_ALIGN: return "SQ_ERR_ALIGN: pointer not 16-byte aligned or N % 8 != 0";
    case SQ_ERR_CUDA: return "SQ_ERR_CUDA: CUDA launch failure";
    case SQ_ERR_WORKSPACE: return "SQ_ERR_WORKSPACE: workspace too small";
    default: return "unknown sq_status";
  }
}

const char* sq_last_error(void) { return g_last_error.c_str(); }

int sq_decode_max_m(void) { return kDecodeMaxM; }

sq_status sq_set_option(int opt, int value) {
  switch (opt) {
    case SQ_OPT_PDL: g_opt_pdl = value ? 1 : 0; return SQ_OK;
    case SQ_OPT_DECODE_SCHEDULE:
      if (value < SQ_SCHED_AUTO || value > SQ_SCHED_ROWBLOCK)
        return fail(SQ_ERR_UNSUPPORTED, "sq_set_option: decode schedule %d", value);
      g_opt_decode_schedule = value;
      return SQ_OK;
    case SQ_OPT_DECODE_GRID_LIMIT:
      if (value < 0) return fail(SQ_ERR_UNSUPPORTED, "sq_set_option: grid limit %d", value);
      g_opt_decode_grid_limit = value;
      return SQ_OK;
    default: return fail(SQ_ERR_UNSUPPORTED, "sq_set_option: unknown option %d", opt);
  }
}

int sq_get_option(int opt) { return option(opt); }

sq_status sq_act_absmax(const void* X, int x_dtype, int64_t T, int64_t K, float* act_max,
                        int accumulate, void* stream) {
  g_last_error.clear();
  if (!X || !act_max) return fail(SQ_ERR_NULL, "sq_act_absmax: null pointer");
  if (T < 0 || K <= 0) return fail(SQ_ERR_SHAPE, "sq_act_absmax: T=%lld K=%lld", (long long)T, (long long)K);
  if (!valid_dtype(x_dtype)) return fail(SQ_ERR_UNSUPPORTED, "sq_act_absmax: dtype %d", x_dtype);
  if (K % 8 != 0 || !aligned16(X) || !aligned16(act_max))
    return fail(SQ_ERR_ALIGN, "sq_act_absmax: K %% 8 != 0 or unaligned pointer");
  cudaStream_t st = (cudaStream_t)stream;
  if (!accumulate) {
    sq_status s = cuda_status(cudaMemsetAsync(act_max, 0, (size_t)K * sizeof(float), st), "memset");
    if (s != SQ_OK) return s;
  }
  if (T == 0) return SQ_OK;
  return cuda_status(launch_colabsmax(X, x_dtype, T, K, act_max, st), "colabsmax");
}

sq_status sq_smooth_scales(const void* W, int w_dtype, int64_t N, int64_t K, const float* act_max,
                           double alpha, double eps, float* s_out, void* stream) {
  g_last_error.clear();
  if (!W || !act_max || !s_out) return fail(SQ_ERR_NULL, "sq_smooth_scales: null pointer");
  if (N <= 0 || K <= 0) return fail(SQ_ERR_SHAPE, "sq_smooth_scales: N=%lld K=%lld", (long long)N, (long long)K);
  if (!valid_dtype(w_dtype)) return fail(SQ_ERR_UNSUPPORTED, "sq_smooth_scales: dtype %d", w_dtype);
  if (!(alpha >= 0.0 && alpha <= 1.0) || !(eps > 0.0))
    return fail(SQ_ERR_UNSUPPORTED, "sq_smooth_scales: alpha=%g eps=%g", alpha, eps);
  if (K % 8 != 0 || !aligned16(W) || !aligned16(s_out) || !aligned16(act_max))
    return fail(SQ_ERR_ALIGN, "sq_smooth_scales: K %% 8 != 0 or unaligned pointer");
  if ((const void*)act_max == (const void*)s_out)
    return fail(SQ_ERR_UNSUPPORTED, "sq_smooth_scales: s_out aliases act_max");
  cudaStream_t st = (cudaStream_t)stream;
  sq_status s = cuda_status(cudaMemsetAsync(s_out, 0, (size_t)K * sizeof(float), st), "memset");
  if (s != SQ_OK) return s;
  s = cuda_status(launch_colabsmax(W, w_dtype, N, K, s_out, st), "colabsmax");
  if (s != SQ_OK) return s;
  return cuda_status(launch_smooth_finalize(act_max, s_out, K, alpha, eps, st), "smooth_finalize");
}

sq_status sq_smooth_scales_wmax(const float* w_max, const float* act_max, int64_t K, double alpha, double eps,
                                float* s_out, void* stream) {
  g_last_error.clear();
  if (!w_max || !act_max || !s_out) return fail(SQ_ERR_NULL, "sq_smooth_scales_wmax: null pointer");
  if (K <= 0) return fail(SQ_ERR_SHAPE, "sq_smooth_scales_wmax: K=%lld", (long long)K);
  if (!(alpha >= 0.0 && alpha <= 1.0) || !(eps > 0.0))
    return fail(SQ_ERR_UNSUPPORTED, "sq_smooth_scales_wmax: alpha=%g eps=%g", alpha, eps);
  if (!aligned16(w_max) || !aligned16(s_out) || !aligned16(act_max))
    return fail(SQ_ERR_ALIGN, "sq_smooth_scales_wmax: unaligned pointer");
  if ((const void*)act_max == (const void*)s_out)
    return fail(SQ_ERR_UNSUPPORTED, "sq_smooth_scales_wmax: s_out aliases act_max");
  cudaStream_t st = (cudaStream_t)stream;
  if ((const void*)w_max != (const void*)s_out) {
    sq_status r = cuda_status(cudaMemcpyAsync(s_out, w_max, (size_t)K * sizeof(float), cudaMemcpyDeviceToDevice, st),
                              "memcpy");
    if (r != SQ_OK) return r;
  }
  return cuda_status(launch_smooth_finalize(act_max, s_out, K, alpha, eps, st), "smooth_finalize");
}

sq_status sq_quantize_pack_groupwise(const void* W, int w_dtype, const float* s, int64_t N,
                                     int64_t K, int group, uint8_t* Wq, uint16_t* scales,
                                     uint16_t* zeros, int* nonfinite_count, void* stream) {
  return sq_quantize_pack_groupwise_ex(W, w_dtype, s, N, K, group, Wq, scales, zeros, nonfinite_count, 0u, stream);
}

sq_status sq_quantize_pack_groupwise_ex(const void* W, int w_dtype, const float* s, int64_t N,
                                        int64_t K, int group, uint8_t* Wq, uint16_t* scales,
                                        void* zeros, int* nonfinite_count, unsigned flags, void* stream) {
  g_last_error.clear();
  if (flags & ~(unsigned)SQ_ZEROS_U4) return fail(SQ_ERR_UNSUPPORTED, "sq_quantize_pack_groupwise: flags 0x%x", flags);
  const bool zu4 = (flags & SQ_ZEROS_U4) != 0;
  if (!W || !Wq || !scales || !zeros) return fail(SQ_ERR_NULL, "sq_quantize_pack_groupwise: null pointer");
  if (N <= 0 || K <= 0) return fail(SQ_ERR_SHAPE, "sq_quantize_pack_groupwise: N=%lld K=%lld", (long long)N, (long long)K);
  if (!valid_group(group) || K % 128 != 0 || !valid_dtype(w_dtype))
    return fail(SQ_ERR_UNSUPPORTED, "sq_quantize_pack_groupwise: group=%d K=%lld dtype=%d", group, (long long)K, w_dtype);
  if (N % 8 != 0 || !aligned16(W) || !aligned16(Wq) || !aligned16(scales) || !aligned16(zeros) ||
      (s && !aligned16(s)) || (zu4 && N % 32 != 0))
    return fail(SQ_ERR_ALIGN, "sq_quantize_pack_groupwise: N %% 8 != 0 (N %% 32 with u4 zeros) or unaligned pointer");
  if (N > (1ll << 30) || K > (1ll << 30)) return fail(SQ_ERR_SHAPE, "sq_quantize_pack_groupwise: too large");
  return cuda_status(launch_quantize(W, w_dtype, s, N, K, group, Wq, scales, zeros, zu4, nonfinite_count,
                                     (cudaStream_t)stream), "quantize");
}

size_t sq_w4a16_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, int group) {
  (void)group;
  if (N <= 0 || K <= 0 || M < 0) return 0;
  // enough for either path, so one buffer serves SQ_PATH_AUTO and the explicit paths
  return std::max(decode_workspace_bytes(N), prefill_workspace_bytes(M, N, K));
}

sq_status sq_workspace_reset(void* workspace, size_t workspace_bytes, void* stream) {
  g_last_error.clear();
  if (workspace_bytes == 0) return SQ_OK;
  if (!workspace) return fail(SQ_ERR_NULL, "sq_workspace_reset: null pointer");
  return cuda_status(cudaMemsetAsync(workspace, 0, workspace_bytes, (cudaStream_t)stream), "sq_workspace_reset");
}

sq_status sq_w4a16_gemm_ex(const void* X, int x_dtype, const uint8_t* Wq, const uint16_t* scales,
                           const uint16_t* zeros, void* Y, int64_t M, int64_t N, int64_t K, int group,
                           void* workspace, size_t workspace_bytes, int path, unsigned flags, void* stream) {
  g_last_error.clear();
  if (M == 0 && N > 0 && K > 0) return SQ_OK;  // no-op; X/Y may be empty (null) tensors
  if (!X || !Wq || !scales || !zeros || !Y) return fail(SQ_ERR_NULL, "sq_w4a16_gemm: null pointer");
  if (M < 0 || N <= 0 || K <= 0) return fail(SQ_ERR_SHAPE, "sq_w4a16_gemm: M=%lld N=%lld K=%lld", (long long)M, (long long)N, (long long)K);
  if (!valid_group(group) || K % 128 != 0 || !valid_dtype(x_dtype))
    return fail(SQ_ERR_UNSUPPORTED, "sq_w4a16_gemm: group=%d K=%lld dtype=%d", group, (long long)K, x_dtype);
  if (flags & ~(unsigned)(SQ_GEMM_WEIGHTS_STATIC | SQ_ZEROS_U4))
    return fail(SQ_ERR_UNSUPPORTED, "sq_w4a16_gemm: flags 0x%x", flags);
  const bool zu4 = (flags & SQ_ZEROS_U4) != 0;
  if (N % 8 != 0 || !aligned16(X) || !aligned16(Wq) || !aligned16(scales) || !aligned16(zeros) ||
      !aligned16(Y) || (zu4 && N % 32 != 0))
    return fail(SQ_ERR_ALIGN, "sq_w4a16_gemm: N %% 8 != 0 (N %% 32 with u4 zeros) or unaligned pointer");
  if (M > (1ll << 30) || N > (1ll << 30) || K > (1ll << 30)) return fail(SQ_ERR_SHAPE, "sq_w4a16_gemm: too large");
  const bool wstatic = (flags & SQ_GEMM_WEIGHTS_STATIC) != 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (path == SQ_PATH_AUTO) path = (M <= kDecodeMaxM) ? SQ_PATH_DECODE : SQ_PATH_PREFILL;
  if (path == SQ_PATH_DECODE) {
    if (M > kDecodeMaxM) return fail(SQ_ERR_UNSUPPORTED, "sq_w4a16_gemm: decode path needs M <= %d", kDecodeMaxM);
    const size_t need = decode_workspace_bytes(N);
    if (workspace == nullptr || workspace_bytes < need || !aligned16(workspace))
      return fail(SQ_ERR_WORKSPACE, "sq_w4a16_gemm: decode needs %zu workspace bytes (16-byte aligned)", need);
    const char* why = nullptr;
    cudaError_t e = launch_decode(X, x_dtype, Wq, scales, zeros, Y, (int)M, (int)N, (int)K, group, workspace, wstatic,
                                  zu4, st, &why);
    if (why) return fail(SQ_ERR_UNSUPPORTED, "sq_w4a16_gemm decode: %s", why);
    return cuda_status(e, "decode");
  }
  if (path == SQ_PATH_PREFILL) {
    const size_t need = prefill_workspace_bytes(M, N, K);
    if (need > 0 && (workspace == nullptr || workspace_bytes < need || !aligned16(workspace)))
      return fail(SQ_ERR_WORKSPACE, "sq_w4a16_gemm: prefill needs %zu workspace bytes (16-byte aligned)", need);
    const char* why = nullptr;
    cudaError_t e = launch_prefill(X, x_dtype, Wq, scales, zeros, Y, (int)M, (int)N, (int)K, group,
                                   workspace, workspace_bytes, wstatic, zu4, st, &why);
    if (why) return fail(SQ_ERR_UNSUPPORTED, "sq_w4a16_gemm prefill: %s", why);
    return cuda_status(e, "prefill");
  }
  return fail(SQ_ERR_UNSUPPORTED, "sq_w4a16_gemm: unknown path %d", path);
}

sq_status sq_w4a16_gemm_path(const void* X, int x_dtype, const uint8_t* Wq, const uint16_t* scales,
                             const uint16_t* zeros, void* Y, int64_t M, int64_t N, int64_t K,
                             int group, void* workspace, size_t workspace_bytes, int path,
                             void* stream) {
  return sq_w4a16_gemm_ex(X, x_dtype, Wq, scales, zeros, Y, M, N, K, group, workspace, workspace_bytes, path, 0u,
                          stream);
}

sq_status sq_w4a16_gemm(const void* X, int x_dtype, const uint8_t* Wq, const uint16_t* scales,
                        const uint16_t* zeros, void* Y, int64_t M, int64_t N, int64_t K, int group,
                        void* workspace, size_t workspace_bytes, void* stream) {
  return sq_w4a16_gemm_ex(X, x_dtype, Wq, scales, zeros, Y, M, N, K, group, workspace, workspace_bytes,
                          SQ_PATH_AUTO, 0u, stream);
}

sq_status sq_smooth_activations(const void* X, int x_dtype, const float* s, int64_t M, int64_t K,
                                void* Xs, void* stream) {
  g_last_error.clear();
  if (M < 0 || K <= 0) return fail(SQ_ERR_SHAPE, "sq_smooth_activations: M=%lld K=%lld", (long long)M, (long long)K);
  if (!valid_dtype(x_dtype)) return fail(SQ_ERR_UNSUPPORTED, "sq_smooth_activations: dtype %d", x_dtype);
  if (M == 0) return SQ_OK;  // no-op (an empty X may have a null data pointer)
  if (!X || !s || !Xs) return fail(SQ_ERR_NULL, "sq_smooth_activations: null pointer");
  if (K % 8 != 0 || !aligned16(X) || !aligned16(Xs))
    return fail(SQ_ERR_ALIGN, "sq_smooth_activations: K %% 8 != 0 or unaligned pointer");
  return cuda_status(launch_smooth_activations(X, x_dtype, s, M, K, Xs, static_cast<cudaStream_t>(stream)),
                     "sq_smooth_activations");
}

sq_status sq_fold_rows(const void* W, int w_dtype, const float* d, int64_t N, int64_t K, void* W_out,
                       void* stream) {
  g_last_error.clear();
  if (N < 0 || K <= 0) return fail(SQ_ERR_SHAPE, "sq_fold_rows: N=%lld K=%lld", (long long)N, (long long)K);
  if (!valid_dtype(w_dtype)) return fail(SQ_ERR_UNSUPPORTED, "sq_fold_rows: dtype %d", w_dtype);
  if (N == 0) return SQ_OK;
  if (!W || !d || !W_out) return fail(SQ_ERR_NULL, "sq_fold_rows: null pointer");
  if (K % 8 != 0 || !aligned16(W) || !aligned16(W_out))
    return fail(SQ_ERR_ALIGN, "sq_fold_rows: K %% 8 != 0 or unaligned pointer");
  return cuda_status(launch_fold_rows(W, w_dtype, d, N, K, W_out, static_cast<cudaStream_t>(stream)),
                     "sq_fold_rows");
}

size_t sq_sq_diff_sum_workspace_bytes(void) { return (size_t)sq_diff_ctas() * sizeof(double); }

sq_status sq_sq_diff_sum(const void* A, const void* B, int dtype, int64_t n, double* out, void* workspace,
                         size_t workspace_bytes, void* stream) {
  g_last_error.clear();
  if ((n > 0 && (!A || !B)) || !out || !workspace) return fail(SQ_ERR_NULL, "sq_sq_diff_sum: null pointer");
  if (n < 0) return fail(SQ_ERR_SHAPE, "sq_sq_diff_sum: n=%lld", (long long)n);
  if (!valid_dtype(dtype)) return fail(SQ_ERR_UNSUPPORTED, "sq_sq_diff_sum: dtype %d", dtype);
  if (workspace_bytes < sq_sq_diff_sum_workspace_bytes())
    return fail(SQ_ERR_WORKSPACE, "sq_sq_diff_sum: workspace %zu < %zu", workspace_bytes,
                sq_sq_diff_sum_workspace_bytes());
  return cuda_status(launch_sq_diff_sum(A, B, dtype, n, static_cast<double*>(workspace), out,
                                        static_cast<cudaStream_t>(stream)),
                     "sq_sq_diff_sum");
}

sq_status sq_w4a16_gemm_allreduce(const void* X, int x_dtype, const uint8_t* Wq, const uint16_t* scales,
                                  const uint16_t* zeros, void* Y, int64_t M, int64_t N, int64_t K, int group,
                                  void* workspace, size_t workspace_bytes, void* const* peer_bufs, int rank,
                                  int world, int64_t n_max, uint32_t epoch, int* error_flag, unsigned flags,
                                  void* stream) {
  g_last_error.clear();
  if (flags & ~(unsigned)(SQ_GEMM_WEIGHTS_STATIC | SQ_ZEROS_U4))
    return fail(SQ_ERR_UNSUPPORTED, "sq_w4a16_gemm_allreduce: flags 0x%x", flags);
  const bool zu4 = (flags & SQ_ZEROS_U4) != 0;
  if (world <= 0 || rank < 0 || rank >= world || M < 0 || N <= 0 || M * N > n_max)
    return fail(SQ_ERR_SHAPE, "sq_w4a16_gemm_allreduce: M=%lld N=%lld n_max=%lld rank=%d world=%d", (long long)M,
                (long long)N, (long long)n_max, rank, world);
  if ((n_max + ar_chunk_elems() - 1) / ar_chunk_elems() > kArMaxChunks || (N + 31) / 32 > kArMaxChunks)
    return fail(SQ_ERR_UNSUPPORTED, "sq_w4a16_gemm_allreduce: n_max or N too large");
  if (M == 0) return SQ_OK;
  if (!peer_bufs || !error_flag) return fail(SQ_ERR_NULL, "sq_w4a16_gemm_allreduce: null pointer");
  if (!aligned16(peer_bufs) || n_max % 8 != 0)
    return fail(SQ_ERR_ALIGN, "sq_w4a16_gemm_allreduce: unaligned peer array or n_max %% 8 != 0");
  if (M > kDecodeMaxM) {
    // prefill-sized: the GEMM, then the one-shot exchange kernel (PDL)
    sq_status st = sq_w4a16_gemm_ex(X, x_dtype, Wq, scales, zeros, Y, M, N, K, group, workspace, workspace_bytes,
                                    SQ_PATH_AUTO, flags, stream);
    if (st != SQ_OK) return st;
    return sq_allreduce_oneshot(Y, x_dtype, Y, M * N, n_max, peer_bufs, rank, world, epoch, error_flag, stream);
  }
  // decode: one kernel -- the epilogue pushes each finished row block to every rank and
  // reduces its own row blocks once every rank's copy has arrived
  if (!X || !Wq || !scales || !zeros || !Y) return fail(SQ_ERR_NULL, "sq_w4a16_gemm_allreduce: null pointer");
  if (K <= 0 || !valid_group(group) || K % 128 != 0 || !valid_dtype(x_dtype))
    return fail(SQ_ERR_UNSUPPORTED, "sq_w4a16_gemm_allreduce: group=%d K=%lld dtype=%d", group, (long long)K, x_dtype);
  if (N % 8 != 0 || !aligned16(X) || !aligned16(Wq) || !aligned16(scales) || !aligned16(zeros) || !aligned16(Y) ||
      (zu4 && N % 32 != 0))
    return fail(SQ_ERR_ALIGN, "sq_w4a16_gemm_allreduce: N %% 8 != 0 (N %% 32 with u4 zeros) or unaligned pointer");
  const size_t need = decode_workspace_bytes(N);
  if (workspace == nullptr || workspace_bytes < need || !aligned16(workspace))
    return fail(SQ_ERR_WORKSPACE, "sq_w4a16_gemm_allreduce: decode needs %zu workspace bytes", need);
  const ArParams ar{reinterpret_cast<uint8_t* const*>(peer_bufs), n_max, error_flag, rank, world, epoch};
  const char* why = nullptr;
  cudaError_t e = launch_decode(X, x_dtype, Wq, scales, zeros, Y, (int)M, (int)N, (int)K, group, workspace,
                                (flags & SQ_GEMM_WEIGHTS_STATIC) != 0, zu4, (cudaStream_t)stream, &why, &ar);
  if (why) return fail(SQ_ERR_UNSUPPORTED, "sq_w4a16_gemm_allreduce: %s", why);
  return cuda_status(e, "sq_w4a16_gemm_allreduce");
}

size_t sq_allreduce_buffer_bytes(int64_t n_max, int world) {
  if (n_max <= 0 || world <= 0) return 0;
  return ar_buffer_bytes(n_max, world);
}

sq_status sq_allreduce_oneshot(const void* y_local, int dtype, void* y_out, int64_t n, int64_t n_max,
                               void* const* peer_bufs, int rank, int world, uint32_t epoch, int* error_flag,
                               void* stream) {
  g_last_error.clear();
  if (n < 0 || n_max < 0 || n > n_max || world <= 0 || rank < 0 || rank >= world)
    return fail(SQ_ERR_SHAPE, "sq_allreduce_oneshot: n=%lld n_max=%lld rank=%d world=%d", (long long)n,
                (long long)n_max, rank, world);
  if (!valid_dtype(dtype)) return fail(SQ_ERR_UNSUPPORTED, "sq_allreduce_oneshot: dtype %d", dtype);
  if ((n_max + ar_chunk_elems() - 1) / ar_chunk_elems() > kArMaxChunks)
    return fail(SQ_ERR_UNSUPPORTED, "sq_allreduce_oneshot: n_max %lld > %lld", (long long)n_max,
                (long long)kArMaxChunks * ar_chunk_elems());
  if (n == 0) return SQ_OK;
  if (!y_local || !y_out || !peer_bufs || !error_flag) return fail(SQ_ERR_NULL, "sq_allreduce_oneshot: null pointer");
  if (!aligned16(y_local) || !aligned16(y_out) || !aligned16(peer_bufs) || n_max % 8 != 0)
    return fail(SQ_ERR_ALIGN, "sq_allreduce_oneshot: unaligned pointer or n_max %% 8 != 0");
  return cuda_status(launch_oneshot_allreduce(y_local, dtype, y_out, n, n_max, peer_bufs, rank, world, epoch,
                                              error_flag, static_cast<cudaStream_t>(stream)),
                     "sq_allreduce_oneshot");
}

size_t sq_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

sq_status sq_ipc_get_handle(void* dev_ptr, void* handle_out, size_t* offset_out) {
  g_last_error.clear();
  if (!dev_ptr || !handle_out || !offset_out) return fail(SQ_ERR_NULL, "sq_ipc_get_handle: null pointer");
  // the handle names the whole cudaMalloc block; report where dev_ptr sits inside it
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(SQ_ERR_CUDA, "sq_ipc_get_handle: cuMemGetAddressRange unavailable");
    get_range = reinterpret_cast<GetRange>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return fail(SQ_ERR_CUDA, "sq_ipc_get_handle: not a device allocation");
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return cuda_status(e, "sq_ipc_get_handle");
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = (size_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return SQ_OK;
}

sq_status sq_ipc_open_handle(const void* handle, void** dev_ptr_out) {
  g_last_error.clear();
  if (!handle || !dev_ptr_out) return fail(SQ_ERR_NULL, "sq_ipc_open_handle: null pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  return cuda_status(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess), "sq_ipc_open_handle");
}

sq_status sq_ipc_close(void* dev_ptr) {
  g_last_error.clear();
  if (!dev_ptr) return fail(SQ_ERR_NULL, "sq_ipc_close: null pointer");
  return cuda_status(cudaIpcCloseMemHandle(dev_ptr), "sq_ipc_close");
}

}  // extern "C"
