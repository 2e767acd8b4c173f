// Internal declarations shared by the libsq translation units (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/libsq.h"

namespace sq {

// ---- launchers (each returns the cudaError_t of its launch) ----
cudaError_t launch_colabsmax(const void* X, int dtype, int64_t rows, int64_t K,
                             float* out_bits_as_float, cudaStream_t st);
cudaError_t launch_smooth_finalize(const float* act_max, float* s_inout, int64_t K,
                                   double alpha, double eps, cudaStream_t st);
// group: 32, 64 or 128 (K % 128 == 0).  zeros_u4: Z packed two per byte along n
// (uint8[G][N/2], low nibble = even n) instead of fp16 bits uint16[G][N] (SQ_ZEROS_U4).
cudaError_t launch_quantize(const void* W, int w_dtype, const float* s, int64_t N, int64_t K, int group,
                            uint8_t* Wq, uint16_t* scales, void* zeros, bool zeros_u4, int* nonfinite,
                            cudaStream_t st);

// GEMM workspace layout: [fp32 partial tiles: ws_partials_bytes()][int counters].  The
// partial region has one fixed size for every shape and path, so no call's counters ever
// overlap another call's partials in a shared workspace.
size_t decode_partials_bytes();
size_t prefill_partials_bytes();
size_t ws_partials_bytes();
// Counter region after the partials: at least 64 KB (16384 row blocks / tiles), so one
// workspace sized for any of the usual shapes serves them all.
inline size_t counter_region_bytes(int64_t counters) {
  const size_t b = (size_t)((counters * 4 + 255) / 256 * 256);
  return b < 65536 ? 65536 : b;
}
bool prefill_streamk(int64_t M, int64_t N, int64_t K);
size_t decode_workspace_bytes(int64_t N);
// Row-parallel all-reduce fused into the decode epilogue (world == 0: plain GEMM).
struct ArParams {
  uint8_t* const* peers;  // device array of `world` symmetric-buffer addresses
  int64_t n_max;
  int* err;
  int rank, world;
  uint32_t epoch;  // 0: device-managed
};
// weights_static: the caller promised (SQ_GEMM_WEIGHTS_STATIC) that the weights are not
// written by the preceding kernels, so with PDL the weight loads may start before the
// previous kernel has finished.
// zeros_u4: zeros is uint8[G][N/2] (two 4-bit Z per byte along n, SQ_ZEROS_U4), else
// fp16 bits uint16[G][N].
cudaError_t launch_decode(const void* X, int x_dtype, const uint8_t* Wq, const uint16_t* scales,
                          const void* zeros, void* Y, int M, int N, int K, int group, void* ws,
                          bool weights_static, bool zeros_u4, cudaStream_t st, const char** why,
                          const ArParams* ar = nullptr);

size_t prefill_workspace_bytes(int64_t M, int64_t N, int64_t K);
cudaError_t launch_prefill(const void* X, int x_dtype, const uint8_t* Wq, const uint16_t* scales,
                           const void* zeros, void* Y, int M, int N, int K, int group,
                           void* workspace, size_t ws_bytes, bool weights_static, bool zeros_u4,
                           cudaStream_t st, const char** why);

int num_sms();
int option(int opt);

// one-shot all-reduce over peer memory (k_allreduce.cu).  Symmetric buffer layout:
//   [header 128 B][flags: 2 parities x world x kArMaxChunks uint32][slots: 2 parities x world
//    slots of n_max elements, each slot 4 * n_max bytes (fp16 partials use the first half,
//    the fused decode path ships bf16 partials as fp32)]
constexpr int kArMaxChunks = 8192;  // 2048 outputs per chunk: n <= 16 Mi outputs per call
constexpr size_t kArHeaderBytes = 128;
__host__ __device__ inline size_t ar_flags_offset() { return kArHeaderBytes; }
__host__ __device__ inline size_t ar_slot_offset(int world, int par, int q, int64_t n_max) {
  return kArHeaderBytes + (size_t)2 * world * kArMaxChunks * sizeof(uint32_t) +
         ((size_t)par * world + q) * (size_t)n_max * 4;
}
int64_t ar_chunk_elems();
size_t ar_buffer_bytes(int64_t n_max, int world);
cudaError_t launch_oneshot_allreduce(const void* y_local, int dtype, void* y_out, int64_t n, int64_t n_max,
                                     void* const* peers_dev, int rank, int world, uint32_t epoch, int* err,
                                     cudaStream_t st);

// calibration / model-level smoothing folds (k_calib.cu)
cudaError_t launch_fold_rows(const void* W, int dtype, const float* d, int64_t N, int64_t K, void* Wo,
                             cudaStream_t st);
int sq_diff_ctas();
cudaError_t launch_smooth_activations(const void* X, int dtype, const float* s, int64_t M, int64_t K,
                                      void* Xs, cudaStream_t st);
cudaError_t launch_sq_diff_sum(const void* A, const void* B, int dtype, int64_t n, double* partials,
                               double* out, cudaStream_t st);

// ---- small device helpers ----
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t and_mask, uint32_t or_mask) {
  uint32_t r;
  // r = (a & b) | c   -> immLut = (0xF0 & 0xCC) | 0xAA = 0xEA
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;\n" : "=r"(r) : "r"(a), "r"(and_mask), "r"(or_mask));
  return r;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;\n" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ uint4 ld_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ uint16_t ld_u16(const uint16_t* p) {
  uint16_t r;
  asm volatile("ld.global.nc.u16 %0, [%1];\n" : "=h"(r) : "l"(p));
  return r;
}

}  // namespace sq
