// K-smooth: column abs-max reductions and the Eq. 6 smoothing factors.
//
//   a1  w_max[k] = max_n |W[n][k]|          PAPER.md:162-164 Eq. 6 "max(|W_j|)"
//   A14 act_max[k] = max_t |X[t][k]|        PAPER.md:162-164 Eq. 6 "max(|X_j|)"
//   a2  s[k] = max(a,eps)^alpha / max(w,eps)^(1-alpha), fp64, RN to fp32
//
// HBM-bound column reduction: each thread owns 8 consecutive columns (one 16-byte
// vector per row), a CTA covers 2048 columns x a slice of rows, and the per-column
// maxima are merged with atomicMax on the fp32 bit pattern (all values >= 0, so
// the unsigned order of the bits is the numeric order; NaN sorts above Inf and so
// propagates, like numpy's max).  Inside a thread the maxima are kept as packed
// 16-bit |x| bit patterns and merged with one SIMD unsigned max per pair
// (exact: fp16/bf16 abs bits are ordered like their values).
#include "sq_internal.cuh"

namespace sq {

namespace {

constexpr int kColsPerThread = 8;
constexpr int kThreads = 256;
constexpr int kColsPerCta = kColsPerThread * kThreads;

__device__ __forceinline__ uint32_t vmaxu2(uint32_t a, uint32_t b) { return __vmaxu2(a, b); }

template <bool kBF16>
__device__ __forceinline__ uint32_t abs16_to_f32bits(uint32_t h) {
  if (kBF16) return h << 16;  // bf16 -> fp32 is a shift
  return __float_as_uint(__half2float(__ushort_as_half(static_cast<unsigned short>(h))));
}

template <bool kBF16>
__global__ void __launch_bounds__(kThreads)
colabsmax_kernel(const uint16_t* __restrict__ X, int64_t rows, int64_t K, int64_t rows_per_cta,
                 unsigned* __restrict__ out) {
  const int64_t col0 = (int64_t)blockIdx.x * kColsPerCta + (int64_t)threadIdx.x * kColsPerThread;
  if (col0 >= K) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_cta;
  const int64_t r1 = min(rows, r0 + rows_per_cta);
  uint32_t m0 = 0, m1 = 0, m2 = 0, m3 = 0;
  const uint16_t* p = X + r0 * K + col0;
  int64_t r = r0;
  // 4 rows in flight per iteration
  for (; r + 4 <= r1; r += 4, p += 4 * K) {
    uint4 v0 = ld_nc_v4(p), v1 = ld_nc_v4(p + K), v2 = ld_nc_v4(p + 2 * K), v3 = ld_nc_v4(p + 3 * K);
    m0 = vmaxu2(m0, vmaxu2(vmaxu2(v0.x & 0x7FFF7FFFu, v1.x & 0x7FFF7FFFu),
                           vmaxu2(v2.x & 0x7FFF7FFFu, v3.x & 0x7FFF7FFFu)));
    m1 = vmaxu2(m1, vmaxu2(vmaxu2(v0.y & 0x7FFF7FFFu, v1.y & 0x7FFF7FFFu),
                           vmaxu2(v2.y & 0x7FFF7FFFu, v3.y & 0x7FFF7FFFu)));
    m2 = vmaxu2(m2, vmaxu2(vmaxu2(v0.z & 0x7FFF7FFFu, v1.z & 0x7FFF7FFFu),
                           vmaxu2(v2.z & 0x7FFF7FFFu, v3.z & 0x7FFF7FFFu)));
    m3 = vmaxu2(m3, vmaxu2(vmaxu2(v0.w & 0x7FFF7FFFu, v1.w & 0x7FFF7FFFu),
                           vmaxu2(v2.w & 0x7FFF7FFFu, v3.w & 0x7FFF7FFFu)));
  }
  for (; r < r1; ++r, p += K) {
    uint4 v = ld_nc_v4(p);
    m0 = vmaxu2(m0, v.x & 0x7FFF7FFFu);
    m1 = vmaxu2(m1, v.y & 0x7FFF7FFFu);
    m2 = vmaxu2(m2, v.z & 0x7FFF7FFFu);
    m3 = vmaxu2(m3, v.w & 0x7FFF7FFFu);
  }
  const uint32_t m[4] = {m0, m1, m2, m3};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    atomicMax(out + col0 + 2 * i, abs16_to_f32bits<kBF16>(m[i] & 0xFFFFu));
    atomicMax(out + col0 + 2 * i + 1, abs16_to_f32bits<kBF16>(m[i] >> 16));
  }
}

__global__ void smooth_finalize_kernel(const float* __restrict__ act_max, float* __restrict__ s,
                                       int64_t K, double alpha, double eps) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const double a = fmax((double)act_max[k], eps);
  const double w = fmax((double)s[k], eps);  // s holds w_max (exact fp16/bf16 values)
  double v;
  if (alpha == 0.5) {
    v = sqrt(a) / sqrt(w);
  } else if (alpha == 1.0) {
    v = a;
  } else if (alpha == 0.0) {
    v = 1.0 / w;
  } else {
    v = pow(a, alpha) / pow(w, 1.0 - alpha);
  }
  // NaN inputs propagate (fmax drops one NaN operand, so re-check explicitly)
  if (isnan(act_max[k]) || isnan(s[k])) v = __longlong_as_double(0x7FF8000000000000ll);
  s[k] = __double2float_rn(v);
}

}  // namespace

cudaError_t launch_colabsmax(const void* X, int dtype, int64_t rows, int64_t K, float* out,
                             cudaStream_t st) {
  const int64_t kblocks = (K + kColsPerCta - 1) / kColsPerCta;
  const int64_t target = 4ll * num_sms();
  int64_t rsplit = (target + kblocks - 1) / kblocks;
  rsplit = std::max<int64_t>(1, std::min<int64_t>(rsplit, (rows + 15) / 16));
  const int64_t rows_per_cta = (rows + rsplit - 1) / rsplit;
  rsplit = (rows + rows_per_cta - 1) / rows_per_cta;
  dim3 grid((unsigned)kblocks, (unsigned)rsplit);
  if (dtype == SQ_BF16)
    colabsmax_kernel<true><<<grid, kThreads, 0, st>>>((const uint16_t*)X, rows, K, rows_per_cta,
                                                      (unsigned*)out);
  else
    colabsmax_kernel<false><<<grid, kThreads, 0, st>>>((const uint16_t*)X, rows, K, rows_per_cta,
                                                       (unsigned*)out);
  return cudaGetLastError();
}

cudaError_t launch_smooth_finalize(const float* act_max, float* s, int64_t K, double alpha,
                                   double eps, cudaStream_t st) {
  const int threads = 256;
  smooth_finalize_kernel<<<(unsigned)((K + threads - 1) / threads), threads, 0, st>>>(act_max, s, K,
                                                                                      alpha, eps);
  return cudaGetLastError();
}

}  // namespace sq
