// K-smooth: column abs-max reductions and the Eq. 6 smoothing factors.
//
//   a1  w_max[k] = max_n |W[n][k]|          PAPER.md:162-164 Eq. 6 "max(|W_j|)"
//   A14 act_max[k] = max_t |X[t][k]|        PAPER.md:162-164 Eq. 6 "max(|X_j|)"
//   a2  s[k] = max(a,eps)^alpha / max(w,eps)^(1-alpha), fp64, RN to fp32
//
// HBM-bound column reduction: each thread owns 8 consecutive columns (one 16-byte
// vector per row) of every kRowLanes-th row of its CTA's row slice; the row lanes of a
// warp are merged with shuffles, and the per-column maxima of the CTAs with atomicMax on the fp32 bit pattern (all values >= 0, so
// the unsigned order of the bits is the numeric order; NaN sorts above Inf and so
// propagates, like numpy's max).  Inside a thread the maxima are kept as packed
// 16-bit |x| bit patterns and merged with one SIMD unsigned max per pair
// (exact: fp16/bf16 abs bits are ordered like their values).
#include "sq_internal.cuh"

namespace sq {

namespace {

constexpr int kColsPerThread = 8;
constexpr int kThreads = 256;
// A warp = kRL row lanes x (32 / kRL) column threads: each row lane walks every kRL-th
// row of the CTA's slice, the lanes are merged with warp shuffles, and then one atomicMax
// per column leaves the CTA.  kRL = 1 (a warp reads 512 contiguous bytes of a row, a CTA
// 4 KB) suits slices of >= 128 rows per CTA; below that the atomics, not the loads, bound
// it and kRL = 8 (8x fewer atomics per byte) wins (profiles/r02/colabsmax_rowlanes_ab.jsonl)
constexpr int kRowsInFlight = 4;  // rows per thread and loop iteration
constexpr int kCtasPerSm = 4;     // grid target (row slices x column blocks)
template <int kRL>
constexpr int cols_per_cta() { return kColsPerThread * (32 / kRL) * (kThreads / 32); }

__device__ __forceinline__ uint32_t vmaxu2(uint32_t a, uint32_t b) { return __vmaxu2(a, b); }

template <bool kBF16>
__device__ __forceinline__ uint32_t abs16_to_f32bits(uint32_t h) {
  if (kBF16) return h << 16;  // bf16 -> fp32 is a shift
  return __float_as_uint(__half2float(__ushort_as_half(static_cast<unsigned short>(h))));
}

template <bool kBF16, int kRowLanes>
__global__ void __launch_bounds__(kThreads)
colabsmax_kernel(const uint16_t* __restrict__ X, int64_t rows, int64_t K, int64_t rows_per_cta,
                 unsigned* __restrict__ out) {
  constexpr int kColThreads = 32 / kRowLanes;  // per warp
  constexpr int kColsPerCta = cols_per_cta<kRowLanes>();
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  const int rl = lane / kColThreads;  // row lane
  const int64_t col0 = (int64_t)blockIdx.x * kColsPerCta +
                       (int64_t)(warp * kColThreads + lane % kColThreads) * kColsPerThread;
  const bool col_ok = col0 < K;  // K % 8 == 0: a thread's 8 columns are all valid or none
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_cta;
  const int64_t r1 = min(rows, r0 + rows_per_cta);
  uint32_t m0 = 0, m1 = 0, m2 = 0, m3 = 0;
  if (col_ok) {
    const uint16_t* p = X + (r0 + rl) * K + col0;
    int64_t r = r0 + rl;
    // kRowsInFlight of this lane's rows per iteration, every load issued before any max
    for (; r + (kRowsInFlight - 1) * kRowLanes < r1; r += kRowsInFlight * kRowLanes, p += kRowsInFlight * kRowLanes * K) {
      uint4 v[kRowsInFlight];
#pragma unroll
      for (int i = 0; i < kRowsInFlight; ++i) v[i] = ld_nc_v4(p + (int64_t)i * kRowLanes * K);
#pragma unroll
      for (int i = 0; i < kRowsInFlight; ++i) {
        m0 = vmaxu2(m0, v[i].x & 0x7FFF7FFFu);
        m1 = vmaxu2(m1, v[i].y & 0x7FFF7FFFu);
        m2 = vmaxu2(m2, v[i].z & 0x7FFF7FFFu);
        m3 = vmaxu2(m3, v[i].w & 0x7FFF7FFFu);
      }
    }
    for (; r < r1; r += kRowLanes, p += kRowLanes * K) {
      uint4 v = ld_nc_v4(p);
      m0 = vmaxu2(m0, v.x & 0x7FFF7FFFu);
      m1 = vmaxu2(m1, v.y & 0x7FFF7FFFu);
      m2 = vmaxu2(m2, v.z & 0x7FFF7FFFu);
      m3 = vmaxu2(m3, v.w & 0x7FFF7FFFu);
    }
  }
  // merge the row lanes (same columns, lanes kColThreads apart)
#pragma unroll
  for (int o = kColThreads; o < 32; o <<= 1) {
    m0 = vmaxu2(m0, __shfl_xor_sync(0xffffffffu, m0, o));
    m1 = vmaxu2(m1, __shfl_xor_sync(0xffffffffu, m1, o));
    m2 = vmaxu2(m2, __shfl_xor_sync(0xffffffffu, m2, o));
    m3 = vmaxu2(m3, __shfl_xor_sync(0xffffffffu, m3, o));
  }
  if (!col_ok || rl != 0) return;
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

template <int kRL>
static cudaError_t launch_colabsmax_rl(const void* X, int dtype, int64_t rows, int64_t K, float* out,
                                       cudaStream_t st) {
  const int64_t kblocks = (K + cols_per_cta<kRL>() - 1) / cols_per_cta<kRL>();
  const int64_t target = (int64_t)kCtasPerSm * num_sms();
  int64_t rsplit = (target + kblocks - 1) / kblocks;
  rsplit = std::max<int64_t>(1, std::min<int64_t>(rsplit, (rows + 15) / 16));
  const int64_t rows_per_cta = (rows + rsplit - 1) / rsplit;
  rsplit = (rows + rows_per_cta - 1) / rows_per_cta;
  dim3 grid((unsigned)kblocks, (unsigned)rsplit);
  if (dtype == SQ_BF16)
    colabsmax_kernel<true, kRL><<<grid, kThreads, 0, st>>>((const uint16_t*)X, rows, K, rows_per_cta,
                                                           (unsigned*)out);
  else
    colabsmax_kernel<false, kRL><<<grid, kThreads, 0, st>>>((const uint16_t*)X, rows, K, rows_per_cta,
                                                            (unsigned*)out);
  return cudaGetLastError();
}

cudaError_t launch_colabsmax(const void* X, int dtype, int64_t rows, int64_t K, float* out,
                             cudaStream_t st) {
  // rows per CTA of the one-row-lane grid: below 128 its atomics dominate, and below 256
  // when >= 128 row slices contend for every column (K <= 8192 on this GPU)
  const int64_t kblocks1 = (K + cols_per_cta<1>() - 1) / cols_per_cta<1>();
  const int64_t slices1 = std::max<int64_t>(
      1, std::min<int64_t>(((int64_t)kCtasPerSm * num_sms() + kblocks1 - 1) / kblocks1, (rows + 15) / 16));
  if ((rows + slices1 - 1) / slices1 >= (slices1 >= 128 ? 256 : 128))
    return launch_colabsmax_rl<1>(X, dtype, rows, K, out, st);
  return launch_colabsmax_rl<8>(X, dtype, rows, K, out, st);
}

cudaError_t launch_smooth_finalize(const float* act_max, float* s, int64_t K, double alpha,
                                   double eps, cudaStream_t st) {
  const int threads = 256;
  smooth_finalize_kernel<<<(unsigned)((K + threads - 1) / threads), threads, 0, st>>>(act_max, s, K,
                                                                                      alpha, eps);
  return cudaGetLastError();
}

}  // namespace sq
