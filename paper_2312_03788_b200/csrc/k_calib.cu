// K-calib: the device steps the single-layer α grid search and the
// model-level smoothing fusion (N3, Fig. 5) add to the hot-path kernels.
//
//  * fold_rows:  W'[n][k] = RN_dtype(W[n][k] / d[n]) -- s^-1 folded into the output rows
//    of the producing linear; fp64 quotient, one rounding.
//  * smooth_activations:  X̂[m][k] = RN_dtype(X[m][k] / s[k])  -- the activation side of
//    Eq. 5, X·diag(s)^-1.  The quotient is taken in fp64 (correctly
//    rounded) and rounded once to fp16/bf16, so the result is bit-identical to the oracle's
//    RN16(fp64(X) / fp64(s)).  HBM-bound: 4 B/element (2 read, 2 written) + 4K for s.
//  * sq_diff_sum:  E = Σ_i (A_i - B_i)^2 in fp64 -- the squared Frobenius norm of Eq. 4
//     over two fp16/bf16 outputs.  Deterministic: a fixed grid, each
//    CTA sums a fixed strided slice in a fixed order (thread-local fp64, then a fixed
//    shuffle/SMEM tree), and one CTA sums the per-CTA partials in index order.
#include <algorithm>

#include "sq_internal.cuh"

namespace sq {

namespace {

constexpr int kCalibThreads = 256;

template <bool kBF16>
__device__ __forceinline__ double load_f64(const uint16_t* p, int64_t i) {
  const uint16_t b = p[i];
  if (kBF16) return (double)__bfloat162float(__ushort_as_bfloat16(b));
  return (double)__half2float(__ushort_as_half(b));
}

template <bool kBF16>
__device__ __forceinline__ uint16_t store_rn(double v) {
  if (kBF16) return __bfloat16_as_ushort(__double2bfloat16(v));
  return __half_as_ushort(__double2half(v));
}

// 8 consecutive elements per thread (one 16-B load and store); K % 8 == 0 so a vector
// never crosses a row.
template <bool kBF16>
__global__ void __launch_bounds__(kCalibThreads)
smooth_activations_kernel(const uint4* X, const float* __restrict__ s, uint4* Xs,  // X, Xs may alias
                          int64_t nvec, int64_t K) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint4 in = X[v];
    const int64_t k0 = (v * 8) % K;
    const uint16_t* e = reinterpret_cast<const uint16_t*>(&in);
    uint4 out;
    uint16_t* o = reinterpret_cast<uint16_t*>(&out);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double x = load_f64<kBF16>(e, i);
      o[i] = store_rn<kBF16>(__ddiv_rn(x, (double)__ldg(s + k0 + i)));
    }
    Xs[v] = out;
  }
}

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kCalibThreads / 32; ++w) t += red[w];  // fixed order
  return t;
}

template <bool kBF16>
__global__ void __launch_bounds__(kCalibThreads)
sq_diff_partials_kernel(const uint16_t* __restrict__ A, const uint16_t* __restrict__ B, int64_t n,
                        double* __restrict__ partials) {
  __shared__ double red[kCalibThreads / 32];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = load_f64<kBF16>(A, i) - load_f64<kBF16>(B, i);  // exact (both fp16/bf16)
    acc = fma(d, d, acc);
  }
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

__global__ void __launch_bounds__(kCalibThreads)
sq_diff_final_kernel(const double* __restrict__ partials, int n, double* __restrict__ out) {
  __shared__ double red[kCalibThreads / 32];
  // each thread sums a fixed strided subset in index order, then the fixed tree
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partials[i];
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) *out = t;
}

// W_out[n][k] = RN_dtype(W[n][k] / d[n]): folding a smoothing factor s^-1 into the OUTPUT
// rows of the linear that produces the smoothed activation (Fig. 5: for
// down_proj, "the operation of dividing its input by the smoothing factor is fused into
// the weights of up_proj").  fp64 quotient, one rounding (bit-identical to the oracle).
template <bool kBF16>
__global__ void __launch_bounds__(kCalibThreads)
fold_rows_kernel(const uint4* W, const float* __restrict__ d, uint4* Wo,  // W, Wo may alias
                 int64_t nvec, int64_t K) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint4 in = W[v];
    const double dn = (double)__ldg(d + (v * 8) / K);
    const uint16_t* e = reinterpret_cast<const uint16_t*>(&in);
    uint4 out;
    uint16_t* o = reinterpret_cast<uint16_t*>(&out);
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = store_rn<kBF16>(__ddiv_rn(load_f64<kBF16>(e, i), dn));
    Wo[v] = out;
  }
}

}  // namespace

cudaError_t launch_fold_rows(const void* W, int dtype, const float* d, int64_t N, int64_t K, void* Wo,
                             cudaStream_t st) {
  const int64_t nvec = N * K / 8;
  if (nvec == 0) return cudaSuccess;
  const int grid = (int)std::min<int64_t>((nvec + kCalibThreads - 1) / kCalibThreads, (int64_t)num_sms() * 16);
  if (dtype == SQ_BF16)
    fold_rows_kernel<true><<<grid, kCalibThreads, 0, st>>>(static_cast<const uint4*>(W), d,
                                                            static_cast<uint4*>(Wo), nvec, K);
  else
    fold_rows_kernel<false><<<grid, kCalibThreads, 0, st>>>(static_cast<const uint4*>(W), d,
                                                             static_cast<uint4*>(Wo), nvec, K);
  return cudaGetLastError();
}

int sq_diff_ctas() { return 4 * num_sms(); }

cudaError_t launch_smooth_activations(const void* X, int dtype, const float* s, int64_t M, int64_t K,
                                      void* Xs, cudaStream_t st) {
  const int64_t nvec = M * K / 8;
  if (nvec == 0) return cudaSuccess;
  const int64_t want = (nvec + kCalibThreads - 1) / kCalibThreads;
  const int grid = (int)std::min<int64_t>(want, (int64_t)num_sms() * 16);
  if (dtype == SQ_BF16)
    smooth_activations_kernel<true><<<grid, kCalibThreads, 0, st>>>(
        static_cast<const uint4*>(X), s, static_cast<uint4*>(Xs), nvec, K);
  else
    smooth_activations_kernel<false><<<grid, kCalibThreads, 0, st>>>(
        static_cast<const uint4*>(X), s, static_cast<uint4*>(Xs), nvec, K);
  return cudaGetLastError();
}

cudaError_t launch_sq_diff_sum(const void* A, const void* B, int dtype, int64_t n, double* partials,
                               double* out, cudaStream_t st) {
  const int P = sq_diff_ctas();
  if (dtype == SQ_BF16)
    sq_diff_partials_kernel<true><<<P, kCalibThreads, 0, st>>>(static_cast<const uint16_t*>(A),
                                                               static_cast<const uint16_t*>(B), n, partials);
  else
    sq_diff_partials_kernel<false><<<P, kCalibThreads, 0, st>>>(static_cast<const uint16_t*>(A),
                                                                static_cast<const uint16_t*>(B), n, partials);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  sq_diff_final_kernel<<<1, kCalibThreads, 0, st>>>(partials, P, out);
  return cudaGetLastError();
}

}  // namespace sq
