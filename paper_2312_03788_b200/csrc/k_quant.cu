// K-quant: Eq. 5 weight-side fold + Eq. 1 group-wise asymmetric INT4 quantization
// and nibble packing (sq_quantize_pack_groupwise).  Bit-exact with oracle/.
//
//   a3  W'[n][k] = RN(W[n][k] * s[k])        PAPER.md:139-141 Eq. 5 "diag(s)W"; reading S13
//   a4  Δ = RZ16((max - min) / 15), Z, codes   PAPER.md:88-93 Eq. 1; readings S1-S4
//       pack: low nibble = even k
//
// Layout: a CTA of 256 threads owns 32 consecutive output channels (rows n) and
// kSlotsPerCta consecutive 128-k slots; 8 lanes share one (row, slot): lane `sub` holds
// elements [16*sub, 16*sub+16) of the slot (two 16-byte loads, all issued before any
// arithmetic).  A group ("different group sizes": GS = 128, 64 or 32) is
// GS/16 consecutive lanes; min/max are reduced with half2 min/max + log2(GS/16)
// xor-shuffles.
//
// Exactness:
//  * fold: fp32 multiply rounded toward zero + FMA residual gives the product
//    rounded-to-odd in fp32 (24 bits >= 11 + 2), so the final RN to fp16/bf16 is the
//    correctly rounded exact product (one rounding, reading S13).
//  * r = hi - lo in fp64 (exact for fp16 inputs), Δ = RZ16(r/15) via fp64 division
//    then RZ->fp32->RZ->fp16 (RZ∘RZ = RZ).
//  * codes (fp16 path): t = v * RN(1/Δ) has |error| <= 2^-19 for |t| < 16 while a
//    non-tie v/Δ is >= 2^-12 from any half-integer (fp16 v, Δ), so trunc(t ± 1/2) is the
//    RHA of v/Δ except at an exact tie that t missed, which one branch-free FMA detects
//    exactly (v - (c ± 1/2)Δ is computed exactly) and moves away from zero.
//  * codes (bf16 path): the gap can be as small as 2^-20, so v/Δ uses fp64 division.
#include <algorithm>

#include "sq_internal.cuh"

namespace sq {

namespace {

constexpr int kThreads = 256;
constexpr int kRowsPerCta = 32;
constexpr int kLanesPerSlot = 8;
constexpr int kSlot = 128;      // k per slot; K % 128 == 0 for every group size
constexpr int kSlotsPerCta = 4;

template <bool kBF16>
struct Fmt;
template <>
struct Fmt<false> {
  static constexpr uint32_t kExpMask = 0x7C00u;
  __device__ static float to_f(uint16_t b) { return __half2float(__ushort_as_half(b)); }
  __device__ static uint16_t from_f_rn(float f) { return __half_as_ushort(__float2half_rn(f)); }
  __device__ static uint32_t min2(uint32_t a, uint32_t b) {
    __half2 r = __hmin2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
  }
  __device__ static uint32_t max2(uint32_t a, uint32_t b) {
    __half2 r = __hmax2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
  }
};
template <>
struct Fmt<true> {
  static constexpr uint32_t kExpMask = 0x7F80u;
  __device__ static float to_f(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }
  __device__ static uint16_t from_f_rn(float f) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(f));
  }
  __device__ static uint32_t min2(uint32_t a, uint32_t b) {
    __nv_bfloat162 r = __hmin2(*reinterpret_cast<__nv_bfloat162*>(&a),
                               *reinterpret_cast<__nv_bfloat162*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
  }
  __device__ static uint32_t max2(uint32_t a, uint32_t b) {
    __nv_bfloat162 r = __hmax2(*reinterpret_cast<__nv_bfloat162*>(&a),
                               *reinterpret_cast<__nv_bfloat162*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
  }
};

// RN_fmt(w * s) with a single rounding (round-to-odd in fp32, then RN).
template <bool kBF16>
__device__ __forceinline__ uint16_t fold1(uint16_t wbits, float s) {
  const float w = Fmt<kBF16>::to_f(wbits);
  float p = __fmul_rz(w, s);
  const float e = __fmaf_rn(w, s, -p);
  if (e != 0.0f) p = __uint_as_float(__float_as_uint(p) | 1u);
  return Fmt<kBF16>::from_f_rn(p);
}

// RHA(v / d) for fp16 v, d (see header comment), as float, branch-free.  t = v * RN(1/d)
// is within 2^-19 of x = v/d (|x| < 16) while a non-tie x is >= 2^-12 from every k + 1/2,
// so c = trunc(t + copysign(1/2, t)) is RHA(x) unless x is an exact tie that t missed by
// rounding toward zero; then v - (c + copysign(1/2, t)) d is exactly 0 (one FMA, the
// product is exact) and c moves one step away from zero.  A nonzero exact difference
// never rounds to 0, so non-ties are never moved.
__device__ __forceinline__ float rha_div_f16(float v, float d, float inv) {
  const float t = v * inv;
  const float h = copysignf(0.5f, t);
  const float c = truncf(t + h);
  return __fmaf_rn(-(c + h), d, v) == 0.0f ? c + 2.0f * h : c;
}

template <bool kBF16, int GS>
__global__ void __launch_bounds__(kThreads)
quantize_kernel(const uint16_t* __restrict__ W, const float* __restrict__ s, int N, int K, int NSL,
                uint8_t* __restrict__ Wq, uint16_t* __restrict__ scales,
                uint16_t* __restrict__ zeros, int* __restrict__ nonfinite) {
  constexpr int kLanesPerGroup = GS / 16;
  const int sub = threadIdx.x % kLanesPerSlot;
  const int n = blockIdx.y * kRowsPerCta + threadIdx.x / kLanesPerSlot;
  const int g0 = blockIdx.x * kSlotsPerCta;  // first slot of the CTA
  const bool row_ok = n < N;

  // issue every load of the CTA's groups first (memory-level parallelism)
  uint4 va[kSlotsPerCta], vb[kSlotsPerCta];
#pragma unroll
  for (int j = 0; j < kSlotsPerCta; ++j) {
    const int g = g0 + j;
    if (row_ok && g < NSL) {
      const uint16_t* p = W + (size_t)n * K + (size_t)g * kSlot + sub * 16;
      va[j] = ld_nc_v4(p);
      vb[j] = ld_nc_v4(p + 8);
    } else {
      va[j] = make_uint4(0, 0, 0, 0);
      vb[j] = va[j];
    }
  }

#pragma unroll
  for (int j = 0; j < kSlotsPerCta; ++j) {
    const int g = g0 + j;
    if (g >= NSL) break;  // uniform across the CTA
    uint32_t w[8] = {va[j].x, va[j].y, va[j].z, va[j].w, vb[j].x, vb[j].y, vb[j].z, vb[j].w};
    if (s != nullptr) {
      const float4* sp = reinterpret_cast<const float4*>(s + (size_t)g * kSlot + sub * 16);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 sv = __ldg(sp + q);
        const uint32_t lo0 = fold1<kBF16>(w[2 * q] & 0xFFFFu, sv.x);
        const uint32_t hi0 = fold1<kBF16>(w[2 * q] >> 16, sv.y);
        const uint32_t lo1 = fold1<kBF16>(w[2 * q + 1] & 0xFFFFu, sv.z);
        const uint32_t hi1 = fold1<kBF16>(w[2 * q + 1] >> 16, sv.w);
        w[2 * q] = lo0 | (hi0 << 16);
        w[2 * q + 1] = lo1 | (hi1 << 16);
      }
    }
    // non-finite detection (abs bits >= exponent mask) and min / max
    uint32_t amax = 0, mn = w[0], mx = w[0];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      amax = __vmaxu2(amax, w[i] & 0x7FFF7FFFu);
      mn = Fmt<kBF16>::min2(mn, w[i]);
      mx = Fmt<kBF16>::max2(mx, w[i]);
    }
#pragma unroll
    for (int o = 1; o < kLanesPerGroup; o <<= 1) {
      amax = __vmaxu2(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      mn = Fmt<kBF16>::min2(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = Fmt<kBF16>::max2(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    bool nf = ((amax & 0xFFFFu) >= Fmt<kBF16>::kExpMask) || ((amax >> 16) >= Fmt<kBF16>::kExpMask);
    const float lo = fminf(Fmt<kBF16>::to_f(mn & 0xFFFFu), Fmt<kBF16>::to_f(mn >> 16));
    const float hi = fmaxf(Fmt<kBF16>::to_f(mx & 0xFFFFu), Fmt<kBF16>::to_f(mx >> 16));

    // Δ (readings S3, S4)
    const double r = (double)hi - (double)lo;
    float d;
    if (r > 0.0) {
      const double q = r / 15.0;
      if (q > 65504.0) nf = true;
      d = __half2float(__float2half_rz(__double2float_rz(q)));
      if (d == 0.0f) d = 0x1p-24f;
    } else {
      d = (lo == 0.0f) ? 1.0f : fabsf(lo);
    }
    if (nf) d = 1.0f;
    // Z (reading S2), once per group: fp64 division (exact-enough for bf16 lo too)
    const float z = (float)fmin(fmax(round(-(double)lo / (double)d), 0.0), 15.0);

    // codes for this lane's 16 elements, packed low nibble = even k
    uint32_t packed[2] = {0u, 0u};
    if (!nf) {
      const float inv = __frcp_rn(d);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t bits = (i & 1) ? (w[i >> 1] >> 16) : (w[i >> 1] & 0xFFFFu);
        const float v = Fmt<kBF16>::to_f((uint16_t)bits);
        float c;
        if (kBF16) {
          c = (float)round((double)v / (double)d);
        } else {
          c = rha_div_f16(v, d, inv);
        }
        c = fminf(fmaxf(c + z, 0.0f), 15.0f);
        // integral c in [0, 15]: c + 2^23 is exact and its low mantissa bits are c (no
        // float->int conversion instruction)
        packed[i >> 3] |= (__float_as_uint(c + 8388608.0f) & 0xFu) << (4 * (i & 7));
      }
    }
    if (row_ok) {
      *reinterpret_cast<uint2*>(Wq + (size_t)n * (K / 2) + (size_t)g * (kSlot / 2) + sub * 8) =
          make_uint2(packed[0], packed[1]);
      if (sub % kLanesPerGroup == 0) {  // first lane of each group
        const size_t gi = (size_t)g * (kSlot / GS) + sub / kLanesPerGroup;
        scales[gi * N + n] = nf ? (uint16_t)0x7E00u : __half_as_ushort(__float2half_rn(d));
        zeros[gi * N + n] = nf ? (uint16_t)0u : __half_as_ushort(__float2half_rn(z));
        if (nf && nonfinite != nullptr) atomicAdd(nonfinite, 1);
      }
    }
  }
}

}  // namespace

template <int GS>
void launch_gs(const void* W, int w_dtype, const float* s, int64_t N, int64_t K, uint8_t* Wq, uint16_t* scales,
               uint16_t* zeros, int* nonfinite, cudaStream_t st) {
  const int NSL = (int)(K / kSlot);
  dim3 grid((unsigned)((NSL + kSlotsPerCta - 1) / kSlotsPerCta), (unsigned)((N + kRowsPerCta - 1) / kRowsPerCta));
  if (w_dtype == SQ_BF16)
    quantize_kernel<true, GS><<<grid, kThreads, 0, st>>>((const uint16_t*)W, s, (int)N, (int)K, NSL, Wq, scales,
                                                         zeros, nonfinite);
  else
    quantize_kernel<false, GS><<<grid, kThreads, 0, st>>>((const uint16_t*)W, s, (int)N, (int)K, NSL, Wq, scales,
                                                          zeros, nonfinite);
}

cudaError_t launch_quantize(const void* W, int w_dtype, const float* s, int64_t N, int64_t K, int group,
                            uint8_t* Wq, uint16_t* scales, uint16_t* zeros, int* nonfinite,
                            cudaStream_t st) {
  if (group == 32)
    launch_gs<32>(W, w_dtype, s, N, K, Wq, scales, zeros, nonfinite, st);
  else if (group == 64)
    launch_gs<64>(W, w_dtype, s, N, K, Wq, scales, zeros, nonfinite, st);
  else
    launch_gs<128>(W, w_dtype, s, N, K, Wq, scales, zeros, nonfinite, st);
  return cudaGetLastError();
}

}  // namespace sq
