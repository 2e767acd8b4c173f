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
//  * codes (fp16 path): a non-tie v/Δ is >= 2^-12 from any half-integer (fp16 v, Δ), so
//    rounding v * RN(1/Δ)(1 + 2^-17) to the nearest integer (one FFMA with the 1.5 * 2^23
//    magic constant) is RHA(v/Δ): the factor pushes exact ties away from zero by more than
//    the product's error and moves non-ties by less than the gap (see the code).  The
//    clamp and the nibble packing then run on two codes per instruction (s16x2).
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
  // NaN-propagating: a NaN anywhere in the group reaches the reduced min and max
  __device__ static uint32_t min2(uint32_t a, uint32_t b) {
    __half2 r = __hmin2_nan(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
  }
  __device__ static uint32_t max2(uint32_t a, uint32_t b) {
    __half2 r = __hmax2_nan(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
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
    __nv_bfloat162 r = __hmin2_nan(*reinterpret_cast<__nv_bfloat162*>(&a),
                                   *reinterpret_cast<__nv_bfloat162*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
  }
  __device__ static uint32_t max2(uint32_t a, uint32_t b) {
    __nv_bfloat162 r = __hmax2_nan(*reinterpret_cast<__nv_bfloat162*>(&a),
                                   *reinterpret_cast<__nv_bfloat162*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
  }
};

// w * s rounded to odd in fp32 (RZ product, sticky bit from the exact FMA residual): its
// RN to fp16/bf16 is the single rounding RN_fmt(w * s) (24 >= 11 + 2 bits)
template <bool kBF16>
__device__ __forceinline__ float fold_odd(uint16_t wbits, float s) {
  const float w = Fmt<kBF16>::to_f(wbits);
  float p = __fmul_rz(w, s);
  const float e = __fmaf_rn(w, s, -p);
  if (e != 0.0f) p = __uint_as_float(__float_as_uint(p) | 1u);
  return p;
}
// two round-to-odd products -> RN pair in one packing conversion (F2FP)
template <bool kBF16>
__device__ __forceinline__ uint32_t pack_rn(float lo, float hi) {
  if (kBF16) {
    const __nv_bfloat162 b = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&b);
  }
  const __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}

template <bool kBF16, int GS>
__global__ void __launch_bounds__(kThreads)
quantize_kernel(const uint16_t* __restrict__ W, const float* __restrict__ s, int N, int K, int NSL,
                uint8_t* __restrict__ Wq, uint16_t* __restrict__ scales,
                void* __restrict__ zeros, int zeros_u4, int* __restrict__ nonfinite) {
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
        w[2 * q] = pack_rn<kBF16>(fold_odd<kBF16>(w[2 * q] & 0xFFFFu, sv.x), fold_odd<kBF16>(w[2 * q] >> 16, sv.y));
        w[2 * q + 1] =
            pack_rn<kBF16>(fold_odd<kBF16>(w[2 * q + 1] & 0xFFFFu, sv.z), fold_odd<kBF16>(w[2 * q + 1] >> 16, sv.w));
      }
    }
    // min / max with NaN propagation; a NaN or ±Inf in the group then shows in mn or mx,
    // so the non-finite test (abs bits >= exponent mask) runs once per group on them
    uint32_t mn = w[0], mx = w[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) {
      mn = Fmt<kBF16>::min2(mn, w[i]);
      mx = Fmt<kBF16>::max2(mx, w[i]);
    }
#pragma unroll
    for (int o = 1; o < kLanesPerGroup; o <<= 1) {
      mn = Fmt<kBF16>::min2(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = Fmt<kBF16>::max2(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const uint32_t amax = __vmaxu2(mn & 0x7FFF7FFFu, mx & 0x7FFF7FFFu);
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
    // fp16: RN(1/Δ)(1 + 2^-17) turns RHA(v / Δ) into one FFMA (see the codes below)
    const float inv = kBF16 ? 0.0f : __fmul_rn(__frcp_rn(d), 1.0f + 0x1p-17f);
    // Z = clamp(RHA(-lo / Δ), 0, 15) (reading S2): for fp16 the same exact one-FFMA rounding
    // (-lo is an fp16 value); bf16 lo needs the fp64 quotient
    float z;
    if (!kBF16) {
      const int zc = __float_as_int(__fmaf_rn(-lo, inv, 12582912.0f)) - 0x4B400000;
      z = (float)min(max(zc, 0), 15);
    } else {
      z = (float)fmin(fmax(round(-(double)lo / (double)d), 0.0), 15.0);
    }

    // codes for this lane's 16 elements, packed low nibble = even k
    uint32_t packed[2] = {0u, 0u};
    if (!nf) {
      if (!kBF16) {
        // RHA(v / Δ) as ONE FFMA per element: RN(v * inv' + 1.5 * 2^23) - 1.5 * 2^23 with
        // inv' = RN(RN(1/Δ) (1 + 2^-17)).  v * inv' = x (1 + 2^-17)(1 + δ), |δ| <= 3 * 2^-24,
        // x = v / Δ.  An exact tie x = k + 1/2 is pushed away from zero by |x| 2^-17, far
        // more than |x| δ, so round-to-nearest of it is RHA; a non-tie (|x| < 16) lies
        // >= 2^-12 from every half-integer (fp16 v and Δ), and |x| (2^-17 + 3 * 2^-24) <
        // 2^-12 cannot cross one.  |x| >= 16 is clamped below whichever way it rounds, and
        // |x| < 2^15 - 16 always (Δ >= (r / 15)(1 - 2^-10) and r >= |v| 2^-11), so the
        // integer c + Z fits the signed 16-bit lanes of the clamp.
        // The magic constant carries + Z: RN(v * inv' + 1.5 * 2^23 + Z) is 1.5 * 2^23 + Z + c
        // (no exact ties remain, see above), whose float bits are 0x4B400000 + (Z + c), so the
        // low 16 bits ARE the signed code Z + c (|Z + c| < 2^15): no subtraction needed.
        const float cz = 12582912.0f + z;
        uint32_t bytes[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {  // element pair (2q, 2q + 1) = the two halves of w[q]
          const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[q]));
          const uint32_t b0 = __float_as_uint(__fmaf_rn(f.x, inv, cz));
          const uint32_t b1 = __float_as_uint(__fmaf_rn(f.y, inv, cz));
          uint32_t cc = __byte_perm(b0, b1, 0x5410);  // (Z + c0, Z + c1) as s16x2
          asm("max.s16x2 %0, %0, %1;" : "+r"(cc) : "r"(0u));
          asm("min.s16x2 %0, %0, %1;" : "+r"(cc) : "r"(0x000F000Fu));
          bytes[q] = (cc | (cc >> 12)) & 0xFFu;  // low nibble = even k
        }
        // gather the eight bytes: two PRMTs per pair of bytes, one per word
        packed[0] = __byte_perm(__byte_perm(bytes[0], bytes[1], 0x0040), __byte_perm(bytes[2], bytes[3], 0x0040),
                                0x5410);
        packed[1] = __byte_perm(__byte_perm(bytes[4], bytes[5], 0x0040), __byte_perm(bytes[6], bytes[7], 0x0040),
                                0x5410);
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint32_t bits = (i & 1) ? (w[i >> 1] >> 16) : (w[i >> 1] & 0xFFFFu);
          const float v = Fmt<kBF16>::to_f((uint16_t)bits);
          float c = (float)round((double)v / (double)d);  // bf16: the gap can be 2^-20, fp64
          c = fminf(fmaxf(c + z, 0.0f), 15.0f);
          packed[i >> 3] |= (__float_as_uint(c + 8388608.0f) & 0xFu) << (4 * (i & 7));
        }
      }
    }
    // packed u4 Z (SQ_ZEROS_U4): rows n and n + 1 of a pair sit 8 lanes apart in the warp
    // (8 lanes per row); the even row's lane writes the byte, low nibble = even n
    const uint32_t zq = nf ? 0u : (uint32_t)z;
    const uint32_t zq_odd = __shfl_down_sync(0xffffffffu, zq, kLanesPerSlot);
    if (row_ok) {
      *reinterpret_cast<uint2*>(Wq + (size_t)n * (K / 2) + (size_t)g * (kSlot / 2) + sub * 8) =
          make_uint2(packed[0], packed[1]);
      if (sub % kLanesPerGroup == 0) {  // first lane of each group
        const size_t gi = (size_t)g * (kSlot / GS) + sub / kLanesPerGroup;
        scales[gi * N + n] = nf ? (uint16_t)0x7E00u : __half_as_ushort(__float2half_rn(d));
        if (!zeros_u4)
          reinterpret_cast<uint16_t*>(zeros)[gi * N + n] = nf ? (uint16_t)0u : __half_as_ushort(__float2half_rn(z));
        else if ((n & 1) == 0)
          reinterpret_cast<uint8_t*>(zeros)[gi * (N / 2) + n / 2] = (uint8_t)(zq | (zq_odd << 4));
        if (nf && nonfinite != nullptr) atomicAdd(nonfinite, 1);
      }
    }
  }
}

}  // namespace

template <int GS>
void launch_gs(const void* W, int w_dtype, const float* s, int64_t N, int64_t K, uint8_t* Wq, uint16_t* scales,
               void* zeros, bool zu4, int* nonfinite, cudaStream_t st) {
  const int NSL = (int)(K / kSlot);
  dim3 grid((unsigned)((NSL + kSlotsPerCta - 1) / kSlotsPerCta), (unsigned)((N + kRowsPerCta - 1) / kRowsPerCta));
  if (w_dtype == SQ_BF16)
    quantize_kernel<true, GS><<<grid, kThreads, 0, st>>>((const uint16_t*)W, s, (int)N, (int)K, NSL, Wq, scales,
                                                         zeros, zu4 ? 1 : 0, nonfinite);
  else
    quantize_kernel<false, GS><<<grid, kThreads, 0, st>>>((const uint16_t*)W, s, (int)N, (int)K, NSL, Wq, scales,
                                                          zeros, zu4 ? 1 : 0, nonfinite);
}

cudaError_t launch_quantize(const void* W, int w_dtype, const float* s, int64_t N, int64_t K, int group,
                            uint8_t* Wq, uint16_t* scales, void* zeros, bool zeros_u4, int* nonfinite,
                            cudaStream_t st) {
  if (group == 32)
    launch_gs<32>(W, w_dtype, s, N, K, Wq, scales, zeros, zeros_u4, nonfinite, st);
  else if (group == 64)
    launch_gs<64>(W, w_dtype, s, N, K, Wq, scales, zeros, zeros_u4, nonfinite, st);
  else
    launch_gs<128>(W, w_dtype, s, N, K, Wq, scales, zeros, zeros_u4, nonfinite, st);
  return cudaGetLastError();
}

}  // namespace sq
