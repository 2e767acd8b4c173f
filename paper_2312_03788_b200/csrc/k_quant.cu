// K-quant: Eq. 5 weight-side fold + Eq. 1 group-wise asymmetric INT4 quantization
// and nibble packing (sq_quantize_pack_groupwise).  Bit-exact with oracle/.
//
//   a3  W'[n][k] = RN(W[n][k] * s[k])        PAPER.md:139-141 Eq. 5 "diag(s)W"; reading S13
//   a4  Δ = RZ16((max - min) / 15), Z, codes   PAPER.md:88-93 Eq. 1; readings S1-S4
//       pack: low nibble = even k
//
// Layout: a CTA of 128 threads owns 16 consecutive output channels (rows n) and
// kSlotsPerCta consecutive 128-k slots; 8 lanes share one (row, slot): lane `sub` holds
// elements [16*sub, 16*sub+16) of the slot (one 32-byte load, all issued before any
// arithmetic).  A group ("different group sizes": GS = 128, 64 or 32) is
// GS/16 consecutive lanes; min/max are reduced with half2 min/max + log2(GS/16)
// xor-shuffles.  Δ, Z and the scale / zero stores then run once per group on one owner
// lane (not on every lane of every slot), and the codes fetch Δ and Z from it.
//
// Exactness:
//  * fold: the odd one of the fp32 products rounded down and up (equal when exact) is the
//    product rounded-to-odd in fp32 (24 bits >= 11 + 2), so the final RN to fp16/bf16 is
//    the correctly rounded exact product (one rounding, reading S13).
//  * r = hi - lo in fp64 (exact for fp16 inputs), Δ = RZ16(r/15) via fp64 division
//    then RZ->fp32->RZ->fp16 (RZ∘RZ = RZ).
//  * codes (fp16 path): a non-tie v/Δ is >= 2^-12 from any half-integer (fp16 v, Δ), so
//    rounding v * RN(1/Δ)(1 + 2^-17) to the nearest integer (one FFMA with the 1.5 * 2^23
//    magic constant) is RHA(v/Δ): the factor pushes exact ties away from zero by more than
//    the product's error and moves non-ties by less than the gap (see the code).  The
//    clamp and the nibble packing then run on two codes per instruction (s16x2).
//  * codes (bf16 path): the gap can be as small as 2^-20, so the rounding of v/Δ is
//    decided exactly by the signs of two FMA residuals at the candidate midpoints.
#include <algorithm>

#include "sq_internal.cuh"

namespace sq {

namespace {

constexpr int kThreads = 128;  // 64 and 512 lose (profiles/r02/quantize_cta_size_ab.jsonl)
constexpr int kRowsPerCta = 16;
constexpr int kLanesPerSlot = 8;
constexpr int kSlot = 128;      // k per slot; K % 128 == 0 for every group size
constexpr int kSlotsPerCta = 4;  // 2 and 8 lose (profiles/r02/quantize_occupancy_ab.jsonl)
constexpr int kMinCtasPerSm = 8; // 64 registers (1024 threads per SM) beat 48, 80 and 128

template <bool kBF16>
struct Fmt;
template <>
struct Fmt<false> {
  static constexpr uint32_t kExpMask = 0x7C00u;
  __device__ static float to_f(uint16_t b) { return __half2float(__ushort_as_half(b)); }
  __device__ static float2 to_f2(uint32_t b) { return __half22float2(*reinterpret_cast<const __half2*>(&b)); }
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
  __device__ static float2 to_f2(uint32_t b) { return make_float2(__uint_as_float(b << 16), __uint_as_float(b & 0xFFFF0000u)); }
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

// 32-byte load (LDG.256): a lane's 16 weights of a slot in one coalesced instruction
__device__ __forceinline__ void ld_nc_v8(const void* p, uint32_t (&r)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "l"(p));
}
// odd one of two adjacent (or equal) fp32 bit patterns: the low bit of RU, sign-extended
// (SGXT), selects RU or RD in one LOP3
__device__ __forceinline__ float odd_of(uint32_t ru, uint32_t rd) {
  int m;
  asm("bfe.s32 %0, %1, 0, 1;" : "=r"(m) : "r"(ru));
  return __uint_as_float((ru & (uint32_t)m) | (rd & ~(uint32_t)m));
}
// w * s rounded to odd in fp32 for an element pair: the products rounded down and up
// (FMUL2.RM / FMUL2.RP) are equal when w * s is exact and adjacent otherwise, and the odd
// one of two adjacent values is the round-to-odd result; its RN to fp16/bf16 is the single
// rounding RN_fmt(w * s) (24 >= 11 + 2 bits)
__device__ __forceinline__ void fold_odd2(float2 w, float s0, float s1, float& p0, float& p1) {
  uint64_t u, d;
  asm("{.reg .b64 w, s;\n\t"
      "mov.b64 w, {%2, %3};\n\t"
      "mov.b64 s, {%4, %5};\n\t"
      "mul.rp.f32x2 %0, w, s;\n\t"
      "mul.rm.f32x2 %1, w, s;}"
      : "=l"(u), "=l"(d)
      : "f"(w.x), "f"(w.y), "f"(s0), "f"(s1));
  p0 = odd_of((uint32_t)u, (uint32_t)d);
  p1 = odd_of((uint32_t)(u >> 32), (uint32_t)(d >> 32));
}
// fp16 pair, s >= 0 (sign bits clear): the product's magnitude |w| * s is formed from |w|
// (the abs is a free operand modifier of the conversion), so its RZ value is RD, RU is RD
// or RD + 1, and the round-to-odd value is RD | (RU & 1) — one LOP3; RN to fp16 commutes
// with the sign, which is w's and is ORed back into the packed pair
__device__ __forceinline__ uint32_t fold_pos2(uint32_t h, float s0, float s1) {
  const __half2 a2 = __habs2(*reinterpret_cast<const __half2*>(&h));
  const float2 a = __half22float2(a2);
  uint64_t u, d;
  asm("{.reg .b64 w, s;\n\t"
      "mov.b64 w, {%2, %3};\n\t"
      "mov.b64 s, {%4, %5};\n\t"
      "mul.rp.f32x2 %0, w, s;\n\t"
      "mul.rm.f32x2 %1, w, s;}"
      : "=l"(u), "=l"(d)
      : "f"(a.x), "f"(a.y), "f"(s0), "f"(s1));
  const uint32_t ru0 = (uint32_t)u, rd0 = (uint32_t)d, ru1 = (uint32_t)(u >> 32), rd1 = (uint32_t)(d >> 32);
  const __half2 r = __floats2half2_rn(__uint_as_float(rd0 | (ru0 & 1u)), __uint_as_float(rd1 | (ru1 & 1u)));
  return *reinterpret_cast<const uint32_t*>(&r) | (h & 0x80008000u);
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
// fp16 codes of an element pair (see the kernel): RN(v * inv' + 1.5 * 2^23 + Z) for both
// halves in one FFMA2, the low 16 bits of each are Z + c; gathered as s16x2 and clamped to
// [0, 15] by one VIMNMX.RELU
__device__ __forceinline__ uint32_t codes2(uint32_t h2, float inv, float cz) {
  const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&h2));
  uint64_t r;
  asm("{.reg .b64 v, a, c;\n\t"
      "mov.b64 v, {%1, %2};\n\t"
      "mov.b64 a, {%3, %3};\n\t"
      "mov.b64 c, {%4, %4};\n\t"
      "fma.rn.f32x2 %0, v, a, c;}"
      : "=l"(r)
      : "f"(f.x), "f"(f.y), "f"(inv), "f"(cz));
  return __vimin_s16x2_relu(__byte_perm((uint32_t)r, (uint32_t)(r >> 32), 0x5410), 0x000F000Fu);
}
// eight nibbles (low nibble = even k) from four clamped code pairs c[q] = (e_2q, e_2q+1):
// t = c0 + (c1 << 8) holds e0 | e2 << 8 | e1 << 16 | e3 << 24, and t + (t >> 12) has
// e0 | e1 << 4 | e2 << 8 | e3 << 12 in its low 16 bits
// (the bit fields of t and t >> 12 are disjoint, so | is +; both steps are integer
// multiply-adds, which issue on the FMA pipe and leave the ALU pipe, the bound, to the rest)
__device__ __forceinline__ uint32_t nib4(uint32_t ca, uint32_t cb) {
  uint32_t t, u;
  asm("mad.lo.u32 %0, %1, 256, %2;" : "=r"(t) : "r"(cb), "r"(ca));
  asm("mad.hi.u32 %0, %1, 1048576, %1;" : "=r"(u) : "r"(t));
  return u;
}
__device__ __forceinline__ uint32_t nibbles8(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) {
  return __byte_perm(nib4(c0, c1), nib4(c2, c3), 0x5410);
}

template <bool kBF16, int GS>
__global__ void __launch_bounds__(kThreads, kMinCtasPerSm)
quantize_kernel(const uint16_t* __restrict__ W, const float* __restrict__ s, int N, int K, int NSL,
                uint8_t* __restrict__ Wq, uint16_t* __restrict__ scales,
                void* __restrict__ zeros, int zeros_u4, int* __restrict__ nonfinite) {
  constexpr int kLanesPerGroup = GS / 16;
  // the per-group work (Δ, Z, the scale / zero stores) runs once per group on one owner
  // lane: in round r lane `sub` owns group sub / kLanesPerGroup of slot
  // r * kLanesPerGroup + sub % kLanesPerGroup, a lane of that very group (it already holds
  // the group's reduced min / max); the codes then fetch Δ and Z from the owner
  constexpr int kRounds = (kSlotsPerCta + kLanesPerGroup - 1) / kLanesPerGroup;
  const int sub = threadIdx.x % kLanesPerSlot;
  const int lane = threadIdx.x % 32;
  const int n = blockIdx.y * kRowsPerCta + threadIdx.x / kLanesPerSlot;
  const int g0 = blockIdx.x * kSlotsPerCta;  // first slot of the CTA
  const bool row_ok = n < N;

  // issue every load of the CTA's groups first (memory-level parallelism)
  uint32_t w[kSlotsPerCta][8];
#pragma unroll
  for (int j = 0; j < kSlotsPerCta; ++j) {
    const int g = g0 + j;
    if (row_ok && g < NSL) {
      ld_nc_v8(W + (size_t)n * K + (size_t)g * kSlot + sub * 16, w[j]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) w[j][i] = 0u;
    }
  }

  // the CTA's s (shared by its 16 rows) staged in shared memory while the weight loads fly,
  // permuted so that float4 q of lane `sub` sits at (q * 8 + sub): one conflict-free
  // wavefront per LDS.128 (the s loads of a slot otherwise wait a full L2 latency)
  __shared__ __align__(16) float4 s_sm[kSlotsPerCta * kSlot / 4];
  bool s_pos = false;  // every staged s has a clear sign bit (CTA-uniform)
  if (s != nullptr) {  // uniform
    uint32_t sign = 0u;
#pragma unroll
    for (int i = threadIdx.x; i < kSlotsPerCta * kSlot / 4; i += kThreads) {
      const int j = i / (kSlot / 4), e = i % (kSlot / 4);  // float4 e of slot j = (sub e/4, q e%4)
      const float4 v = g0 + j < NSL ? __ldg(reinterpret_cast<const float4*>(s + (size_t)(g0 + j) * kSlot) + e)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
      sign |= __float_as_uint(v.x) | __float_as_uint(v.y) | __float_as_uint(v.z) | __float_as_uint(v.w);
      s_sm[j * (kSlot / 4) + (e % 4) * 8 + e / 4] = v;
    }
    s_pos = !__syncthreads_or((int)(sign >> 31));
  }

  // fold (a3) and the group min / max of every slot
  uint32_t mn[kSlotsPerCta], mx[kSlotsPerCta];
#pragma unroll
  for (int j = 0; j < kSlotsPerCta; ++j) {
    const int g = g0 + j;
    if (!kBF16 && s_pos && g < NSL) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 sv = s_sm[j * (kSlot / 4) + q * 8 + sub];
        w[j][2 * q] = fold_pos2(w[j][2 * q], sv.x, sv.y);
        w[j][2 * q + 1] = fold_pos2(w[j][2 * q + 1], sv.z, sv.w);
      }
    } else if (s != nullptr && g < NSL) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 sv = s_sm[j * (kSlot / 4) + q * 8 + sub];
        float p0, p1, p2, p3;
        fold_odd2(Fmt<kBF16>::to_f2(w[j][2 * q]), sv.x, sv.y, p0, p1);
        fold_odd2(Fmt<kBF16>::to_f2(w[j][2 * q + 1]), sv.z, sv.w, p2, p3);
        w[j][2 * q] = pack_rn<kBF16>(p0, p1);
        w[j][2 * q + 1] = pack_rn<kBF16>(p2, p3);
      }
    }
    // min / max with NaN propagation; a NaN or ±Inf in the group then shows in mn or mx,
    // so the non-finite test (abs bits >= exponent mask) runs once per group on them
    mn[j] = w[j][0], mx[j] = w[j][0];
#pragma unroll
    for (int i = 1; i < 8; ++i) {
      mn[j] = Fmt<kBF16>::min2(mn[j], w[j][i]);
      mx[j] = Fmt<kBF16>::max2(mx[j], w[j][i]);
    }
#pragma unroll
    for (int o = 1; o < kLanesPerGroup; o <<= 1) {
      mn[j] = Fmt<kBF16>::min2(mn[j], __shfl_xor_sync(0xffffffffu, mn[j], o));
      mx[j] = Fmt<kBF16>::max2(mx[j], __shfl_xor_sync(0xffffffffu, mx[j], o));
    }
  }

  // per group: Δ, Z and their stores, on the owner lane
  float gv[kRounds];  // fp16: inv' (see the codes); bf16: Δ
  float gz[kRounds];  // fp16: 1.5 * 2^23 + Z; bf16: Z; -1 marks a non-finite group
#pragma unroll
  for (int rd = 0; rd < kRounds; ++rd) {
    const int j = rd * kLanesPerGroup + sub % kLanesPerGroup;
    uint32_t gmn = mn[0], gmx = mx[0];
#pragma unroll
    for (int jj = 1; jj < kSlotsPerCta; ++jj)
      if (jj == j) gmn = mn[jj], gmx = mx[jj];
    const int g = g0 + j;
    const bool live = j < kSlotsPerCta && g < NSL;

    const uint32_t amax = __vmaxu2(gmn & 0x7FFF7FFFu, gmx & 0x7FFF7FFFu);
    bool nf = ((amax & 0xFFFFu) >= Fmt<kBF16>::kExpMask) || ((amax >> 16) >= Fmt<kBF16>::kExpMask);
    const float lo = fminf(Fmt<kBF16>::to_f(gmn & 0xFFFFu), Fmt<kBF16>::to_f(gmn >> 16));
    const float hi = fmaxf(Fmt<kBF16>::to_f(gmx & 0xFFFFu), Fmt<kBF16>::to_f(gmx >> 16));

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

    // packed u4 Z (SQ_ZEROS_U4): rows n and n + 1 of a pair sit 8 lanes apart in the warp
    // (8 lanes per row) with the same owned group; the even row's lane writes the byte,
    // low nibble = even n
    const uint32_t zq = nf ? 0u : (uint32_t)z;
    const uint32_t zq_odd = __shfl_down_sync(0xffffffffu, zq, kLanesPerSlot);
    if (row_ok && live) {
      const size_t gi = (size_t)g * (kSlot / GS) + sub / kLanesPerGroup;
      scales[gi * N + n] = nf ? (uint16_t)0x7E00u : __half_as_ushort(__float2half_rn(d));
      if (!zeros_u4)
        reinterpret_cast<uint16_t*>(zeros)[gi * N + n] = nf ? (uint16_t)0u : __half_as_ushort(__float2half_rn(z));
      else if ((n & 1) == 0)
        reinterpret_cast<uint8_t*>(zeros)[gi * (N / 2) + n / 2] = (uint8_t)(zq | (zq_odd << 4));
      if (nf && nonfinite != nullptr) atomicAdd(nonfinite, 1);
    }
    gv[rd] = kBF16 ? d : inv;
    gz[rd] = nf ? -1.0f : (kBF16 ? z : 12582912.0f + z);
  }

  // codes (a4) of every slot, packed low nibble = even k
  uint8_t* const wq_row = Wq + (size_t)n * (K / 2) + (size_t)g0 * (kSlot / 2) + sub * 8;
#pragma unroll
  for (int j = 0; j < kSlotsPerCta; ++j) {
    if (g0 + j >= NSL) break;  // uniform across the CTA
    const int owner = (lane & ~(kLanesPerGroup - 1)) + j % kLanesPerGroup;
    const float gvj = __shfl_sync(0xffffffffu, gv[j / kLanesPerGroup], owner);
    const float gzj = __shfl_sync(0xffffffffu, gz[j / kLanesPerGroup], owner);
    uint32_t packed[2] = {0u, 0u};
    if (gzj >= 0.0f) {
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
        uint32_t cc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) cc[q] = codes2(w[j][q], gvj, gzj);
        packed[0] = nibbles8(cc[0], cc[1], cc[2], cc[3]);
        packed[1] = nibbles8(cc[4], cc[5], cc[6], cc[7]);
      } else {
        // bf16: a non-tie v / Δ can lie 2^-20 from a half-integer, too close for the one-FFMA
        // rounding.  c0 = rint(v * RN(1/Δ)) is within 1 of RHA(v / Δ) (|v / Δ| < 2^13 in a
        // finite group, relative error < 2^-22), and the two candidate midpoints are decided
        // exactly: fma(-(c0 ± 1/2), Δ, v) is v - (c0 ± 1/2) Δ rounded once, so its sign is
        // exact and it is 0 only at an exact tie (the exact value is a multiple of 2^-133,
        // far above fp32's 2^-149 underflow), which RHA sends away from zero
        const float inv = __frcp_rn(gvj);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint32_t bits = (i & 1) ? (w[j][i >> 1] >> 16) : (w[j][i >> 1] & 0xFFFFu);
          const float v = Fmt<kBF16>::to_f((uint16_t)bits);
          const float c0 = rintf(v * inv);
          const float th = __fmaf_rn(-(c0 + 0.5f), gvj, v);  // v/Δ - (c0 + 1/2), scaled by Δ
          const float tl = __fmaf_rn(-(c0 - 0.5f), gvj, v);  // v/Δ - (c0 - 1/2), scaled by Δ
          float c = c0;
          if (th > 0.0f || (th == 0.0f && c0 >= 0.0f)) c = c0 + 1.0f;
          else if (tl < 0.0f || (tl == 0.0f && c0 <= 0.0f)) c = c0 - 1.0f;
          c = fminf(fmaxf(c + gzj, 0.0f), 15.0f);
          packed[i >> 3] |= (__float_as_uint(c + 8388608.0f) & 0xFu) << (4 * (i & 7));
        }
      }
    }
    if (row_ok) *reinterpret_cast<uint2*>(wq_row + j * (kSlot / 2)) = make_uint2(packed[0], packed[1]);
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
