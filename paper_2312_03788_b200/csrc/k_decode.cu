// K-dec: W4A16 GEMM for small M (decode, M <= 16) -- HBM-bound.
//
//   Y[m][n] = sum_gi Δ[gi][n] * sum_{k in gi} X[m][k] * (q[n][k] - Z[gi][n])
//   PAPER.md:104-106 Eq. 3 with Ŵ of Eq. 1 line 2; fp32 accumulation.
//
// Design:
//  * Persistent stream-K: the (64-row block x 4-group stage) units of the whole GEMM
//    are split into equal contiguous ranges, one per resident CTA (one wave, no
//    tail); a row block cut between CTAs is finished by a deterministic fixup (the
//    last contributor sums the fp32 partials in CTA order).
//  * One producer warp streams each unit with TMA into a 4-stage SMEM ring: packed
//    codes (3-D box 64 B x 64 rows x 4 groups), the scale/zero rows and the matching
//    X slice (4-D box, SWIZZLE_128B so the fragment reads are bank-conflict free) --
//    about 100 KB per SM in flight, which is what HBM's latency-bandwidth product
//    asks for.
//  * Four consumer warps: warp w takes group w of every stage for all 64 rows (4
//    row tiles of 16), so its X fragment is loaded (and k-permuted with PRMT) once
//    and reused four times.  Codes are turned into the EXACT integer (q - Z) in
//    fp16/bf16 with the lop3 magic-number trick and fed to mma.sync.m16n8k16 with
//    fp32 accumulation; Δ is applied once per group to the accumulator fragment.
//  * Row-block results of the 4 consumer warps are summed through shared memory.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "sq_internal.cuh"

namespace sq {

namespace {

constexpr int kGroup = 128;
#ifndef SQ_DEC_BN
#define SQ_DEC_BN 64
#endif
#ifndef SQ_DEC_CTAS
#define SQ_DEC_CTAS 2
#endif
#ifndef SQ_DEC_NS1
#define SQ_DEC_NS1 4
#endif
#ifndef SQ_DEC_NS2
#define SQ_DEC_NS2 3
#endif
#ifndef SQ_DEC_ROWMAJOR
#define SQ_DEC_ROWMAJOR 0  // 1: codes box traversed row by row (256 contiguous bytes per row)
#endif
#ifndef SQ_DEC_NOLOAD
#define SQ_DEC_NOLOAD 0  // experiment: after the first NS stages, recompute on resident data (compute ceiling)
#endif
#ifndef SQ_DEC_NOCOMPUTE
#define SQ_DEC_NOCOMPUTE 0  // experiment: stream the operands but skip the math (bandwidth ceiling)
#endif
#ifndef SQ_DEC_ABLATE
#define SQ_DEC_ABLATE 0  // experiment only: 1 = skip the MMAs, 2 = skip the dequant (wrong results)
#endif
#ifndef SQ_DEC_CHAINS
#define SQ_DEC_CHAINS 1  // independent MMA accumulator chains per row tile (1, 2 or 4)
#endif
#ifndef SQ_DEC_IL
#define SQ_DEC_IL 0  // 1: load all 4 row tiles' codes first, then interleave their MMA chains
#endif
#ifndef SQ_DEC_SX
#define SQ_DEC_SX 0  // 1: magic-offset MMAs + activation-sum correction (no per-code hsub/hfma)
#endif
#ifndef SQ_DEC_PF
#define SQ_DEC_PF 0   // L2 prefetch distance in units ahead of the SMEM ring (0 = off)
#endif
constexpr int BN = SQ_DEC_BN;   // rows per row block (multiple of 16)
constexpr int kRT = BN / 16;    // 16-row tiles per consumer warp
#ifndef SQ_DEC_GPW
#define SQ_DEC_GPW 1  // groups per consumer warp per stage
#endif
constexpr int GPW = SQ_DEC_GPW;
constexpr int GPS = 4 * GPW;    // groups per stage (4 consumer warps x GPW)
constexpr int kConsumerWarps = 4;
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr int kMaxCtasPerSm = SQ_DEC_CTAS;

template <int MT>
struct Cfg {
  static constexpr int MPAD = 8 * MT;
  static constexpr int NS = MT == 1 ? SQ_DEC_NS1 : SQ_DEC_NS2;
  static constexpr int CODES = GPS * BN * (kGroup / 2);  // 16 KB
  static constexpr int XB = GPS * MPAD * kGroup * 2;      // 8 / 16 KB
  static constexpr int SZ = GPS * BN * 2;                 // 512 B
  static constexpr int STAGE = CODES + XB + 2 * SZ;
  static constexpr int OFF_RED = NS * STAGE;
  static constexpr int RED = (kConsumerWarps - 1) * MPAD * BN * 4;
  static constexpr int OFF_BAR = OFF_RED + RED;
  static constexpr int OFF_FLAG = OFF_BAR + 2 * NS * 8;
  static constexpr int SMEM = OFF_FLAG + 16;
  static constexpr int SMEM_ALLOC = SMEM + 1024;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void tma_4d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];\n"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* m, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];\n"
               ::"l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* m, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];\n"
               ::"l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(kConsumerWarps * 32) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  // not volatile: ptxas/NVVM may schedule it early; the "memory" clobber keeps it after
  // the mbarrier wait that makes the TMA data visible
  asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ uint16_t lds16(uint32_t addr) {
  uint16_t v;
  asm("ld.shared.u16 %0, [%1];\n" : "=h"(v) : "r"(addr) : "memory");
  return v;
}

__device__ __forceinline__ void mma_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint32_t b0, uint32_t b1, bool bf16) {
  if (bf16) {
    asm(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  } else {
    asm(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
}

__device__ __forceinline__ void mma_16816_zc(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                             uint32_t a3, uint32_t b0, uint32_t b1, bool bf16) {
  const float z = 0.0f;
  if (bf16) {
    asm(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%10,%10,%10,%10};\n"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(z));
  } else {
    asm(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%10,%10,%10,%10};\n"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(z));
  }
}

__device__ __forceinline__ uint32_t hsub2_u(uint32_t a, uint32_t b, bool bf16) {
  if (bf16) {
    __nv_bfloat162 r = __hsub2(*reinterpret_cast<__nv_bfloat162*>(&a),
                               *reinterpret_cast<__nv_bfloat162*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
  }
  __half2 r = __hsub2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t hfma2_u(uint32_t a, uint32_t b, uint32_t c) {
  __half2 r = __hfma2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b),
                      *reinterpret_cast<__half2*>(&c));
  return *reinterpret_cast<uint32_t*>(&r);
}

// One 32-bit word of codes (k offsets 0..7 of one row) -> the exact (q - Z) pairs
// (e0,e4), (e1,e5), (e2,e6), (e3,e7) in fp16 / bf16.
template <bool kBF16>
__device__ __forceinline__ void dequant_word(uint32_t w, uint32_t zsub, uint32_t zfma, uint32_t (&h)[4]) {
  if (!kBF16) {
    const uint32_t t = w >> 8;
    h[0] = hsub2_u(lop3_and_or(w, 0x000F000Fu, 0x64006400u), zsub, false);  // 1024+q - (1024+Z)
    h[2] = hsub2_u(lop3_and_or(t, 0x000F000Fu, 0x64006400u), zsub, false);
    h[1] = hfma2_u(lop3_and_or(w, 0x00F000F0u, 0x64006400u), 0x2C002C00u, zfma);  // (1024+16q)/16-(64+Z)
    h[3] = hfma2_u(lop3_and_or(t, 0x00F000F0u, 0x64006400u), 0x2C002C00u, zfma);
  } else {
    h[0] = hsub2_u(lop3_and_or(w, 0x000F000Fu, 0x43004300u), zsub, true);  // 128+q - (128+Z)
    h[1] = hsub2_u(lop3_and_or(w >> 4, 0x000F000Fu, 0x43004300u), zsub, true);
    h[2] = hsub2_u(lop3_and_or(w >> 8, 0x000F000Fu, 0x43004300u), zsub, true);
    h[3] = hsub2_u(lop3_and_or(w >> 12, 0x000F000Fu, 0x43004300u), zsub, true);
  }
}

// zero-point constants from the fp16 bits of Z (an integer 0..15)
template <bool kBF16>
__device__ __forceinline__ void zero_consts(uint16_t zbits, uint32_t& zsub, uint32_t& zfma) {
  const uint32_t z = (uint32_t)__half2int_rn(__ushort_as_half(zbits));
  if (!kBF16) {
    zsub = z * 0x00010001u + 0x64006400u;         // fp16x2(1024 + Z): ulp of 1024 is 1
    zfma = z * 0x00100010u + 0xD400D400u;         // fp16x2(-(64 + Z)): ulp of 64 is 1/16
  } else {
    zsub = z * 0x00010001u + 0x43004300u;         // bf16x2(128 + Z): ulp of 128 is 1
    zfma = 0;
  }
}

struct Work {
  int units, upb, cta_q, cta_r;  // total units, units per row block, units per CTA (q, remainder)
  __device__ __forceinline__ int start(int c) const { return c * cta_q + min(c, cta_r); }
  __device__ __forceinline__ int cta_of(int u) const {
    const int big = (cta_q + 1) * cta_r;
    return u < big ? u / (cta_q + 1) : cta_r + (u - big) / cta_q;
  }
};

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

template <int MT, bool kBF16>
__global__ void __launch_bounds__(kThreads, kMaxCtasPerSm)
decode_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
              const __grid_constant__ CUtensorMap tm_s, const __grid_constant__ CUtensorMap tm_z,
              uint16_t* __restrict__ Y, int* __restrict__ counters, float* __restrict__ partials,
              int M, int N, Work wk, int early_weights) {
  using C = Cfg<MT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_full = sbase + C::OFF_BAR;
  const uint32_t bar_empty = bar_full + 8 * C::NS;
  int* flag = reinterpret_cast<int*>(smem + C::OFF_FLAG);
  float* red = reinterpret_cast<float*>(smem + C::OFF_RED);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int c = blockIdx.x;
  const int u0 = wk.start(c), u1 = wk.start(c + 1);

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NS; ++i) {
      mbar_init(bar_full + 8 * i, 1);
      mbar_init(bar_empty + 8 * i, kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // the next kernel in the stream may start its prologue as our CTAs retire
  pdl_launch_dependents();

  if (warp == kConsumerWarps) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      prefetch_tmap(&tm_w);
      prefetch_tmap(&tm_x);
      prefetch_tmap(&tm_s);
      prefetch_tmap(&tm_z);
      // Weights (codes, Δ, Z) never depend on the previous kernel when the caller
      // declared them static: stream the first stages before waiting on it.
      int pre = 0;
      // L2 prefetch cursor, SQ_DEC_PF units ahead of the SMEM ring: more bytes in flight
      // from HBM than the shared-memory ring alone can hold
      int pf_u = u0, pf_rb = u0 / wk.upb, pf_g0 = (u0 % wk.upb) * GPS;
      auto prefetch_next = [&]() {
        if (SQ_DEC_PF > 0 && pf_u < u1) {
          if (SQ_DEC_ROWMAJOR) tma_prefetch_3d(&tm_w, 0, pf_g0, pf_rb * BN);
          else tma_prefetch_3d(&tm_w, 0, pf_rb * BN, pf_g0);
          tma_prefetch_2d(&tm_s, pf_rb * BN, pf_g0);
          tma_prefetch_2d(&tm_z, pf_rb * BN, pf_g0);
          ++pf_u;
          pf_g0 += GPS;
          if (pf_g0 >= wk.upb * GPS) { pf_g0 = 0; ++pf_rb; }
        }
      };
      if (SQ_DEC_PF > 0 && early_weights)
        for (int q = 0; q < C::NS + SQ_DEC_PF; ++q) prefetch_next();
      if (early_weights) {
        int rb = u0 / wk.upb, g0 = (u0 % wk.upb) * GPS;
        for (; pre < C::NS && u0 + pre < u1; ++pre) {
          const uint32_t st = sbase + pre * C::STAGE;
          const uint32_t fb = bar_full + 8 * pre;
          mbar_expect_tx(fb, C::STAGE);
          if (SQ_DEC_ROWMAJOR) tma_3d(st, &tm_w, fb, 0, g0, rb * BN);
          else tma_3d(st, &tm_w, fb, 0, rb * BN, g0);
          tma_2d(st + C::CODES + C::XB, &tm_s, fb, rb * BN, g0);
          tma_2d(st + C::CODES + C::XB + C::SZ, &tm_z, fb, rb * BN, g0);
          g0 += GPS;
          if (g0 >= wk.upb * GPS) { g0 = 0; ++rb; }
        }
      }
      pdl_wait();  // X (and everything after) may be the previous kernel's output
      if (SQ_DEC_PF > 0 && !early_weights)
        for (int q = 0; q < C::NS + SQ_DEC_PF; ++q) prefetch_next();
      int rb = u0 / wk.upb, g0 = (u0 % wk.upb) * GPS;
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; u0 + i < u1; ++i) {
        const uint32_t st = sbase + s * C::STAGE;
        const uint32_t fb = bar_full + 8 * s;
        if (i < pre) {
          tma_4d(st + C::CODES, &tm_x, fb, 0, 0, 0, g0);
        } else if (SQ_DEC_NOLOAD && i >= C::NS) {
          mbar_wait(bar_empty + 8 * s, ph ^ 1);
          mbar_arrive(fb);
        } else {
          mbar_wait(bar_empty + 8 * s, ph ^ 1);
          mbar_expect_tx(fb, C::STAGE);
          if (SQ_DEC_ROWMAJOR) tma_3d(st, &tm_w, fb, 0, g0, rb * BN);
          else tma_3d(st, &tm_w, fb, 0, rb * BN, g0);
          tma_4d(st + C::CODES, &tm_x, fb, 0, 0, 0, g0);
          tma_2d(st + C::CODES + C::XB, &tm_s, fb, rb * BN, g0);
          tma_2d(st + C::CODES + C::XB + C::SZ, &tm_z, fb, rb * BN, g0);
          prefetch_next();
        }
        if (++s == C::NS) { s = 0; ph ^= 1; }
        g0 += GPS;
        if (g0 >= wk.upb * GPS) { g0 = 0; ++rb; }
      }
    }
    return;
  }

  // ===================== consumers: warp w = group w of each stage =====================
  const int r = lane / 4, j = lane % 4;
  float acc[kRT][MT][4];
#pragma unroll
  for (int rt = 0; rt < kRT; ++rt)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[rt][mt][i] = 0.0f;

  int s = 0;
  uint32_t ph = 0;
  int rb = u0 / wk.upb;            // current row block
  int pos = u0 - rb * wk.upb;      // unit index inside the row block
  int seg_begin_pos = pos;
  bool first_seg = true;
  bool waited = false;
  for (int u = u0; u < u1; ++u) {
    mbar_wait(bar_full + 8 * s, ph);
    const uint32_t st = sbase + s * C::STAGE;
#if SQ_DEC_NOCOMPUTE
    if (true) {
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_empty + 8 * s);
      if (++s == C::NS) { s = 0; ph ^= 1; }
      ++pos;
      if (pos == wk.upb) { ++rb; pos = 0; seg_begin_pos = 0; first_seg = false; }
      continue;
    }
#endif

#pragma unroll
    for (int gi = 0; gi < GPW; ++gi) {
    const int grp = warp + kConsumerWarps * gi;  // group of the stage this pass works on
    // ---- X fragments of this warp's group: token t = r + 8 mt, k = 32 j + [0, 32)
    uint32_t xb[MT][4][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int R = (grp * C::MPAD + r + 8 * mt) * 2 + (j >> 1);  // 128-byte row of the swizzled box
      const uint32_t rowaddr = st + C::CODES + R * 128;
      uint32_t xv[16];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 v = lds128(rowaddr + ((((j & 1) * 4 + i) ^ (R & 7)) << 4));
        xv[4 * i] = v.x; xv[4 * i + 1] = v.y; xv[4 * i + 2] = v.z; xv[4 * i + 3] = v.w;
      }
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        xb[mt][w][0] = prmt(xv[4 * w], xv[4 * w + 2], 0x5410u);      // (x0, x4)
        xb[mt][w][1] = prmt(xv[4 * w], xv[4 * w + 2], 0x7632u);      // (x1, x5)
        xb[mt][w][2] = prmt(xv[4 * w + 1], xv[4 * w + 3], 0x5410u);  // (x2, x6)
        xb[mt][w][3] = prmt(xv[4 * w + 1], xv[4 * w + 3], 0x7632u);  // (x3, x7)
      }
    }
#if SQ_DEC_SX
    // activation sums of this group for this lane's tokens: even-k and odd-k positions
    float sxe[MT][2], sxo[MT][2];
    {
      const uint32_t kOnes = kBF16 ? 0x3F803F80u : 0x3C003C00u;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        float se[4], so[4];
        mma_16816_zc(se, kOnes, kOnes, kOnes, kOnes, xb[mt][0][0], xb[mt][0][2], kBF16);
        mma_16816_zc(so, kOnes, kOnes, kOnes, kOnes, xb[mt][0][1], xb[mt][0][3], kBF16);
#pragma unroll
        for (int w = 1; w < 4; ++w) {
          mma_16816(se, kOnes, kOnes, kOnes, kOnes, xb[mt][w][0], xb[mt][w][2], kBF16);
          mma_16816(so, kOnes, kOnes, kOnes, kOnes, xb[mt][w][1], xb[mt][w][3], kBF16);
        }
        sxe[mt][0] = se[0]; sxe[mt][1] = se[1];
        sxo[mt][0] = so[0]; sxo[mt][1] = so[1];
      }
    }
#endif
    // codes of this warp's group: [group][row][64 B] (default) or [row][group][64 B]
    const uint32_t cbase = SQ_DEC_ROWMAJOR ? st + grp * 64 + r * (GPS * 64) + j * 16
                                           : st + grp * (BN * 64) + r * 64 + j * 16;
    constexpr int kRowStride = SQ_DEC_ROWMAJOR ? GPS * 64 : 64;
    const uint32_t sbs = st + C::CODES + C::XB + grp * (BN * 2) + r * 2;
    const uint32_t sbz = sbs + C::SZ;
#if SQ_DEC_IL
    {
      uint32_t wa[kRT][4], wb[kRT][4], zsA[kRT], zfA[kRT], zsB[kRT], zfB[kRT];
      float dA[kRT], dB[kRT];
#pragma unroll
      for (int rt = 0; rt < kRT; ++rt) {
        const uint4 ca = lds128(cbase + rt * 16 * kRowStride);
        const uint4 cb = lds128(cbase + (rt * 16 + 8) * kRowStride);
        wa[rt][0] = ca.x; wa[rt][1] = ca.y; wa[rt][2] = ca.z; wa[rt][3] = ca.w;
        wb[rt][0] = cb.x; wb[rt][1] = cb.y; wb[rt][2] = cb.z; wb[rt][3] = cb.w;
        dA[rt] = __half2float(__ushort_as_half(lds16(sbs + rt * 32)));
        dB[rt] = __half2float(__ushort_as_half(lds16(sbs + rt * 32 + 16)));
        zero_consts<kBF16>(lds16(sbz + rt * 32), zsA[rt], zfA[rt]);
        zero_consts<kBF16>(lds16(sbz + rt * 32 + 16), zsB[rt], zfB[rt]);
      }
      float g[kRT][MT][4];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
#pragma unroll
        for (int rt = 0; rt < kRT; ++rt) {
          uint32_t hA[4], hB[4];
          dequant_word<kBF16>(wa[rt][w], zsA[rt], zfA[rt], hA);
          dequant_word<kBF16>(wb[rt][w], zsB[rt], zfB[rt], hB);
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            if (w == 0) {
              mma_16816_zc(g[rt][mt], hA[0], hB[0], hA[1], hB[1], xb[mt][w][0], xb[mt][w][1], kBF16);
            } else {
              mma_16816(g[rt][mt], hA[0], hB[0], hA[1], hB[1], xb[mt][w][0], xb[mt][w][1], kBF16);
            }
            mma_16816(g[rt][mt], hA[2], hB[2], hA[3], hB[3], xb[mt][w][2], xb[mt][w][3], kBF16);
          }
        }
      }
#pragma unroll
      for (int rt = 0; rt < kRT; ++rt)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          acc[rt][mt][0] = fmaf(g[rt][mt][0], dA[rt], acc[rt][mt][0]);
          acc[rt][mt][1] = fmaf(g[rt][mt][1], dA[rt], acc[rt][mt][1]);
          acc[rt][mt][2] = fmaf(g[rt][mt][2], dB[rt], acc[rt][mt][2]);
          acc[rt][mt][3] = fmaf(g[rt][mt][3], dB[rt], acc[rt][mt][3]);
        }
    }
    if (false)
#endif
#pragma unroll
    for (int rt = 0; rt < kRT; ++rt) {
      const uint4 ca = lds128(cbase + rt * 16 * kRowStride);
      const uint4 cb = lds128(cbase + (rt * 16 + 8) * kRowStride);
      const float dA = __half2float(__ushort_as_half(lds16(sbs + rt * 32)));
      const float dB = __half2float(__ushort_as_half(lds16(sbs + rt * 32 + 16)));
#if SQ_DEC_SX
      {
        const float zA = __half2float(__ushort_as_half(lds16(sbz + rt * 32)));
        const float zB = __half2float(__ushort_as_half(lds16(sbz + rt * 32 + 16)));
        const uint32_t wa[4] = {ca.x, ca.y, ca.z, ca.w};
        const uint32_t wb[4] = {cb.x, cb.y, cb.z, cb.w};
        float ge[MT][4], go[MT][4];
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          uint32_t la0, la1, ha0, ha1, lb0, lb1, hb0, hb1;
          if (!kBF16) {
            const uint32_t ta = wa[w] >> 8, tb = wb[w] >> 8;
            la0 = lop3_and_or(wa[w], 0x000F000Fu, 0x64006400u);  // 1024 + (e0, e4)
            la1 = lop3_and_or(ta, 0x000F000Fu, 0x64006400u);     // 1024 + (e2, e6)
            ha0 = lop3_and_or(wa[w], 0x00F000F0u, 0x64006400u);  // 1024 + 16 (e1, e5)
            ha1 = lop3_and_or(ta, 0x00F000F0u, 0x64006400u);     // 1024 + 16 (e3, e7)
            lb0 = lop3_and_or(wb[w], 0x000F000Fu, 0x64006400u);
            lb1 = lop3_and_or(tb, 0x000F000Fu, 0x64006400u);
            hb0 = lop3_and_or(wb[w], 0x00F000F0u, 0x64006400u);
            hb1 = lop3_and_or(tb, 0x00F000F0u, 0x64006400u);
          } else {
            la0 = lop3_and_or(wa[w], 0x000F000Fu, 0x43004300u);
            la1 = lop3_and_or(wa[w] >> 8, 0x000F000Fu, 0x43004300u);
            ha0 = lop3_and_or(wa[w] >> 4, 0x000F000Fu, 0x43004300u);
            ha1 = lop3_and_or(wa[w] >> 12, 0x000F000Fu, 0x43004300u);
            lb0 = lop3_and_or(wb[w], 0x000F000Fu, 0x43004300u);
            lb1 = lop3_and_or(wb[w] >> 8, 0x000F000Fu, 0x43004300u);
            hb0 = lop3_and_or(wb[w] >> 4, 0x000F000Fu, 0x43004300u);
            hb1 = lop3_and_or(wb[w] >> 12, 0x000F000Fu, 0x43004300u);
          }
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            if (w == 0) {
              mma_16816_zc(ge[mt], la0, lb0, la1, lb1, xb[mt][w][0], xb[mt][w][2], kBF16);
              mma_16816_zc(go[mt], ha0, hb0, ha1, hb1, xb[mt][w][1], xb[mt][w][3], kBF16);
            } else {
              mma_16816(ge[mt], la0, lb0, la1, lb1, xb[mt][w][0], xb[mt][w][2], kBF16);
              mma_16816(go[mt], ha0, hb0, ha1, hb1, xb[mt][w][1], xb[mt][w][3], kBF16);
            }
          }
        }
        // sum_k X (q - Z) = ge + go/16 - (1024+Z) SXe - (64+Z) SXo   (fp16 magic)
        //                 = ge + go    - (128+Z) (SXe + SXo)          (bf16 magic)
        const float osc = kBF16 ? 1.0f : 0.0625f;
        const float ceA = -((kBF16 ? 128.0f : 1024.0f) + zA), coA = -((kBF16 ? 128.0f : 64.0f) + zA);
        const float ceB = -((kBF16 ? 128.0f : 1024.0f) + zB), coB = -((kBF16 ? 128.0f : 64.0f) + zB);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float ce = i < 2 ? ceA : ceB, co = i < 2 ? coA : coB, d = i < 2 ? dA : dB;
            float v = fmaf(go[mt][i], osc, ge[mt][i]);
            v = fmaf(ce, sxe[mt][i & 1], v);
            v = fmaf(co, sxo[mt][i & 1], v);
            acc[rt][mt][i] = fmaf(v, d, acc[rt][mt][i]);
          }
        }
        continue;
      }
#endif
      uint32_t zsA, zfA, zsB, zfB;
      zero_consts<kBF16>(lds16(sbz + rt * 32), zsA, zfA);
      zero_consts<kBF16>(lds16(sbz + rt * 32 + 16), zsB, zfB);
      const uint32_t wa[4] = {ca.x, ca.y, ca.z, ca.w};
      const uint32_t wb[4] = {cb.x, cb.y, cb.z, cb.w};
      constexpr int NC = SQ_DEC_CHAINS;
      float gc[MT][NC][4];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        uint32_t hA[4], hB[4];
#if SQ_DEC_ABLATE == 2
        hA[0] = wa[w]; hA[1] = wa[w] >> 8; hA[2] = wa[w] >> 4; hA[3] = wa[w] >> 12;
        hB[0] = wb[w]; hB[1] = wb[w] >> 8; hB[2] = wb[w] >> 4; hB[3] = wb[w] >> 12;
#else
        dequant_word<kBF16>(wa[w], zsA, zfA, hA);
        dequant_word<kBF16>(wb[w], zsB, zfB, hB);
#endif
#if SQ_DEC_ABLATE == 1
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int i = 0; i < 4; ++i)
            gc[mt][0][i] = (w == 0 ? 0.0f : gc[mt][0][i]) +
                           __uint_as_float((hA[i] ^ hB[i] ^ xb[mt][w][i]) & 0x3FFFFFFFu);
        if (false)
#endif
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int q = 2 * w + h, ch = q % NC;  // q-th MMA of the group -> chain ch
            if (q < NC) {
              mma_16816_zc(gc[mt][ch], hA[2 * h], hB[2 * h], hA[2 * h + 1], hB[2 * h + 1],
                           xb[mt][w][2 * h], xb[mt][w][2 * h + 1], kBF16);
            } else {
              mma_16816(gc[mt][ch], hA[2 * h], hB[2 * h], hA[2 * h + 1], hB[2 * h + 1],
                        xb[mt][w][2 * h], xb[mt][w][2 * h + 1], kBF16);
            }
          }
        }
      }
      float g[MT][4];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float v = gc[mt][0][i];
#pragma unroll
          for (int ch = 1; ch < NC; ++ch) v += gc[mt][ch][i];
          g[mt][i] = v;
        }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        acc[rt][mt][0] = fmaf(g[mt][0], dA, acc[rt][mt][0]);
        acc[rt][mt][1] = fmaf(g[mt][1], dA, acc[rt][mt][1]);
        acc[rt][mt][2] = fmaf(g[mt][2], dB, acc[rt][mt][2]);
        acc[rt][mt][3] = fmaf(g[mt][3], dB, acc[rt][mt][3]);
      }
    }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(bar_empty + 8 * s);
    if (++s == C::NS) { s = 0; ph ^= 1; }

    // ---- end of this CTA's segment of row block rb?
    ++pos;
    const bool rb_done = pos == wk.upb;
    if (!rb_done && u + 1 != u1) continue;

    if (!waited) {  // global writes below must follow the previous kernel (PDL)
      pdl_wait();
      waited = true;
    }
    // sum the 4 consumer warps through shared memory: warps 1..3 park, warp 0 adds
    if (warp > 0) {
      float* rw = red + (warp - 1) * C::MPAD * BN;
#pragma unroll
      for (int rt = 0; rt < kRT; ++rt)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int t0 = 8 * mt + 2 * j, ra = rt * 16 + r;
          rw[t0 * BN + ra] = acc[rt][mt][0];
          rw[(t0 + 1) * BN + ra] = acc[rt][mt][1];
          rw[t0 * BN + ra + 8] = acc[rt][mt][2];
          rw[(t0 + 1) * BN + ra + 8] = acc[rt][mt][3];
        }
    }
    consumer_sync();
    if (warp == 0) {
#pragma unroll
      for (int rt = 0; rt < kRT; ++rt)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int t0 = 8 * mt + 2 * j, ra = rt * 16 + r;
          float v[4] = {acc[rt][mt][0], acc[rt][mt][1], acc[rt][mt][2], acc[rt][mt][3]};
#pragma unroll
          for (int w = 0; w < kConsumerWarps - 1; ++w) {
            const float* rw = red + w * C::MPAD * BN;
            v[0] += rw[t0 * BN + ra];
            v[1] += rw[(t0 + 1) * BN + ra];
            v[2] += rw[t0 * BN + ra + 8];
            v[3] += rw[(t0 + 1) * BN + ra + 8];
          }
          red[t0 * BN + ra] = v[0];  // total parked in slot 0 (each lane owns its entries)
          red[(t0 + 1) * BN + ra] = v[1];
          red[t0 * BN + ra + 8] = v[2];
          red[(t0 + 1) * BN + ra + 8] = v[3];
        }
    }
    consumer_sync();
#pragma unroll
    for (int rt = 0; rt < kRT; ++rt)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[rt][mt][i] = 0.0f;

    const int n0 = rb * BN;
    const bool full = (seg_begin_pos == 0) && rb_done;
    auto to_out = [](float v) -> uint16_t {
      if (kBF16) return __bfloat16_as_ushort(__float2bfloat16_rn(v));
      return __half_as_ushort(__float2half_rn(v));
    };
    if (full) {
      for (int idx = threadIdx.x; idx < M * BN; idx += kConsumerWarps * 32) {
        const int t = idx / BN, row = idx % BN;
        if (n0 + row < N) Y[(size_t)t * N + n0 + row] = to_out(red[t * BN + row]);
      }
    } else {
      // stream-K fixup: park the partial; the last contributor sums them in CTA order
      const int e = first_seg ? 0 : 1;
      float* slot = partials + ((size_t)c * 2 + e) * (16 * BN);
      for (int idx = threadIdx.x; idx < M * BN; idx += kConsumerWarps * 32) __stcg(slot + idx, red[idx]);
      consumer_sync();
      const int c0 = wk.cta_of(rb * wk.upb), c1 = wk.cta_of((rb + 1) * wk.upb - 1);
      if (threadIdx.x == 0) {
        __threadfence();
        const int prev = atomicAdd(counters + rb, 1);
        __threadfence();
        *flag = (prev == c1 - c0) ? 1 : 0;
      }
      consumer_sync();
      if (*flag) {
        for (int idx = threadIdx.x; idx < M * BN; idx += kConsumerWarps * 32) {
          float part[8];
          float v = 0.0f;
          int cc = c0;
          while (cc <= c1) {  // batch the L2 reads, add in fixed CTA order
            const int nb = min(8, c1 - cc + 1);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (q < nb) {
                const int ee = (wk.start(cc + q) / wk.upb == rb) ? 0 : 1;
                part[q] = __ldcg(partials + ((size_t)(cc + q) * 2 + ee) * (16 * BN) + idx);
              }
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (q < nb) v += part[q];
            cc += nb;
          }
          const int t = idx / BN, row = idx % BN;
          if (n0 + row < N) Y[(size_t)t * N + n0 + row] = to_out(v);
        }
        if (threadIdx.x == 0) counters[rb] = 0;  // leave the workspace zeroed
      }
    }
    consumer_sync();  // red[] and flag are reused by the next segment
    first_seg = false;
    if (rb_done) { ++rb; pos = 0; }
    seg_begin_pos = pos;
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool encode(CUtensorMap* map, CUtensorMapDataType dt, int rank, const void* base, const uint64_t* dims,
            const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle sw) {
  auto fn = get_encode();
  if (!fn) return false;
  cuuint64_t d[5], s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) { d[i] = dims[i]; b[i] = box[i]; e[i] = 1; }
  for (int i = 0; i < rank - 1; ++i) s[i] = strides_bytes[i];
  return fn(map, dt, rank, const_cast<void*>(base), d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int MT, bool kBF16>
int ctas_per_sm() {
  static int cached = -1;
  if (cached < 0) {
    int n = 0;
    cudaFuncSetAttribute(decode_kernel<MT, kBF16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Cfg<MT>::SMEM_ALLOC);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, decode_kernel<MT, kBF16>, kThreads,
                                                      Cfg<MT>::SMEM_ALLOC) != cudaSuccess || n < 1)
      n = 1;
    cached = std::min(n, kMaxCtasPerSm);
  }
  return cached;
}

template <int MT, bool kBF16>
cudaError_t launch_t(const void* X, const uint8_t* Wq, const uint16_t* scales, const uint16_t* zeros,
                     void* Y, int M, int N, int K, void* ws, cudaStream_t st, const char** why) {
  using C = Cfg<MT>;
  const int G = K / kGroup;
  CUtensorMap tw, tx, ts, tz;
  {
    const uint64_t d[3] = {64, SQ_DEC_ROWMAJOR ? (uint64_t)G : (uint64_t)N, SQ_DEC_ROWMAJOR ? (uint64_t)N : (uint64_t)G};
    const uint64_t s[2] = {SQ_DEC_ROWMAJOR ? 64 : (uint64_t)K / 2, SQ_DEC_ROWMAJOR ? (uint64_t)K / 2 : 64};
    const uint32_t b[3] = {64, SQ_DEC_ROWMAJOR ? (uint32_t)GPS : (uint32_t)BN, SQ_DEC_ROWMAJOR ? (uint32_t)BN : (uint32_t)GPS};
    if (!encode(&tw, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, Wq, d, s, b, CU_TENSOR_MAP_SWIZZLE_NONE)) {
      *why = "tensor map (codes)";
      return cudaErrorInvalidValue;
    }
  }
  {
    const uint64_t d[4] = {64, 2, (uint64_t)M, (uint64_t)G};
    const uint64_t s[3] = {128, (uint64_t)K * 2, 256};
    const uint32_t b[4] = {64, 2, (uint32_t)C::MPAD, GPS};
    if (!encode(&tx, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, X, d, s, b, CU_TENSOR_MAP_SWIZZLE_128B)) {
      *why = "tensor map (X)";
      return cudaErrorInvalidValue;
    }
  }
  {
    const uint64_t d[2] = {(uint64_t)N, (uint64_t)G};
    const uint64_t s[1] = {(uint64_t)N * 2};
    const uint32_t b[2] = {BN, GPS};
    if (!encode(&ts, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, scales, d, s, b, CU_TENSOR_MAP_SWIZZLE_NONE) ||
        !encode(&tz, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, zeros, d, s, b, CU_TENSOR_MAP_SWIZZLE_NONE)) {
      *why = "tensor map (scales/zeros)";
      return cudaErrorInvalidValue;
    }
  }
  const int RB = (N + BN - 1) / BN;
  Work wk;
  wk.upb = (G + GPS - 1) / GPS;
  wk.units = RB * wk.upb;
  const int P = std::min(wk.units, num_sms() * ctas_per_sm<MT, kBF16>());
  wk.cta_q = wk.units / P;
  wk.cta_r = wk.units % P;
  int* counters = reinterpret_cast<int*>(ws);
  float* partials = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + decode_counter_bytes(N));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)P, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM_ALLOC;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = option(SQ_OPT_PDL) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int early = option(SQ_OPT_PDL) && option(SQ_OPT_WEIGHTS_STATIC);
  return cudaLaunchKernelEx(&cfg, decode_kernel<MT, kBF16>, tw, tx, ts, tz, (uint16_t*)Y, counters,
                            partials, M, N, wk, early);
}

}  // namespace

size_t decode_counter_bytes(int64_t N) {
  const int64_t RB = (N + BN - 1) / BN;
  return (size_t)((RB * 4 + 255) / 256 * 256);
}

size_t decode_workspace_bytes(int64_t N) {
  return decode_counter_bytes(N) + (size_t)num_sms() * kMaxCtasPerSm * 2 * 16 * BN * sizeof(float);
}

cudaError_t launch_decode(const void* X, int x_dtype, const uint8_t* Wq, const uint16_t* scales,
                          const uint16_t* zeros, void* Y, int M, int N, int K, void* ws,
                          cudaStream_t st, const char** why) {
  const bool bf16 = x_dtype == SQ_BF16;
  if (M <= 8)
    return bf16 ? launch_t<1, true>(X, Wq, scales, zeros, Y, M, N, K, ws, st, why)
                : launch_t<1, false>(X, Wq, scales, zeros, Y, M, N, K, ws, st, why);
  return bf16 ? launch_t<2, true>(X, Wq, scales, zeros, Y, M, N, K, ws, st, why)
              : launch_t<2, false>(X, Wq, scales, zeros, Y, M, N, K, ws, st, why);
}

}  // namespace sq
