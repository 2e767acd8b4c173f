// K-dec-tc: W4A16 decode GEMM (M <= 16) on the 5th-gen tensor cores.
//
//   Y[m][n] = sum_gi Δ[gi][n] * sum_{k in gi} X[m][k] * (q[n][k] - Z[gi][n])
//   PAPER.md:104-106 Eq. 3 with Ŵ of Eq. 1 line 2; fp32 accumulation.
//
// Swap-AB: D[row][token] = A[row][k] * X[token][k]^T with tcgen05.mma.cta_group::1.kind::f16,
// M_mma = 128 weight rows (TMEM lanes), N_mma = 16 tokens, K = 16 per instruction.
//  * A = the EXACT integer (q - Z) in fp16/bf16 (lop3 magic number + hsub2/hfma2, 9 ops per
//    8 codes), written by the dequant warps into TMEM with tcgen05.st.  The lop3 trick
//    yields k-pairs (k, k+4) of every 8-code word, so the activations are k-permuted the
//    same way in shared memory (one warp, 4 PRMT per 16 bytes) before the MMA reads them.
//  * Every group (128 k) accumulates into its own small TMEM accumulator (16 columns); the
//    dequant warps read it back (tcgen05.ld), multiply by Δ and add into fp32 registers --
//    Δ is applied once per group, as in the mma.sync kernel, not once per weight.
//  * Two sets of four dequant warps (one per TMEM lane quarter) take alternate groups, so
//    two groups are in flight; A and the per-group accumulators are double-buffered per set.
//  * Persistent stream-K over units of (128-row block x 4 groups); one CTA per SM; TMA
//    producer warp; epilogue warp for the cross-set sum, the Y store and the deterministic
//    stream-K fixup (same protocol as k_decode.cu).
//  * The MMA warp issues from warp-uniform control flow with elect.sync (see k_prefill.cu).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "sq_internal.cuh"

namespace sq {

namespace {

constexpr int kGroup = 128;
constexpr int BM = 128;      // weight rows per row block (MMA M, TMEM lanes)
constexpr int NT = 16;       // tokens (MMA N); M <= 16
constexpr int GPS = 4;       // groups per stage (unit)
constexpr int kProducerWarp = 0, kMmaWarp = 1, kEpilogueWarp = 2, kDqWarp0 = 4;
constexpr int kSets = 2;     // dequant warp sets, alternate groups
constexpr int kThreads = (kDqWarp0 + 4 * kSets) * 32;

constexpr int CODES = GPS * BM * 64;           // 32 KB: [group][row][64 B], SWIZZLE_64B
constexpr int XB = GPS * 2 * NT * 128;          // 16 KB: [64-k atom][token][128 B], SWIZZLE_128B
constexpr int SZ = GPS * BM * 2;                // 1 KB: [group][row] fp16
constexpr int TX = CODES + XB + 2 * SZ;         // bytes per stage the TMA delivers
constexpr int STAGE = (TX + 1023) / 1024 * 1024;
constexpr int NS = 4;
constexpr int SLOT = kSets * NT * BM * 4;       // parked partial sums [set][token][row] fp32
constexpr int OFF_SLOT = NS * STAGE;
constexpr int OFF_BAR = OFF_SLOT + SLOT;
// barriers: full[NS] empty[NS] a_full[4] a_empty[4] d_full[4] d_empty[4] red_full red_empty
constexpr int NBARS = 2 * NS + 16 + 2;
constexpr int OFF_TMEM = OFF_BAR + NBARS * 8;
constexpr int SMEM = OFF_TMEM + 16;
constexpr int SMEM_ALLOC = SMEM + 1024;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t A_COL = 0;     // A[set][buf]: 64 columns each (128 k as fp16 pairs)
constexpr uint32_t D_COL = 256;   // D[set][buf]: NT columns each (fp32)

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_wait_idle(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(bar), "r"(parity), "r"(100000) : "memory");
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
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
// issued by a whole warp; elect.sync picks the lane that executes the tcgen05 instruction
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accum) {
  asm volatile(
      "{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
      ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum) : "memory");
}
__device__ __forceinline__ void tmem_st_x32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31, %32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
      "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]),
      "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]),
      "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_ld_x16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row groups 1024 B apart, version 1.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// Instruction descriptor: D fp32, A/B fp16 or bf16 (K-major), M = 128, N = NT.
__device__ __forceinline__ uint32_t make_idesc(bool bf16) {
  return (1u << 4) | ((bf16 ? 1u : 0u) << 7) | ((bf16 ? 1u : 0u) << 10) | ((uint32_t)(NT >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ uint32_t hsub2_u(uint32_t a, uint32_t b, bool bf16) {
  if (bf16) {
    __nv_bfloat162 r = __hsub2(*reinterpret_cast<__nv_bfloat162*>(&a), *reinterpret_cast<__nv_bfloat162*>(&b));
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
__device__ __forceinline__ void dequant_word(uint32_t w, uint32_t zsub, uint32_t zfma, uint32_t* h) {
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
template <bool kBF16>
__device__ __forceinline__ void zero_consts(uint16_t zbits, uint32_t& zsub, uint32_t& zfma) {
  const uint32_t z = (uint32_t)__half2int_rn(__ushort_as_half(zbits));
  if (!kBF16) {
    zsub = z * 0x00010001u + 0x64006400u;  // fp16x2(1024 + Z)
    zfma = z * 0x00100010u + 0xD400D400u;  // fp16x2(-(64 + Z))
  } else {
    zsub = z * 0x00010001u + 0x43004300u;  // bf16x2(128 + Z)
    zfma = 0;
  }
}

// Stream-K work split over units u = rb * upb + pos (row block rb of 128 rows, stage pos).
struct Work {
  int units, upb, cta_q, cta_r;
  __device__ __forceinline__ int start(int c) const { return c * cta_q + min(c, cta_r); }
  __device__ __forceinline__ int cta_of(int u) const {
    const int big = (cta_q + 1) * cta_r;
    return u < big ? u / (cta_q + 1) : cta_r + (u - big) / cta_q;
  }
};

template <bool kBF16>
__global__ void __launch_bounds__(kThreads, 1)
decode_tc_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
                 const __grid_constant__ CUtensorMap tm_s, const __grid_constant__ CUtensorMap tm_z,
                 uint16_t* __restrict__ Y, int* __restrict__ counters, float* __restrict__ partials,
                 int M, int N, Work wk, int early_weights) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = sbase + OFF_BAR;
  auto full = [&](int s) { return bar0 + 8u * s; };
  auto empty = [&](int s) { return bar0 + 8u * (NS + s); };
  auto a_full = [&](int i) { return bar0 + 8u * (2 * NS + i); };
  auto a_empty = [&](int i) { return bar0 + 8u * (2 * NS + 4 + i); };
  auto d_full = [&](int i) { return bar0 + 8u * (2 * NS + 8 + i); };
  auto d_empty = [&](int i) { return bar0 + 8u * (2 * NS + 12 + i); };
  const uint32_t red_full = bar0 + 8u * (2 * NS + 16);
  const uint32_t red_empty = red_full + 8u;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);
  float* slot = reinterpret_cast<float*>(smem + OFF_SLOT);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int c = blockIdx.x;
  const int u0 = wk.start(c), u1 = wk.start(c + 1);

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(full(i), 1);
      mbar_init(empty(i), 4 * kSets + 1);  // dequant warps (codes read) + MMA commit (X read)
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(a_full(i), 4);
      mbar_init(a_empty(i), 1);
      mbar_init(d_full(i), 1);
      mbar_init(d_empty(i), 4);
    }
    mbar_init(red_full, 4 * kSets);
    mbar_init(red_empty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  pdl_launch_dependents();

  if (warp == kProducerWarp) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      prefetch_tmap(&tm_w);
      prefetch_tmap(&tm_x);
      prefetch_tmap(&tm_s);
      prefetch_tmap(&tm_z);
      auto load_weights = [&](uint32_t st, uint32_t fb, int u) {
        const int rb = u / wk.upb, g0 = (u % wk.upb) * GPS;
        tma_3d(st, &tm_w, fb, 0, rb * BM, g0);
        tma_2d(st + CODES + XB, &tm_s, fb, rb * BM, g0);
        tma_2d(st + CODES + XB + SZ, &tm_z, fb, rb * BM, g0);
      };
      int pre = 0;
      if (early_weights) {  // static weights: stream the first stages before waiting on PDL
        for (; pre < NS && u0 + pre < u1; ++pre) {
          mbar_expect_tx(full(pre), TX);
          load_weights(sbase + pre * STAGE, full(pre), u0 + pre);
        }
      }
      pdl_wait();  // X may be the previous kernel's output
      int s = 0;
      uint32_t ph = 0;
      for (int u = u0, i = 0; u < u1; ++u, ++i) {
        const uint32_t st = sbase + s * STAGE;
        if (i >= pre) {
          mbar_wait_idle(empty(s), ph ^ 1);
          mbar_expect_tx(full(s), TX);
          load_weights(st, full(s), u);
        }
        tma_3d(st + CODES, &tm_x, full(s), 0, 0, (u % wk.upb) * GPS * 2);  // 8 atoms of 64 k
        if (++s == NS) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == kMmaWarp) {
    // ===================== X k-permutation + MMA issue (whole warp, warp-uniform) =====================
    const uint32_t idesc = make_idesc(kBF16);
    int s = 0;
    uint32_t ph = 0;
    int j = 0;  // running group index of this CTA
    for (int u = u0; u < u1; ++u) {
      mbar_wait(full(s), ph);
      const uint32_t xbase = sbase + s * STAGE + CODES;
      // (x0..x7) -> (x0, x4, x1, x5, x2, x6, x3, x7) in every 16-byte chunk: the k order of
      // the A pairs the lop3 dequantization produces (the swizzle moves whole chunks only)
#pragma unroll 4
      for (int ch = lane; ch < XB / 16; ch += 32) {
        uint4 v;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(xbase + ch * 16) : "memory");
        const uint32_t o0 = prmt(v.x, v.z, 0x5410u), o1 = prmt(v.x, v.z, 0x7632u);
        const uint32_t o2 = prmt(v.y, v.w, 0x5410u), o3 = prmt(v.y, v.w, 0x7632u);
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(xbase + ch * 16), "r"(o0), "r"(o1),
                     "r"(o2), "r"(o3) : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> MMA reads
      __syncwarp();
#pragma unroll 1
      for (int gi = 0; gi < GPS; ++gi, ++j) {
        const int set = j & 1, buf = (j >> 1) & 1, ab = set * 2 + buf;
        const uint32_t par = (uint32_t)(j >> 2) & 1u;
        mbar_wait(a_full(ab), par);
        mbar_wait(d_empty(ab), par ^ 1u);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // 8 x K=16 = the group's 128 k
          const uint32_t a_t = tmem + A_COL + (uint32_t)ab * 64 + (uint32_t)kk * 8;
          const uint32_t xatom = xbase + (uint32_t)(2 * gi + (kk >> 2)) * (NT * 128) + (uint32_t)(kk & 3) * 32;
          tc_mma(tmem + D_COL + (uint32_t)ab * NT, a_t, sw128_desc(xatom), idesc, kk ? 1u : 0u);
        }
        tc_commit(d_full(ab));
        tc_commit(a_empty(ab));
      }
      tc_commit(empty(s));  // X of this stage consumed once these MMAs complete
      if (++s == NS) { s = 0; ph ^= 1; }
    }
  } else if (warp == kEpilogueWarp) {
    // ===================== epilogue: cross-set sum, Y store or stream-K fixup =====================
    constexpr int E = NT * BM / 32;  // elements per lane
    uint32_t redph = 0;
    int seg_begin_pos = u0 % wk.upb;
    bool first_seg = true, waited = false;
    auto to_out = [](float v) -> uint16_t {
      return kBF16 ? __bfloat16_as_ushort(__float2bfloat16_rn(v)) : __half_as_ushort(__float2half_rn(v));
    };
    for (int u = u0; u < u1; ++u) {
      const int rb = u / wk.upb, pos = u % wk.upb;
      const bool rb_done = pos + 1 == wk.upb;
      if (!(rb_done || u + 1 == u1)) continue;
      mbar_wait_idle(red_full, redph);
      float v[E];
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int idx = lane + 32 * i;
        v[i] = slot[idx] + slot[NT * BM + idx];  // set 0 + set 1, fixed order
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(red_empty);
      if (!waited) {  // global accesses must follow the previous kernel (PDL)
        pdl_wait();
        waited = true;
      }
      const int n0 = rb * BM;
      if (seg_begin_pos == 0 && rb_done) {
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int idx = lane + 32 * i, t = idx / BM, row = idx % BM;
          if (t < M && n0 + row < N) Y[(size_t)t * N + n0 + row] = to_out(v[i]);
        }
      } else {
        float* mine = partials + ((size_t)c * 2 + (first_seg ? 0 : 1)) * (NT * BM);
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int idx = lane + 32 * i;
          if (idx < M * BM) __stcg(mine + idx, v[i]);
        }
        __syncwarp();
        const int c0 = wk.cta_of(rb * wk.upb), c1 = wk.cta_of((rb + 1) * wk.upb - 1);
        int last = 0;
        if (lane == 0) {
          int prev;
          asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;\n" : "=r"(prev) : "l"(counters + rb) : "memory");
          last = prev == c1 - c0;
        }
        if (__shfl_sync(0xffffffffu, last, 0)) {
          float tot[E];
#pragma unroll
          for (int i = 0; i < E; ++i) tot[i] = 0.0f;
          for (int cc = c0; cc <= c1; ++cc) {  // fixed CTA order
            const int e = (wk.start(cc) / wk.upb == rb) ? 0 : 1;
            const float* src = partials + ((size_t)cc * 2 + e) * (NT * BM);
            float part[E];
#pragma unroll
            for (int i = 0; i < E; ++i) {
              const int idx = lane + 32 * i;
              part[i] = idx < M * BM ? __ldcg(src + idx) : 0.0f;
            }
#pragma unroll
            for (int i = 0; i < E; ++i) tot[i] += part[i];
          }
#pragma unroll
          for (int i = 0; i < E; ++i) {
            const int idx = lane + 32 * i, t = idx / BM, row = idx % BM;
            if (t < M && n0 + row < N) Y[(size_t)t * N + n0 + row] = to_out(tot[i]);
          }
          if (lane == 0) counters[rb] = 0;
        }
      }
      first_seg = false;
      seg_begin_pos = 0;
      redph ^= 1;
    }
  } else if (warp >= kDqWarp0) {
    // ===================== dequant (thread = weight row = TMEM lane) =====================
    const int q = (warp - kDqWarp0) % 4, set = (warp - kDqWarp0) / 4;
    const int row = q * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const int sw = (row >> 1) & 3;  // SWIZZLE_64B chunk permutation of this row
    float acc[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[t] = 0.0f;
    int s = 0;
    uint32_t ph = 0;
    int jn = 0;             // this set's running group count (buffer / phase)
    int pend = -1;          // buffer index of a group whose accumulator is still to be read
    float pend_d = 0.0f;    // its Δ
    uint32_t pend_par = 0;
    uint32_t redph = 0;
    auto drain = [&]() {  // read back the pending group's accumulator, scale by Δ, add
      mbar_wait(d_full(pend), pend_par);
      tc_fence_after();
      uint32_t d[16];
      tmem_ld_x16(tmem + lane_addr + D_COL + (uint32_t)pend * NT, d);
      tmem_ld_wait();
#pragma unroll
      for (int t = 0; t < NT; ++t) acc[t] = fmaf(__uint_as_float(d[t]), pend_d, acc[t]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(d_empty(pend));
      pend = -1;
    };
    for (int u = u0; u < u1; ++u) {
      mbar_wait(full(s), ph);
      const uint8_t* st = smem + s * STAGE;
      // this set's two groups of the stage: set, set + 2
      uint4 cw[2][4];
      uint16_t sb[2], zb[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int g = set + 2 * h;
        const uint8_t* crow = st + g * (BM * 64) + row * 64;
#pragma unroll
        for (int cidx = 0; cidx < 4; ++cidx) cw[h][cidx] = *reinterpret_cast<const uint4*>(crow + ((cidx ^ sw) << 4));
        sb[h] = *reinterpret_cast<const uint16_t*>(st + CODES + XB + g * (BM * 2) + row * 2);
        zb[h] = *reinterpret_cast<const uint16_t*>(st + CODES + XB + SZ + g * (BM * 2) + row * 2);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty(s));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t zsub, zfma;
        zero_consts<kBF16>(zb[h], zsub, zfma);
        const int ab = set * 2 + (jn & 1);
        const uint32_t par = (uint32_t)(jn >> 1) & 1u;
        uint32_t a[2][32];
#pragma unroll
        for (int cidx = 0; cidx < 4; ++cidx) {
          const uint32_t w4[4] = {cw[h][cidx].x, cw[h][cidx].y, cw[h][cidx].z, cw[h][cidx].w};
#pragma unroll
          for (int wd = 0; wd < 4; ++wd) dequant_word<kBF16>(w4[wd], zsub, zfma, &a[cidx >> 1][(cidx & 1) * 16 + wd * 4]);
        }
        mbar_wait(a_empty(ab), par ^ 1u);
        tc_fence_after();
        tmem_st_x32(tmem + lane_addr + A_COL + (uint32_t)ab * 64, a[0]);
        tmem_st_x32(tmem + lane_addr + A_COL + (uint32_t)ab * 64 + 32, a[1]);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(a_full(ab));
        if (pend >= 0) drain();  // the previous group's MMAs ran while this one was dequantized
        pend = ab;
        pend_par = par;
        pend_d = __half2float(__ushort_as_half(sb[h]));
        ++jn;
      }
      if (++s == NS) { s = 0; ph ^= 1; }
      // ---- end of a row-block segment: park the partial sums for the epilogue warp
      const bool rb_done = (u % wk.upb) + 1 == wk.upb;
      if (rb_done || u + 1 == u1) {
        if (pend >= 0) drain();
        mbar_wait(red_empty, redph ^ 1u);
        float* mine = slot + set * (NT * BM);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          mine[t * BM + row] = acc[t];
          acc[t] = 0.0f;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(red_full);
        redph ^= 1u;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
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

}  // namespace

cudaError_t launch_decode_tc(const void* X, int x_dtype, const uint8_t* Wq, const uint16_t* scales,
                             const uint16_t* zeros, void* Y, int M, int N, int K, void* ws,
                             cudaStream_t st, const char** why) {
  const int G = K / kGroup;
  CUtensorMap tw, tx, ts, tz;
  bool ok;
  {
    const uint64_t d[3] = {64, (uint64_t)N, (uint64_t)G};
    const uint64_t s[2] = {(uint64_t)K / 2, 64};
    const uint32_t b[3] = {64, (uint32_t)BM, (uint32_t)GPS};
    ok = encode(&tw, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, Wq, d, s, b, CU_TENSOR_MAP_SWIZZLE_64B);
  }
  {
    // X [M][K] viewed as {64 elements, M rows, K/64 atoms}; box = 8 atoms (4 groups) x NT rows
    const uint64_t d[3] = {64, (uint64_t)M, (uint64_t)K / 64};
    const uint64_t s[2] = {(uint64_t)K * 2, 128};
    const uint32_t b[3] = {64, (uint32_t)NT, (uint32_t)(2 * GPS)};
    ok = ok && encode(&tx, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, X, d, s, b, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  {
    const uint64_t d[2] = {(uint64_t)N, (uint64_t)G};
    const uint64_t s[1] = {(uint64_t)N * 2};
    const uint32_t b[2] = {(uint32_t)BM, (uint32_t)GPS};
    ok = ok && encode(&ts, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, scales, d, s, b, CU_TENSOR_MAP_SWIZZLE_NONE) &&
         encode(&tz, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, zeros, d, s, b, CU_TENSOR_MAP_SWIZZLE_NONE);
  }
  if (!ok) {
    *why = "cuTensorMapEncodeTiled failed";
    return cudaErrorInvalidValue;
  }
  Work wk;
  wk.upb = (G + GPS - 1) / GPS;
  wk.units = ((N + BM - 1) / BM) * wk.upb;
  const int P = std::min(wk.units, num_sms());
  wk.cta_q = wk.units / P;
  wk.cta_r = wk.units % P;
  float* partials = reinterpret_cast<float*>(ws);
  int* counters = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(ws) + ws_partials_bytes());
  auto kern = x_dtype == SQ_BF16 ? decode_tc_kernel<true> : decode_tc_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ALLOC);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)P, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = SMEM_ALLOC;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = option(SQ_OPT_PDL) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int early = option(SQ_OPT_PDL) && option(SQ_OPT_WEIGHTS_STATIC);
  return cudaLaunchKernelEx(&cfg, kern, tw, tx, ts, tz, (uint16_t*)Y, counters, partials, M, N, wk, early);
}

size_t decode_tc_partials_bytes() { return (size_t)num_sms() * 2 * NT * BM * sizeof(float); }

}  // namespace sq
