// K-dtc: W4A16 GEMM for 9 <= M <= 64 (batched decode) on the
// 5th-generation tensor cores.
//
//   Y[m][n] = sum_gi Δ[gi][n] * sum_{k in gi} X[m][k] * (q[n][k] - Z[gi][n])
//   PAPER.md:104-106 Eq. 3 with Ŵ of Eq. 1 line 2; fp32 accumulation.
//
// Why a second decode kernel: the mma.sync kernel (k_decode.cu) issues its MMAs from the
// dequantizing warps; at M = 9-16 it needs two m16n8k16 per 256 weights and the SM's
// HMMA pipe saturates before HBM does, and at M = 17-64 the prefill kernel (which rounds
// Ŵ = RN((q-Z)Δ) into TMEM and keeps one accumulator) is capped by its dequant rate.
// Here the dequantizing warps only produce operands; the MMA is asynchronous.
//
// Design:
//  * MMA: tcgen05.mma.cta_group::1.kind::f16, M = 128 weight rows (TMEM lanes), N = NT
//    tokens (16/32/64), K = 16.  A = the EXACT integer (q - Z) in fp16/bf16, written into
//    TMEM by the dequant warps (tcgen05.st); B = X from SMEM (TMA, SWIZZLE_128B).
//  * Δ is per (row, group), so every group accumulates into its OWN TMEM accumulator
//    D_g [128 x NT] (a ring of ND slots); the dequant warps read it back (tcgen05.ld) a
//    few groups later and add Δ · D_g into fp32 registers -- Δ is applied once per group
//    in fp32, as in the mma.sync kernel, so only fp32 rounding remains.
//  * The lop3 magic-number dequant yields k pairs (k, k+4) of every 8-code word; the X
//    rows are permuted the same way inside each 16-byte chunk by one warp after the TMA
//    lands (the swizzle only moves whole chunks), so the MMA's K order matches.
//  * Warps: 0 TMA producer, 1 TMEM allocator + MMA issuer, 2 X permuter, 3 epilogue,
//    4-11 dequant (two sets of four, one warp per TMEM lane quarter; the sets take
//    alternate groups, and the epilogue adds their two partial sums per row block).
//  * Persistent stream-K over units of (128-row block x 4 groups), one CTA per SM, the
//    schedule and deterministic fixup of k_decode.cu; the epilogue warp takes finished
//    row-block segments from SMEM (Y store or fixup) off the dequant warps' path.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "decode_common.cuh"
#include "sm100.cuh"
#include "sq_internal.cuh"

namespace sq {

bool encode_tmap(CUtensorMap* map, CUtensorMapDataType dt, int rank, const void* base, const uint64_t* dims,
                 const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle sw);

namespace {

using namespace dec;
using namespace ptx;

constexpr int kGroup = 128;
constexpr int GPS = 4;        // groups per unit
constexpr int BM = 128;       // weight rows per row block (MMA M, TMEM lanes)
constexpr int kDqWarp0 = 4;

template <int NT>
struct TC {
  // dequant warp sets (4 warps each, one per TMEM lane quarter) taking groups round-robin
  static constexpr int SETS = NT == 16 ? 3 : 2;
  static constexpr int THREADS = (kDqWarp0 + 4 * SETS) * 32;
  static constexpr int CODES = GPS * BM * 64;       // [group][row][64 B], SWIZZLE_64B
  static constexpr int SZB = GPS * BM * 2;          // [group][row] fp16
  static constexpr int CST = CODES + 2 * SZB;       // 34 KB, a multiple of 1 KB
  static constexpr int NSC = NT <= 16 ? 4 : 3;      // unit stages (codes + Δ + Z)
  static constexpr int ATOM = NT * 128;             // one SWIZZLE_128B atom: NT rows x 64 k
  static constexpr int XG = 2 * ATOM;               // X of one group (128 k)
  static constexpr int NSX = NT == 16 ? 8 : NT == 32 ? 6 : 3;
  // TMEM: NA A slots of 64 columns + ND accumulator slots of NT columns <= 512.  The
  // dequant warps read D_g back LAG groups after storing A_g, so LAG groups' MMAs (issue,
  // execution, commit) are in flight behind the dequant work
  static constexpr int NA = NT == 16 ? 6 : NT == 32 ? 5 : 3;
  static constexpr int ND = NT == 16 ? 8 : NT == 32 ? 5 : 4;
  static constexpr int LAG = ND - 1;                // groups (both sets) between A store and read-back
  static constexpr int NE = NT == 64 ? 1 : 2;       // epilogue buffers
  static constexpr int EPI = SETS * NT * BM * 4;    // [set][token][row] fp32
  static constexpr int OFF_X = NSC * CST;
  static constexpr int OFF_E = OFF_X + NSX * XG;
  static constexpr int OFF_DR = OFF_E + NE * EPI;   // Δ of the groups awaiting read-back: [ND][row]
  static constexpr int OFF_BAR = OFF_DR + ND * BM * 4;
  static constexpr int NBAR = 2 * NSC + 3 * NSX + 2 * NA + 2 * ND + 2 * NE;
  static constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
  static constexpr int SMEM = OFF_TMEM + 16;
  static constexpr int SMEM_ALLOC = SMEM + 1024;
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr uint32_t A_COL = 0;              // A slots: [0, 256)
  static constexpr uint32_t D_COL = 256;            // D slots: [256, 256 + ND * NT)
  static_assert(D_COL + ND * NT <= TMEM_COLS, "TMEM");
  static_assert(SMEM_ALLOC <= 227 * 1024, "SMEM");
};

template <int N>
__device__ __forceinline__ void tmem_ld_n(uint32_t taddr, uint32_t (&v)[N]) {
  if constexpr (N == 8) {
    tmem_ld_x8(taddr, v);
  } else if constexpr (N == 16) {
    tmem_ld_x16(taddr, v);
  } else {
    static_assert(N == 32, "8, 16 or 32 columns");
    tmem_ld_x16(taddr, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
    tmem_ld_x16(taddr + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
  }
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

template <int NT, bool kBF16>
__global__ void __launch_bounds__(TC<NT>::THREADS, 1)
dtc_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
           const __grid_constant__ CUtensorMap tm_s, const __grid_constant__ CUtensorMap tm_z,
           uint16_t* __restrict__ Y, int* __restrict__ counters, float* __restrict__ partials, int M, int N, int G,
           Work wk, int early_weights) {
  using C = TC<NT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = sbase + C::OFF_BAR;
  auto c_full = [&](int i) { return bar0 + 8u * i; };
  auto c_empty = [&](int i) { return bar0 + 8u * (C::NSC + i); };
  auto x_full = [&](int i) { return bar0 + 8u * (2 * C::NSC + i); };
  auto x_ready = [&](int i) { return bar0 + 8u * (2 * C::NSC + C::NSX + i); };
  auto x_empty = [&](int i) { return bar0 + 8u * (2 * C::NSC + 2 * C::NSX + i); };
  auto a_full = [&](int i) { return bar0 + 8u * (2 * C::NSC + 3 * C::NSX + i); };
  auto a_empty = [&](int i) { return bar0 + 8u * (2 * C::NSC + 3 * C::NSX + C::NA + i); };
  auto d_full = [&](int i) { return bar0 + 8u * (2 * C::NSC + 3 * C::NSX + 2 * C::NA + i); };
  auto d_empty = [&](int i) { return bar0 + 8u * (2 * C::NSC + 3 * C::NSX + 2 * C::NA + C::ND + i); };
  auto e_full = [&](int i) { return bar0 + 8u * (2 * C::NSC + 3 * C::NSX + 2 * C::NA + 2 * C::ND + i); };
  auto e_empty = [&](int i) { return bar0 + 8u * (2 * C::NSC + 3 * C::NSX + 2 * C::NA + 2 * C::ND + C::NE + i); };
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEM);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int c = blockIdx.x, P = gridDim.x;
  constexpr int kDq = 4 * C::SETS;  // dequant warps

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NSC; ++i) { mbar_init(c_full(i), 1); mbar_init(c_empty(i), kDq); }
    for (int i = 0; i < C::NSX; ++i) { mbar_init(x_full(i), 1); mbar_init(x_ready(i), 1); mbar_init(x_empty(i), 1); }
    for (int i = 0; i < C::NA; ++i) { mbar_init(a_full(i), 4); mbar_init(a_empty(i), 1); }   // one set writes A_g
    for (int i = 0; i < C::ND; ++i) { mbar_init(d_full(i), 1); mbar_init(d_empty(i), 4); }   // one set reads D_g
    for (int i = 0; i < C::NE; ++i) { mbar_init(e_full(i), kDq * 32); mbar_init(e_empty(i), 1); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) tmem_alloc(smem_u32(tmem_holder), C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  pdl_launch_dependents();

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      prefetch_tmap(&tm_w);
      prefetch_tmap(&tm_x);
      prefetch_tmap(&tm_s);
      prefetch_tmap(&tm_z);
      const uint64_t wpol = l2_evict_first_policy();
      auto load_unit = [&](int slot, int rb, int pos) {
        const int g0 = pos * GPS;
        const uint32_t st = sbase + slot * C::CST;
        mbar_expect_tx(c_full(slot), C::CST);
        tma_3d_hint(st, &tm_w, c_full(slot), 0, rb * BM, g0, wpol);
        tma_2d(st + C::CODES, &tm_s, c_full(slot), rb * BM, g0);
        tma_2d(st + C::CODES + C::SZB, &tm_z, c_full(slot), rb * BM, g0);
      };
      int pre = 0;
      if (early_weights) {  // weights never depend on the previous kernel: stream them now
        Sched sc(wk, c, P);
        for (; pre < C::NSC && sc.valid(); ++pre, sc.next(wk)) load_unit(pre, sc.rb, sc.pos);
      }
      pdl_wait();  // X may be the previous kernel's output
      int ui = 0, j = 0;
      for (Sched sc(wk, c, P); sc.valid(); sc.next(wk), ++ui) {
        const int cs = ui % C::NSC;
        if (ui >= pre) {
          mbar_wait_idle(c_empty(cs), ((ui / C::NSC) & 1) ^ 1);
          load_unit(cs, sc.rb, sc.pos);
        }
        const int gq = sc.pos * GPS;
        const int ng = min(GPS, G - gq);
        for (int g = 0; g < ng; ++g, ++j) {
          const int xs = j % C::NSX;
          mbar_wait_idle(x_empty(xs), ((j / C::NSX) & 1) ^ 1);
          mbar_expect_tx(x_full(xs), C::XG);
          const uint32_t xd = sbase + C::OFF_X + xs * C::XG;
          tma_2d(xd, &tm_x, x_full(xs), (gq + g) * kGroup, 0);
          tma_2d(xd + C::ATOM, &tm_x, x_full(xs), (gq + g) * kGroup + 64, 0);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (whole warp, elect.sync issues) =====================
    constexpr uint32_t idesc = f16_idesc(kBF16, BM, NT);
    int j = 0;
    for (Sched sc(wk, c, P); sc.valid(); sc.next(wk)) {
      const int ng = min(GPS, G - sc.pos * GPS);
      for (int g = 0; g < ng; ++g, ++j) {
        const int xs = j % C::NSX, as = j % C::NA, ds = j % C::ND;
        mbar_wait(x_ready(xs), (j / C::NSX) & 1);
        mbar_wait(a_full(as), (j / C::NA) & 1);
        mbar_wait(d_empty(ds), ((j / C::ND) & 1) ^ 1);
        tc_fence_after();
        const uint32_t xaddr = sbase + C::OFF_X + xs * C::XG;
#pragma unroll
        for (int kk = 0; kk < kGroup / 16; ++kk) {
          const uint64_t bdesc = sw128_desc(xaddr + (kk >> 2) * C::ATOM + (kk & 3) * 32);
          tc_mma_ts(tmem + C::D_COL + ds * NT, tmem + C::A_COL + as * 64 + kk * 8, bdesc, idesc, kk > 0 ? 1u : 0u);
        }
        tc_commit(x_empty(xs));
        tc_commit(a_empty(as));
        tc_commit(d_full(ds));
      }
    }
  } else if (warp == 2) {
    // ===================== X permuter: (x0..x7) -> (x0,x4,x1,x5,x2,x6,x3,x7) per 16-B chunk =====
    // (the order of the dequantized k pairs); rows >= M are the TMA's zero fill
    int j = 0;
    const int per_atom = min(M, NT) * 8;  // 16-B chunks of the real token rows in one atom
    for (Sched sc(wk, c, P); sc.valid(); sc.next(wk)) {
      const int ng = min(GPS, G - sc.pos * GPS);
      for (int g = 0; g < ng; ++g, ++j) {
        const int xs = j % C::NSX;
        mbar_wait_idle(x_full(xs), (j / C::NSX) & 1);
        const uint32_t xaddr = sbase + C::OFF_X + xs * C::XG;
        for (int i = lane; i < 2 * per_atom; i += 32) {
          const int atom = i >= per_atom ? 1 : 0, rem = i - atom * per_atom;
          const uint32_t a = xaddr + atom * C::ATOM + (rem >> 3) * 128 + (rem & 7) * 16;
          const uint4 v = lds128(a);
          uint4 o;
          o.x = prmt(v.x, v.z, 0x5410u);
          o.y = prmt(v.x, v.z, 0x7632u);
          o.z = prmt(v.y, v.w, 0x5410u);
          o.w = prmt(v.y, v.w, 0x7632u);
          sts128(a, o);
        }
        // generic-proxy writes -> visible to the tensor core's (async proxy) reads
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(x_ready(xs));
      }
    }
  } else if (warp == 3) {
    // ===================== epilogue: finished row-block segments, off the dequant path ====
    auto to_out = [](float v) -> uint16_t {
      if (kBF16) return __bfloat16_as_ushort(__float2bfloat16_rn(v));
      return __half_as_ushort(__float2half_rn(v));
    };
    const int mt = min(M, NT);
    bool waited = false;
    int sgc = 0;  // segment counter
    for (Sched sc(wk, c, P); sc.valid(); sc.next(wk)) {
      if (!sc.range_last()) continue;
      const int e = sgc % C::NE;
      mbar_wait_idle(e_full(e), (sgc / C::NE) & 1);
      ++sgc;
      if (!waited) {  // global writes must follow the previous kernel (PDL)
        pdl_wait();
        waited = true;
      }
      // the two sets' partial sums of this segment, [set][token][row]
      const float* ep = reinterpret_cast<const float*>(smem + C::OFF_E + e * C::EPI);
      auto val = [&](int t, int r) {
        float v = ep[t * BM + r];
#pragma unroll
        for (int k = 1; k < C::SETS; ++k) v += ep[(k * NT + t) * BM + r];
        return v;
      };
      const int rb = sc.rb, n0 = rb * BM;
      if (sc.full) {
        for (int t = 0; t < mt; ++t)
#pragma unroll
          for (int i = 0; i < BM / 32; ++i) {
            const int r = lane + 32 * i;
            if (n0 + r < N) Y[(size_t)t * N + n0 + r] = to_out(val(t, r));
          }
        __syncwarp();
        if (lane == 0) mbar_arrive(e_empty(e));
        continue;
      }
      // stream-K fixup: park the partial; the last contributor sums them in CTA order
      float* slot = partials + ((size_t)c * 2 + sc.e) * (NT * BM);
      for (int t = 0; t < mt; ++t)
#pragma unroll
        for (int i = 0; i < BM / 32; ++i) __stcg(slot + t * BM + lane + 32 * i, val(t, lane + 32 * i));
      __syncwarp();
      if (lane == 0) mbar_arrive(e_empty(e));
      const int c0 = wk.cta_of(rb * wk.upb), c1 = wk.cta_of((rb + 1) * wk.upb - 1);
      int last = 0;
      if (lane == 0) {
        int prev;
        asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;\n" : "=r"(prev) : "l"(counters + rb) : "memory");
        last = prev == c1 - c0;
      }
      if (__shfl_sync(0xffffffffu, last, 0)) {
        for (int t = 0; t < mt; ++t) {
          float tot[BM / 32];
#pragma unroll
          for (int i = 0; i < BM / 32; ++i) tot[i] = 0.0f;
          for (int cc = c0; cc <= c1; ++cc) {
            const int ee = (wk.start(cc) / wk.upb == rb) ? 0 : 1;
            const float* src = partials + ((size_t)cc * 2 + ee) * (NT * BM) + t * BM;
#pragma unroll
            for (int i = 0; i < BM / 32; ++i) tot[i] += __ldcg(src + lane + 32 * i);
          }
#pragma unroll
          for (int i = 0; i < BM / 32; ++i) {
            const int r = lane + 32 * i;
            if (n0 + r < N) Y[(size_t)t * N + n0 + r] = to_out(tot[i]);
          }
        }
        if (lane == 0) counters[rb] = 0;  // leave the workspace zeroed
      }
    }
  } else {
    // ===================== dequant warps: thread = weight row = TMEM lane =====================
    const int q = warp % 4;                     // TMEM lane quarter (warp % 4 by hardware rule)
    const int s = (warp - kDqWarp0) / 4;        // set: groups j with j % SETS == s
    const int row = q * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const int sw = (row >> 1) & 3;              // SWIZZLE_64B: chunk c of this row sits at c ^ sw
    float* dring = reinterpret_cast<float*>(smem + C::OFF_DR);  // Δ of groups awaiting read-back
    float acc[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[t] = 0.0f;
    // Read-backs trail the A stores by LAG groups, on a second cursor over the same schedule
    // (all groups in order: the set reads back its own groups and hands its partial sum of
    // every row-block segment to the epilogue warp when the cursor passes the segment's end).
    Sched rsc(wk, c, P);
    int rg = 0, jr = 0, sgc = 0;
    auto readback = [&]() {
      const int rng = min(GPS, G - rsc.pos * GPS);
      const bool seg_end = rsc.range_last() && rg == rng - 1;
      if (jr % C::SETS == s) {
        const int ds = jr % C::ND;
        const float d = dring[ds * BM + row];
        mbar_wait(d_full(ds), (jr / C::ND) & 1);
        tc_fence_after();
        uint32_t v[NT];
#pragma unroll
        for (int h = 0; h < NT / 16; ++h)
          tmem_ld_x16(tmem + lane_addr + C::D_COL + ds * NT + 16 * h, *reinterpret_cast<uint32_t(*)[16]>(&v[16 * h]));
        tmem_ld_wait();
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[t] = fmaf(d, __uint_as_float(v[t]), acc[t]);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(d_empty(ds));
      }
      ++jr;
      if (++rg == rng) {
        rg = 0;
        rsc.next(wk);
      }
      if (seg_end) {  // this set's share of the segment is complete: hand it to the epilogue warp
        const int e = sgc % C::NE;
        mbar_wait(e_empty(e), ((sgc / C::NE) & 1) ^ 1);
        ++sgc;
        float* ep = reinterpret_cast<float*>(smem + C::OFF_E + e * C::EPI) + s * NT * BM;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          ep[t * BM + row] = acc[t];
          acc[t] = 0.0f;
        }
        mbar_arrive(e_full(e));  // every lane, after its own writes (release)
      }
    };
    int ui = 0, j = 0;
    for (Sched sc(wk, c, P); sc.valid(); sc.next(wk), ++ui) {
      const int cs = ui % C::NSC;
      const int ng = min(GPS, G - sc.pos * GPS);
      const uint32_t st = sbase + cs * C::CST;
      mbar_wait(c_full(cs), (ui / C::NSC) & 1);
      for (int g = 0; g < ng; ++g, ++j) {
        if (j % C::SETS == s) {
          const uint32_t crow = st + g * (BM * 64) + row * 64;
          uint32_t w[16];
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            const uint4 v = lds128(crow + ((ch ^ sw) << 4));
            w[4 * ch] = v.x; w[4 * ch + 1] = v.y; w[4 * ch + 2] = v.z; w[4 * ch + 3] = v.w;
          }
          const uint16_t dbits = *reinterpret_cast<const uint16_t*>(smem + cs * C::CST + C::CODES + (g * BM + row) * 2);
          const uint16_t zbits =
              *reinterpret_cast<const uint16_t*>(smem + cs * C::CST + C::CODES + C::SZB + (g * BM + row) * 2);
          dring[(j % C::ND) * BM + row] = __half2float(__ushort_as_half(dbits));
          uint32_t zsub, zfma;
          zero_consts<kBF16>(zbits, zsub, zfma);
          uint32_t a[64];
#pragma unroll
          for (int k = 0; k < 16; ++k)
            dequant_word<kBF16>(w[k], zsub, zfma, *reinterpret_cast<uint32_t(*)[4]>(&a[4 * k]));
          const int as = j % C::NA;
          mbar_wait(a_empty(as), ((j / C::NA) & 1) ^ 1);
          tc_fence_after();
          tmem_st_x32(tmem + lane_addr + C::A_COL + as * 64, a);
          tmem_st_x32(tmem + lane_addr + C::A_COL + as * 64 + 32, a + 32);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(a_full(as));
        }
        if (g == ng - 1) {  // every dequant warp releases the unit's stage once
          __syncwarp();
          if (lane == 0) mbar_arrive(c_empty(cs));
        }
        if (j >= C::LAG) readback();
      }
    }
    while (jr < j) readback();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

template <int NT, bool kBF16>
cudaError_t launch_nt(const void* X, const uint8_t* Wq, const uint16_t* scales, const uint16_t* zeros, void* Y, int M,
                      int N, int K, void* ws, bool weights_static, cudaStream_t st, const char** why) {
  using C = TC<NT>;
  const int G = K / kGroup;
  CUtensorMap tw, tx, ts, tz;
  {
    const uint64_t d[3] = {64, (uint64_t)N, (uint64_t)G};
    const uint64_t s[2] = {(uint64_t)K / 2, 64};
    const uint32_t b[3] = {64, (uint32_t)BM, (uint32_t)GPS};
    if (!encode_tmap(&tw, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, Wq, d, s, b, CU_TENSOR_MAP_SWIZZLE_64B)) {
      *why = "tensor map (codes)";
      return cudaErrorInvalidValue;
    }
  }
  {
    const uint64_t d[2] = {(uint64_t)K, (uint64_t)M};
    const uint64_t s[1] = {(uint64_t)K * 2};
    const uint32_t b[2] = {64, (uint32_t)NT};
    if (!encode_tmap(&tx, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, X, d, s, b, CU_TENSOR_MAP_SWIZZLE_128B)) {
      *why = "tensor map (X)";
      return cudaErrorInvalidValue;
    }
  }
  {
    const uint64_t d[2] = {(uint64_t)N, (uint64_t)G};
    const uint64_t s[1] = {(uint64_t)N * 2};
    const uint32_t b[2] = {(uint32_t)BM, GPS};
    if (!encode_tmap(&ts, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, scales, d, s, b, CU_TENSOR_MAP_SWIZZLE_NONE) ||
        !encode_tmap(&tz, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, zeros, d, s, b, CU_TENSOR_MAP_SWIZZLE_NONE)) {
      *why = "tensor map (scales/zeros)";
      return cudaErrorInvalidValue;
    }
  }
  Work wk;
  wk.rbs = (N + BM - 1) / BM;
  wk.upb = (G + GPS - 1) / GPS;
  wk.units = wk.rbs * wk.upb;
  wk.dp = 0;
  int slots = num_sms();
  if (option(SQ_OPT_DECODE_GRID_LIMIT) > 0) slots = std::min(slots, option(SQ_OPT_DECODE_GRID_LIMIT));
  const int P = std::min(wk.units, slots);
  wk.cta_q = wk.units / P;
  wk.cta_r = wk.units % P;
  float* partials = reinterpret_cast<float*>(ws);
  int* counters = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(ws) + ws_partials_bytes());
  auto kern = dtc_kernel<NT, kBF16>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_ALLOC);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)P, 1, 1);
  cfg.blockDim = dim3(C::THREADS, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM_ALLOC;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = option(SQ_OPT_PDL) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int early = option(SQ_OPT_PDL) && weights_static;
  return cudaLaunchKernelEx(&cfg, kern, tw, tx, ts, tz, (uint16_t*)Y, counters, partials, M, N, G, wk, early);
}

}  // namespace

size_t dtc_partials_bytes() { return (size_t)num_sms() * 2 * 64 * BM * sizeof(float); }

size_t dtc_workspace_bytes(int64_t N) { return ws_partials_bytes() + counter_region_bytes((N + BM - 1) / BM); }

cudaError_t launch_dtc(const void* X, int x_dtype, const uint8_t* Wq, const uint16_t* scales, const uint16_t* zeros,
                       void* Y, int M, int N, int K, void* ws, bool weights_static, cudaStream_t st,
                       const char** why) {
  const bool bf16 = x_dtype == SQ_BF16;
  if (M <= 16)
    return bf16 ? launch_nt<16, true>(X, Wq, scales, zeros, Y, M, N, K, ws, weights_static, st, why)
                : launch_nt<16, false>(X, Wq, scales, zeros, Y, M, N, K, ws, weights_static, st, why);
  if (M <= 32)
    return bf16 ? launch_nt<32, true>(X, Wq, scales, zeros, Y, M, N, K, ws, weights_static, st, why)
                : launch_nt<32, false>(X, Wq, scales, zeros, Y, M, N, K, ws, weights_static, st, why);
  if (M <= 64)
    return bf16 ? launch_nt<64, true>(X, Wq, scales, zeros, Y, M, N, K, ws, weights_static, st, why)
                : launch_nt<64, false>(X, Wq, scales, zeros, Y, M, N, K, ws, weights_static, st, why);
  *why = "tcgen05 decode path needs M <= 64";
  return cudaErrorInvalidValue;
}

}  // namespace sq
