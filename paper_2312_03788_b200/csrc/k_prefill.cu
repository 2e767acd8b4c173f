// K-pre: W4A16 GEMM for large M (prefill) on the 5th-generation tensor cores.
//
//   Y[m][n] = sum_k X[m][k] * Ŵ[n][k],  Ŵ = RN((q - Z) * Δ)      PAPER.md:104-106 Eq. 3,
//                                                             PAPER.md:90 Eq. 1 line 2
// Design -- "swap-AB, weights in TMEM":
//  * The MMA computes D[n][m] = Ŵ_tile[n][:] · X_tile[m][:]^T with tcgen05.mma
//    .cta_group::1.kind::f16, M_mma = 128 weight rows, N_mma = up to 256 tokens,
//    K = 16 per instruction, fp32 accumulator D in TMEM (256 columns).
//  * Operand A (the dequantized weights) lives in TMEM: the dequant warps turn
//    packed codes into fp16/bf16 with register math and write them with
//    tcgen05.st straight into a 4-stage ring of TMEM A buffers -- the dequantized
//    tile never touches shared memory, so SMEM bandwidth is spent only on the X
//    operand (TMA, 128B swizzle) and the packed codes.
//  * Operand B (activations X[M][K]) is loaded by TMA into a 4-stage SMEM ring in
//    the canonical K-major SWIZZLE_128B layout the UMMA descriptor expects.
//  * Packed codes (64 bytes/row/group, SWIZZLE_64B to keep the per-row LDS
//    conflict-free) and the group's Δ/Z rows arrive by TMA into a separate ring.
//  * Warp roles: warp 0 = TMA producer, warp 1 = TMEM allocator + single-thread MMA
//    issuer, warps 4-7 = dequant (thread = TMEM lane = weight row) and epilogue
//    (tcgen05.ld -> fp16/bf16 -> coalesced stores along n).
//  * Persistent: one CTA per SM walks the (n-tile, m-tile) list.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "sq_internal.cuh"

namespace sq {

namespace {

constexpr int BM = 128;        // weight rows per tile (MMA M, TMEM lanes)
constexpr int kGroup = 128;    // k per code stage (one quantization-group column), A stage and X stage
constexpr int kBTMax = 256;    // tokens per tile, widest configuration (MMA N max)
constexpr int kDequantWarp0 = 4;
constexpr int C_STAGE_BYTES = BM * kGroup / 2;  // packed codes of a stage, 64 B per row
constexpr int SZ_BYTES = (kGroup / 32) * BM * 2;  // Δ (or Z) rows of a stage: [128 / GS][BM] fp16, GS >= 32

// Tile configuration by token-tile width BT.  A 128-k code stage (packed
// codes + Δ/Z rows, one TMA box each) holds 128 / KA "A stages" of KA k; each A stage is
// converted into KA / 2 TMEM columns by one set of four dequant warps (one per TMEM lane
// quarter) and consumed with KA / 16 MMAs against an X stage of KA k.  The R warp sets take
// the A stages of the CTA's sequence round robin (i = r, r + R, ...), so R stages are in
// conversion at once and one set's barrier hand-offs overlap the others' arithmetic.  The
// accumulator takes BT TMEM columns, the A ring the rest.
//  * BT = 256 (large M, tensor-bound): KA = 64, R = 2 -- the two sets split every code stage.
//  * BT = 64 / 128 (one token tile, M <= 128: weight streaming, bound by the dequant warps):
//    KA = 128, R = 3 (16 warps, 128 registers/thread).  With two sets each warp spent
//    ~850-1050 cycles converting a stage and ~650 more in barrier checks and hand-offs
//    (profiles/r02/prefill_midm_trace.txt); whole-group stages halve the hand-offs per weight
//    and the third set fills the sub-partition while another waits.
template <int kBT, int kR = (kBT == kBTMax ? 2 : 3)>
struct PCfg {
  static constexpr int BT = kBT;
  static constexpr int KA = kBT == kBTMax ? 64 : 128;  // k per A stage and per X stage
  static constexpr int APS = kGroup / KA;               // A stages per code stage
  // dequant warp sets: 4 when the token tile is more than three quarters full (M = 49-64 at
  // BT = 64, 97-128 at BT = 128) -- the wider MMAs and X stages slow the MMA side and a fourth
  // set keeps more A stages converted (3-10 % on the 34B shapes but gate|up, unchanged) --
  // else 3 (a fourth set costs 2-4 % there); profiles/r02/prefill_four_sets_ab.jsonl
  static constexpr int R = kR;
  static constexpr int DQW = 4 * R;                     // dequant / epilogue warps
  static constexpr int THREADS = (kDequantWarp0 + DQW) * 32;
  static constexpr int X_SUB_BYTES = BT * 128;          // one 64-k SWIZZLE_128B box of BT rows
  static constexpr int X_STAGE_BYTES = (KA / 64) * X_SUB_BYTES;
  static constexpr int NSX = kBT == kBTMax ? 4 : kBT == 128 ? 3 : 6;    // X stages (SMEM)
  static constexpr int NSC = kBT == kBTMax ? 8 : kBT == 128 ? 10 : 12;  // code stages (SMEM)
  static constexpr int NSA = kBT == kBTMax ? 4 : (512 - kBT) / (KA / 2);  // A stages (TMEM)
  static_assert(APS == 1 || APS == R, "each set takes one A stage of every code stage, or whole code stages");
  static constexpr int OFF_X = 0;
  static constexpr int OFF_C = OFF_X + NSX * X_STAGE_BYTES;
  static constexpr int OFF_S = OFF_C + NSC * C_STAGE_BYTES;
  static constexpr int OFF_Z = OFF_S + NSC * SZ_BYTES;
  static constexpr int OFF_BAR = OFF_Z + NSC * SZ_BYTES;
  static constexpr int NUM_BARS = 2 * NSX + 2 * NSC + 2 * NSA + 2;
  static constexpr int OFF_TMEM = OFF_BAR + NUM_BARS * 8;
  static constexpr int SMEM_BYTES = OFF_TMEM + 16;
  static constexpr int SMEM_ALLOC = SMEM_BYTES + 1024;  // slack for 1024 B alignment
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr uint32_t D_COL = 0;   // accumulator: columns [0, BT)
  static constexpr uint32_t A_COL = BT;  // A stages: columns [BT, BT + NSA * KA / 2)
  static_assert(A_COL + NSA * (KA / 2) <= TMEM_COLS, "TMEM budget");
  static_assert(SMEM_ALLOC <= 227 * 1024, "SMEM budget");
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
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// The MMA issuer is a whole warp in warp-uniform control flow and the tcgen05 instructions
// are predicated on elect.sync: the descriptors then live in uniform registers and one MMA
// issues every few cycles.  Issued from a divergent single-lane branch instead, every MMA
// pays a per-instruction uniform-register round trip (~160-220 cycles per MMA,
// profiles/r02/tcgen05_mma_issue_rate.txt, vs the 128-cycle tensor floor of a 128x256x16 MMA).
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(bar)
      : "memory");
}
// One A stage's worth of MMAs (KA / 16 of them, K = 16 each) under a single elect.sync: the
// A address steps 8 TMEM columns and the B descriptor 32 bytes (2 in its >> 4 address field)
// per MMA, with a jump to the second 64-k X box after four.  One asm block keeps the issue
// stream at a few uniform-datapath instructions per MMA -- the MMA warp shares its SM
// sub-partition with two dequant warps, so every instruction it issues costs about three
// cycles (profiles/r02/prefill_midm_trace.txt).
template <int NMMA>
__device__ __forceinline__ void tc_mma_ts_stage(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc0, uint64_t b_desc1,
                                                uint32_t idesc, uint32_t accum) {
  static_assert(NMMA == 4 || NMMA == 8, "64 or 128 k per A stage");
#define SQ_MMA_I(A, B, P) "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [" A "], " B ", %4, " P ";\n"
#define SQ_MMA_NEXT "add.u32 a, a, 8;\nadd.u64 b, b, 2;\n"
  if constexpr (NMMA == 4) {
    asm volatile(
        "{\n.reg .pred e, p, t;\n.reg .b32 a;\n.reg .b64 b;\n"
        "elect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %5, 0;\nsetp.eq.b32 t, 0, 0;\n"
        "mov.b32 a, %1;\nmov.b64 b, %2;\n" SQ_MMA_I("a", "b", "p") SQ_MMA_NEXT SQ_MMA_I("a", "b", "t")
        SQ_MMA_NEXT SQ_MMA_I("a", "b", "t") SQ_MMA_NEXT SQ_MMA_I("a", "b", "t") "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc0), "l"(b_desc1), "r"(idesc), "r"(accum)
        : "memory");
  } else {
    asm volatile(
        "{\n.reg .pred e, p, t;\n.reg .b32 a;\n.reg .b64 b;\n"
        "elect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %5, 0;\nsetp.eq.b32 t, 0, 0;\n"
        "mov.b32 a, %1;\nmov.b64 b, %2;\n" SQ_MMA_I("a", "b", "p") SQ_MMA_NEXT SQ_MMA_I("a", "b", "t")
        SQ_MMA_NEXT SQ_MMA_I("a", "b", "t") SQ_MMA_NEXT SQ_MMA_I("a", "b", "t")
        "add.u32 a, a, 8;\nmov.b64 b, %3;\n" SQ_MMA_I("a", "b", "t") SQ_MMA_NEXT SQ_MMA_I("a", "b", "t")
        SQ_MMA_NEXT SQ_MMA_I("a", "b", "t") SQ_MMA_NEXT SQ_MMA_I("a", "b", "t") "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc0), "l"(b_desc1), "r"(idesc), "r"(accum)
        : "memory");
  }
#undef SQ_MMA_I
#undef SQ_MMA_NEXT
}
__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&v)[32]) {
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
__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// shared-window loads: the 1024-aligned dynamic-smem pointer is generic to the compiler, and
// generic loads of the code stage would take the long-scoreboard path
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint16_t lds16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];\n" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];\n" : "=r"(v) : "r"(a));
  return v;
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row core-matrix groups
// 1024 bytes apart (SBO), sm_100 descriptor version 1.
__device__ __forceinline__ uint64_t make_sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);  // start address
  d |= (uint64_t)1 << 16;                    // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;          // SBO
  d |= (uint64_t)1 << 46;                    // version
  d |= (uint64_t)2 << 61;                    // SWIZZLE_128B
  return d;
}

// Instruction descriptor: D fp32, A/B fp16 or bf16, both K-major, M = 128, N = n.
__device__ __forceinline__ uint32_t make_idesc(bool bf16, int n) {
  uint32_t d = 0;
  d |= 1u << 4;                          // D format f32
  d |= (bf16 ? 1u : 0u) << 7;            // A format
  d |= (bf16 ? 1u : 0u) << 10;           // B format
  d |= (uint32_t)(n >> 3) << 17;         // N >> 3
  d |= (uint32_t)(BM >> 4) << 24;        // M >> 4
  return d;
}

__device__ __forceinline__ uint32_t hsub2_f16(uint32_t a, uint32_t b) {
  __half2 r = __hsub2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t hmul2_f16(uint32_t a, uint32_t b) {
  __half2 r = __hmul2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}

// 8 codes (k0..k7, natural order) of one row -> 4 words of Ŵ = RN((q - Z) Δ) pairs
// (k0,k1), (k2,k3), (k4,k5), (k6,k7) in the MMA's natural k order.
// kSat (fp16 only, groups with Δ > 65504 / 15): |(q - Z) Δ| may exceed the fp16 range, so
// the product is formed in fp32 (exact: 5 x 11 bits) and rounded with saturation to
// ±65504 instead of overflowing to Inf (include/libsq.h).  Never taken for real weights
// (|W| < 2.5); the branch is per (row, group), uniform in practice.
template <bool kBF16, bool kSat = false>
__device__ __forceinline__ void dequant8(uint32_t w, uint32_t zc, uint32_t d2, float df,
                                         uint32_t* out) {
  const uint32_t u = w >> 4;
  const uint32_t sel[4] = {0x0400u, 0x0501u, 0x0602u, 0x0703u};  // byte i of w -> b0, of w>>4 -> b2
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    // low nibble of w.byte(i) -> half 0, low nibble of (w>>4).byte(i) -> half 1
    const uint32_t p = lop3_and_or(prmt(w, u, sel[i]), 0x000F000Fu, 0x64006400u);
    const uint32_t qz = hsub2_f16(p, zc);  // exact (q - Z) in fp16
    if (!kBF16 && kSat) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&qz));
      const float lo = fminf(fmaxf(f.x * df, -65504.0f), 65504.0f);
      const float hi = fminf(fmaxf(f.y * df, -65504.0f), 65504.0f);
      const __half2 h = __floats2half2_rn(lo, hi);  // RN of the clamped exact product
      out[i] = *reinterpret_cast<const uint32_t*>(&h);
    } else if (!kBF16) {
      out[i] = hmul2_f16(qz, d2);           // RN16((q - Z) Δ)
    } else {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&qz));
      const __nv_bfloat162 b = __floats2bfloat162_rn(f.x * df, f.y * df);  // exact product, one RN
      out[i] = *reinterpret_cast<const uint32_t*>(&b);
    }
  }
}

// Work split of one CTA into segments (tile, groups [g0, g1)).  Tiles are (128-row
// n-block, BT-token m-block), m fastest.  Without stream-K a CTA takes whole tiles c, c+P,
// ...; with stream-K the (tile x group) units are split into equal contiguous ranges and a
// tile cut between CTAs is finished by a fixup (last contributor sums the fp32 partials in
// CTA order).
struct PSched {
  int c, P, G, tiles, sk, q, r;
  int u, ue, tile, g0, g1;
  bool first;
  __device__ __forceinline__ int start(int cc) const { return cc * q + min(cc, r); }
  __device__ __forceinline__ int cta_of(int v) const {
    const int big = (q + 1) * r;
    return v < big ? v / (q + 1) : r + (v - big) / q;
  }
  __device__ __forceinline__ PSched(int c_, int P_, int G_, int tiles_, int sk_, int q_, int r_)
      : c(c_), P(P_), G(G_), tiles(tiles_), sk(sk_), q(q_), r(r_), first(true) {
    if (sk) {
      u = start(c);
      ue = start(c + 1);
      set();
    } else {
      tile = c;
      g0 = 0;
      g1 = G;
    }
  }
  __device__ __forceinline__ void set() {
    tile = u / G;
    g0 = u % G;
    g1 = min(G, g0 + (ue - u));
  }
  __device__ __forceinline__ bool valid() const { return sk ? u < ue : tile < tiles; }
  __device__ __forceinline__ void next() {
    first = false;
    if (sk) {
      u += g1 - g0;
      set();
    } else {
      tile += P;
    }
  }
};

template <bool kBF16, int GS, int kBT, int kR>
__global__ void __launch_bounds__(PCfg<kBT, kR>::THREADS, 1)
prefill_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
               const __grid_constant__ CUtensorMap tm_s, const __grid_constant__ CUtensorMap tm_z,
               uint16_t* __restrict__ Y, int M, int N, int K, int early_weights, int x_bytes,
               int sk, int cta_q, int cta_r, float* __restrict__ partials, int* __restrict__ counters,
               int zu4) {
  using C = PCfg<kBT, kR>;
  constexpr int BT = C::BT, KA = C::KA, APS = C::APS, R = C::R, DQW = C::DQW;
  constexpr int NSX = C::NSX, NSC = C::NSC, NSA = C::NSA;
  constexpr int SUBS = kGroup / GS;  // Δ/Z rows per stage
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = sbase + C::OFF_BAR;
  auto x_full = [&](int i) { return bar0 + 8u * i; };
  auto x_empty = [&](int i) { return bar0 + 8u * (NSX + i); };
  auto c_full = [&](int i) { return bar0 + 8u * (2 * NSX + i); };
  auto c_empty = [&](int i) { return bar0 + 8u * (2 * NSX + NSC + i); };
  auto a_full = [&](int i) { return bar0 + 8u * (2 * NSX + 2 * NSC + i); };
  auto a_empty = [&](int i) { return bar0 + 8u * (2 * NSX + 2 * NSC + NSA + i); };
  const uint32_t d_full = bar0 + 8u * (2 * NSX + 2 * NSC + 2 * NSA);
  const uint32_t d_empty = d_full + 8u;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEM);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n_tiles = (N + BM - 1) / BM;
  const int m_tiles = (M + BT - 1) / BT;
  const int num_tiles = n_tiles * m_tiles;
  const int G = K / kGroup;  // stages per tile (the schedule's unit)

  if (threadIdx.x == 0) {
    for (int i = 0; i < NSX; ++i) { mbar_init(x_full(i), 1); mbar_init(x_empty(i), 1); }
    for (int i = 0; i < NSC; ++i) { mbar_init(c_full(i), 1); mbar_init(c_empty(i), 4 * APS); }
    for (int i = 0; i < NSA; ++i) { mbar_init(a_full(i), 4); mbar_init(a_empty(i), 1); }
    mbar_init(d_full, 1);
    mbar_init(d_empty, DQW);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_x);
    prefetch_tmap(&tm_w);
    prefetch_tmap(&tm_s);
    prefetch_tmap(&tm_z);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_launch_dependents();

  if (warp == 0) {
    // ===================== TMA producer: activations, one X stage per A stage =====================
    if (lane == 0) {
      pdl_wait();  // X may be the previous kernel's output
      int xs = 0;
      uint32_t xph = 0;
      for (PSched sc(blockIdx.x, gridDim.x, G, num_tiles, sk, cta_q, cta_r); sc.valid(); sc.next()) {
        const int tile = sc.tile;
        const int m0 = (tile % m_tiles) * BT;
        for (int kb = APS * sc.g0; kb < APS * sc.g1; ++kb) {
          mbar_wait(x_empty(xs), xph ^ 1);
          mbar_expect_tx(x_full(xs), x_bytes);
#pragma unroll
          for (int h = 0; h < KA / 64; ++h)
            tma_load_2d(sbase + C::OFF_X + xs * C::X_STAGE_BYTES + h * C::X_SUB_BYTES, &tm_x, x_full(xs),
                        kb * KA + h * 64, m0);
          if (++xs == NSX) { xs = 0; xph ^= 1; }
        }
      }
    }
  } else if (warp == 2) {
    // ===================== TMA producer: packed codes + Δ/Z rows (own ring, runs ahead) ====
    if (lane == 0) {
      if (!early_weights) pdl_wait();
      int cs = 0;
      uint32_t cph = 0;
      for (PSched sc(blockIdx.x, gridDim.x, G, num_tiles, sk, cta_q, cta_r); sc.valid(); sc.next()) {
        const int tile = sc.tile;
        const int n0 = (tile / m_tiles) * BM;
        for (int g = sc.g0; g < sc.g1; ++g) {
          mbar_wait(c_empty(cs), cph ^ 1);
          // packed u4 zero rows (SQ_ZEROS_U4) are BM / 2 bytes, at the start of the same slot
          mbar_expect_tx(c_full(cs), C_STAGE_BYTES + SUBS * BM * 2 + (zu4 ? SUBS * BM / 2 : SUBS * BM * 2));
          tma_load_2d(sbase + C::OFF_C + cs * C_STAGE_BYTES, &tm_w, c_full(cs), g * (kGroup / 2), n0);
          tma_load_2d(sbase + C::OFF_S + cs * SZ_BYTES, &tm_s, c_full(cs), n0, g * SUBS);
          tma_load_2d(sbase + C::OFF_Z + cs * SZ_BYTES, &tm_z, c_full(cs), zu4 ? n0 / 2 : n0, g * SUBS);
          if (++cs == NSC) { cs = 0; cph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer: the whole warp, warp-uniform, elect.sync issues =====
    {
      int xs = 0, as = 0;
      uint32_t xph = 0, aph = 0, dph = 0;
      for (PSched sc(blockIdx.x, gridDim.x, G, num_tiles, sk, cta_q, cta_r); sc.valid(); sc.next()) {
        const int tile = sc.tile;
        const int m0 = (tile % m_tiles) * BT;
        const int n_mma = min(BT, ((M - m0) + 15) & ~15);
        const uint32_t idesc = make_idesc(kBF16, n_mma);
        mbar_wait(d_empty, dph ^ 1);  // epilogue has drained the accumulator
        dph ^= 1;
        tc_fence_after();
        for (int kb = APS * sc.g0; kb < APS * sc.g1; ++kb) {
          mbar_wait(a_full(as), aph);
          mbar_wait(x_full(xs), xph);
          tc_fence_after();
          const uint32_t xaddr = sbase + C::OFF_X + xs * C::X_STAGE_BYTES;
          tc_mma_ts_stage<KA / 16>(tmem_base + C::D_COL, tmem_base + C::A_COL + (uint32_t)as * (KA / 2),
                                   make_sw128_desc(xaddr), make_sw128_desc(xaddr + C::X_SUB_BYTES), idesc,
                                   kb != APS * sc.g0 ? 1u : 0u);
          tc_commit(x_empty(xs));
          tc_commit(a_empty(as));
          if (++xs == NSX) { xs = 0; xph ^= 1; }
          if (++as == NSA) { as = 0; aph ^= 1; }
        }
        tc_commit(d_full);
      }
    }
  } else if (warp >= kDequantWarp0) {
    // ===================== dequant + epilogue (thread = weight row = TMEM lane) =====
    const int q = (warp - kDequantWarp0) % 4;   // TMEM sub-partition (warp % 4)
    const int ch = (warp - kDequantWarp0) / 4;  // warp set: stages j = ch (mod R) of the CTA's sequence
    const int row = q * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const int sw = (row >> 1) & 3;  // SWIZZLE_64B: 16-byte chunk c of the row sits at c ^ ((row >> 1) & 3)
    uint32_t dph = 0;
    int j = 0;  // code-stage counter over the CTA's whole sequence (ring slot j % NSC, phase (j / NSC) & 1)
    // APS == 1: this set's next stage jn = ch, ch + R, ... and its code / A ring slots and phases
    static_assert(R < NSC && R < NSA, "one wrap per step");
    int jn = ch, cs_n = ch % NSC, sl_n = ch % NSA;
    uint32_t cph_n = (uint32_t)((ch / NSC) & 1), aph_n = (uint32_t)((ch / NSA) & 1);
    for (PSched sc(blockIdx.x, gridDim.x, G, num_tiles, sk, cta_q, cta_r); sc.valid(); sc.next()) {
      const int tile = sc.tile;
      const int n0 = (tile / m_tiles) * BM;
      const int m0 = (tile % m_tiles) * BT;
      // convert one A stage: code-ring slot cs (phase cph), A stage t of it, TMEM A slot (phase aph)
      auto convert = [&](int cs, uint32_t cph, int t, int slot, uint32_t aph) {
        mbar_wait(c_full(cs), cph);
        const uint32_t crow = sbase + C::OFF_C + cs * C_STAGE_BYTES + row * (kGroup / 2);
        constexpr int NCH = KA / 32;  // 16-byte chunks of the A stage in the row
        uint32_t words[KA / 8];
#pragma unroll
        for (int u = 0; u < NCH; ++u) {
          const uint4 v = lds128(crow + (((t * NCH + u) ^ sw) << 4));
          words[4 * u] = v.x; words[4 * u + 1] = v.y; words[4 * u + 2] = v.z; words[4 * u + 3] = v.w;
        }
        constexpr int NG = KA >= GS ? KA / GS : 1;  // quantization groups in the A stage
        constexpr int GSPAN = KA >= GS ? GS : KA;   // k of the A stage in each
        uint16_t sbits[NG];
        uint32_t zq[NG];  // Z (integer 0..15) from fp16 bits or a packed u4 nibble
#pragma unroll
        for (int h = 0; h < NG; ++h) {
          const int sub = (t * KA + h * GSPAN) / GS;
          sbits[h] = lds16(sbase + C::OFF_S + cs * SZ_BYTES + (sub * BM + row) * 2);
          if (zu4)
            zq[h] = (lds8(sbase + C::OFF_Z + cs * SZ_BYTES + sub * (BM / 2) + (row >> 1)) >> (4 * (row & 1))) & 0xFu;
          else
            zq[h] = (uint32_t)__half2int_rn(__ushort_as_half(lds16(sbase + C::OFF_Z + cs * SZ_BYTES + (sub * BM + row) * 2)));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(c_empty(cs));
        uint32_t zc[NG], d2[NG];
        float df[NG];
        bool sat = false;  // fp16 groups with Δ > 65504 / 15 take the saturating conversion
#pragma unroll
        for (int h = 0; h < NG; ++h) {
          const __half2 d2h = __half2half2(__ushort_as_half(sbits[h]));
          zc[h] = (0x6400u + zq[h]) * 0x00010001u;  // fp16x2(1024 + Z): ulp of 1024 is 1
          d2[h] = *reinterpret_cast<const uint32_t*>(&d2h);
          df[h] = __half2float(__ushort_as_half(sbits[h]));
          sat |= !kBF16 && df[h] > 4366.0f;
        }
        mbar_wait(a_empty(slot), aph ^ 1);
        tc_fence_after();
        // dequantize and store 64 k (32 TMEM columns) at a time
#pragma unroll
        for (int part = 0; part < KA / 64; ++part) {
          uint32_t a[32];
          if (sat) {
#pragma unroll
            for (int wd = 0; wd < 8; ++wd) {
              const int h = ((part * 8 + wd) * 8) / GSPAN;  // quantization group of this word
              dequant8<kBF16, true>(words[part * 8 + wd], zc[h], d2[h], df[h], &a[4 * wd]);
            }
          } else {
#pragma unroll
            for (int wd = 0; wd < 8; ++wd) {
              const int h = ((part * 8 + wd) * 8) / GSPAN;
              dequant8<kBF16>(words[part * 8 + wd], zc[h], d2[h], df[h], &a[4 * wd]);
            }
          }
          tmem_st_32x32b_x32(tmem_base + lane_addr + C::A_COL + (uint32_t)slot * (KA / 2) + (uint32_t)part * 32, a);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(a_full(slot));
      };
      const int jend = j + (sc.g1 - sc.g0);
      if constexpr (APS == 1) {
        // whole code stages, this set's every R-th one: running ring indices, no per-stage
        // division (the skip loop and its modulo were ~5 % of the kernel's instructions)
        for (; jn < jend; jn += R) {
          convert(cs_n, cph_n, 0, sl_n, aph_n);
          cs_n += R;
          if (cs_n >= NSC) { cs_n -= NSC; cph_n ^= 1u; }
          sl_n += R;
          if (sl_n >= NSA) { sl_n -= NSA; aph_n ^= 1u; }
        }
      } else {
        for (int jj = j; jj < jend; ++jj) {
          const int i = jj * APS + ch;  // A-stage counter
          convert(jj % NSC, (jj / NSC) & 1, ch, i % NSA, (i / NSA) & 1);
        }
      }
      j = jend;
      // ---- epilogue: D[row][token] -> Y[m0 + token][n0 + row]
      pdl_wait();  // (returns at once after the first tile) Y may be read by the previous kernel
      mbar_wait(d_full, dph);
      dph ^= 1;
      tc_fence_after();
      const int n = n0 + row;
      const int mt = min(BT, M - m0);
      auto to_out = [](float f) -> uint16_t {
        return kBF16 ? __bfloat16_as_ushort(__float2bfloat16_rn(f)) : __half_as_ushort(__float2half_rn(f));
      };
      const bool full = sc.g0 == 0 && sc.g1 == G;
      // stream-K partial tile: fp32 [token][row] slot of this CTA (0: first segment, 1: last)
      float* slot = partials + ((size_t)blockIdx.x * 2 + (sc.first ? 0 : 1)) * (BT * BM);
      // warps sharing a lane quarter take alternating 16-token column blocks
      for (int c0 = ch * 16; c0 < mt; c0 += 16 * R) {
        uint32_t v[16];
        tmem_ld_32x32b_x16(tmem_base + lane_addr + C::D_COL + (uint32_t)c0, v);
        tmem_ld_wait();
        if (full) {
          if (n < N) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (c0 + i < mt) Y[(size_t)(m0 + c0 + i) * N + n] = to_out(__uint_as_float(v[i]));
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (c0 + i < mt) __stcg(slot + (c0 + i) * BM + row, __uint_as_float(v[i]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(d_empty);  // the accumulator is free for the next segment
      if (!full) {
        // fixup, overlapping the next segment's MMAs: the dequant warps' partial stores are
        // published by one acq_rel atomic after a barrier among them
        int* flag = reinterpret_cast<int*>(smem + C::OFF_TMEM + 8);
        asm volatile("bar.sync 1, %0;\n" ::"n"(DQW * 32) : "memory");
        const int c_lo = sc.cta_of(tile * G), c_hi = sc.cta_of(tile * G + G - 1);
        if (threadIdx.x == kDequantWarp0 * 32) {
          int prev;
          asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;\n"
                       : "=r"(prev) : "l"(counters + tile) : "memory");
          *flag = prev == c_hi - c_lo;
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(DQW * 32) : "memory");
        if (*flag) {
          if (n < N) {
            for (int c0 = ch * 16; c0 < mt; c0 += 16 * R) {
              float acc[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) acc[i] = 0.0f;
              for (int cc = c_lo; cc <= c_hi; ++cc) {
                const int e = (sc.start(cc) / G == tile) ? 0 : 1;
                const float* src = partials + ((size_t)cc * 2 + e) * (BT * BM) + row;
                float pv[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) pv[i] = (c0 + i < mt) ? __ldcg(src + (c0 + i) * BM) : 0.0f;
#pragma unroll
                for (int i = 0; i < 16; ++i) acc[i] += pv[i];
              }
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (c0 + i < mt) Y[(size_t)(m0 + c0 + i) * N + n] = to_out(acc[i]);
            }
          }
          if (threadIdx.x == kDequantWarp0 * 32) counters[tile] = 0;  // leave the workspace zeroed
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(DQW * 32) : "memory");  // flag reuse
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base),
                 "r"(C::TMEM_COLS));
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool encode_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t inner,
               uint64_t outer, uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
               CUtensorMapSwizzle sw) {
  auto fn = get_encode();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

size_t prefill_partials_bytes() { return (size_t)num_sms() * 2 * kBTMax * BM * sizeof(float); }

// Token-tile width: the narrowest configuration that holds M in one tile, else 256.
static int prefill_bt(int64_t M) { return M <= 64 ? 64 : M <= 128 ? 128 : kBTMax; }
static int64_t prefill_tiles(int64_t M, int64_t N) {
  const int64_t bt = prefill_bt(M);
  return ((N + BM - 1) / BM) * ((M + bt - 1) / bt);
}
static int64_t prefill_stages(int64_t, int64_t K) { return K / kGroup; }  // schedule units per tile

// Stream-K over (tile x code stage) units when whole tiles would leave > 5 % of the last
// wave idle at mid M (one token tile), or > 10 % on a long-K shape at large M (down_proj at
// M = 2048).  Elsewhere the CTAs sweeping k in lockstep share X and W tiles in L2, which
// stream-K's staggered ranges give up (measured: o_proj/qkv at M = 2048 are faster without).
bool prefill_streamk(int64_t M, int64_t N, int64_t K) {
  const int64_t tiles = prefill_tiles(M, N);
  const int64_t P = num_sms();
  const int64_t waves = (tiles + P - 1) / P;
  const double eff = (double)tiles / (double)(waves * P);
  if (tiles * prefill_stages(M, K) < P) return false;
  return M <= kBTMax ? eff < 0.95 : (eff < 0.9 && K >= 16384);
}

size_t prefill_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  if (!prefill_streamk(M, N, K)) return 0;
  return ws_partials_bytes() + counter_region_bytes(prefill_tiles(M, N));
}

namespace {
template <bool kBF16, int kBT, int kR>
auto pick_kernel(int group) {
  return group == 32 ? prefill_kernel<kBF16, 32, kBT, kR>
                     : group == 64 ? prefill_kernel<kBF16, 64, kBT, kR> : prefill_kernel<kBF16, 128, kBT, kR>;
}

template <int kBT, int kR = (kBT == kBTMax ? 2 : 3)>
cudaError_t launch_bt(const void* X, int x_dtype, const uint8_t* Wq, const uint16_t* scales, const void* zeros,
                      void* Y, int M, int N, int K, int group, void* ws, bool weights_static, bool zu4,
                      cudaStream_t st, const char** why) {
  using C = PCfg<kBT, kR>;
  alignas(64) CUtensorMap tm_x, tm_w, tm_s, tm_z;
  const int G = (int)prefill_stages(M, K);
  // X box: 64 k (one SWIZZLE_128B row) of only as many token rows as the problem has (OOB
  // rows would still cross the crossbar as zero fill)
  const int x_rows = std::min(kBT, (M + 15) / 16 * 16);
  bool ok = encode_2d(&tm_x, CU_TENSOR_MAP_DATA_TYPE_UINT16, X, (uint64_t)K, (uint64_t)M,
                      (uint64_t)K * 2, 64, x_rows, CU_TENSOR_MAP_SWIZZLE_128B);
  ok = ok && encode_2d(&tm_w, CU_TENSOR_MAP_DATA_TYPE_UINT8, Wq, (uint64_t)K / 2, (uint64_t)N,
                       (uint64_t)K / 2, kGroup / 2, BM, CU_TENSOR_MAP_SWIZZLE_64B);
  const int sub = kGroup / group;  // scale / zero rows per 128 k
  const int subs = sub;
  ok = ok && encode_2d(&tm_s, CU_TENSOR_MAP_DATA_TYPE_UINT16, scales, (uint64_t)N, (uint64_t)(K / kGroup) * sub,
                       (uint64_t)N * 2, BM, subs, CU_TENSOR_MAP_SWIZZLE_NONE);
  ok = ok && (zu4 ? encode_2d(&tm_z, CU_TENSOR_MAP_DATA_TYPE_UINT8, zeros, (uint64_t)N / 2,
                              (uint64_t)(K / kGroup) * sub, (uint64_t)N / 2, BM / 2, subs, CU_TENSOR_MAP_SWIZZLE_NONE)
                  : encode_2d(&tm_z, CU_TENSOR_MAP_DATA_TYPE_UINT16, zeros, (uint64_t)N, (uint64_t)(K / kGroup) * sub,
                              (uint64_t)N * 2, BM, subs, CU_TENSOR_MAP_SWIZZLE_NONE));
  if (!ok) {
    *why = "cuTensorMapEncodeTiled failed";
    return cudaErrorInvalidValue;
  }
  const int num_tiles = (int)prefill_tiles(M, N);
  const bool sk = prefill_streamk(M, N, K);
  const int units = num_tiles * G;
  const int grid = sk ? std::min(units, num_sms()) : std::min(num_tiles, num_sms());
  const int cta_q = units / grid, cta_r = units % grid;
  float* partials = reinterpret_cast<float*>(ws);
  int* counters = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(ws) + ws_partials_bytes());
  auto kern = x_dtype == SQ_BF16 ? pick_kernel<true, kBT, kR>(group) : pick_kernel<false, kBT, kR>(group);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_ALLOC);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid, 1, 1);
  cfg.blockDim = dim3(C::THREADS, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM_ALLOC;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = option(SQ_OPT_PDL) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int early = option(SQ_OPT_PDL) && weights_static;
  e = cudaLaunchKernelEx(&cfg, kern, tm_x, tm_w, tm_s, tm_z, (uint16_t*)Y, M, N, K, early,
                         x_rows * C::KA * 2, sk ? 1 : 0, cta_q, cta_r, partials, counters, zu4 ? 1 : 0);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_prefill(const void* X, int x_dtype, const uint8_t* Wq, const uint16_t* scales,
                           const void* zeros, void* Y, int M, int N, int K, int group, void* ws, size_t,
                           bool weights_static, bool zu4, cudaStream_t st, const char** why) {
  switch (prefill_bt(M)) {
    case 64:
      if (M > 48)  // four dequant warp sets when the 64-token tile is > 3/4 full (PCfg)
        return launch_bt<64, 4>(X, x_dtype, Wq, scales, zeros, Y, M, N, K, group, ws, weights_static, zu4, st, why);
      return launch_bt<64>(X, x_dtype, Wq, scales, zeros, Y, M, N, K, group, ws, weights_static, zu4, st, why);
    case 128:
      if (M > 96)  // four dequant warp sets when the 128-token tile is > 3/4 full (PCfg)
        return launch_bt<128, 4>(X, x_dtype, Wq, scales, zeros, Y, M, N, K, group, ws, weights_static, zu4, st, why);
      return launch_bt<128>(X, x_dtype, Wq, scales, zeros, Y, M, N, K, group, ws, weights_static, zu4, st, why);
    default:
      return launch_bt<kBTMax>(X, x_dtype, Wq, scales, zeros, Y, M, N, K, group, ws, weights_static, zu4, st, why);
  }
}

}  // namespace sq

