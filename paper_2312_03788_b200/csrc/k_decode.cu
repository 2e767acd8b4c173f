// K-dec: W4A16 GEMM for small M (decode, M <= 16) -- HBM-bound.
//
//   Y[m][n] = sum_gi Δ[gi][n] * sum_{k in gi} X[m][k] * (q[n][k] - Z[gi][n])
//   PAPER.md:104-106 Eq. 3 with Ŵ of Eq. 1 line 2; fp32 accumulation.
//
// Design:
//  * Persistent kernel, one wave of resident CTAs.  The weight matrix is cut into
//    units of (BN-row block x 4 groups).  Two schedules (SQ_OPT_DECODE_SCHEDULE):
//    stream-K (equal contiguous unit ranges per CTA; a row block cut between CTAs is
//    finished by a deterministic fixup: the last contributor sums the fp32 partials
//    in CTA order) and row-block (whole 32- or 64-row blocks per CTA, no fixup),
//    chosen per shape by wave quantization.
//  * One producer warp streams each unit with TMA into an SMEM ring: packed codes
//    (3-D box 64 B x BN rows x 4 groups), the scale/zero rows and the matching X
//    slice (4-D box, SWIZZLE_128B so the fragment reads are bank-conflict free).  At M = 1
//    the box stages the one real token row (the MMA's other seven B columns are zeros
//    supplied in registers), so a stage is 17.5 KB instead of 24.5 KB.
//  * Four consumer warps: warp w takes group w of every stage for all BN rows, so
//    its X fragment is loaded (and k-permuted with PRMT) once and reused BN/16
//    times.  Codes are turned into the EXACT integer (q - Z) in fp16/bf16 with the
//    lop3 magic-number trick and fed to mma.sync.m16n8k16 with fp32 accumulation;
//    Δ is applied once per group to the accumulator fragment.
//  * At the end of a row-block segment the consumer warps park their fp32 partial
//    sums in SMEM (over their own, already consumed, activation slice of the stage)
//    and go on; a sixth warp (epilogue) sums the four in fixed order, hands the stage
//    back to the producer and does the global work (Y store or stream-K fixup) off
//    the consumers' critical path.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "decode_common.cuh"
#include "sq_internal.cuh"

namespace sq {

namespace {

using namespace dec;

constexpr int kGroup = 128;
constexpr int GPS = 4;             // groups per stage (unit)
constexpr int kConsumerWarps = 4;  // one per group of a stage; warp roles: consumers 0..3, TMA producer 4, epilogue 5
constexpr int kCtasPerSm = 2;      // M >= 2 (and M = 1 outside the 3-CTA rule): two ~112-KB CTAs per SM
// M = 1: three 74-KB CTAs per SM for 32-48 MB layers with K < 8192 that two CTAs would stream-K
// (7B gate|up -12 %; profiles/decode_m1_ct3_ab_r01.jsonl); larger / longer-K layers take two CTAs
// with 128-row blocks (launch_m)
constexpr int kMaxCtasPerSm = 3;   // workspace partial slots are sized for the most CTAs a launch can have
constexpr int kMaxBN = 64;         // row-block heights: 32 or 64 (128 at M = 1, within the same partial slots)
constexpr int kMinBN = 32;
// try_wait suspend-time hint of the producer / epilogue waits (ns)
constexpr uint32_t kIdleWaitNs = 100000;

// MT: 8-token MMA n-tiles; XR: token rows of the activation box actually staged (M = 1 stages
// one row, the MMA sees zeros for the other seven); CT: resident CTAs per SM (smem budget);
// GS: quantization group size (128, or 64 / 32: "different group sizes")
template <int MT, int BN, int XR, int CT, int GS = 128>
struct Cfg {
  static constexpr int SUB = kGroup / GS;                 // groups per 128-k slot
  static constexpr int MPAD = 8 * MT;
  static constexpr int CW = kConsumerWarps;
  static constexpr int THREADS = (CW + 2) * 32;
  static_assert(CT == 2 || CT == 3, "two or three CTAs per SM");
  static constexpr int kSmemBudget = (CT == 2 ? 112 : 74) * 1024;  // per CTA
  static constexpr int RT = BN / 16;                      // 16-row tiles per consumer warp
  static constexpr int CODES = GPS * BN * (kGroup / 2);  // 16 KB at BN = 64
  static constexpr int XB = GPS * XR * kGroup * 2;        // 1 / 8 / 16 KB
  static constexpr int SZ = GPS * SUB * BN * 2;           // Δ (or Z) rows of the stage: [slot][sub][row]
  // stage bases stay 1024-B aligned (SWIZZLE_128B destination of the X box)
  static constexpr int TX = CODES + XB + 2 * SZ;  // bytes the TMA delivers per stage
  static constexpr int STAGE = (TX + 1023) / 1024 * 1024;
  static constexpr int NS = std::min(8, (kSmemBudget - 1024 - 256) / STAGE);
  // At a segment end each consumer warp parks its fp32 partial sums (MPAD x BN) over its
  // own group's activation slice of the stage, which only that warp reads.
  static constexpr int XSLICE = XB / GPS;
  // partial sums are parked over the group's activation slice, or over its codes slab when
  // the slice is too small (M = 1 stages one token row); both were fully read before the park
  static constexpr bool kParkCodes = XR * BN * 4 > XSLICE;
  static constexpr int PARK_OFF = kParkCodes ? 0 : CODES;
  static constexpr int PARK_STRIDE = kParkCodes ? BN * 64 : XSLICE;
  static_assert(XR * BN * 4 <= PARK_STRIDE, "partial-sum slot must fit");
  static_assert(XR * BN >= 32, "epilogue lanes");
  static_assert(XR * BN <= 16 * kMaxBN, "stream-K partial slot (16 x kMaxBN fp32) must hold a row block");
  static constexpr int OFF_BAR = NS * STAGE;  // full[NS], empty[NS], red_full[NS]
  static constexpr int SMEM = OFF_BAR + 3 * NS * 8;
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
__device__ __forceinline__ void mbar_arrive_cnt(uint32_t bar, uint32_t cnt) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(cnt) : "memory");
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
// Same, for warps that wait long (producer, epilogue): the suspend-time hint lets the
// hardware park the warp until the phase completes instead of re-polling, so the
// wait loop does not take issue slots from the consumer warps on the same SMSP.
__device__ __forceinline__ void mbar_wait_idle(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity), "r"(kIdleWaitNs)
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
// weights are streamed exactly once: load them with an L2 evict-first policy so they do
// not push the activations / partials (re-read across CTAs and kernels) out of L2
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_3d_hint(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1, int c2,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;\n"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "l"(policy) : "memory");
}
__device__ __forceinline__ void tma_4d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];\n"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
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

// h[i] (exact (q - Z) pairs) <- RN((q - Z) Δ) in the activation format, Δ = fp16 bits.
// fp16: one HMUL2 per pair; a Δ above 65504 / 15 could overflow, so such a (row, group) --
// impossible for real weights -- takes the fp32 product clamped to ±65504.
template <bool kBF16>
__device__ __forceinline__ void scale_pairs(uint32_t (&h)[4], uint16_t dbits) {
  const float df = __half2float(__ushort_as_half(dbits));
  if (kBF16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&h[i]));
      const __nv_bfloat162 b = __floats2bfloat162_rn(f.x * df, f.y * df);  // exact product, one RN
      h[i] = *reinterpret_cast<const uint32_t*>(&b);
    }
  } else if (df > 4366.0f) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&h[i]));
      const __half2 r = __floats2half2_rn(fminf(fmaxf(f.x * df, -65504.0f), 65504.0f),
                                          fminf(fmaxf(f.y * df, -65504.0f), 65504.0f));
      h[i] = *reinterpret_cast<const uint32_t*>(&r);
    }
  } else {
    const __half2 d2 = __half2half2(__ushort_as_half(dbits));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __half2 r = __hmul2(*reinterpret_cast<const __half2*>(&h[i]), d2);
      h[i] = *reinterpret_cast<const uint32_t*>(&r);
    }
  }
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// Row-parallel all-reduce fused into the epilogue (sq_w4a16_gemm_allreduce; the buffer
// layout and protocol are those of k_allreduce.cu: header, flags[2][world][kArMaxChunks],
// slots[2][world][n_max] with a 4-byte slot stride; here a "chunk" is a row block).
// world == 0: off.  fp16 partials travel as fp16, bf16 partials as fp32 (SURVEY.md §8(e):
// reduce bf16 in fp32), and the rank-ordered sum is always taken in fp32.
__device__ __forceinline__ uint32_t* ar_flags(uint8_t* base, int world, int par) {
  return reinterpret_cast<uint32_t*>(base + ar_flags_offset()) + (size_t)par * world * kArMaxChunks;
}
__device__ __forceinline__ uint8_t* ar_slot(uint8_t* base, int world, int par, int q, int64_t n_max) {
  return base + ar_slot_offset(world, par, q, n_max);
}
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

template <int MT, bool kBF16, int BN, int XR, int CT, bool kAR, int GS>
__global__ void __launch_bounds__(Cfg<MT, BN, XR, CT, GS>::THREADS, CT)
decode_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
              const __grid_constant__ CUtensorMap tm_s, const __grid_constant__ CUtensorMap tm_z,
              uint16_t* __restrict__ Y, int* __restrict__ counters, float* __restrict__ partials,
              int M, int N, Work wk, int early_weights, int zu4, const ArParams ar) {
  using C = Cfg<MT, BN, XR, CT, GS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_full = sbase + C::OFF_BAR;
  const uint32_t bar_empty = bar_full + 8 * C::NS;
  const uint32_t red_full = bar_empty + 8 * C::NS;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int c = blockIdx.x, P = gridDim.x;
  // bytes the TMA delivers per stage: packed u4 zero rows (SQ_ZEROS_U4) are a quarter of
  // the fp16 ones; they land at the start of the same zero-row region, [slot][sub][BN / 2]
  const uint32_t tx = zu4 ? (uint32_t)(C::TX - C::SZ + C::SZ / 4) : (uint32_t)C::TX;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NS; ++i) {
      mbar_init(bar_full + 8 * i, 1);
      mbar_init(bar_empty + 8 * i, C::CW);
      mbar_init(red_full + 8 * i, C::CW * 32);  // every consumer lane arrives after its parked writes
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // the next kernel in the stream may start its prologue as our CTAs retire
  pdl_launch_dependents();

  if (warp == C::CW) {  // producer
    // ===================== TMA producer =====================
    if (lane == 0) {
      prefetch_tmap(&tm_w);
      prefetch_tmap(&tm_x);
      prefetch_tmap(&tm_s);
      prefetch_tmap(&tm_z);
      // codes are streamed exactly once: L2 evict-first keeps the activations and the
      // stream-K partials resident (0.3-2 %, profiles/decode_evict_first_ab_r01.jsonl)
      const uint64_t wpol = l2_evict_first_policy();
      auto load_weights = [&](uint32_t st, uint32_t fb, int u) {
        const int rb = u / wk.upb, g0 = (u % wk.upb) * GPS;
        tma_3d_hint(st, &tm_w, fb, 0, rb * BN, g0, wpol);
        tma_2d(st + C::CODES + C::XB, &tm_s, fb, rb * BN, g0 * C::SUB);
        tma_2d(st + C::CODES + C::XB + C::SZ, &tm_z, fb, zu4 ? rb * (BN / 2) : rb * BN, g0 * C::SUB);
      };
      // Weights (codes, Δ, Z) never depend on the previous kernel when the caller
      // declared them static (SQ_GEMM_WEIGHTS_STATIC): stream the first stages before
      // waiting on it.
      int pre = 0;
      if (early_weights) {
        Sched sc(wk, c, P);
        for (; pre < C::NS && sc.valid(); ++pre, sc.next(wk)) {
          const uint32_t fb = bar_full + 8 * pre;
          mbar_expect_tx(fb, tx);
          load_weights(sbase + pre * C::STAGE, fb, sc.u);
        }
      }
      pdl_wait();  // X (and everything after) may be the previous kernel's output
      int s = 0;
      uint32_t ph = 0;
      int i = 0;
      for (Sched sc(wk, c, P); sc.valid(); sc.next(wk), ++i) {
        const uint32_t st = sbase + s * C::STAGE;
        const uint32_t fb = bar_full + 8 * s;
        if (i >= pre) {
          mbar_wait_idle(bar_empty + 8 * s, ph ^ 1);
          mbar_expect_tx(fb, tx);
          load_weights(st, fb, sc.u);
        }
        tma_4d(st + C::CODES, &tm_x, fb, 0, 0, 0, (sc.u % wk.upb) * GPS);
        if (++s == C::NS) { s = 0; ph ^= 1; }
      }
    }
    return;
  }

  auto to_out = [](float v) -> uint16_t {
    if (kBF16) return __bfloat16_as_ushort(__float2bfloat16_rn(v));
    return __half_as_ushort(__float2half_rn(v));
  };

  if (warp == C::CW + 1) {  // epilogue
    // ===================== epilogue: one warp, off the consumers' critical path =====================
    // Walks the same schedule as the consumers.  At each segment end it sums the four
    // warps' parked partials (fixed warp order), hands the stage back to the producer,
    // then writes Y (whole row block) or runs the stream-K fixup (partial row block).
    constexpr int E = XR * BN / 32;  // elements per lane
    int s = 0;
    uint32_t redph = 0;                   // phase bit per stage
    bool waited = false;
    // fused all-reduce: this CTA's finalized row blocks are pushed to every rank as they
    // complete and reduced after the CTA has pushed all of them (waiting only at the end
    // keeps the cross-GPU waits acyclic)
    __shared__ int fin_list[64];
    int n_fin = 0;
    uint32_t epoch = ar.epoch;
    if (kAR && epoch == 0) {
      // the device-managed epoch is advanced by the previous call's last CTA: read it only
      // after that grid has completed (PDL lets this kernel start while it still runs)
      pdl_wait();
      waited = true;
      const uint32_t cur = *reinterpret_cast<volatile uint32_t*>(ar.peers[ar.rank]);
      epoch = cur == 0xFFFFFFFFu ? 2u : cur + 1u;
    }
    const int par = epoch & 1;
    auto emit = [&](int rb, const float (&val)[E]) {  // final values of row block rb
      const int n0 = rb * BN;
      if constexpr (!kAR) {
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int idx = lane + 32 * i, t = idx / BN, row = idx % BN;
          if (t < M && n0 + row < N) Y[(size_t)t * N + n0 + row] = to_out(val[i]);
        }
        return;
      } else {
        for (int p = 0; p < ar.world; ++p) {
          uint8_t* dst = ar_slot(ar.peers[p], ar.world, par, ar.rank, ar.n_max);
#pragma unroll
          for (int i = 0; i < E; ++i) {
            const int idx = lane + 32 * i, t = idx / BN, row = idx % BN;
            if (t < M && n0 + row < N) {
              const size_t o = (size_t)t * N + n0 + row;
              if (kBF16)
                reinterpret_cast<float*>(dst)[o] = val[i];
              else
                reinterpret_cast<uint16_t*>(dst)[o] = to_out(val[i]);
            }
          }
        }
        __threadfence_system();
        __syncwarp();
        if (lane < ar.world) {
          uint32_t* f = ar_flags(ar.peers[lane], ar.world, par) + (size_t)ar.rank * kArMaxChunks + rb;
          asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(f), "r"(epoch) : "memory");
        }
        if (n_fin < 64) {
          if (lane == 0) fin_list[n_fin] = rb;
        } else if (lane == 0) {
          atomicExch(ar.err, 2);  // more finalized row blocks than the list holds
        }
        ++n_fin;
        __syncwarp();
      }
    };
    for (Sched sc(wk, c, P); sc.valid(); sc.next(wk)) {
      const int rb = sc.u / wk.upb;
      if (sc.range_last()) {
        mbar_wait_idle(red_full + 8 * s, (redph >> s) & 1u);
        redph ^= 1u << s;
        const float* sl = reinterpret_cast<const float*>(smem + s * C::STAGE + C::PARK_OFF);
        constexpr int W = C::PARK_STRIDE / 4;  // floats per group slot
        float v[E];
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int idx = lane + 32 * i;
          v[i] = ((sl[idx] + sl[W + idx]) + sl[2 * W + idx]) + sl[3 * W + idx];
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive_cnt(bar_empty + 8 * s, C::CW);  // stage back to the producer
        if (!waited) {  // global accesses below must follow the previous kernel (PDL)
          pdl_wait();
          waited = true;
        }
        if (sc.full) {
          emit(rb, v);
        } else {
          // stream-K fixup: park the partial; the last contributor sums them in CTA order
          float* slot = partials + ((size_t)c * 2 + sc.e) * (16 * kMaxBN);
#pragma unroll
          for (int i = 0; i < E; ++i) {
            const int idx = lane + 32 * i;
            if (idx < M * BN) __stcg(slot + idx, v[i]);
          }
          __syncwarp();
          const int c0 = wk.cta_of(rb * wk.upb), c1 = wk.cta_of((rb + 1) * wk.upb - 1);
          int last = 0;
          if (lane == 0) {
            // acq_rel: publishes this warp's partial (ordered by __syncwarp) and, for the
            // last contributor, makes the others' partials visible to the loads below
            int prev;
            asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;\n"
                         : "=r"(prev) : "l"(counters + rb) : "memory");
            last = prev == c1 - c0;
          }
          if (__shfl_sync(0xffffffffu, last, 0)) {
            // sum in fixed CTA order; each CTA's E loads are independent (one L2 round trip per CTA)
            float tot[E];
#pragma unroll
            for (int i = 0; i < E; ++i) tot[i] = 0.0f;
            for (int cc = c0; cc <= c1; ++cc) {
              const int e = (wk.start(cc) / wk.upb == rb) ? 0 : 1;
              const float* src = partials + ((size_t)cc * 2 + e) * (16 * kMaxBN);
              float part[E];
#pragma unroll
              for (int i = 0; i < E; ++i) {
                const int idx = lane + 32 * i;
                part[i] = idx < M * BN ? __ldcg(src + idx) : 0.0f;
              }
#pragma unroll
              for (int i = 0; i < E; ++i) tot[i] += part[i];
            }
            emit(rb, tot);
            if (lane == 0) counters[rb] = 0;  // leave the workspace zeroed
          }
        }
      }
      if (++s == C::NS) s = 0;
    }
    if (kAR) {
      // reduce the row blocks this CTA finalized: wait for every rank's copy (bounded),
      // sum in rank order in fp32 (bit-identical Y on every rank), store
      const int nf = n_fin < 64 ? n_fin : 64;
      bool timed_out = false;
      for (int f = 0; f < nf && !timed_out; ++f) {
        const int rb = fin_list[f], n0 = rb * BN;
        if (lane < ar.world) {
          const uint32_t* fl = ar_flags(ar.peers[ar.rank], ar.world, par) + (size_t)lane * kArMaxChunks + rb;
          uint32_t v, polls = 0;
          while (true) {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(fl) : "memory");
            if (v == epoch) break;
            if (++polls > (1u << 24)) {
              atomicExch(ar.err, 1);
              break;
            }
            if (polls > 64) __nanosleep(polls > 4096 ? 1000 : 64);
          }
          if (v != epoch) timed_out = true;
        }
        timed_out = __any_sync(0xffffffffu, timed_out);
        if (timed_out) break;
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int idx = lane + 32 * i, t = idx / BN, row = idx % BN;
          if (t < M && n0 + row < N) {
            const size_t o = (size_t)t * N + n0 + row;
            float acc = 0.0f;
            for (int q = 0; q < ar.world; ++q) {
              const uint8_t* src = ar_slot(ar.peers[ar.rank], ar.world, par, q, ar.n_max);
              if (kBF16)
                acc += __ldcv(reinterpret_cast<const float*>(src) + o);
              else
                acc += __half2float(__ushort_as_half(__ldcv(reinterpret_cast<const uint16_t*>(src) + o)));
            }
            Y[o] = to_out(acc);
          }
        }
      }
      // the last CTA to finish advances the device-managed epoch (also after a timeout, so
      // the header stays consistent; the error word reports the failure)
      if (ar.epoch == 0 && lane == 0) {
        uint32_t* hdr = reinterpret_cast<uint32_t*>(ar.peers[ar.rank]);
        __threadfence();
        if (atomicAdd(hdr + 1, 1u) == gridDim.x - 1) {
          hdr[1] = 0;
          __threadfence();
          *reinterpret_cast<volatile uint32_t*>(hdr) = epoch;
        }
      }
    }
    return;
  }

  // ===== consumers: warp w = group w of each stage, all BN rows =====
  const int r = lane / 4, j = lane % 4;
  const int grp = warp;
  float acc[C::RT][MT][4];
#pragma unroll
  for (int rt = 0; rt < C::RT; ++rt)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[rt][mt][i] = 0.0f;

  int s = 0;
  uint32_t ph = 0;
  for (Sched sc(wk, c, P); sc.valid(); sc.next(wk)) {
    mbar_wait(bar_full + 8 * s, ph);
    const uint32_t st = sbase + s * C::STAGE;
    // ---- X fragments of this warp's group: token t = r + 8 mt, k = 32 j + [0, 32)
    uint32_t xb[MT][4][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int t = r + 8 * mt;
      const int R = (grp * XR + t) * 2 + (j >> 1);  // 128-byte row of the swizzled box
      const uint32_t rowaddr = st + C::CODES + R * 128;
      uint32_t xv[16];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (XR >= C::MPAD || t < XR) v = lds128(rowaddr + ((((j & 1) * 4 + i) ^ (R & 7)) << 4));
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
    // codes of this warp's group: [group][row][64 B]
    const uint32_t cbase = st + grp * (BN * 64) + r * 64 + j * 16;
    const uint32_t sbs = st + C::CODES + C::XB + grp * (BN * 2) + r * 2;
    // this warp's group row of the zero region (fp16: BN x 2 B per group, u4: BN / 2 B)
    const uint32_t zrow = st + C::CODES + C::XB + C::SZ + grp * (zu4 ? BN / 2 : BN * 2);
    if constexpr (GS < kGroup) {
      // groups of 64 / 32 k: one MMA's 16 k span the four lanes' 32-k ranges, i.e. up to
      // four groups, so Δ cannot be applied to the fp32 sum; the operand is the rounded
      // Ŵ = RN((q - Z) Δ) instead (the value the prefill path feeds its MMA, P13) and the
      // MMA accumulates Ŵ·X directly.  Lane j's k range lies in group (32 j) / GS.
      const uint32_t sbg = st + C::CODES + C::XB + ((grp * C::SUB + (32 * j) / GS) * BN + r) * 2;
      const uint32_t zrow_g = st + C::CODES + C::XB + C::SZ + (grp * C::SUB + (32 * j) / GS) * (zu4 ? BN / 2 : BN * 2);
#pragma unroll
      for (int rt = 0; rt < C::RT; ++rt) {
        const uint4 ca = lds128(cbase + rt * 16 * 64);
        const uint4 cb = lds128(cbase + (rt * 16 + 8) * 64);
        const uint16_t dA = lds16(sbg + rt * 32), dB = lds16(sbg + rt * 32 + 16);
        uint32_t zsA, zfA, zsB, zfB;
        zero_consts_q<kBF16>(load_zero(zrow_g, rt * 16 + r, zu4), zsA, zfA);
        zero_consts_q<kBF16>(load_zero(zrow_g, rt * 16 + r + 8, zu4), zsB, zfB);
        const uint32_t wa[4] = {ca.x, ca.y, ca.z, ca.w};
        const uint32_t wb[4] = {cb.x, cb.y, cb.z, cb.w};
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          uint32_t hA[4], hB[4];
          dequant_word<kBF16>(wa[w], zsA, zfA, hA);
          dequant_word<kBF16>(wb[w], zsB, zfB, hB);
          scale_pairs<kBF16>(hA, dA);
          scale_pairs<kBF16>(hB, dB);
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            mma_16816(acc[rt][mt], hA[0], hB[0], hA[1], hB[1], xb[mt][w][0], xb[mt][w][1], kBF16);
            mma_16816(acc[rt][mt], hA[2], hB[2], hA[3], hB[3], xb[mt][w][2], xb[mt][w][3], kBF16);
          }
        }
      }
    } else
#pragma unroll
    for (int rt = 0; rt < C::RT; ++rt) {
      const uint4 ca = lds128(cbase + rt * 16 * 64);
      const uint4 cb = lds128(cbase + (rt * 16 + 8) * 64);
      const float dA = __half2float(__ushort_as_half(lds16(sbs + rt * 32)));
      const float dB = __half2float(__ushort_as_half(lds16(sbs + rt * 32 + 16)));
      const uint32_t wa[4] = {ca.x, ca.y, ca.z, ca.w};
      const uint32_t wb[4] = {cb.x, cb.y, cb.z, cb.w};
      uint32_t zsA, zfA, zsB, zfB;
      zero_consts_q<kBF16>(load_zero(zrow, rt * 16 + r, zu4), zsA, zfA);
      zero_consts_q<kBF16>(load_zero(zrow, rt * 16 + r + 8, zu4), zsB, zfB);
      float g[MT][4];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        uint32_t hA[4], hB[4];
        dequant_word<kBF16>(wa[w], zsA, zfA, hA);
        dequant_word<kBF16>(wb[w], zsB, zfB, hB);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          // A = rows (r, r+8) x k pairs; B = the same k pairs of this lane's token
          if (w == 0)
            mma_16816_zc(g[mt], hA[0], hB[0], hA[1], hB[1], xb[mt][w][0], xb[mt][w][1], kBF16);
          else
            mma_16816(g[mt], hA[0], hB[0], hA[1], hB[1], xb[mt][w][0], xb[mt][w][1], kBF16);
          mma_16816(g[mt], hA[2], hB[2], hA[3], hB[3], xb[mt][w][2], xb[mt][w][3], kBF16);
        }
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        acc[rt][mt][0] = fmaf(g[mt][0], dA, acc[rt][mt][0]);
        acc[rt][mt][1] = fmaf(g[mt][1], dA, acc[rt][mt][1]);
        acc[rt][mt][2] = fmaf(g[mt][2], dB, acc[rt][mt][2]);
        acc[rt][mt][3] = fmaf(g[mt][3], dB, acc[rt][mt][3]);
      }
    }

    // ---- end of a row-block segment?
    const bool seg_end = sc.range_last();
    __syncwarp();
    if (!seg_end) {
      if (lane == 0) mbar_arrive(bar_empty + 8 * s);
    } else {
      // park this warp's partial sums over its own activation slice of the stage and hand
      // them to the epilogue warp, which also releases the stage; no CTA-wide barrier
      float* slot = reinterpret_cast<float*>(smem + s * C::STAGE + C::PARK_OFF + grp * C::PARK_STRIDE);
#pragma unroll
      for (int rt = 0; rt < C::RT; ++rt)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int t0 = 8 * mt + 2 * j, ra = rt * 16 + r;
          if (XR >= C::MPAD || t0 < XR) {
            slot[t0 * BN + ra] = acc[rt][mt][0];
            slot[t0 * BN + ra + 8] = acc[rt][mt][2];
          }
          if (XR >= C::MPAD || t0 + 1 < XR) {
            slot[(t0 + 1) * BN + ra] = acc[rt][mt][1];
            slot[(t0 + 1) * BN + ra + 8] = acc[rt][mt][3];
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[rt][mt][i] = 0.0f;
        }
      // the stage is refilled by TMA (async proxy) after the epilogue releases it: order
      // these generic-proxy writes before that.  Every lane arrives (release) after its own
      // writes, so the epilogue's acquire covers all of them directly.
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_arrive(red_full + 8 * s);
    }
    if (++s == C::NS) { s = 0; ph ^= 1; }
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

// Resident CTAs per SM of one kernel instance (occupancy query), cached per device: the
// dynamic-smem attribute is per device context, so it is set on each device before use.
template <int MT, bool kBF16, int BN, int XR, int CT, int GS>
int ctas_per_sm() {
  static int cached[64];
  static std::once_flag once[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  std::call_once(once[dev], [] {
    int d = 0, n = 0;
    cudaGetDevice(&d);
    using C = Cfg<MT, BN, XR, CT, GS>;
    cudaFuncSetAttribute(decode_kernel<MT, kBF16, BN, XR, CT, false, GS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         C::SMEM_ALLOC);
    cudaFuncSetAttribute(decode_kernel<MT, kBF16, BN, XR, CT, true, GS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         C::SMEM_ALLOC);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, decode_kernel<MT, kBF16, BN, XR, CT, false, GS>, C::THREADS,
                                                      C::SMEM_ALLOC) != cudaSuccess || n < 1)
      n = 1;
    cached[d < 64 && d >= 0 ? d : 0] = std::min(n, CT);
  });
  return cached[dev];
}

template <int MT, bool kBF16, int BN, int XR, int CT, int GS = 128>
cudaError_t launch_t(const void* X, const uint8_t* Wq, const uint16_t* scales, const void* zeros,
                     void* Y, int M, int N, int K, void* ws, bool dp, const ArParams& ar, bool weights_static,
                     bool zu4, int grid_per_sm, cudaStream_t st, const char** why) {
  using C = Cfg<MT, BN, XR, CT, GS>;
  const int G = K / kGroup;  // 128-k slots
  CUtensorMap tw, tx, ts, tz;
  {
    const uint64_t d[3] = {64, (uint64_t)N, (uint64_t)G};
    const uint64_t s[2] = {(uint64_t)K / 2, 64};
    const uint32_t b[3] = {64, (uint32_t)BN, (uint32_t)GPS};
    if (!encode(&tw, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, Wq, d, s, b, CU_TENSOR_MAP_SWIZZLE_NONE)) {
      *why = "tensor map (codes)";
      return cudaErrorInvalidValue;
    }
  }
  {
    const uint64_t d[4] = {64, 2, (uint64_t)M, (uint64_t)G};
    const uint64_t s[3] = {128, (uint64_t)K * 2, 256};
    const uint32_t b[4] = {64, 2, (uint32_t)XR, GPS};
    if (!encode(&tx, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, X, d, s, b, CU_TENSOR_MAP_SWIZZLE_128B)) {
      *why = "tensor map (X)";
      return cudaErrorInvalidValue;
    }
  }
  {
    const uint64_t d[2] = {(uint64_t)N, (uint64_t)G * C::SUB};  // [K / GS][N]
    const uint64_t s[1] = {(uint64_t)N * 2};
    const uint32_t b[2] = {(uint32_t)BN, (uint32_t)(GPS * C::SUB)};
    // packed u4 zeros: uint8[K / GS][N / 2], a box of BN / 2 bytes per zero row (a multiple of
    // 16 bytes: every row-block height the dispatch uses with u4 zeros -- 32, 64, 96, 128)
    const uint64_t dz[2] = {(uint64_t)N / 2, (uint64_t)G * C::SUB};
    const uint64_t sz[1] = {(uint64_t)N / 2};
    const uint32_t bz[2] = {(uint32_t)BN / 2, (uint32_t)(GPS * C::SUB)};
    if (!encode(&ts, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, scales, d, s, b, CU_TENSOR_MAP_SWIZZLE_NONE) ||
        !(zu4 ? encode(&tz, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, zeros, dz, sz, bz, CU_TENSOR_MAP_SWIZZLE_NONE)
              : encode(&tz, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, zeros, d, s, b, CU_TENSOR_MAP_SWIZZLE_NONE))) {
      *why = "tensor map (scales/zeros)";
      return cudaErrorInvalidValue;
    }
  }
  Work wk;
  wk.rbs = (N + BN - 1) / BN;
  wk.upb = (G + GPS - 1) / GPS;
  wk.units = wk.rbs * wk.upb;
  wk.dp = dp ? 1 : 0;
  int slots = num_sms() * std::min(grid_per_sm, ctas_per_sm<MT, kBF16, BN, XR, CT, GS>());
  if (option(SQ_OPT_DECODE_GRID_LIMIT) > 0) slots = std::min(slots, option(SQ_OPT_DECODE_GRID_LIMIT));
  const int P = dp ? std::min(wk.rbs, slots) : std::min(wk.units, slots);
  wk.cta_q = wk.units / P;
  wk.cta_r = wk.units % P;
  // partial slots first (fixed size), counters after: the counter region of one shape
  // never overlaps another shape's partials in a shared workspace
  float* partials = reinterpret_cast<float*>(ws);
  int* counters = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(ws) + ws_partials_bytes());
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
  if (ar.world > 0)
    return cudaLaunchKernelEx(&cfg, decode_kernel<MT, kBF16, BN, XR, CT, true, GS>, tw, tx, ts, tz, (uint16_t*)Y,
                              counters, partials, M, N, wk, early, zu4 ? 1 : 0, ar);
  return cudaLaunchKernelEx(&cfg, decode_kernel<MT, kBF16, BN, XR, CT, false, GS>, tw, tx, ts, tz, (uint16_t*)Y,
                            counters, partials, M, N, wk, early, zu4 ? 1 : 0, ar);
}

// Fraction of the resident CTA slots kept busy by whole row blocks of height bn.
double rowblock_utilization(int N, int bn, int slots) {
  const int rbs = (N + bn - 1) / bn;
  const int waves = (rbs + slots - 1) / slots;
  return (double)rbs / ((double)waves * slots);
}

// The AUTO row-block decision (see launch_m): true and the row height if whole row blocks win.
bool auto_rowblock(int N, int K, int slots, int* bn_out) {
  const int G = K / kGroup;
  const double sk_bytes_per_cta = (double)N * K / 2 / std::min<double>((double)slots,
      (double)((N + 63) / 64) * ((G + GPS - 1) / GPS));
  for (int cand : {32, 64}) {
    const int rbs = (N + cand - 1) / cand;
    const double rb_bytes = (double)cand * K / 2;
    if (rbs <= slots && rb_bytes - sk_bytes_per_cta <= 48.0 * 1024 && rb_bytes <= 192.0 * 1024) {
      *bn_out = cand;
      return true;
    }
  }
  return false;
}

template <int MT, bool kBF16, int XR, int CT>
cudaError_t launch_m(const void* X, const uint8_t* Wq, const uint16_t* scales, const void* zeros,
                     void* Y, int M, int N, int K, void* ws, const ArParams& ar, bool weights_static,
                     bool zu4, cudaStream_t st, const char** why, int grid_per_sm = CT) {
  const int sched = option(SQ_OPT_DECODE_SCHEDULE);
  const int slots = num_sms() * grid_per_sm;
  // AUTO (measured on the 34B and 7B shapes, 48-launch chains): whole row
  // blocks (no stream-K fixups) when one wave of them fits the resident CTA slots, a CTA's
  // row block exceeds the stream-K share by at most what the fixups cost (~2.5 µs at a CTA's
  // ~19 GB/s: 48 KB of codes), and the row block is short (<= 192 KB: longer ones stream
  // below the HBM rate with fewer CTAs busy).  The shorter qualifying row height wins.
  // 34B o_proj 8192 x 8192 (+15 KB, 128 KB), 7B qkv 4096 x 12288 (+46 KB, 128 KB) and 7B
  // o_proj 4096 x 4096 (+36 KB, 64 KB) take row blocks; 34B qkv (+114 KB), 34B down_proj
  // (+47 KB but 352 KB per CTA) and the rest stay stream-K.
  bool dp = sched == SQ_SCHED_ROWBLOCK;
  // stream-K row-block height: 32 rows for M = 9..16 on layers below 48 MB of codes (half
  // the cut row blocks' fixup work; measured -8..-13 % on the 7B shapes, +2 % on 34B qkv),
  // 64 otherwise (larger stages stream faster)
  // ... and at M = 2-8 on layers below 32 MB (7B down, 8192 x 4096: -8-9 %; +3-11 % at M = 1,
  // profiles/r02/decode_bn32_small_ab.jsonl)
  const double codes_m = (double)N * K / 2;
  int bn = (MT == 2 && codes_m < 48.0 * 1024 * 1024) || (MT == 1 && XR > 1 && codes_m < 32.0 * 1024 * 1024) ? 32 : 64;
  if (sched == SQ_SCHED_ROWBLOCK) {
    bn = rowblock_utilization(N, 64, slots) >= rowblock_utilization(N, 32, slots) ? 64 : 32;
  } else if (sched == SQ_SCHED_AUTO) {
    int rbn = 64;
    if (auto_rowblock(N, K, slots, &rbn)) {
      dp = true;
      bn = rbn;
    }
  }
  if (ar.world > 0) {
    // fused all-reduce: flags are per row block, so every rank must cut N the same way.
    // Decide from N alone (K differs between row-parallel shards): stream-K, 64-row blocks.
    dp = false;
    bn = 64;
  }
  // M = 1-4 on layers of >= 48 MB of codes, or >= 32 MB with K >= 8192 (stream-K, two CTAs
  // per SM): 128-row blocks -- a stage then carries 32 KB of codes per barrier round and X
  // fragment, and each consumer warp runs eight row tiles per stage; 4-6 % faster at M = 1 on
  // the 34B gate|up, gate, down and qkv shapes (profiles/r02/decode_bn128_ab.jsonl,
  // decode_bn128_threshold_ab.jsonl), 1-5 % at M = 2-4 with four staged activation rows
  // (decode_bn128_m4_ab.jsonl); with eight rows the stages get too deep for the ring (M = 5-8)
  if constexpr (XR <= 4 && CT == 2) {
    const double codes = (double)N * K / 2;
    // (96-row blocks for the 32-48 MB ones at M = 1: 34B qkv -5 % against 128, every larger
    // layer +1.5-7 %; profiles/r02/decode_bn96_ab.jsonl)
    if (XR == 1 && !dp && bn == 64 && ar.world == 0 && codes >= 32.0 * 1024 * 1024 &&
        codes < 48.0 * 1024 * 1024 && K >= 8192)
      return launch_t<MT, kBF16, 96, XR, CT>(X, Wq, scales, zeros, Y, M, N, K, ws, dp, ar, weights_static, zu4,
                                             grid_per_sm, st, why);
    if (!dp && bn == 64 && ar.world == 0 &&
        (codes >= 48.0 * 1024 * 1024 || (codes >= 32.0 * 1024 * 1024 && K >= 8192)))
      return launch_t<MT, kBF16, 128, XR, CT>(X, Wq, scales, zeros, Y, M, N, K, ws, dp, ar, weights_static, zu4,
                                              grid_per_sm, st, why);
  }
  // M = 9-16, stream-K, 32-128 MB layers with 8192 <= K < 16384 (34B qkv, gate): 48-row
  // blocks, between the 32-row (shallower work per stage) and 64-row (fewer, larger stages)
  // choices: qkv -4-5 %, gate -3 %; gate|up (180 MB), down (K = 22016) and the 7B shapes do not
  // gain (profiles/r02/decode_bn48_ab.jsonl)
  // (not with packed u4 zero points: a 48-row block's zero rows are 24 bytes, and a TMA box
  // must span a multiple of 16 bytes)
  if (MT == 2 && !dp && ar.world == 0 && !zu4 && codes_m >= 32.0 * 1024 * 1024 && codes_m < 128.0 * 1024 * 1024 &&
      K >= 8192 && K < 16384)
    return launch_t<MT, kBF16, 48, XR, CT>(X, Wq, scales, zeros, Y, M, N, K, ws, dp, ar, weights_static, zu4,
                                           grid_per_sm, st, why);
  if (bn == 32)
    return launch_t<MT, kBF16, 32, XR, CT>(X, Wq, scales, zeros, Y, M, N, K, ws, dp, ar, weights_static, zu4, grid_per_sm,
                                           st, why);
  return launch_t<MT, kBF16, 64, XR, CT>(X, Wq, scales, zeros, Y, M, N, K, ws, dp, ar, weights_static, zu4, grid_per_sm, st,
                                         why);
}

}  // namespace

bool encode_tmap(CUtensorMap* map, CUtensorMapDataType dt, int rank, const void* base, const uint64_t* dims,
                 const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle sw) {
  return encode(map, dt, rank, base, dims, strides_bytes, box, sw);
}

size_t decode_partials_bytes() {
  return (size_t)num_sms() * kMaxCtasPerSm * 2 * 16 * kMaxBN * sizeof(float);
}

size_t decode_workspace_bytes(int64_t N) {
  const int64_t RB = (N + kMinBN - 1) / kMinBN;
  return ws_partials_bytes() + counter_region_bytes(RB);
}

template <int GS>
cudaError_t launch_small_group(const void* X, bool bf16, const uint8_t* Wq, const uint16_t* scales,
                               const void* zeros, void* Y, int M, int N, int K, void* ws, const ArParams& ar,
                               bool weights_static, bool zu4, cudaStream_t st, const char** why) {
  // group sizes 64 / 32: one configuration per M class (stream-K, 64-row blocks, two CTAs per SM)
  constexpr int C2 = kCtasPerSm;
  if (M == 1)
    return bf16 ? launch_t<1, true, 64, 1, C2, GS>(X, Wq, scales, zeros, Y, M, N, K, ws, false, ar, weights_static, zu4, C2,
                                                   st, why)
                : launch_t<1, false, 64, 1, C2, GS>(X, Wq, scales, zeros, Y, M, N, K, ws, false, ar, weights_static, zu4,
                                                    C2, st, why);
  if (M <= 8)
    return bf16 ? launch_t<1, true, 64, 8, C2, GS>(X, Wq, scales, zeros, Y, M, N, K, ws, false, ar, weights_static, zu4, C2,
                                                   st, why)
                : launch_t<1, false, 64, 8, C2, GS>(X, Wq, scales, zeros, Y, M, N, K, ws, false, ar, weights_static, zu4,
                                                    C2, st, why);
  return bf16 ? launch_t<2, true, 64, 16, C2, GS>(X, Wq, scales, zeros, Y, M, N, K, ws, false, ar, weights_static, zu4, C2,
                                                  st, why)
              : launch_t<2, false, 64, 16, C2, GS>(X, Wq, scales, zeros, Y, M, N, K, ws, false, ar, weights_static, zu4, C2,
                                                   st, why);
}

cudaError_t launch_decode(const void* X, int x_dtype, const uint8_t* Wq, const uint16_t* scales,
                          const void* zeros, void* Y, int M, int N, int K, int group, void* ws,
                          bool weights_static, bool zu4, cudaStream_t st, const char** why, const ArParams* ar_in) {
  const ArParams ar = ar_in ? *ar_in : ArParams{nullptr, 0, nullptr, 0, 0, 0u};
  const bool bf16 = x_dtype == SQ_BF16;
  if (group == 64)
    return launch_small_group<64>(X, bf16, Wq, scales, zeros, Y, M, N, K, ws, ar, weights_static, zu4, st, why);
  if (group == 32)
    return launch_small_group<32>(X, bf16, Wq, scales, zeros, Y, M, N, K, ws, ar, weights_static, zu4, st, why);
  if (M == 1) {  // batch-1 decode: stage one activation row, smaller stages
    // three 74-KB CTAs per SM for mid-sized layers (32-48 MB of codes, K < 8192) that two CTAs
    // per SM would stream-K: more CTAs in flight (or a one-wave row-block split at 444 slots);
    // measured -12 % on 7B gate|up (profiles/decode_m1_ct3_ab_r01.jsonl).  Not for the fused
    // all-reduce (its row-block cut must not depend on the rank's K).
    const double codes = (double)N * K / 2;
    int rbn = 64;
    // (K >= 8192 layers of this size take two CTAs per SM with 128-row blocks instead, launch_m)
    if (ar.world == 0 && option(SQ_OPT_DECODE_SCHEDULE) == SQ_SCHED_AUTO && codes >= 32.0 * 1024 * 1024 &&
        codes < 48.0 * 1024 * 1024 && K < 8192 && !auto_rowblock(N, K, num_sms() * kCtasPerSm, &rbn))
      return bf16 ? launch_m<1, true, 1, 3>(X, Wq, scales, zeros, Y, M, N, K, ws, ar, weights_static, zu4, st, why)
                  : launch_m<1, false, 1, 3>(X, Wq, scales, zeros, Y, M, N, K, ws, ar, weights_static, zu4, st, why);
    return bf16 ? launch_m<1, true, 1, kCtasPerSm>(X, Wq, scales, zeros, Y, M, N, K, ws, ar, weights_static, zu4, st, why)
                : launch_m<1, false, 1, kCtasPerSm>(X, Wq, scales, zeros, Y, M, N, K, ws, ar, weights_static, zu4, st, why);
  }
  // M = 2-4 on whole-row-block layers and K < 8192 layers: stage only four activation rows
  // (4-KB X slices, a deeper ring): 34B o_proj -2 %, the 7B shapes -5 %; the big stream-K
  // 34B layers stay on eight rows (+1-2 % with four; profiles/r02/decode_xr4_ab.jsonl)
  int rbn4 = 64;
  // The large K >= 8192 stream-K layers (>= 32 MB) stage four rows too, in 128-row blocks (launch_m)
  const bool big4 = M <= 4 && ar.world == 0 && option(SQ_OPT_DECODE_SCHEDULE) == SQ_SCHED_AUTO &&
                    K >= 8192 && !auto_rowblock(N, K, num_sms() * kCtasPerSm, &rbn4) &&
                    (double)N * K / 2 >= 32.0 * 1024 * 1024;
  const bool xr4 = big4 || (M <= 4 && ar.world == 0 && option(SQ_OPT_DECODE_SCHEDULE) == SQ_SCHED_AUTO &&
                            (K < 8192 || auto_rowblock(N, K, num_sms() * kCtasPerSm, &rbn4)));
  // ... and, like M = 1, three CTAs per SM on the 32-48 MB, K < 8192 stream-K layers (7B gate|up
  // -10 % at M = 2-4; every other shape slower, profiles/r02/decode_ct3_m4_ab.jsonl)
  int rbn3 = 64;
  const double codes4 = (double)N * K / 2;
  if (xr4 && codes4 >= 32.0 * 1024 * 1024 && codes4 < 48.0 * 1024 * 1024 && K < 8192 &&
      !auto_rowblock(N, K, num_sms() * kCtasPerSm, &rbn3))
    return bf16 ? launch_m<1, true, 4, 3>(X, Wq, scales, zeros, Y, M, N, K, ws, ar, weights_static, zu4, st, why)
                : launch_m<1, false, 4, 3>(X, Wq, scales, zeros, Y, M, N, K, ws, ar, weights_static, zu4, st, why);
  if (xr4)
    return bf16 ? launch_m<1, true, 4, kCtasPerSm>(X, Wq, scales, zeros, Y, M, N, K, ws, ar, weights_static, zu4, st, why)
                : launch_m<1, false, 4, kCtasPerSm>(X, Wq, scales, zeros, Y, M, N, K, ws, ar, weights_static, zu4, st, why);
  if (M <= 8)
    return bf16 ? launch_m<1, true, 8, kCtasPerSm>(X, Wq, scales, zeros, Y, M, N, K, ws, ar, weights_static, zu4, st, why)
                : launch_m<1, false, 8, kCtasPerSm>(X, Wq, scales, zeros, Y, M, N, K, ws, ar, weights_static, zu4, st, why);
  return bf16 ? launch_m<2, true, 16, kCtasPerSm>(X, Wq, scales, zeros, Y, M, N, K, ws, ar, weights_static, zu4, st, why)
              : launch_m<2, false, 16, kCtasPerSm>(X, Wq, scales, zeros, Y, M, N, K, ws, ar, weights_static, zu4, st, why);
}

}  // namespace sq
