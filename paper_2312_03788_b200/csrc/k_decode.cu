// K-dec: W4A16 GEMM for small M (decode, M <= 16) -- HBM-bound.
//
//   Y[m][n] = sum_gi Δ[gi][n] * sum_{k in gi} X[m][k] * (q[n][k] - Z[gi][n])
//   PAPER.md:104-106 Eq. 3 with Ŵ of Eq. 1 line 2; fp32 accumulation.
//
// Design:
//  * A warp owns 16 output channels; lane (r = lane/4, j = lane%4) streams 16 bytes
//    (32 codes) of row r and 16 bytes of row r+8 per group with 128-bit
//    ld.global.nc.L1::no_allocate loads (4 lanes -> 64 contiguous bytes per row).
//    One (16-row x 128-k) group = two loads per lane = 8 mma.sync.m16n8k16.
//  * Register dequant to the EXACT integer (q - Z) in fp16/bf16 with the
//    lop3 magic-number trick; Δ is applied once per group to the fp32 accumulator
//    fragment (so the MMA sees exact operands and only fp32 rounding remains).
//  * The MMA's k order is permuted (nibble pairs (e0,e4),(e1,e5),...): X is loaded in
//    natural order (L1-resident, shared by all warps) and permuted with PRMT.
//  * Tokens are the MMA's N = 8 (MT = 2 tiles for M <= 16).
//  * Split-K over a thread-block cluster of S CTAs along K; the S fp32 partial
//    tiles are reduced through distributed shared memory by the cluster's rank-0
//    CTA in fixed rank order (deterministic, no global workspace, no atomics).
#include <algorithm>
#include <cooperative_groups.h>

#include "sq_internal.cuh"

namespace cg = cooperative_groups;

namespace sq {

namespace {

constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
constexpr int kRowsPerCta = kWarps * 16;
constexpr int kGroup = 128;

struct WFrag {
  uint4 a, b;       // 32 codes of row r and of row r+8
  uint32_t sa, sb;  // (scale bits) | (zero bits << 16) for rows r and r+8
};

__device__ __forceinline__ void mma_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint32_t b0, uint32_t b1, bool bf16) {
  if (bf16) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
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

// Dequantize one 32-bit word (8 codes, k offsets 0..7) of one row into the four
// exact (q - Z) pairs (e0,e4), (e1,e5), (e2,e6), (e3,e7).
template <bool kBF16>
__device__ __forceinline__ void dequant_word(uint32_t w, uint32_t zsub, uint32_t zfma,
                                             uint32_t (&h)[4]) {
  if (!kBF16) {
    const uint32_t t = w >> 8;
    h[0] = hsub2_u(lop3_and_or(w, 0x000F000Fu, 0x64006400u), zsub, false);   // 1024+e0,e4
    h[2] = hsub2_u(lop3_and_or(t, 0x000F000Fu, 0x64006400u), zsub, false);   // 1024+e2,e6
    // 1024+16e1 -> (x/16) - (64+Z)
    h[1] = hfma2_u(lop3_and_or(w, 0x00F000F0u, 0x64006400u), 0x2C002C00u, zfma);
    h[3] = hfma2_u(lop3_and_or(t, 0x00F000F0u, 0x64006400u), 0x2C002C00u, zfma);
  } else {
    h[0] = hsub2_u(lop3_and_or(w, 0x000F000Fu, 0x43004300u), zsub, true);   // 128+e0,e4
    h[1] = hsub2_u(lop3_and_or(w >> 4, 0x000F000Fu, 0x43004300u), zsub, true);
    h[2] = hsub2_u(lop3_and_or(w >> 8, 0x000F000Fu, 0x43004300u), zsub, true);
    h[3] = hsub2_u(lop3_and_or(w >> 12, 0x000F000Fu, 0x43004300u), zsub, true);
  }
}

template <bool kBF16>
__device__ __forceinline__ void zero_consts(uint32_t szbits, uint32_t& zsub, uint32_t& zfma,
                                            float& d) {
  const __half z = __ushort_as_half((unsigned short)(szbits >> 16));
  d = __half2float(__ushort_as_half((unsigned short)(szbits & 0xFFFFu)));
  if (!kBF16) {
    const __half c1 = __hadd(__float2half(1024.0f), z);           // exact
    const __half c2 = __hneg(__hadd(__float2half(64.0f), z));     // exact
    const __half2 p1 = __half2half2(c1), p2 = __half2half2(c2);
    zsub = *reinterpret_cast<const uint32_t*>(&p1);
    zfma = *reinterpret_cast<const uint32_t*>(&p2);
  } else {
    const __nv_bfloat16 c1 = __float2bfloat16_rn(128.0f + __half2float(z));  // exact (<= 143)
    const __nv_bfloat162 p1 = __bfloat162bfloat162(c1);
    zsub = *reinterpret_cast<const uint32_t*>(&p1);
    zfma = 0;
  }
}

template <int MT, bool kBF16>
__global__ void __launch_bounds__(kThreads)
decode_kernel(const uint16_t* __restrict__ X, const uint8_t* __restrict__ Wq,
              const uint16_t* __restrict__ scales, const uint16_t* __restrict__ zeros,
              uint16_t* __restrict__ Y, int M, int N, int K, int splits) {
  __shared__ float part[MT * 8][kRowsPerCta];

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int r = lane / 4, j = lane % 4;
  const int split = blockIdx.x;  // == rank in the cluster (cluster dims = (splits,1,1))
  const int n0 = blockIdx.y * kRowsPerCta + warp * 16;
  const int rowA = n0 + r, rowB = n0 + r + 8;
  const bool okA = rowA < N, okB = rowB < N;
  const int G = K / kGroup;
  const int gbeg = (int)(((long long)G * split) / splits);
  const int gend = (int)(((long long)G * (split + 1)) / splits);

  const uint8_t* pA = Wq + (size_t)rowA * (K / 2) + j * 16;
  const uint8_t* pB = Wq + (size_t)rowB * (K / 2) + j * 16;

  auto load = [&](int g) {
    WFrag f;
    if (okA) {
      f.a = ld_nc_v4(pA + (size_t)g * 64);
      f.sa = (uint32_t)ld_u16(scales + (size_t)g * N + rowA) |
             ((uint32_t)ld_u16(zeros + (size_t)g * N + rowA) << 16);
    } else {
      f.a = make_uint4(0, 0, 0, 0);
      f.sa = 0;
    }
    if (okB) {
      f.b = ld_nc_v4(pB + (size_t)g * 64);
      f.sb = (uint32_t)ld_u16(scales + (size_t)g * N + rowB) |
             ((uint32_t)ld_u16(zeros + (size_t)g * N + rowB) << 16);
    } else {
      f.b = make_uint4(0, 0, 0, 0);
      f.sb = 0;
    }
    return f;
  };

  float acc[MT][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[mt][i] = 0.0f;

  auto compute = [&](const WFrag& f, int g) {
    // X fragments: token t = r + 8 mt, k = g*128 + 32 j + [0, 32)
    uint32_t xv[MT][16];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int t = r + 8 * mt;
      if (t < M) {
        const uint4* xp = reinterpret_cast<const uint4*>(X + (size_t)t * K + (size_t)g * kGroup + j * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 v = __ldg(xp + q);
          xv[mt][4 * q + 0] = v.x;
          xv[mt][4 * q + 1] = v.y;
          xv[mt][4 * q + 2] = v.z;
          xv[mt][4 * q + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) xv[mt][q] = 0u;
      }
    }
    uint32_t zsubA, zfmaA, zsubB, zfmaB;
    float dA, dB;
    zero_consts<kBF16>(f.sa, zsubA, zfmaA, dA);
    zero_consts<kBF16>(f.sb, zsubB, zfmaB, dB);
    float gacc[MT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int i = 0; i < 4; ++i) gacc[mt][i] = 0.0f;
    const uint32_t wa[4] = {f.a.x, f.a.y, f.a.z, f.a.w};
    const uint32_t wb[4] = {f.b.x, f.b.y, f.b.z, f.b.w};
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      uint32_t hA[4], hB[4];
      dequant_word<kBF16>(wa[w], zsubA, zfmaA, hA);
      dequant_word<kBF16>(wb[w], zsubB, zfmaB, hB);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const uint32_t x01 = xv[mt][4 * w], x23 = xv[mt][4 * w + 1];
        const uint32_t x45 = xv[mt][4 * w + 2], x67 = xv[mt][4 * w + 3];
        const uint32_t p0 = prmt(x01, x45, 0x5410u), p1 = prmt(x01, x45, 0x7632u);
        const uint32_t p2 = prmt(x23, x67, 0x5410u), p3 = prmt(x23, x67, 0x7632u);
        mma_16816(gacc[mt], hA[0], hB[0], hA[1], hB[1], p0, p1, kBF16);
        mma_16816(gacc[mt], hA[2], hB[2], hA[3], hB[3], p2, p3, kBF16);
      }
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      acc[mt][0] = fmaf(gacc[mt][0], dA, acc[mt][0]);
      acc[mt][1] = fmaf(gacc[mt][1], dA, acc[mt][1]);
      acc[mt][2] = fmaf(gacc[mt][2], dB, acc[mt][2]);
      acc[mt][3] = fmaf(gacc[mt][3], dB, acc[mt][3]);
    }
  };

  // software pipeline: up to three groups of codes in flight per warp
  {
    int g = gbeg;
    WFrag f0 = {}, f1 = {};
    if (g < gend) f0 = load(g);
    if (g + 1 < gend) f1 = load(g + 1);
    for (; g < gend; g += 2) {
      WFrag n0 = {};
      if (g + 2 < gend) n0 = load(g + 2);
      compute(f0, g);
      WFrag n1 = {};
      if (g + 3 < gend) n1 = load(g + 3);
      if (g + 1 < gend) compute(f1, g + 1);
      f0 = n0;
      f1 = n1;
    }
  }

  auto to_out = [](float v) -> uint16_t {
    if (kBF16) return __bfloat16_as_ushort(__float2bfloat16_rn(v));
    return __half_as_ushort(__float2half_rn(v));
  };

  if (splits == 1) {
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int t0 = 8 * mt + 2 * j, t1 = t0 + 1;
      if (t0 < M) {
        if (okA) Y[(size_t)t0 * N + rowA] = to_out(acc[mt][0]);
        if (okB) Y[(size_t)t0 * N + rowB] = to_out(acc[mt][2]);
      }
      if (t1 < M) {
        if (okA) Y[(size_t)t1 * N + rowA] = to_out(acc[mt][1]);
        if (okB) Y[(size_t)t1 * N + rowB] = to_out(acc[mt][3]);
      }
    }
    return;
  }

  // ---- split-K: stage this CTA's fp32 partial tile, reduce over the cluster ----
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int t0 = 8 * mt + 2 * j;
    part[t0][warp * 16 + r] = acc[mt][0];
    part[t0 + 1][warp * 16 + r] = acc[mt][1];
    part[t0][warp * 16 + r + 8] = acc[mt][2];
    part[t0 + 1][warp * 16 + r + 8] = acc[mt][3];
  }
  cg::cluster_group cluster = cg::this_cluster();
  cluster.sync();
  if (cluster.block_rank() == 0) {
    const int nblk = blockIdx.y * kRowsPerCta;
    for (int idx = threadIdx.x; idx < M * kRowsPerCta; idx += kThreads) {
      const int t = idx / kRowsPerCta, row = idx % kRowsPerCta;
      float s = 0.0f;
      for (int rk = 0; rk < splits; ++rk) {
        const float* peer = cluster.map_shared_rank(&part[0][0], rk);
        s += peer[t * kRowsPerCta + row];
      }
      if (nblk + row < N) Y[(size_t)t * N + nblk + row] = to_out(s);
    }
  }
  cluster.sync();
}

template <int MT, bool kBF16>
cudaError_t launch_t(const void* X, const uint8_t* Wq, const uint16_t* scales,
                     const uint16_t* zeros, void* Y, int M, int N, int K, const DecodePlan& p,
                     cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.splits, (unsigned)p.row_blocks, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)p.splits;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, decode_kernel<MT, kBF16>, (const uint16_t*)X, Wq, scales, zeros,
                            (uint16_t*)Y, M, N, K, p.splits);
}

}  // namespace

DecodePlan plan_decode(int64_t M, int64_t N, int64_t K) {
  (void)M;
  DecodePlan p;
  p.rows_per_cta = kRowsPerCta;
  p.row_blocks = (int)((N + kRowsPerCta - 1) / kRowsPerCta);
  const int G = (int)(K / kGroup);
  // CTAs resident at once (4 warps each, ~4 per SM); split K over a cluster only as
  // far as the whole grid still fits in one wave, and keep >= 4 groups per CTA.
  const int slots = 4 * num_sms();
  int s = 1;
  while (s * 2 <= 8 && (int64_t)p.row_blocks * s * 2 <= slots && G / (s * 2) >= 4) s *= 2;
  p.splits = s;
  return p;
}

cudaError_t launch_decode(const void* X, int x_dtype, const uint8_t* Wq, const uint16_t* scales,
                          const uint16_t* zeros, void* Y, int M, int N, int K,
                          const DecodePlan& plan, cudaStream_t st) {
  const bool bf16 = x_dtype == SQ_BF16;
  if (M <= 8)
    return bf16 ? launch_t<1, true>(X, Wq, scales, zeros, Y, M, N, K, plan, st)
                : launch_t<1, false>(X, Wq, scales, zeros, Y, M, N, K, plan, st);
  return bf16 ? launch_t<2, true>(X, Wq, scales, zeros, Y, M, N, K, plan, st)
              : launch_t<2, false>(X, Wq, scales, zeros, Y, M, N, K, plan, st);
}

}  // namespace sq
