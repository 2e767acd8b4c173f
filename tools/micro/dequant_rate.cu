// Microbenchmark: consumer-side throughput of the decode GEMM's per-stage math with no
// memory traffic (codes / X / scale / zero read from a small SMEM ring that stays
// resident), to find which dequant formulation the ALU / FMA / HMMA pipes allow.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dequant_rate dequant_rate.cu
//   ./dequant_rate            -> one line per variant: G weights/s and the equivalent
//                                 W4 stream rate (0.53125 B/weight) in TB/s
//
// Variants (per stage = 64 rows x 4 groups of 128 k; one consumer warp per group):
//   0  current: exact (q - Z) fp16 via lop3 + hsub2/hfma2, Z from F2I per row tile
//   1  magic:  lop3 only (1024 + q, 1024 + 16 q), odd-k activations pre-scaled by 1/16,
//              one accumulator, zero point / offset removed per row tile with the
//              per-group activation sums (FFMA); shift by SHF
//   2  as 1 with the >> 8 done by IMAD.HI (fma pipe) instead of SHF (alu pipe)
//   3  as 2 without the per-row-tile scale/zero loads (upper bound)
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t m, uint32_t o) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;\n" : "=r"(r) : "r"(a), "r"(m), "r"(o));
  return r;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;\n" : "=r"(r) : "r"(a), "r"(b), "r"(s));
  return r;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint16_t lds16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];\n" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                    uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t hsub2u(uint32_t a, uint32_t b) {
  __half2 r = __hsub2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t hfma2u(uint32_t a, uint32_t b, uint32_t c) {
  __half2 r = __hfma2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b), *reinterpret_cast<__half2*>(&c));
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t hmul2u(uint32_t a, uint32_t b) {
  __half2 r = __hmul2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}

constexpr int BN = 64, GPS = 4, NS = 2;
constexpr int CODES = GPS * BN * 64;  // 16 KB
constexpr int XB = GPS * 8 * 128 * 2;  // 8 token rows
constexpr int SZ = GPS * BN * 2;
constexpr int STAGE = CODES + XB + 2 * SZ;

template <int V, int MT, int CW>
__global__ void __launch_bounds__(CW * 32) kern(int iters, float* out, long long* clk) {
  long long t0 = clock64();
  extern __shared__ __align__(1024) uint8_t smem[];
  for (int i = threadIdx.x; i < NS * STAGE / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3C003C00u ^ (i * 2654435761u & 0x03FF03FFu);
  __syncthreads();
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int r = lane / 4, j = lane % 4, grp = warp % GPS;
  constexpr int RS = CW / GPS;
  constexpr int RT = BN / 16 / RS;
  const int roff = (warp / GPS) * (BN / RS);
  float acc[RT][MT][4];
#pragma unroll
  for (int a = 0; a < RT; ++a)
#pragma unroll
    for (int b = 0; b < MT; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.f;
  for (int it = 0; it < iters; ++it) {
    const uint32_t st = sbase + (it % NS) * STAGE;
    uint32_t xb[MT][4][4];
    float sxe[MT][2], sxo[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int t = r + 8 * mt;
      const int R = (grp * 8 + (t & 7)) * 2 + (j >> 1);
      const uint32_t rowaddr = st + CODES + R * 128;
      uint32_t xv[16];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 v = lds128(rowaddr + ((((j & 1) * 4 + i) ^ (R & 7)) << 4));
        xv[4 * i] = v.x; xv[4 * i + 1] = v.y; xv[4 * i + 2] = v.z; xv[4 * i + 3] = v.w;
      }
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        if (V == 4 || V == 7) { xb[mt][w][0] = xv[4 * w]; xb[mt][w][1] = xv[4 * w + 1]; xb[mt][w][2] = xv[4 * w + 2]; xb[mt][w][3] = xv[4 * w + 3]; continue; }
        xb[mt][w][0] = prmt(xv[4 * w], xv[4 * w + 2], 0x5410u);
        xb[mt][w][1] = prmt(xv[4 * w], xv[4 * w + 2], 0x7632u);
        xb[mt][w][2] = prmt(xv[4 * w + 1], xv[4 * w + 3], 0x5410u);
        xb[mt][w][3] = prmt(xv[4 * w + 1], xv[4 * w + 3], 0x7632u);
      }
      if (V >= 1 && V != 6) {
        // odd k (hi nibbles, 1024 + 16 q) see x / 16; sums of the fed values per token
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          xb[mt][w][1] = hmul2u(xb[mt][w][1], 0x2C002C00u);
          xb[mt][w][3] = hmul2u(xb[mt][w][3], 0x2C002C00u);
        }
        __half2 se = __hadd2(*reinterpret_cast<__half2*>(&xb[mt][0][0]), *reinterpret_cast<__half2*>(&xb[mt][0][2]));
        __half2 so = __hadd2(*reinterpret_cast<__half2*>(&xb[mt][0][1]), *reinterpret_cast<__half2*>(&xb[mt][0][3]));
        float2 fe = __half22float2(se), fo = __half22float2(so);
        float e = fe.x + fe.y, o = fo.x + fo.y;
#pragma unroll
        for (int w = 1; w < 4; ++w) {
          float2 a = __half22float2(*reinterpret_cast<__half2*>(&xb[mt][w][0]));
          float2 b = __half22float2(*reinterpret_cast<__half2*>(&xb[mt][w][2]));
          float2 c = __half22float2(*reinterpret_cast<__half2*>(&xb[mt][w][1]));
          float2 d = __half22float2(*reinterpret_cast<__half2*>(&xb[mt][w][3]));
          e += (a.x + a.y) + (b.x + b.y);
          o += (c.x + c.y) + (d.x + d.y);
        }
        e += __shfl_xor_sync(0xffffffffu, e, 1);
        e += __shfl_xor_sync(0xffffffffu, e, 2);
        o += __shfl_xor_sync(0xffffffffu, o, 1);
        o += __shfl_xor_sync(0xffffffffu, o, 2);
        sxe[mt][0] = e; sxe[mt][1] = e;
        sxo[mt][0] = o; sxo[mt][1] = o;
      }
    }
    if (V == 12) {
      const uint32_t cb0 = st + grp * (BN * 64) + (roff + r) * 64 + j * 16;
      const uint32_t sb0 = st + CODES + XB + grp * (BN * 2) + (roff + r) * 2;
      uint4 ca[RT], cbv[RT];
      uint32_t zs[RT][2], zf[RT][2];
      float d[RT][2];
#pragma unroll
      for (int rt = 0; rt < RT; ++rt) {
        ca[rt] = lds128(cb0 + rt * 16 * 64);
        cbv[rt] = lds128(cb0 + (rt * 16 + 8) * 64);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t zq = (uint32_t)__half2int_rn(__ushort_as_half(lds16(sb0 + SZ + rt * 32 + 16 * h)));
          zs[rt][h] = zq * 0x00010001u + 0x64006400u;
          zf[rt][h] = zq * 0x00100010u + 0xD400D400u;
          d[rt][h] = __half2float(__ushort_as_half(lds16(sb0 + rt * 32 + 16 * h)));
        }
      }
      float g[RT][MT][4];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
#pragma unroll
        for (int rt = 0; rt < RT; ++rt) {
          const uint32_t wa = w == 0 ? ca[rt].x : w == 1 ? ca[rt].y : w == 2 ? ca[rt].z : ca[rt].w;
          const uint32_t wb = w == 0 ? cbv[rt].x : w == 1 ? cbv[rt].y : w == 2 ? cbv[rt].z : cbv[rt].w;
          uint32_t hA[4], hB[4];
          const uint32_t ta = wa >> 8, tb = wb >> 8;
          hA[0] = hsub2u(lop3_and_or(wa, 0x000F000Fu, 0x64006400u), zs[rt][0]);
          hA[2] = hsub2u(lop3_and_or(ta, 0x000F000Fu, 0x64006400u), zs[rt][0]);
          hA[1] = hfma2u(lop3_and_or(wa, 0x00F000F0u, 0x64006400u), 0x2C002C00u, zf[rt][0]);
          hA[3] = hfma2u(lop3_and_or(ta, 0x00F000F0u, 0x64006400u), 0x2C002C00u, zf[rt][0]);
          hB[0] = hsub2u(lop3_and_or(wb, 0x000F000Fu, 0x64006400u), zs[rt][1]);
          hB[2] = hsub2u(lop3_and_or(tb, 0x000F000Fu, 0x64006400u), zs[rt][1]);
          hB[1] = hfma2u(lop3_and_or(wb, 0x00F000F0u, 0x64006400u), 0x2C002C00u, zf[rt][1]);
          hB[3] = hfma2u(lop3_and_or(tb, 0x00F000F0u, 0x64006400u), 0x2C002C00u, zf[rt][1]);
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            if (w == 0)
#pragma unroll
              for (int q = 0; q < 4; ++q) g[rt][mt][q] = 0.f;
            mma(g[rt][mt], hA[0], hB[0], hA[1], hB[1], xb[mt][w][0], xb[mt][w][1]);
            mma(g[rt][mt], hA[2], hB[2], hA[3], hB[3], xb[mt][w][2], xb[mt][w][3]);
          }
        }
      }
#pragma unroll
      for (int rt = 0; rt < RT; ++rt)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          acc[rt][mt][0] = fmaf(g[rt][mt][0], d[rt][0], acc[rt][mt][0]);
          acc[rt][mt][1] = fmaf(g[rt][mt][1], d[rt][0], acc[rt][mt][1]);
          acc[rt][mt][2] = fmaf(g[rt][mt][2], d[rt][1], acc[rt][mt][2]);
          acc[rt][mt][3] = fmaf(g[rt][mt][3], d[rt][1], acc[rt][mt][3]);
        }
      continue;
    }
    const uint32_t cbase = st + grp * (BN * 64) + (roff + r) * 64 + j * 16;
    const uint32_t sbs = st + CODES + XB + grp * (BN * 2) + (roff + r) * 2;
    const uint32_t sbz = sbs + SZ;
#pragma unroll
    for (int rt = 0; rt < RT; ++rt) {
      const uint4 ca = lds128(cbase + rt * 16 * 64);
      const uint4 cb = lds128(cbase + (rt * 16 + 8) * 64);
      const uint32_t wa[4] = {ca.x, ca.y, ca.z, ca.w};
      const uint32_t wb[4] = {cb.x, cb.y, cb.z, cb.w};
      float dA = 1.f, dB = 1.f, zA = 3.f, zB = 5.f;
      if (V != 3) {
        dA = __half2float(__ushort_as_half(lds16(sbs + rt * 32)));
        dB = __half2float(__ushort_as_half(lds16(sbs + rt * 32 + 16)));
      }
      float g[MT][4];
      if (V == 0 || V == 8 || V == 9 || V == 10) {
        const uint32_t zqa = (uint32_t)__half2int_rn(__ushort_as_half(lds16(sbz + rt * 32)));
        const uint32_t zqb = (uint32_t)__half2int_rn(__ushort_as_half(lds16(sbz + rt * 32 + 16)));
        const uint32_t zsA = zqa * 0x00010001u + 0x64006400u, zfA = zqa * 0x00100010u + 0xD400D400u;
        const uint32_t zsB = zqb * 0x00010001u + 0x64006400u, zfB = zqb * 0x00100010u + 0xD400D400u;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          uint32_t hA[4], hB[4];
          if (V == 9) {
            hA[0] = wa[w]; hA[1] = wa[w] >> 8; hA[2] = wa[w] ^ zsA; hA[3] = wa[w] + zfA;
            hB[0] = wb[w]; hB[1] = wb[w] >> 8; hB[2] = wb[w] ^ zsB; hB[3] = wb[w] + zfB;
          } else {
            const uint32_t t = wa[w] >> 8;
            hA[0] = hsub2u(lop3_and_or(wa[w], 0x000F000Fu, 0x64006400u), zsA);
            hA[2] = hsub2u(lop3_and_or(t, 0x000F000Fu, 0x64006400u), zsA);
            hA[1] = hfma2u(lop3_and_or(wa[w], 0x00F000F0u, 0x64006400u), 0x2C002C00u, zfA);
            hA[3] = hfma2u(lop3_and_or(t, 0x00F000F0u, 0x64006400u), 0x2C002C00u, zfA);
            {
            const uint32_t t = wb[w] >> 8;
            hB[0] = hsub2u(lop3_and_or(wb[w], 0x000F000Fu, 0x64006400u), zsB);
            hB[2] = hsub2u(lop3_and_or(t, 0x000F000Fu, 0x64006400u), zsB);
            hB[1] = hfma2u(lop3_and_or(wb[w], 0x00F000F0u, 0x64006400u), 0x2C002C00u, zfB);
            hB[3] = hfma2u(lop3_and_or(t, 0x00F000F0u, 0x64006400u), 0x2C002C00u, zfB);
          }
          }
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            if (w == 0)
#pragma unroll
              for (int i = 0; i < 4; ++i) g[mt][i] = 0.f;
            if (V == 10) {  // dequant only: results stored to SMEM (stands in for tcgen05.st to TMEM)
              if (mt == 0) {
                const uint32_t dst = sbase + NS * STAGE + (warp * 32 + lane) * 32;
                asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};\n" :: "r"(dst), "r"(hA[0]), "r"(hA[1]), "r"(hA[2]), "r"(hA[3]) : "memory");
                asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};\n" :: "r"(dst + 16), "r"(hB[0]), "r"(hB[1]), "r"(hB[2]), "r"(hB[3]) : "memory");
              }
              continue;
            }
            if (V == 8) {
              uint32_t t0 = hfma2u(hA[0], xb[mt][w][0], hB[0]);
              uint32_t t1 = hfma2u(hA[1], xb[mt][w][1], hB[1]);
              uint32_t t2 = hfma2u(hA[2], xb[mt][w][2], hB[2]);
              uint32_t t3 = hfma2u(hA[3], xb[mt][w][3], hB[3]);
              g[mt][0] += __uint_as_float(t0 ^ t2);
              g[mt][1] += __uint_as_float(t1 ^ t3);
              continue;
            }
            mma(g[mt], hA[0], hB[0], hA[1], hB[1], xb[mt][w][0], xb[mt][w][1]);
            mma(g[mt], hA[2], hB[2], hA[3], hB[3], xb[mt][w][2], xb[mt][w][3]);
          }
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          acc[rt][mt][0] = fmaf(g[mt][0], dA, acc[rt][mt][0]);
          acc[rt][mt][1] = fmaf(g[mt][1], dA, acc[rt][mt][1]);
          acc[rt][mt][2] = fmaf(g[mt][2], dB, acc[rt][mt][2]);
          acc[rt][mt][3] = fmaf(g[mt][3], dB, acc[rt][mt][3]);
        }
      } else {
        if (V != 3) {
          zA = __half2float(__ushort_as_half(lds16(sbz + rt * 32)));
          zB = __half2float(__ushort_as_half(lds16(sbz + rt * 32 + 16)));
        }
        // accumulator starts at -(1024 (se + so) + Z (se + 16 so)) so g ends as sum x (q - Z)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float z = i < 2 ? zA : zB;
            const float e = sxe[mt][i & 1], o = sxo[mt][i & 1];
            g[mt][i] = -fmaf(z + 1024.f, e, (16.f * z + 1024.f) * o);
          }
        if (V == 6) {  // exact (q - Z) without activation sums: 4 ALU + 6 FMA per 8 codes
          const float zz[2] = {zA, zB};
          uint32_t zs[2], z16[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t zi = (uint32_t)zz[h];
            zs[h] = zi * 0x00010001u + 0x64006400u;   // 1024 + Z
            z16[h] = __half_as_ushort(__float2half(16.f * zz[h])) * 0x00010001u;
          }
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int i = 0; i < 4; ++i) g[mt][i] = 0.f;
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            uint32_t lo0[2], hi0[2], lo1[2], hi1[2];
            const uint32_t ww[2] = {wa[w], wb[w]};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t c02 = lop3_and_or(ww[h], 0x00FF00FFu, 0x64006400u);
              const uint32_t l02 = lop3_and_or(ww[h], 0x000F000Fu, 0x64006400u);
              const uint32_t c13 = prmt(ww[h], 0x64646464u, 0x4341u);
              const uint32_t l13 = lop3_and_or(c13, 0xFF0FFF0Fu, 0u);
              lo0[h] = hsub2u(l02, zs[h]);
              lo1[h] = hsub2u(l13, zs[h]);
              hi0[h] = hsub2u(hsub2u(c02, l02), z16[h]);
              hi1[h] = hsub2u(hsub2u(c13, l13), z16[h]);
            }
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              mma(g[mt], lo0[0], lo0[1], lo1[0], lo1[1], xb[mt][w][0], xb[mt][w][2]);
              mma(g[mt], hi0[0], hi0[1], hi1[0], hi1[1], xb[mt][w][1], xb[mt][w][3]);
            }
          }
        } else if (V == 5 || V == 7) {  // 4 ALU + 2 FMA per 8 codes, activation-sum correction
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float z = i < 2 ? zA : zB;
              g[mt][i] = -fmaf(z + 1024.f, sxe[mt][i & 1], 16.f * z * sxo[mt][i & 1]);
            }
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            uint32_t lo0[2], hi0[2], lo1[2], hi1[2];
            const uint32_t ww[2] = {wa[w], wb[w]};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t c02 = lop3_and_or(ww[h], 0x00FF00FFu, 0x64006400u);
              lo0[h] = lop3_and_or(ww[h], 0x000F000Fu, 0x64006400u);
              const uint32_t c13 = prmt(ww[h], 0x64646464u, 0x4341u);
              lo1[h] = lop3_and_or(c13, 0xFF0FFF0Fu, 0u);
              hi0[h] = hsub2u(c02, lo0[h]);
              hi1[h] = hsub2u(c13, lo1[h]);
            }
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              mma(g[mt], lo0[0], lo0[1], lo1[0], lo1[1], xb[mt][w][0], xb[mt][w][2]);
              mma(g[mt], hi0[0], hi0[1], hi1[0], hi1[1], xb[mt][w][1], xb[mt][w][3]);
            }
          }
        } else
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          uint32_t ta, tb;
          if (V == 1 || V == 4) {
            ta = wa[w] >> 8;
            tb = wb[w] >> 8;
          } else {
            ta = __umulhi(wa[w], 0x1000000u);
            tb = __umulhi(wb[w], 0x1000000u);
          }
          const uint32_t la0 = lop3_and_or(wa[w], 0x000F000Fu, 0x64006400u);
          const uint32_t la1 = lop3_and_or(ta, 0x000F000Fu, 0x64006400u);
          const uint32_t ha0 = lop3_and_or(wa[w], 0x00F000F0u, 0x64006400u);
          const uint32_t ha1 = lop3_and_or(ta, 0x00F000F0u, 0x64006400u);
          const uint32_t lb0 = lop3_and_or(wb[w], 0x000F000Fu, 0x64006400u);
          const uint32_t lb1 = lop3_and_or(tb, 0x000F000Fu, 0x64006400u);
          const uint32_t hb0 = lop3_and_or(wb[w], 0x00F000F0u, 0x64006400u);
          const uint32_t hb1 = lop3_and_or(tb, 0x00F000F0u, 0x64006400u);
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            mma(g[mt], la0, lb0, la1, lb1, xb[mt][w][0], xb[mt][w][2]);
            mma(g[mt], ha0, hb0, ha1, hb1, xb[mt][w][1], xb[mt][w][3]);
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
    }
  }
  float s = 0.f;
#pragma unroll
  for (int a = 0; a < RT; ++a)
#pragma unroll
    for (int b = 0; b < MT; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) s += acc[a][b][c];
  if (s == 1234.5f) out[0] = s;
  long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int V, int MT, int CW>
void run(int sms, int ctas_per_sm, float* out, long long* clk) {
  const int smem = NS * STAGE + CW * 32 * 32;
  cudaFuncSetAttribute(kern<V, MT, CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000;
  const int grid = sms * ctas_per_sm;
  kern<V, MT, CW><<<grid, CW * 32, smem>>>(100, out, clk);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<V, MT, CW><<<grid, CW * 32, smem>>>(iters, out, clk);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  static long long h[4096];
  cudaMemcpy(h, clk, grid * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  const double weights = (double)grid * iters * BN * GPS * 128;
  const double gw = weights / (ms * 1e-3) / 1e9;
  printf("variant %d MT=%d CW=%d ctas/SM=%d: %8.1f Gw/s = %5.2f TB/s W4   %5.1f weights/clk/SM (%.0f MHz)  %s\n", V, MT, CW,
         ctas_per_sm, gw, gw * 0.53125 / 1e3, weights / sms / mx, (double)mx / (ms * 1e3),
         cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* clk;
  cudaMalloc(&out, 16);
  cudaMalloc(&clk, 4096 * sizeof(long long));
  if (argc == 3) {  // single config for ncu: variant, ctas/SM (MT = 1, CW = 4)
    const int v = atoi(argv[1]), c = atoi(argv[2]);
    if (v == 0) run<0, 1, 4>(sms, c, out, clk);
    if (v == 1) run<1, 1, 4>(sms, c, out, clk);
    if (v == 4) run<4, 1, 4>(sms, c, out, clk);
    if (v == 5) run<5, 1, 4>(sms, c, out, clk);
    if (v == 6) run<6, 1, 4>(sms, c, out, clk);
    if (v == 7) run<7, 1, 4>(sms, c, out, clk);
    return 0;
  }
  for (int c = 2; c <= 4; c += 1) {
    run<0, 1, 4>(sms, c, out, clk);
    run<12, 1, 4>(sms, c, out, clk);
    run<0, 2, 4>(sms, c, out, clk);
    run<12, 2, 4>(sms, c, out, clk);
  }
  return 0;
}
