// Shared pieces of the decode kernel (k_decode.cu) and its variants: the exact
// int4 -> (q - Z) conversion and the persistent stream-K / row-block work split.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "sq_internal.cuh"

namespace sq {
namespace dec {

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

// zero-point constants from the integer Z (0..15)
template <bool kBF16>
__device__ __forceinline__ void zero_consts_q(uint32_t z, uint32_t& zsub, uint32_t& zfma) {
  if (!kBF16) {
    zsub = z * 0x00010001u + 0x64006400u;         // fp16x2(1024 + Z): ulp of 1024 is 1
    zfma = z * 0x00100010u + 0xD400D400u;         // fp16x2(-(64 + Z)): ulp of 64 is 1/16
  } else {
    zsub = z * 0x00010001u + 0x43004300u;         // bf16x2(128 + Z): ulp of 128 is 1
    zfma = 0;
  }
}
// Z of weight row `row` in a stage's zero rows: fp16 bits (uint16 per row), or packed u4
// (SQ_ZEROS_U4: uint8 per row pair, low nibble = even row).  zrow: shared address of the
// stage's zero row (fp16: row 0's element; u4: row 0's byte).
__device__ __forceinline__ uint32_t load_zero(uint32_t zrow, int row, bool u4) {
  if (u4) {
    uint32_t b;
    asm("ld.shared.u8 %0, [%1];\n" : "=r"(b) : "r"(zrow + (uint32_t)(row >> 1)) : "memory");
    return (b >> (4 * (row & 1))) & 0xFu;
  }
  uint16_t h;
  asm("ld.shared.u16 %0, [%1];\n" : "=h"(h) : "r"(zrow + 2u * (uint32_t)row) : "memory");
  return (uint32_t)__half2int_rn(__ushort_as_half(h));
}

// Work split.  Units are numbered u = rb * upb + pos (row block rb, stage pos).
//  stream-K (dp = 0): CTA c owns the contiguous range [start(c), start(c + 1)).
//  row-block (dp = 1): CTA c owns row blocks c, c + P, c + 2P, ... (each a full range).
struct Work {
  int units, upb, cta_q, cta_r, rbs, dp;
  __device__ __forceinline__ int start(int c) const { return c * cta_q + min(c, cta_r); }
  __device__ __forceinline__ int cta_of(int u) const {
    const int big = (cta_q + 1) * cta_r;
    return u < big ? u / (cta_q + 1) : cta_r + (u - big) / cta_q;
  }
};

// Walks the units of one CTA in processing order (identical in all three warp roles) as
// segments: contiguous unit ranges inside one row block.  Stream-K processes a CTA's
// partial row blocks (the head and tail of its range) FIRST and its whole row blocks
// after them, so the fixups of cut row blocks overlap the rest of the stream and the
// kernel ends on plain Y stores instead of fixup round trips.
struct Sched {
  int c, P, ri, nr, u, ue;
  int u0, u1, hp, tp, nparts, f_lo;
  bool full;  // the segment is a whole row block (direct Y store)
  int e;      // partial-slot index: 0 = head of the CTA's range, 1 = tail
  int rb;     // row block of the current segment
  int pos;    // stage (group quad) of the current unit inside its row block: u - rb * upb
  __device__ __forceinline__ Sched(const Work& wk, int c_, int P_) : c(c_), P(P_), ri(0) {
    if (wk.dp) {
      nr = (wk.rbs - c + P - 1) / P;
    } else {
      u0 = wk.start(c);
      u1 = wk.start(c + 1);
      const int rb_a = u0 / wk.upb, rb_b = (u1 - 1) / wk.upb;
      if (rb_a == rb_b) {
        hp = 1;
        tp = 0;
        nparts = 1;
        nr = 1;
      } else {
        hp = u0 % wk.upb != 0;
        tp = u1 % wk.upb != 0;
        nparts = hp + tp;
        f_lo = hp ? rb_a + 1 : rb_a;
        const int f_hi = tp ? rb_b - 1 : rb_b;
        nr = nparts + max(0, f_hi - f_lo + 1);
      }
    }
    load(wk);
  }
  __device__ __forceinline__ void load(const Work& wk) {
    if (ri >= nr) return;
    set_unit(wk);
    rb = u / wk.upb;  // one division per segment
    pos = u - rb * wk.upb;
  }
  __device__ __forceinline__ void set_unit(const Work& wk) {
    if (wk.dp) {
      u = (c + ri * P) * wk.upb;
      ue = u + wk.upb;
      full = true;
      e = 0;
    } else if (nr == 1 && nparts == 1 && hp && (u1 - 1) / wk.upb == u0 / wk.upb) {
      u = u0;  // the whole range lies in one row block
      ue = u1;
      full = (u0 % wk.upb == 0) && (u1 - u0 == wk.upb);
      e = 0;
    } else if (ri < nparts) {
      if (hp && ri == 0) {
        u = u0;
        ue = (u0 / wk.upb + 1) * wk.upb;
        e = 0;
      } else {
        u = ((u1 - 1) / wk.upb) * wk.upb;
        ue = u1;
        e = 1;
      }
      full = false;
    } else {
      u = (f_lo + ri - nparts) * wk.upb;
      ue = u + wk.upb;
      full = true;
      e = 0;
    }
  }
  __device__ __forceinline__ bool valid() const { return ri < nr; }
  __device__ __forceinline__ bool range_last() const { return u + 1 == ue; }
  __device__ __forceinline__ void next(const Work& wk) {
    ++pos;
    if (++u == ue) {
      ++ri;
      load(wk);
    }
  }
};

}  // namespace dec
}  // namespace sq
