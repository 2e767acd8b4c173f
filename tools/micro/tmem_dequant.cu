// Microbenchmark: throughput of the per-row dequant of a tcgen05 decode design (thread =
// weight row = TMEM lane, one 128-k group per iteration): 4 LDS.128 of the row's codes
// (SWIZZLE_64B-style addressing), exact (q - Z) fp16 pairs (lop3 magic + hsub2/hfma2),
// two tcgen05.st.32x32b.x32 into a TMEM A ring, wait::st, and the per-group readback of
// an N-token accumulator (tcgen05.ld + N FFMA with Δ).  No MMA, no global memory.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_dequant tmem_dequant.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t m, uint32_t o) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;\n" : "=r"(r) : "r"(a), "r"(m), "r"(o));
  return r;
}
__device__ __forceinline__ uint32_t hsub2u(uint32_t a, uint32_t b) {
  __half2 r = __hsub2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t hfma2u(uint32_t a, uint32_t b, uint32_t c) {
  __half2 r = __hfma2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b), *reinterpret_cast<__half2*>(&c));
  return *reinterpret_cast<uint32_t*>(&r);
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
__device__ __forceinline__ void tst32(uint32_t taddr, const uint32_t* v) {
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
__device__ __forceinline__ void tld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}

template <int NT>  // tokens read back per group (0: no readback)
__global__ void kern(int iters, int tmem_cols, float* out, long long* clk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t holder;
  long long t0 = clock64();
  for (int i = threadIdx.x; i < 4 * 8192 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x76543210u ^ (i * 2654435761u);
  for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x)
    reinterpret_cast<uint16_t*>(smem + 4 * 8192)[i] = (i & 1) ? 0x4400 : 0x2E66;  // Z = 4, Δ ~ 0.1
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&holder)), "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = holder;
  const int q = warp % 4, set = warp / 4;
  const int row = q * 32 + lane;
  const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const int nsets = blockDim.x / 128;
  const int abufs = (tmem_cols - 64) / 64 / nsets;  // A ring per set (64 columns per group)
  float acc[NT > 0 ? NT : 1];
#pragma unroll
  for (int t = 0; t < (NT > 0 ? NT : 1); ++t) acc[t] = 0.f;
  for (int it = 0; it < iters; ++it) {
    const int st = it & 3;  // 4 code stages of 8 KB ([row][64 B], 64B-swizzled chunks)
    const uint32_t crow = sbase + st * 8192 + row * 64;
    const int sw = (row >> 1) & 3;
    uint32_t w[16];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 v = lds128(crow + ((c ^ sw) << 4));
      w[4 * c] = v.x; w[4 * c + 1] = v.y; w[4 * c + 2] = v.z; w[4 * c + 3] = v.w;
    }
    const uint32_t zq = (uint32_t)__half2int_rn(__ushort_as_half(lds16(sbase + 4 * 8192 + st * 512 + row * 2 + 256)));
    const float d = __half2float(__ushort_as_half(lds16(sbase + 4 * 8192 + st * 512 + row * 2)));
    const uint32_t zs = zq * 0x00010001u + 0x64006400u, zf = zq * 0x00100010u + 0xD400D400u;
    uint32_t a[64];
    uint32_t v[NT > 0 ? NT : 1];
    if (NT > 0) {  // readback of an older group's accumulator, issued before this group's math
#pragma unroll
      for (int h = 0; h < NT / 8; ++h)
        tld8(tmem + lane_addr + (uint32_t)(h * 8), *reinterpret_cast<uint32_t(*)[8]>(&v[h * 8]));
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const uint32_t t = w[k] >> 8;
      a[4 * k + 0] = hsub2u(lop3_and_or(w[k], 0x000F000Fu, 0x64006400u), zs);
      a[4 * k + 1] = hfma2u(lop3_and_or(w[k], 0x00F000F0u, 0x64006400u), 0x2C002C00u, zf);
      a[4 * k + 2] = hsub2u(lop3_and_or(t, 0x000F000Fu, 0x64006400u), zs);
      a[4 * k + 3] = hfma2u(lop3_and_or(t, 0x00F000F0u, 0x64006400u), 0x2C002C00u, zf);
    }
    const uint32_t abase = tmem + lane_addr + 64 + (uint32_t)((set * abufs + it % abufs) * 64);
    tst32(abase, a);
    tst32(abase + 32, a + 32);
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    if (NT > 0) {
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int t = 0; t < NT; ++t) acc[t] = fmaf(__uint_as_float(v[t]), d, acc[t]);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int t = 0; t < (NT > 0 ? NT : 1); ++t) s += acc[t];
  if (s == 1234.5f) out[0] = s;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(tmem_cols));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int NT>
void run(int sms, int warps, int ctas, float* out, long long* clk) {
  const int smem = 4 * 8192 + 4 * 512;
  const int cols = ctas == 1 ? 512 : 256;
  cudaFuncSetAttribute(kern<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 20000, grid = sms * ctas;
  kern<NT><<<grid, warps * 32, smem>>>(100, cols, out, clk);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<NT><<<grid, warps * 32, smem>>>(iters, cols, out, clk);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  static long long h[4096];
  cudaMemcpy(h, clk, grid * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  const double weights = (double)grid * warps * 32 * iters * 128;
  const double gw = weights / (ms * 1e-3) / 1e9;
  printf("NT=%2d warps=%2d ctas/SM=%d: %8.1f Gw/s = %5.2f TB/s W4  %6.1f weights/clk/SM  %s\n", NT, warps, ctas, gw,
         gw * 0.53125 / 1e3, weights / sms / mx, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* clk;
  cudaMalloc(&out, 16);
  cudaMalloc(&clk, 4096 * sizeof(long long));
  for (int w : {4, 8, 12}) {
    run<0>(sms, w, 1, out, clk);
    run<8>(sms, w, 1, out, clk);
    run<16>(sms, w, 1, out, clk);
  }
  for (int w : {4, 8}) {
    run<8>(sms, w, 2, out, clk);
    run<16>(sms, w, 2, out, clk);
  }
  return 0;
}
