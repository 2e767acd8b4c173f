// Microbenchmark: issue rate of tcgen05.mma.cta_group::1.kind::f16 (M = 128, K = 16) with
// A from TMEM ("ts") or SMEM ("ss") and N in {16, 32, 64, 128, 256}; one CTA per SM,
// one issuing thread, R MMAs back to back, optional tcgen05.commit + mbarrier wait every
// `every` MMAs.  Prints cycles per MMA (development tool; nvcc -arch=sm_100a).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ uint32_t idesc(int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__global__ void kern(int R, int n, int ts, int every, int nacc, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&holder)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = holder;
  if (every < 0 && warp == 0) {
    // warp-uniform loop: descriptors precomputed, per-step increments only, one elected lane issues
    const uint32_t sb = smem_u32(smem);
    const uint32_t id = idesc(n);
    const uint64_t b0 = desc_sw128(sb);
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int i = 0; i < R; i += 4) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t bdesc = b0 + (uint64_t)(kk * 2);  // +32 B per k-step (addr >> 4)
        const uint32_t a = tmem + 480 + kk * 8;
        const uint32_t dcol = (uint32_t)((kk % nacc) * n);
        const uint32_t acc = (i | kk) >= nacc ? 1u : 0u;
        asm volatile("{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(tmem + dcol), "r"(a), "l"(bdesc), "r"(id), "r"(acc) : "memory");
      }
    }
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(smem_u32(&bar)), "r"(ph) : "memory");
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
  } else if (every >= 0 && threadIdx.x == 0) {
    const uint32_t sb = smem_u32(smem);
    const uint32_t id = idesc(n);
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int i = 0; i < R; ++i) {
      const uint64_t bdesc = desc_sw128(sb + (i & 3) * 32);
      const uint32_t acc = i >= nacc ? 1u : 0u;
      const uint32_t dcol = (uint32_t)((i % nacc) * n);  // independent accumulators
      if (ts) {
        const uint32_t a = tmem + 480 + (i & 3) * 8;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(tmem + dcol), "r"(a), "l"(bdesc), "r"(id), "r"(acc) : "memory");
      } else {
        const uint64_t adesc = desc_sw128(sb + 65536 + (i & 3) * 32);
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tmem + dcol), "l"(adesc), "l"(bdesc), "r"(id), "r"(acc) : "memory");
      }
      if (every && (i + 1) % every == 0) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(smem_u32(&bar)), "r"(ph) : "memory");
        ph ^= 1;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(smem_u32(&bar)), "r"(ph) : "memory");
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  const int R = 4096;
  for (int nacc : {1, 2})
    for (int n : {16, 64, 128, 256}) {
      if (nacc * n > 480) continue;
      for (int rep = 0; rep < 2; ++rep) kern<<<148, 128, 140 * 1024>>>(R, n, 1, -1, nacc, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h = 0;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("warp-uniform A=TMEM N=%3d accumulators %d: %7.1f cyc/MMA (floor %5.1f) %s\n", n, nacc,
             (double)h / R, 128.0 * n / 256.0, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  for (int ts = 1; ts >= 0; --ts)
    for (int nacc : {1, 2, 4})
      for (int n : {16, 64, 128, 256}) {
        if (nacc * n > 480 && ts) continue;
        if (nacc * n > 512) continue;
        for (int rep = 0; rep < 2; ++rep) kern<<<148, 128, 140 * 1024>>>(R, n, ts, 0, nacc, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h = 0;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        const double floor_c = 128.0 * n / 256.0;
        printf("%s N=%3d accumulators %d: %7.1f cyc/MMA (floor %5.1f) %s\n", ts ? "A=TMEM" : "A=SMEM", n,
               nacc, (double)h / R, floor_c, e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
