// Microbenchmark: read-only HBM streaming ceiling on B200 for the access patterns a
// W4A16 decode kernel can use over packed codes Wq[N][K/2] (development tool).
//   ldg    : grid-stride LDG.128 (ld.global.nc.L1::no_allocate), U loads in flight
//   ldgrow : the mma.sync fragment pattern straight from global: lane (r, j) of a warp
//            loads rows r and r+8, 16 B at j*16 of one 64-B group slice
//   tma3   : TMA 3-D box (64 B x BN rows x GPS groups) into an NS-stage ring, producer warp
//            + 4 consumer warps that only touch one word per stage (current decode pattern)
//   bulk   : cp.async.bulk 1-D of contiguous chunks, same ring
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_pattern hbm_pattern.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint4 ldg_nc(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

template <int U>
__global__ void __launch_bounds__(256) k_ldg(const uint4* __restrict__ a, size_t n16, uint32_t* out) {
  const size_t T = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (; i + (U - 1) * T < n16; i += U * T) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldg_nc(a + i + u * T);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n16; i += T) { uint4 v = ldg_nc(a + i); acc ^= v.x ^ v.w; }
  if (acc == 0x12345678u) out[0] = acc;
}

// rows x (K/2) bytes; work item = (16-row tile, group of 64 B); warps take contiguous ranges
template <int U>
__global__ void __launch_bounds__(256) k_ldgrow(const uint8_t* __restrict__ w, int N, int K, uint32_t* out) {
  const int lane = threadIdx.x & 31, r = lane >> 2, j = lane & 3;
  const int G = K / 128;
  const long long items = (long long)(N / 16) * G;
  const long long W = (long long)gridDim.x * (blockDim.x / 32);
  const long long wid = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const long long q = items / W, rem = items % W;
  const long long b = wid * q + (wid < rem ? wid : rem), e = b + q + (wid < rem ? 1 : 0);
  uint32_t acc = 0;
  long long it = b;
  for (; it + U <= e; it += U) {
    uint4 va[U], vb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long x = it + u;
      const int rt = (int)(x / G), g = (int)(x % G);
      const uint8_t* p = w + (size_t)(rt * 16 + r) * (K / 2) + g * 64 + j * 16;
      va[u] = ldg_nc(p);
      vb[u] = ldg_nc(p + (size_t)8 * (K / 2));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= va[u].x ^ vb[u].y ^ va[u].z ^ vb[u].w;
  }
  for (; it < e; ++it) {
    const int rt = (int)(it / G), g = (int)(it % G);
    const uint8_t* p = w + (size_t)(rt * 16 + r) * (K / 2) + g * 64 + j * 16;
    uint4 v = ldg_nc(p);
    acc ^= v.x;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(bar), "r"(ph) : "memory");
}

// mode 0: TMA 3-D box (64, BN, GPS) over dims (64, N, G); mode 1: 1-D bulk of STAGE bytes
template <int NS>
__global__ void __launch_bounds__(160) k_ring(const __grid_constant__ CUtensorMap tm, const uint8_t* w, int mode,
                                              int N, int G, int BN, int GPS, long long total_bytes, uint32_t* out, int hold) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const int STAGE = 64 * BN * GPS;
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;\n" ::"r"(smem_u32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const long long units = mode == 0 ? (long long)(N / BN) * (G / GPS) : total_bytes / STAGE;
  const long long P = gridDim.x, c = blockIdx.x;
  const long long q = units / P, rem = units % P;
  const long long ub = c * q + (c < rem ? c : rem), ue = ub + q + (c < rem ? 1 : 0);
  if (warp == 4) {
    if (lane == 0) {
      int s = 0; uint32_t ph = 0;
      for (long long u = ub; u < ue; ++u) {
        mbar_wait(smem_u32(&empty[s]), ph ^ 1);
        const uint32_t fb = smem_u32(&full[s]);
        const uint32_t dst = smem_u32(sm + s * STAGE);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(fb), "r"(STAGE) : "memory");
        if (mode == 0) {
          const int upb = G / GPS;
          const int rb = (int)(u / upb), g0 = (int)(u % upb) * GPS;
          asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n"
                       ::"r"(dst), "l"((uint64_t)&tm), "r"(fb), "r"(0), "r"(rb * BN), "r"(g0) : "memory");
        } else {
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                       ::"r"(dst), "l"(w + u * STAGE), "r"(STAGE), "r"(fb) : "memory");
        }
        if (++s == NS) { s = 0; ph ^= 1; }
      }
    }
    return;
  }
  uint32_t acc = 0;
  int s = 0; uint32_t ph = 0;
  for (long long u = ub; u < ue; ++u) {
    mbar_wait(smem_u32(&full[s]), ph);
    acc ^= *(volatile uint32_t*)(sm + s * STAGE + warp * 64 + lane * 4);
    if (hold) { const long long t0 = clock64(); while (clock64() - t0 < hold) {} }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&empty[s])) : "memory");
    if (++s == NS) { s = 0; ph ^= 1; }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return (PFN_cuTensorMapEncodeTiled_v12000)p;
}

int main(int argc, char** argv) {
  const int N = 44032, K = 8192;
  const size_t bytes = (size_t)N * K / 2;  // 180 MB, one buffer
  const int NB = 3;
  uint8_t* buf[NB];
  for (int i = 0; i < NB; ++i) { CK(cudaMalloc(&buf[i], bytes)); CK(cudaMemset(buf[i], i + 1, bytes)); }
  uint32_t* out; CK(cudaMalloc(&out, 4));
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int R = 30;
  auto report = [&](const char* name, auto&& launch) {
    for (int i = 0; i < 3; ++i) launch(buf[i % NB]);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int i = 0; i < R; ++i) launch(buf[i % NB]);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("%-48s %8.1f GB/s  (%.1f us/launch)\n", name, bytes * (double)R / (ms * 1e-3) / 1e9, ms * 1e3 / R);
  };
  char nm[128];
  for (int occ : {4}) {
    snprintf(nm, sizeof nm, "ldg U=4 grid=%dx%d", sms, occ);
    report(nm, [&](uint8_t* b) { k_ldg<4><<<sms * occ, 256>>>((const uint4*)b, bytes / 16, out); });
    snprintf(nm, sizeof nm, "ldg U=8 grid=%dx%d", sms, occ);
    report(nm, [&](uint8_t* b) { k_ldg<8><<<sms * occ, 256>>>((const uint4*)b, bytes / 16, out); });
  }
  for (int occ : {8}) {
    snprintf(nm, sizeof nm, "ldgrow U=4 grid=%dx%d", sms, occ);
    report(nm, [&](uint8_t* b) { k_ldgrow<4><<<sms * occ, 256>>>(b, N, K, out); });
    snprintf(nm, sizeof nm, "ldgrow U=8 grid=%dx%d", sms, occ);
    report(nm, [&](uint8_t* b) { k_ldgrow<8><<<sms * occ, 256>>>(b, N, K, out); });
  }
  auto encf = enc();
  struct Cfg { int mode, BN, GPS, occ, ns, hold; };
  Cfg cfgs[64]; int nc = 0;
  if (argc > 1 && !strcmp(argv[1], "prefill")) {
    // the prefill codes ring: one group per box (64-B rows) vs several groups per box
    cfgs[nc++] = {0, 128, 1, 1, 12, 0};
    cfgs[nc++] = {0, 128, 1, 1, 24, 0};
    cfgs[nc++] = {0, 128, 2, 1, 12, 0};
    cfgs[nc++] = {0, 128, 4, 1, 6, 0};
    cfgs[nc++] = {0, 64, 4, 2, 4, 0};
  } else {
    const int holds[] = {0, 500, 1000, 1500};
    for (int h : holds) {
      for (int ns : {3, 4, 6}) cfgs[nc++] = {0, 64, 4, 2, ns, h};
      cfgs[nc++] = {0, 64, 4, 1, 12, h};
      cfgs[nc++] = {1, 64, 4, 2, 6, h};
    }
  }
  for (int ci = 0; ci < nc; ++ci) {
    Cfg cf = cfgs[ci];
    CUtensorMap tm[NB];
    for (int i = 0; i < NB; ++i) {
      cuuint64_t d[3] = {64, (cuuint64_t)N, (cuuint64_t)(K / 128)};
      cuuint64_t st[2] = {(cuuint64_t)K / 2, 64};
      cuuint32_t bx[3] = {64, (cuuint32_t)cf.BN, (cuuint32_t)cf.GPS}, es[3] = {1, 1, 1};
      if (encf(&tm[i], CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, buf[i], d, st, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed\n"); return 1;
      }
    }
    const int STAGE = 64 * cf.BN * cf.GPS;
    const int smem = cf.ns * STAGE + 1024;
    void (*kp)(CUtensorMap, const uint8_t*, int, int, int, int, int, long long, uint32_t*, int) =
        cf.ns == 3 ? k_ring<3> : cf.ns == 4 ? k_ring<4> : cf.ns == 6 ? k_ring<6> : cf.ns == 12 ? k_ring<12> : k_ring<24>;
    CK(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    snprintf(nm, sizeof nm, "%s BN=%d GPS=%d (%d KB) NS=%d occ=%d hold=%d", cf.mode ? "bulk" : "tma3", cf.BN, cf.GPS,
             STAGE / 1024, cf.ns, cf.occ, cf.hold);
    report(nm, [&](uint8_t* b) {
      int i = b == buf[0] ? 0 : b == buf[1] ? 1 : 2;
      kp<<<sms * cf.occ, 160, smem>>>(tm[i], b, cf.mode, N, K / 128, cf.BN, cf.GPS, (long long)bytes, out, cf.hold);
    });
  }
  return 0;
}
