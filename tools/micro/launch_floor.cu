// Microbenchmark: per-launch floor of a dependent kernel chain on B200 (development tool).
// 48 launches in a CUDA graph, each kernel waits on its predecessor (griddepcontrol.wait)
// and writes one value; variants: PDL on/off, grid 1 / 148 / 296 CTAs, dynamic smem 0 /
// 112 KB per CTA (the decode kernel's footprint), optional L2 read of a 16-KB input after
// the wait (the decode kernel's activation fetch).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_floor launch_floor.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void chain_kernel(const float* __restrict__ in, float* __restrict__ out, int read_in) {
  extern __shared__ float sm[];
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  float v = 0.0f;
  if (read_in) {
    // every CTA reads the same 16 KB (like X at M = 1, K = 8192), 16 B per thread
    const float4* p = reinterpret_cast<const float4*>(in);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
      float4 t = p[i];
      v += t.x + t.y + t.z + t.w;
    }
    sm[threadIdx.x] = v;
    __syncthreads();
    v = sm[(threadIdx.x + 1) % blockDim.x];
  }
  if (threadIdx.x == 0) out[blockIdx.x] = v + 1.0f;
}

int main() {
  float *in, *out;
  CK(cudaMalloc(&in, 1 << 20));
  CK(cudaMalloc(&out, 1 << 20));
  CK(cudaMemset(in, 0, 1 << 20));
  CK(cudaFuncSetAttribute(chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 114 * 1024));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int L = 48;
  for (int pdl = 0; pdl < 2; ++pdl)
    for (int grid : {1, 148, 296})
      for (int smem : {0, 112 * 1024})
        for (int rd = 0; rd < 2; ++rd) {
          cudaGraph_t g;
          cudaGraphExec_t ge;
          CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
          for (int i = 0; i < L; ++i) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(192);
            cfg.dynamicSmemBytes = smem + 192 * 4;
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = pdl;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            CK(cudaLaunchKernelEx(&cfg, chain_kernel, (const float*)in, out, rd));
          }
          CK(cudaStreamEndCapture(st, &g));
          CK(cudaGraphInstantiate(&ge, g, 0));
          for (int w = 0; w < 3; ++w) CK(cudaGraphLaunch(ge, st));
          CK(cudaStreamSynchronize(st));
          float best = 1e30f;
          for (int r = 0; r < 10; ++r) {
            CK(cudaEventRecord(e0, st));
            CK(cudaGraphLaunch(ge, st));
            CK(cudaEventRecord(e1, st));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (ms < best) best = ms;
          }
          printf("pdl=%d grid=%3d smem=%6d read16KB=%d : %.2f us/launch\n", pdl, grid, smem, rd,
                 best * 1e3f / L);
          CK(cudaGraphExecDestroy(ge));
          CK(cudaGraphDestroy(g));
        }
  return 0;
}
