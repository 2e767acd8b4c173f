// K-ar: one-shot all-reduce of row-parallel partial outputs over peer memory
// (the collective after o_proj / down_proj, §8(e)).
//
// Every rank owns a symmetric buffer (the same layout on every rank, opened by its peers
// through CUDA IPC, i.e. NVLink/NVSwitch loads and stores between GPUs):
//
//   [header 128 B: epoch counter, done counter][flags: 2 parities x world x kArMaxChunks
//    uint32][slots: 2 parities x world x n_max elements, 4-byte stride] (sq_internal.cuh)
//
// Call `epoch` e on rank r (e > 0 given by the caller, +1 per call; or e == 0: taken from
// the rank's own device counter + 1 and stored back by the last CTA, so a CUDA graph that
// replays the launch advances it -- the counters of all ranks move in lock step because
// every rank makes the same sequence of calls), chunk c of the
// n outputs (one CTA per chunk, no grid-wide barrier):
//   1. push: copy the chunk of r's partial Y into slot[e & 1][r] of EVERY rank's buffer
//      (16-B peer stores);
//   2. publish: a system-scope fence per thread, a CTA barrier, then flag[e & 1][r][c] = e
//      on every rank (st.release.sys);
//   3. wait: until flag[e & 1][q][c] == e in r's own buffer for every rank q (ld.acquire.sys);
//   4. reduce: Y[c] = RN( sum_q slot[e & 1][q][c] ) in fp32, q = 0 .. world-1 in rank
//      order, so every rank computes the bit-identical result.
// Double buffering by epoch parity makes back-to-back calls safe: rank r can only push call
// e+2 into parity e & 1 after every rank has published call e+1, i.e. finished reading e.
// The wait is bounded (~2^24 polls with backoff): on timeout the kernel records an error
// code in the rank's error word instead of hanging the GPU.
#include "sq_internal.cuh"

namespace sq {

namespace {

constexpr int kArThreads = 256;
constexpr int kArChunkVec = kArThreads;           // 16-B vectors per chunk (4 KB of outputs)
constexpr int kArChunkElems = kArChunkVec * 8;    // 2048 fp16 / bf16 outputs per chunk

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <bool kBF16>
__device__ __forceinline__ float to_f(uint16_t b) {
  return kBF16 ? __bfloat162float(__ushort_as_bfloat16(b)) : __half2float(__ushort_as_half(b));
}
template <bool kBF16>
__device__ __forceinline__ uint16_t from_f(float v) {
  return kBF16 ? __bfloat16_as_ushort(__float2bfloat16_rn(v)) : __half_as_ushort(__float2half_rn(v));
}

template <bool kBF16>
__global__ void __launch_bounds__(kArThreads)
oneshot_allreduce_kernel(const uint16_t* y_local, uint16_t* y_out, int64_t n,  // may alias
                         int64_t n_max, uint8_t* const* __restrict__ peers, int rank, int world,
                         uint32_t epoch, int* __restrict__ err) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");  // y_local is the previous kernel's output
  const bool device_epoch = epoch == 0;
  const int c = blockIdx.x;
  uint32_t* hdr = reinterpret_cast<uint32_t*>(peers[rank]);
  if (epoch == 0) {  // device-managed epoch (graph replays)
    const uint32_t cur = *reinterpret_cast<volatile uint32_t*>(hdr);
    epoch = cur == 0xFFFFFFFFu ? 2u : cur + 1u;  // never 0; parity alternates across the wrap
  }
  const int par = epoch & 1;
  const int64_t e0 = (int64_t)c * kArChunkElems;
  const int64_t e1 = min(n, e0 + kArChunkElems);
  auto flags_of = [&](uint8_t* base) {
    return reinterpret_cast<uint32_t*>(base + ar_flags_offset()) + (size_t)par * world * kArMaxChunks;
  };
  auto slots_of = [&](uint8_t* base, int q) {
    return reinterpret_cast<uint16_t*>(base + ar_slot_offset(world, par, q, n_max));
  };
  // 1. push this rank's chunk to every rank's slot [par][rank]
  const int64_t i = e0 + (int64_t)threadIdx.x * 8;
  uint4 v = make_uint4(0, 0, 0, 0);
  const bool full_vec = i + 8 <= e1;
  if (full_vec) v = *reinterpret_cast<const uint4*>(y_local + i);
  for (int p = 0; p < world; ++p) {
    uint16_t* dst = slots_of(peers[p], rank);
    if (full_vec) {
      *reinterpret_cast<uint4*>(dst + i) = v;
    } else {
      for (int64_t t = i; t < e1; ++t) dst[t] = y_local[t];
    }
  }
  // 2. publish: every thread's peer stores are ordered (system scope) before the CTA
  //    barrier, the barrier before the flag stores (release, system scope)
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < world)
    st_release_sys(flags_of(peers[threadIdx.x]) + (size_t)rank * kArMaxChunks + c, epoch);
  // 3. wait for every rank's chunk c in this rank's buffer
  __shared__ int timed_out;
  if (threadIdx.x == 0) timed_out = 0;
  __syncthreads();
  if (threadIdx.x < world) {
    const uint32_t* f = flags_of(peers[rank]) + (size_t)threadIdx.x * kArMaxChunks + c;
    uint32_t polls = 0;
    while (ld_acquire_sys(f) != epoch) {
      if (++polls > (1u << 24)) {
        atomicExch(err, 1);
        timed_out = 1;
        break;
      }
      if (polls > 64) __nanosleep(polls > 4096 ? 1000 : 64);
    }
  }
  __syncthreads();
  // 4. reduce in rank order (bit-identical on every rank); skipped after a timeout (the
  //    error word reports it), but the CTA still counts itself done below so the header
  //    stays consistent for the next call
  if (i < e1 && !timed_out) {
    float acc[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) acc[t] = 0.0f;
    for (int q = 0; q < world; ++q) {
      const uint16_t* src = slots_of(peers[rank], q);
      if (full_vec) {
        const uint4 w = __ldcv(reinterpret_cast<const uint4*>(src + i));
        const uint16_t* h = reinterpret_cast<const uint16_t*>(&w);
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[t] += to_f<kBF16>(h[t]);
      } else {
        for (int64_t t = i; t < e1; ++t) acc[t - i] += to_f<kBF16>(__ldcv(src + t));
      }
    }
    if (full_vec) {
      uint4 o;
      uint16_t* h = reinterpret_cast<uint16_t*>(&o);
#pragma unroll
      for (int t = 0; t < 8; ++t) h[t] = from_f<kBF16>(acc[t]);
      *reinterpret_cast<uint4*>(y_out + i) = o;
    } else {
      for (int64_t t = i; t < e1; ++t) y_out[t] = from_f<kBF16>(acc[t - i]);
    }
  }
  if (device_epoch) {  // the last CTA to finish advances the device epoch
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(hdr + 1, 1u) == gridDim.x - 1) {
      hdr[1] = 0;
      __threadfence();
      *reinterpret_cast<volatile uint32_t*>(hdr) = epoch;
    }
  }
}

}  // namespace

int64_t ar_chunk_elems() { return kArChunkElems; }

size_t ar_buffer_bytes(int64_t n_max, int world) { return ar_slot_offset(world, 2, 0, n_max); }

cudaError_t launch_oneshot_allreduce(const void* y_local, int dtype, void* y_out, int64_t n, int64_t n_max,
                                     void* const* peers_dev, int rank, int world, uint32_t epoch, int* err,
                                     cudaStream_t st) {
  const int chunks = (int)((n + kArChunkElems - 1) / kArChunkElems);
  if (chunks == 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)chunks, 1, 1);
  cfg.blockDim = dim3(kArThreads, 1, 1);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = option(SQ_OPT_PDL) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  uint8_t* const* peers = reinterpret_cast<uint8_t* const*>(peers_dev);
  if (dtype == SQ_BF16)
    return cudaLaunchKernelEx(&cfg, oneshot_allreduce_kernel<true>, static_cast<const uint16_t*>(y_local),
                              static_cast<uint16_t*>(y_out), n, n_max, peers, rank, world, epoch, err);
  return cudaLaunchKernelEx(&cfg, oneshot_allreduce_kernel<false>, static_cast<const uint16_t*>(y_local),
                            static_cast<uint16_t*>(y_out), n, n_max, peers, rank, world, epoch, err);
}

}  // namespace sq
