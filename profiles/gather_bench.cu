// gather_bench.cu — microbenchmark of the access pattern that bounds HiP's kernels: random 512-byte
// key blocks (2 rows x 256 B) gathered from a buffer into shared memory (16-byte cp.async,
// 16 threads per row, like mask_tc.cu), with the buffer either L2-resident (one head's K at 32k =
// 8 MB) or HBM-resident.  Reports achieved GB/s for several (CTAs/SM, tiles in flight) settings.
// Profiling tool only: built by profiles/gather_bench.py into its own .so, never by the product.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

// Each CTA: `iters` tiles of 128 rows (64 random blocks of 2 rows) into a ring of NBUF 32 KB slots.
template <int NBUF>
__global__ void __launch_bounds__(256) gather_kernel(const char* __restrict__ buf, uint32_t nblocks, int iters,
                                                     unsigned long long* sink) {
  extern __shared__ __align__(128) char smem[];
  const int tid = threadIdx.x, c16 = tid & 15, r0 = tid >> 4;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  uint32_t seed = blockIdx.x * 7919u + 17u;
  auto issue = [&](int it) {
    const uint32_t slot = sbase + (it % NBUF) * 32768;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = r0 + 16 * i;
      const uint32_t blk = hash32(seed + (uint32_t)it * 64u + (uint32_t)(r >> 1)) % nblocks;
      const char* src = buf + ((uint64_t)blk * 2 + (r & 1)) * 256 + c16 * 16;
      cp_async16(slot + r * 256 + c16 * 16, src);
    }
  };
#pragma unroll
  for (int i = 0; i < NBUF - 1; ++i) {
    issue(i);
    commit();
  }
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    issue(it + NBUF - 1);
    commit();
    wait_group<NBUF - 1>();
    __syncthreads();
    acc += *reinterpret_cast<const unsigned int*>(smem + (it % NBUF) * 32768 + tid * 4);
    __syncthreads();
  }
  wait_group<0>();
  if (acc == 0x123456789ull) *sink = acc;
}

extern "C" int gather_bench(const char* buf, unsigned long long bytes, int nbuf, int ctas_per_sm, int iters,
                            float* ms_out) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t nblocks = (uint32_t)(bytes / 512);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const int grid = sms * ctas_per_sm;
  const size_t smem = (size_t)nbuf * 32768;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](void (*k)(const char*, uint32_t, int, unsigned long long*)) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, 256, smem>>>(buf, nblocks, 8, sink);
    cudaEventRecord(a);
    k<<<grid, 256, smem>>>(buf, nblocks, iters, sink);
    cudaEventRecord(b);
  };
  if (nbuf == 1) run(gather_kernel<1>);
  else if (nbuf == 2) run(gather_kernel<2>);
  else if (nbuf == 3) run(gather_kernel<3>);
  else run(gather_kernel<4>);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(ms_out, a, b);
  cudaFree(sink);
  return (int)cudaGetLastError();
}
