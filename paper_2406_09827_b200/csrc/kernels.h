// kernels.h — internal launchers (C++), called by api.cu after argument validation.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "common.cuh"

namespace hip {

// Resident CTAs per SM for a persistent launch, computed from the real limits (shared memory with
// the per-block reservation, registers, threads, TMEM columns) instead of the occupancy API, and
// with the shared-memory carveout forced to the maximum.  Sets the dynamic-smem attribute.
template <typename K>
inline cudaError_t persistent_ctas(K kernel, int threads, size_t smem, int tmem_cols, int* per_sm) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  int dev = 0, smem_sm = 0, reserved = 0, regs_sm = 0, thr_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev);
  cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&thr_sm, cudaDevAttrMaxThreadsPerMultiProcessor, dev);
  cudaFuncAttributes fa{};
  e = cudaFuncGetAttributes(&fa, kernel);
  if (e != cudaSuccess) return e;
  const size_t per_block = smem + fa.sharedSizeBytes + (size_t)reserved;
  int n = (int)(smem_sm / std::max<size_t>(per_block, 1));
  const int regs = std::max(fa.numRegs, 1) * threads;
  n = std::min(n, regs_sm / regs);
  n = std::min(n, thr_sm / threads);
  if (tmem_cols > 0) n = std::min(n, 512 / tmem_cols);
  n = std::min(n, 32);
#ifdef HIPATTN_TUNING  // profiling builds only: cap the residency, print the launch shape
  if (const char* cap = getenv("HIPATTN_CTAS_PER_SM")) n = std::min(n, atoi(cap));
  fprintf(stderr, "[hipattn] launch: threads=%d smem=%zu regs=%d -> %d CTAs/SM\n", threads, smem, fa.numRegs,
          std::max(n, 1));
#endif
  *per_sm = std::max(n, 1);
  return cudaSuccess;
}

// Split-K of single-row attention units (attn_row1): at most kSplitMax splits (= the cluster size), only
// for launches of at most kSplitMaxUnits units; a chunk state is kSplitStride floats (O[128], max, sum,
// pad) in the CTA's shared memory.
constexpr int kSplitMax = 8, kSplitMaxUnits = 4096, kSplitStride = 132;

// Dynamic job claiming (common.cuh JobQueue) only pays when there are more jobs than resident
// CTAs; then the launch's counter (sh.sched, caller workspace) is zeroed on the launch stream.
inline cudaError_t setup_queue(Shape& sh, int64_t jobs, int64_t grid, cudaStream_t stream) {
  if (!sh.sched || jobs <= grid) {
    sh.sched = nullptr;
    return cudaSuccess;
  }
  return cudaMemsetAsync(sh.sched, 0, sizeof(unsigned int), stream);
}

// CUDA-core mask estimation (exact sequential fp32 scores), contiguous or paged keys.
cudaError_t launch_mask_cc(const Shape& sh, const QSrc& qs, const RowSrc& ks, bool bf16, int32_t* idx, int32_t* cnt,
                           cudaStream_t stream, int num_sms);

// Short query blocks (decode, <= 4 rows): direct-load GEMV scoring, exact sequential fp32.
bool mask_decode_supported(const Shape& sh);
cudaError_t launch_mask_decode(const Shape& sh, const QSrc& qs, const RowSrc& ks, bool bf16, int32_t* idx,
                               int32_t* cnt, cudaStream_t stream, int num_sms);

// tcgen05 mask estimation (bf16, d = 128, b_q <= 32, b_k | 32), contiguous or paged keys.
bool mask_tc_supported(const Shape& sh);
cudaError_t launch_mask_tc(const Shape& sh, const QSrc& qs, const RowSrc& ks, int32_t* idx, int32_t* cnt,
                           cudaStream_t stream, int num_sms);

// CUDA-core block-sparse attention (fp32 or bf16), contiguous or paged K/V.
cudaError_t launch_attn_cc(const Shape& sh, const QSrc& qs, const RowSrc& ks, const RowSrc& vs, bool bf16,
                           const int32_t* idx, const int32_t* cnt, float sm_scale, char* o, int64_t osb, int64_t osh,
                           int64_t ost, float* lse, cudaStream_t stream, int num_sms);

// Short query blocks (decode, <= 4 rows): half-warp-per-key GEMV attention, online softmax.
bool attn_decode_supported(const Shape& sh);
cudaError_t launch_attn_decode(const Shape& sh, const QSrc& qs, const RowSrc& ks, const RowSrc& vs, bool bf16,
                               const int32_t* idx, const int32_t* cnt, float sm_scale, char* o, int64_t osb,
                               int64_t osh, int64_t ost, float* lse, cudaStream_t stream, int num_sms);

// tcgen05 block-sparse attention prefill (bf16, d = 128, b_q <= 32, 128 % b_k == 0).
bool attn_tc_supported(const Shape& sh);
cudaError_t launch_attn_tc(const Shape& sh, const QSrc& qs, const RowSrc& ks, const RowSrc& vs, const int32_t* idx,
                           const int32_t* cnt, float sm_scale, char* o, int64_t osb, int64_t osh, int64_t ost,
                           float* lse, cudaStream_t stream, int num_sms);

// Single-row query blocks (decode, b_q = 1), bf16, d = 128: CUDA-core GEMV attention over a
// 3-slot cp.async ring with mbarrier completion, warp-owned online softmax, split-K to fill idle
// CTA slots (attn_row1.cu).
bool attn_row1_supported(const Shape& sh);
cudaError_t launch_attn_row1(const Shape& sh, const QSrc& qs, const RowSrc& ks, const RowSrc& vs, const int32_t* idx,
                             const int32_t* cnt, float sm_scale, char* o, int64_t osb, int64_t osh, int64_t ost,
                             float* lse, cudaStream_t stream, int num_sms);

// Ensemble vote (vote.cu).
cudaError_t launch_vote(int n_e, int64_t units, int n_in, const int32_t* idx, const int32_t* cnt, int theta, int tau,
                        int n_out, int32_t* out_idx, int32_t* out_cnt, cudaStream_t stream, int num_sms);

}  // namespace hip
