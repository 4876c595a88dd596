// kernels.h — internal launchers (C++), called by api.cu after argument validation.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace hip {

// CUDA-core mask estimation (exact sequential fp32 scores), contiguous or paged keys.
cudaError_t launch_mask_cc(const Shape& sh, const QSrc& qs, const RowSrc& ks, bool bf16, int32_t* idx, int32_t* cnt,
                           cudaStream_t stream, int num_sms);

// tcgen05 mask estimation (bf16, d = 128, b_q <= 32, b_k | 32), contiguous or paged keys.
bool mask_tc_supported(const Shape& sh);
cudaError_t launch_mask_tc(const Shape& sh, const QSrc& qs, const RowSrc& ks, int32_t* idx, int32_t* cnt,
                           cudaStream_t stream, int num_sms);

// CUDA-core block-sparse attention (fp32 or bf16), contiguous or paged K/V.
cudaError_t launch_attn_cc(const Shape& sh, const QSrc& qs, const RowSrc& ks, const RowSrc& vs, bool bf16,
                           const int32_t* idx, const int32_t* cnt, float sm_scale, char* o, int64_t osb, int64_t osh,
                           int64_t ost, float* lse, cudaStream_t stream, int num_sms);

// tcgen05 block-sparse attention prefill (bf16, d = 128, b_q <= 32, 128 % b_k == 0).
bool attn_tc_supported(const Shape& sh);
cudaError_t launch_attn_tc(const Shape& sh, const QSrc& qs, const RowSrc& ks, const RowSrc& vs, const int32_t* idx,
                           const int32_t* cnt, float sm_scale, char* o, int64_t osb, int64_t osh, int64_t ost,
                           float* lse, cudaStream_t stream, int num_sms);

}  // namespace hip
