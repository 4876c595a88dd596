// topr.cuh — top-r approximation of the branch scores, shared by the mask kernels.
//
// "instead of fetching all d components of the key vectors, we only fetch r << d most prominent
// components estimated by the query vector q": q.k ~ sum_{l=1..r} q_{p_l} k_{p_l} with
// {p_l} = argtop_r(|q|).  Reading G22: a query block reduces |q_c| by the max over its rows, ties go
// to the smaller component, and the r terms are summed in ascending component order.  The kernels
// realise the restricted sum by ZEROING the other components of the staged query block: every
// dropped term then contributes an exact 0 (fmaf(0, k, acc) == acc for finite k; a tensor-core
// product 0 * k == 0), so each fp32 evaluation order of the full dot product computes the
// restricted sum in the same order — bit-for-bit what the oracle sums over {p_l}.  Key chunks whose
// components are all dropped are not fetched at all (mask_tc: cp.async with src-size 0 zero-fills
// the shared tile without a global read).
#pragma once

#include "common.cuh"

namespace hip {

// Keep flag of component c among a[0..d): rank by (a desc, c asc) < r.
__device__ __forceinline__ bool top_r_keep(const float* a, int d, int c, int r) {
  const float ac = a[c];
  int rank = 0;
  for (int j = 0; j < d; ++j) {
    const float aj = a[j];
    rank += (aj > ac) || (aj == ac && j < c);
  }
  return rank < r;
}

// fp32 query block staged in shared memory (rows x d, row pitch `pitch`): zero every component
// outside argtop_r.  `scratch` holds d floats.  All NT threads call it; it ends with a barrier.
template <int NT>
__device__ void top_r_zero_f32(float* qs, int pitch, int rows, int d, int r, float* scratch) {
  for (int c = threadIdx.x; c < d; c += NT) {
    float a = 0.f;
    for (int t = 0; t < rows; ++t) a = fmaxf(a, fabsf(qs[t * pitch + c]));
    scratch[c] = a;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += NT)
    if (!top_r_keep(scratch, d, c, r))
      for (int t = 0; t < rows; ++t) qs[t * pitch + c] = 0.f;
  __syncthreads();
}

}  // namespace hip
