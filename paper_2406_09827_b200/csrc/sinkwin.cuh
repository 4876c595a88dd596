// sinkwin.cuh — StreamingLLM sink + sliding-window tokens fused into the block-sparse attention
// kernels ("local sliding window and global sink attention are also added
// during block sparse flash attention", sizes (128, 32); the EffectiveMask union of S:285-301;
// reading G14).  Row t of a query block, at key position p_t = t + T_k - T_q, attends to
//     (tokens of its selected blocks)  U  [0, sink)  U  (p_t - window, p_t]
// intersected with [0, T_k) and, if causal, with s <= p_t — each token once.  Per query block the
// kernels append to the selected keys the "extra" tokens: the sink range and the union of the
// rows' windows (p_first - window, p_last], minus every token a selected block already covers
// (dedup).  For each (row, extra token) the sink / window / causal condition is re-checked.
#pragma once

#include "select.cuh"

namespace hip {

constexpr int kMaxExtra = 256;        // sink + window + b_q - 1 <= 256 (checked on the host)
constexpr int kExtraBit = 1 << 30;    // marks an extra token in the kernels' staged token lists

// Is key block j among the ascending selected blocks blk[0, c)?  (blk in global memory, read
// through the read-only path, or staged in shared memory: kShared.)
template <bool kShared = false>
__device__ __forceinline__ int blk_at(const int32_t* blk, int i) {
  if constexpr (kShared) return blk[i];
  else return __ldg(blk + i);
}
template <bool kShared = false>
__device__ __forceinline__ bool blk_selected(const int32_t* blk, int c, int j) {
  int lo = 0, hi = c;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const int v = blk_at<kShared>(blk, mid);
    if (v < j) lo = mid + 1; else hi = mid;
  }
  return lo < c && blk_at<kShared>(blk, lo) == j;
}

// Row at position p sees extra token s (s < T_k by construction): a sink token, or inside the
// row's window (p - window, p] (the window ends at the row's own position even when not causal).
__device__ __forceinline__ bool extra_visible(int s, int64_t p, int causal, int sink, int window) {
  return (!causal || s <= p) && (s < sink || ((int64_t)s > p - window && (int64_t)s <= p));
}

// The extra tokens of one query block (rows at positions p_first..p_last), ascending, into
// list[0, return).  Block-wide (all NT threads of the CTA call it); ends with a barrier.  Blocks
// must be ascending in blk (hip_mask_estimate's output format).
template <int NT, bool kShared = false>
__device__ int build_extra(const int32_t* blk, int c, int lbk, int Tk, int64_t p_first, int64_t p_last, int causal,
                           int sink, int window, int* list, int* warp_tot) {
  const int tid = threadIdx.x;
  int64_t a1 = min((int64_t)sink, (int64_t)Tk);  // sink range [0, a1)
  if (causal) a1 = min(a1, p_last + 1);
  a1 = max(a1, (int64_t)0);
  int64_t w0 = max((int64_t)0, p_first - window + 1), w1 = min((int64_t)Tk, p_last + 1);
  if (window <= 0) w0 = w1 = 0;
  const int64_t r2 = max(w0, a1);                  // window part outside the sink range: [r2, w1)
  const int L = (int)(a1 + max((int64_t)0, w1 - r2));
  int total = 0;
  for (int base = 0; base < L; base += NT) {
    const int i = base + tid;
    int s = 0, keep = 0;
    if (i < L) {
      s = i < a1 ? i : (int)(r2 + (i - a1));
      keep = !blk_selected<kShared>(blk, c, s >> lbk);
    }
    int cnt_round;
    const int pos = block_excl_scan<NT, CtaSync>(keep, warp_tot, cnt_round);
    if (keep && total + pos < kMaxExtra) list[total + pos] = s;
    total += cnt_round;
    __syncthreads();
  }
  if (L == 0) __syncthreads();
  return min(total, kMaxExtra);
}

}  // namespace hip
