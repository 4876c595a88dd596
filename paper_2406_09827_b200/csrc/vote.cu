// vote.cu — the HiP ensemble vote (Appendix D): per query block an index survives iff
// at least theta of the n_e sample masks contain it; tau = 1 truncates the survivors to n_in,
// preferring more votes and then the smaller block (reading G24); output ascending, -1 padded.
//
// One CTA per unit (persistent, grid-stride).  The n_e ascending sample lists are staged in shared
// memory; every entry finds its rank in each list by binary search, which gives at once its vote
// count and its position in the stable merge of all lists (entries equal to x in earlier lists go
// first), so the merged order is built without sorting and the first copy of each index carries its
// vote.  Survivors are then compacted in ascending order by block scans; tau = 1 resolves the
// truncation with a vote histogram (the level where the count from the top reaches n_in) and a
// rank among the entries of that level.
#include "kernels.h"
#include "select.cuh"

namespace hip {

constexpr int kVoteThreads = 256;
constexpr int kVoteMaxE = 16;
constexpr int kVoteMaxEntries = 4096;

__global__ void __launch_bounds__(kVoteThreads) vote_kernel(int n_e, int64_t units, int n_in, const int32_t* __restrict__ idx,
                                                           const int32_t* __restrict__ cnt, int theta, int tau, int n_out,
                                                           int32_t* __restrict__ out_idx, int32_t* __restrict__ out_cnt) {
  __shared__ int L[kVoteMaxEntries];   // the sample lists, packed
  __shared__ int mx[kVoteMaxEntries];  // merged entries: index << 5 | vote of its first copy (0 for later copies)
  __shared__ int off[kVoteMaxE + 1];
  __shared__ int hist[kVoteMaxE + 1];
  __shared__ int warp_tot[32];
  const int tid = threadIdx.x;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    if (tid == 0) {
      int o = 0;
      for (int e = 0; e < n_e; ++e) {
        off[e] = o;
        o += min(max(__ldg(cnt + (int64_t)e * units + u), 0), n_in);
      }
      off[n_e] = o;
    }
    if (tid <= kVoteMaxE) hist[tid] = 0;
    __syncthreads();
    const int M = off[n_e];
    for (int p = tid; p < M; p += kVoteThreads) {
      int e = 0;
      while (off[e + 1] <= p) ++e;
      L[p] = __ldg(idx + ((int64_t)e * units + u) * n_in + (p - off[e]));
    }
    __syncthreads();
    for (int p = tid; p < M; p += kVoteThreads) {
      int e = 0;
      while (off[e + 1] <= p) ++e;
      const int x = L[p];
      int pos = 0, votes = 0, before = 0;
      for (int f = 0; f < n_e; ++f) {
        int lo = off[f], hi = off[f + 1];  // lower bound of x in list f
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (L[mid] < x) lo = mid + 1;
          else hi = mid;
        }
        const int eq = lo < off[f + 1] && L[lo] == x;
        pos += lo - off[f];
        votes += eq;
        if (f < e) before += eq;
      }
      pos += before;
      mx[pos] = (x << 5) | (before == 0 ? votes : 0);
      if (tau && before == 0 && votes >= theta) atomicAdd(&hist[votes], 1);
    }
    __syncthreads();
    // truncation level (tau = 1): keep votes > vstar, and the first `rem` (ascending) of votes == vstar
    int vstar = 0, rem = 0;
    if (tau) {
      int acc = 0;
      vstar = 0;
      for (int v = n_e; v >= theta; --v) {
        if (acc + hist[v] >= n_in) {
          vstar = v;
          rem = n_in - acc;
          break;
        }
        acc += hist[v];
      }
    }
    int carry_eq = 0, carry_out = 0;
    for (int base = 0; base < M; base += kVoteThreads) {
      const int p = base + tid;
      const int v = p < M ? (mx[p] & 31) : 0;
      bool keep = v >= theta;
      int r_eq = 0, tot_eq = 0;
      if (tau && vstar > 0) {  // rank among the survivors at the truncation level
        const int is_eq = keep && v == vstar;
        r_eq = carry_eq + block_excl_scan<kVoteThreads, CtaSync>(is_eq, warp_tot, tot_eq);
        __syncthreads();
        keep = keep && (v > vstar || (is_eq && r_eq < rem));
      }
      int tot;
      const int w = carry_out + block_excl_scan<kVoteThreads, CtaSync>(keep ? 1 : 0, warp_tot, tot);
      __syncthreads();
      if (keep) out_idx[u * n_out + w] = mx[p] >> 5;
      carry_eq += tot_eq;
      carry_out += tot;
    }
    for (int j = carry_out + tid; j < n_out; j += kVoteThreads) out_idx[u * n_out + j] = -1;
    if (tid == 0) out_cnt[u] = carry_out;
    __syncthreads();
  }
}

cudaError_t launch_vote(int n_e, int64_t units, int n_in, const int32_t* idx, const int32_t* cnt, int theta, int tau,
                        int n_out, int32_t* out_idx, int32_t* out_cnt, cudaStream_t stream, int num_sms) {
  if (units == 0) return cudaSuccess;
  const int64_t grid = std::min<int64_t>(units, (int64_t)num_sms * 8);
  vote_kernel<<<(unsigned)grid, kVoteThreads, 0, stream>>>(n_e, units, n_in, idx, cnt, theta, tau, n_out, out_idx,
                                                          out_cnt);
  return cudaGetLastError();
}

}  // namespace hip
