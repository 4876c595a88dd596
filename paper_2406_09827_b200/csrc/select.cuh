// select.cuh — the tree-search control of HiP mask estimation for one query block, run by one CTA
// (Alg. 1 lines 4-17).  Scoring of the representative key blocks is delegated to a
// Scorer (CUDA-core sequential fp32 in mask_cc.cu, tcgen05 in mask_tc.cu).
//
// Data layout in shared memory (SelState): the n current nodes (f, l, score) are kept SORTED by
// the ranking key (score desc, first block asc; reading G10).  Splitting a node at
// m = floor((f + l + 1) / 2) (reading G3) turns it into a left child (f, m - 1) that keeps the
// node's key (same first block => same representative => same score, exact) and a right child
// (m, l) that needs a fresh score.  So each iteration the left children form a list A that is
// already sorted, the right children a list B of <= n fresh scores: B is bitonic-sorted and
// merged with A by rank (binary search), keeping the top n.  On the first
// iteration A's scores are fresh too (2n scored blocks, PIN-7) and A is sorted as well.
#pragma once

#include "common.cuh"

namespace hip {

template <int NMAX>
struct SelState {
  int f[2][NMAX];
  int l[2][NMAX];
  float s[2][NMAX];
  int bf[NMAX];
  int bl[NMAX];
  float bs[NMAX];
  int rep[2 * NMAX];      // representative blocks to score this iteration
  float rep_s[2 * NMAX];  // their scores (written by the Scorer)
  int warp_tot[32];
  int total;
};

template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int* warp_tot, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    constexpr int NW = NT / 32;
    int t = lane < NW ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < NW) warp_tot[lane] = t;  // inclusive
    if (lane == NW - 1) *total = t;
  }
  __syncthreads();
  int base = warp ? warp_tot[warp - 1] : 0;
  return base + x - v;
}

// NaN never occurs for finite inputs; mapping it to -inf keeps the ranking a total order.
__device__ __forceinline__ float nan_to_ninf(float x) { return x != x ? -INFINITY : x; }

__device__ __forceinline__ int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Bitonic sort of P = next_pow2(cnt) entries by key descending; entries [cnt, P) are padded with
// (-inf, INT_MAX) which rank below every real candidate.  Ends with __syncthreads().
template <int NT>
__device__ void bitonic_desc(float* s, int* f, int* l, int cnt) {
  const int P = next_pow2(cnt);
  for (int i = cnt + threadIdx.x; i < P; i += NT) {
    s[i] = -INFINITY;
    f[i] = 0x7fffffff;
    l[i] = 0x7fffffff;
  }
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += NT) {
        int ixj = i ^ j;
        if (ixj > i) {
          bool up = (i & k) == 0;
          float si = s[i], sj = s[ixj];
          int fi = f[i], fj = f[ixj];
          bool jg = key_greater(sj, fj, si, fi);
          if (jg == up) {
            s[i] = sj; s[ixj] = si;
            f[i] = fj; f[ixj] = fi;
            int li = l[i]; l[i] = l[ixj]; l[ixj] = li;
          }
        }
      }
      __syncthreads();
    }
  }
}

template <int NT>
__device__ void bitonic_asc_int(int* f, int cnt) {
  const int P = next_pow2(cnt);
  for (int i = cnt + threadIdx.x; i < P; i += NT) f[i] = 0x7fffffff;
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += NT) {
        int ixj = i ^ j;
        if (ixj > i) {
          bool up = (i & k) == 0;
          int a = f[i], b = f[ixj];
          if ((a > b) == up) { f[i] = b; f[ixj] = a; }
        }
      }
      __syncthreads();
    }
  }
}

// Number of entries of the descending-sorted list (s, f)[0, cnt) whose key is greater than (x, y).
__device__ __forceinline__ int count_greater(const float* s, const int* f, int cnt, float x, int y) {
  int lo = 0, hi = cnt;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (key_greater(s[mid], f[mid], x, y)) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Runs the tree search of one query block with B_q visible key blocks and writes the n selected
// blocks (ascending, -1 padded) to out_idx and the count to *out_cnt.  All NT threads call it.
// Scorer::score(rep, n_rep, rep_s) must fill rep_s[i] = tile score of key block rep[i] and end
// with a __syncthreads().
template <int NMAX, int NT, class Scorer>
__device__ void tree_search(SelState<NMAX>& st, int n, int Bq, Scorer& scorer, int32_t* out_idx, int32_t* out_cnt) {
  const int tid = threadIdx.x;
  if (Bq <= n) {  // exact case (G1): every visible block
    for (int j = tid; j < n; j += NT) out_idx[j] = j < Bq ? j : -1;
    if (tid == 0) *out_cnt = Bq;
    return;
  }
  // Initial nodes (Alg. 1 line 4, readings G1-G3): f_j = floor((2 j B_q + n) / (2 n)).
  for (int j = tid; j < n; j += NT) {
    int64_t fj = (2 * (int64_t)j * Bq + n) / (2 * (int64_t)n);
    int64_t fj1 = (2 * (int64_t)(j + 1) * Bq + n) / (2 * (int64_t)n);
    st.f[0][j] = (int)fj;
    st.l[0][j] = (int)fj1 - 1;
    st.s[0][j] = 0.f;
  }
  __syncthreads();
  constexpr int PER = (NMAX + NT - 1) / NT;
  int cur = 0;
  bool first = true;
  // Every iteration at least halves the largest node, so ceil(log2(B_q)) <= 31 iterations end the
  // search; the cap only guards against non-finite inputs (NaN scores are mapped to -inf below).
  for (int iter = 0; iter < 40; ++iter) {
    // --- branching (Alg. 1 lines 6-9): count the nodes that split, compact the right children
    const int j0 = tid * PER;
    int mine = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      int j = j0 + i;
      if (j < n && st.l[cur][j] > st.f[cur][j]) ++mine;
    }
    int pos = block_excl_scan<NT>(mine, st.warp_tot, &st.total);
    const int nB = st.total;
    if (nB == 0) break;  // every node is a single block (G5/G6)
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      int j = j0 + i;
      if (j < n) {
        int f = st.f[cur][j], l = st.l[cur][j];
        if (l > f) {
          int m = (f + l + 1) >> 1;
          st.bf[pos] = m;
          st.bl[pos] = l;
          st.rep[(first ? n : 0) + pos] = m;
          ++pos;
          st.l[cur][j] = m - 1;  // left child keeps (score, first)
        }
        if (first) st.rep[j] = f;
      }
    }
    __syncthreads();
    // --- representative scores (Alg. 1 lines 10-13)
    const int n_rep = first ? n + nB : nB;
    scorer.score(st.rep, n_rep, st.rep_s);
    for (int i = tid; i < nB; i += NT) st.bs[i] = nan_to_ninf(st.rep_s[(first ? n : 0) + i]);
    if (first)
      for (int j = tid; j < n; j += NT) st.s[cur][j] = nan_to_ninf(st.rep_s[j]);
    __syncthreads();
    // --- top-n (Alg. 1 lines 14-15)
    if (first) bitonic_desc<NT>(st.s[cur], st.f[cur], st.l[cur], n);
    bitonic_desc<NT>(st.bs, st.bf, st.bl, nB);
    const int nxt = cur ^ 1;
    for (int i = tid; i < n; i += NT) {
      float s = st.s[cur][i];
      int f = st.f[cur][i];
      int r = i + count_greater(st.bs, st.bf, nB, s, f);
      if (r < n) { st.s[nxt][r] = s; st.f[nxt][r] = f; st.l[nxt][r] = st.l[cur][i]; }
    }
    for (int i = tid; i < nB; i += NT) {
      float s = st.bs[i];
      int f = st.bf[i];
      int r = i + count_greater(st.s[cur], st.f[cur], n, s, f);
      if (r < n) { st.s[nxt][r] = s; st.f[nxt][r] = f; st.l[nxt][r] = st.bl[i]; }
    }
    __syncthreads();
    cur = nxt;
    first = false;
  }
  // --- output (Alg. 1 line 17): first blocks of the final single-block nodes, ascending (G18)
  bitonic_asc_int<NT>(st.f[cur], n);
  for (int j = tid; j < n; j += NT) out_idx[j] = st.f[cur][j];
  if (tid == 0) *out_cnt = n;
}

}  // namespace hip
