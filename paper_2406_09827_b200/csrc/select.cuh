// select.cuh — the tree-search control of HiP mask estimation for one query block, run by one CTA
// (Alg. 1 lines 4-17).  Scoring of the representative key blocks is delegated to a
// Scorer (CUDA-core sequential fp32 in mask_cc.cu, GEMV in mask_decode.cu, tcgen05 in mask_tc.cu).
//
// Ranking key (reading G10): larger score first, equal scores -> smaller first block.
// It is packed into one 64-bit integer
//     key = orderable(score) << 32 | (kFirstMax - first) << kSlotBits | slot
// so ranking is a plain unsigned compare (+0 and -0 normalised to one key; NaN, impossible for
// finite inputs, mapped to -inf so the order is total).  `slot` is the entry's position in the
// unsorted array it was built from; first blocks are unique among candidates, so the slot never
// decides an order — it only lets the sort move 64-bit keys alone (no payload) and the merge find
// each entry's last block afterwards.
//
// The n current nodes are kept SORTED by key.  Splitting a node at m = floor((f + l + 1) / 2)
// (reading G3) gives a left child (f, m - 1) that keeps the node's key (same first block => same
// representative => same score, exact) and a right child (m, l) that needs a fresh score.  So
// each iteration the left children form a list A that is already sorted and the right children a
// list B of <= n fresh keys: B is sorted with a register/shuffle bitonic network (only the strides
// that cross warps go through shared memory), then A and B are merged by rank (binary search) and
// the first n kept.  On the first iteration A's scores are fresh too (2n scored
// blocks, PIN-7) and A is sorted the same way.
#pragma once

#include "common.cuh"

namespace hip {

constexpr int kFirstBits = 22;                       // first block < 2^22 (T_k <= 4M * b_k)
constexpr uint32_t kFirstMax = (1u << kFirstBits) - 1;

template <int NMAX>
struct SelState {
  static constexpr int kSlotBits = 32 - kFirstBits;  // 10 bits: NMAX <= 1024
  static_assert(NMAX <= (1 << kSlotBits), "slot field too small");
  uint64_t key[2][NMAX];   // nodes, sorted by key (descending)
  int l[2][NMAX];          // last block of each node, aligned with key
  uint64_t bkey[NMAX];     // right children (B list)
  int bl[NMAX];            // their last blocks, indexed by slot
  int ltmp[NMAX];
  int rep[2 * NMAX];       // representative blocks to score this iteration
  float rep_s[2 * NMAX];   // their scores (written by the Scorer)
  int warp_tot[32];
  int total;
};

__device__ __forceinline__ uint32_t ord_score(float s) {
  s = (s != s) ? -INFINITY : s;  // NaN -> -inf
  s = (s == 0.f) ? 0.f : s;      // -0 -> +0
  uint32_t u = __float_as_uint(s);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ uint64_t make_key(float s, int first, int slot) {
  constexpr int kSlotBits = 32 - kFirstBits;
  return ((uint64_t)ord_score(s) << 32) | ((uint32_t)(kFirstMax - (uint32_t)first) << kSlotBits) | (uint32_t)slot;
}
__device__ __forceinline__ int key_first(uint64_t k) {
  constexpr int kSlotBits = 32 - kFirstBits;
  return (int)(kFirstMax - ((uint32_t)k >> kSlotBits));
}
__device__ __forceinline__ int key_slot(uint64_t k) {
  constexpr int kSlotBits = 32 - kFirstBits;
  return (int)((uint32_t)k & ((1u << kSlotBits) - 1));
}

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

// One compare-exchange of the network: element e against e ^ J inside blocks of K; the pair
// ends descending inside blocks with (e & K) == 0, ascending otherwise.
template <int K, int J>
__device__ __forceinline__ uint64_t bitonic_pick(uint64_t key, uint64_t pk, int e) {
  const bool want_max = ((e & K) == 0) == ((e & J) == 0);
  return want_max ? (pk > key ? pk : key) : (pk < key ? pk : key);
}

template <int P, int NT, int K, int J>
__device__ __forceinline__ void bitonic_stage(uint64_t (&key)[(P + NT - 1) / NT], uint64_t* skey) {
  constexpr int E = P >= NT ? P / NT : 1;
  const int tid = threadIdx.x;
  const bool active = tid < P;
  if constexpr (J >= NT) {  // partner in the same thread
    constexpr int JR = J / NT;
#pragma unroll
    for (int r = 0; r < E; ++r) {
      if ((r & JR) == 0) {
        const int e = r * NT + tid;
        const uint64_t a = key[r], b = key[r | JR];
        const bool desc_seg = (e & K) == 0;  // e is the lower index of the pair
        const bool swap = desc_seg ? (b > a) : (b < a);
        key[r] = swap ? b : a;
        key[r | JR] = swap ? a : b;
      }
    }
  } else if constexpr (J >= 32) {  // partner in another warp: through shared memory
    __syncthreads();
#pragma unroll
    for (int r = 0; r < E; ++r)
      if (active) skey[r * NT + tid] = key[r];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < E; ++r)
      if (active) {
        const int e = r * NT + tid;
        key[r] = bitonic_pick<K, J>(key[r], skey[e ^ J], e);
      }
  } else if (active) {  // partner in the same warp
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)key[r], J);
      const uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(key[r] >> 32), J);
      key[r] = bitonic_pick<K, J>(key[r], ((uint64_t)hi << 32) | lo, r * NT + tid);
    }
  }
}

template <int P, int NT, int K, int J>
__device__ __forceinline__ void bitonic_stages(uint64_t (&key)[(P + NT - 1) / NT], uint64_t* skey) {
  bitonic_stage<P, NT, K, J>(key, skey);
  if constexpr (J > 1) bitonic_stages<P, NT, K, J / 2>(key, skey);
  else if constexpr (K < P) bitonic_stages<P, NT, 2 * K, K>(key, skey);
}

// Bitonic sort, descending, of cnt <= P 64-bit keys held in shared memory (P a power of two >= 32,
// compile-time: the whole network is unrolled); the result is written back to the first cnt slots,
// entries past cnt are padded with key 0 (ranks below every real key).  Element e = r*NT + tid
// lives in register r of its thread: strides < 32 are warp shuffles, strides >= NT in-thread,
// only strides in [32, NT) go through shared memory.  All NT threads call it.
template <int P, int NT>
__device__ void bitonic_desc(uint64_t* skey, int cnt) {
  static_assert(P >= 32 && (P & (P - 1)) == 0, "P must be a power of two >= 32");
  constexpr int E = P >= NT ? P / NT : 1;
  const int tid = threadIdx.x;
  const bool active = tid < P;
  uint64_t key[E];
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int e = r * NT + tid;
    key[r] = (active && e < cnt) ? skey[e] : 0ull;
  }
  bitonic_stages<P, NT, 2, 1>(key, skey);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int e = r * NT + tid;
    if (active && e < cnt) skey[e] = key[r];
  }
  __syncthreads();
}

// Number of entries of the descending list key[0, cnt) strictly greater than x.
__device__ __forceinline__ int count_greater(const uint64_t* key, int cnt, uint64_t x) {
  int lo = 0, hi = cnt;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (key[mid] > x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Runs the tree search of one query block with B_q visible key blocks and writes the n selected
// blocks (ascending, -1 padded) to out_idx and the count to *out_cnt.  All NT threads call it.
// Scorer::score(rep, n_rep, rep_s) must fill rep_s[i] = tile score of key block rep[i] and end
// with a __syncthreads(); Scorer::mark(p) is a profiling hook (no-op in product builds).
template <int NMAX, int NT, class Scorer>
__device__ void tree_search(SelState<NMAX>& st, int n, int Bq, Scorer& scorer, int32_t* out_idx, int32_t* out_cnt) {
  constexpr int EMAX = (NMAX + NT - 1) / NT;
  static_assert(NMAX >= 32 && (NMAX & (NMAX - 1)) == 0, "NMAX must be a power of two >= 32");
  const int tid = threadIdx.x;
  if (Bq <= n) {  // exact case (G1): every visible block
    for (int j = tid; j < n; j += NT) out_idx[j] = j < Bq ? j : -1;
    if (tid == 0) *out_cnt = Bq;
    return;
  }
  // Initial nodes (Alg. 1 line 4, readings G1-G3): f_j = floor((2 j B_q + n) / (2 n)).
  for (int j = tid; j < n; j += NT) {
    const int64_t fj = (2 * (int64_t)j * Bq + n) / (2 * (int64_t)n);
    const int64_t fj1 = (2 * (int64_t)(j + 1) * Bq + n) / (2 * (int64_t)n);
    st.key[0][j] = make_key(0.f, (int)fj, j);
    st.l[0][j] = (int)fj1 - 1;
  }
  __syncthreads();
  constexpr int PER = EMAX;
  int cur = 0;
  bool first = true;
  // Every iteration at least halves the largest node, so <= 31 iterations end the search; the cap
  // only guards against non-finite inputs.
  for (int iter = 0; iter < 40; ++iter) {
    // --- branching (Alg. 1 lines 6-9): count the nodes that split, compact the right children
    const int j0 = tid * PER;
    int mine = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int j = j0 + i;
      if (j < n && st.l[cur][j] > key_first(st.key[cur][j])) ++mine;
    }
    int pos = block_excl_scan<NT>(mine, st.warp_tot, &st.total);
    const int nB = st.total;
    if (nB == 0) break;  // every node is a single block (G5/G6)
    const int boff = first ? n : 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int j = j0 + i;
      if (j < n) {
        const int f = key_first(st.key[cur][j]), l = st.l[cur][j];
        if (l > f) {
          const int m = (f + l + 1) >> 1;
          st.bl[pos] = l;
          st.rep[boff + pos] = m;
          ++pos;
          st.l[cur][j] = m - 1;  // left child keeps (score, first)
        }
        if (first) st.rep[j] = f;
      }
    }
    __syncthreads();
    scorer.mark(0);  // split + scan
    // --- representative scores (Alg. 1 lines 10-13)
    scorer.score(st.rep, boff + nB, st.rep_s);
    for (int i = tid; i < nB; i += NT) st.bkey[i] = make_key(st.rep_s[boff + i], st.rep[boff + i], i);
    if (first)
      for (int j = tid; j < n; j += NT) st.key[cur][j] = make_key(st.rep_s[j], st.rep[j], j);
    __syncthreads();
    // --- top-n (Alg. 1 lines 14-15)
    if (first) {  // A is unsorted on the first iteration: sort it, then realign its last blocks
      bitonic_desc<NMAX, NT>(st.key[cur], n);
      for (int i = tid; i < n; i += NT) st.ltmp[i] = st.l[cur][key_slot(st.key[cur][i])];
      __syncthreads();
      for (int i = tid; i < n; i += NT) st.l[cur][i] = st.ltmp[i];
    }
    bitonic_desc<NMAX, NT>(st.bkey, nB);
    scorer.mark(4);  // keys + sorts
    const int nxt = cur ^ 1;
    for (int i = tid; i < n; i += NT) {
      const uint64_t k = st.key[cur][i];
      const int r = i + count_greater(st.bkey, nB, k);
      if (r < n) { st.key[nxt][r] = k; st.l[nxt][r] = st.l[cur][i]; }
    }
    for (int i = tid; i < nB; i += NT) {
      const uint64_t k = st.bkey[i];
      const int r = i + count_greater(st.key[cur], n, k);
      if (r < n) { st.key[nxt][r] = k; st.l[nxt][r] = st.bl[key_slot(k)]; }
    }
    __syncthreads();
    scorer.mark(5);  // rank merge
    cur = nxt;
    first = false;
  }
  // --- output (Alg. 1 line 17): first blocks of the final single-block nodes, ascending (G18)
  for (int j = tid; j < n; j += NT) st.bkey[j] = 0xFFFFFFFFull - (uint32_t)key_first(st.key[cur][j]);
  __syncthreads();
  bitonic_desc<NMAX, NT>(st.bkey, n);  // descending key = ascending block
  for (int j = tid; j < n; j += NT) out_idx[j] = (int)(0xFFFFFFFFull - st.bkey[j]);
  if (tid == 0) *out_cnt = n;
  scorer.mark(6);  // output sort
}

}  // namespace hip
