// select.cuh — the tree-search control of HiP mask estimation for one query block, run by one CTA
// (Alg. 1 lines 4-17).  Scoring of the representative key blocks is delegated to a
// Scorer (CUDA-core sequential fp32 in mask_cc.cu, GEMV in mask_decode.cu, tcgen05 in mask_tc.cu).
//
// The nodes are kept in POSITION order (ascending first block), not in score order.  Splitting a
// node (f, l) at m = floor((f + l + 1) / 2) (reading G3) gives two adjacent children (f, m - 1) and
// (m, l), so the children of the position-ordered nodes are again position ordered: one block-wide
// exclusive scan places them.  The left child keeps its parent's score (same first block => same
// representative => same score, exact); only the right children are scored (all 2n children on
// the first iteration, PIN-7).  The n best children are then found by a block-wide
// radix select over their ranking keys and compacted in place by a second scan, which keeps the
// position order — so the final nodes are already the ascending block list Alg. 1 line 17 returns
// (G18) and no sort is ever needed.
//
// Ranking key (reading G10): larger score first, equal scores -> smaller first block:
//     key = orderable(score) << 22 | (kFirstMax - first)
// a plain unsigned compare (+0 and -0 normalised to one key; NaN, impossible for finite inputs,
// mapped to -inf so the order is total).  First blocks are unique among candidates, so keys are
// unique and "the n largest keys" is exactly one set.
#pragma once

#include "common.cuh"

namespace hip {

constexpr int kFirstBits = 22;                       // first block < 2^22 (T_k <= 4M * b_k)
constexpr uint32_t kFirstMax = (1u << kFirstBits) - 1;

// Selection state of one unit in shared memory.  NW = warps of the team.  The representatives'
// scores (2 NMAX floats, written by the Scorer) alias the node arrays nf / nl: nodes are read into
// registers at the start of an iteration and rewritten only by the compaction, after every score has
// been turned into a ranking key, so the two never live at the same time.
template <int NMAX, int NW = 32>
struct SelState {
  static constexpr int kRep = 2 * NMAX > 384 ? 2 * NMAX : 384;
  int nf[NMAX], nl[NMAX];            // nodes (first, last block), position order | scores (scoring)
  uint32_t ns[NMAX];                 // their orderable scores
  int rep[kRep];                     // representative blocks to score; 3 packed radix histograms after
  unsigned long long red[2 * NW];    // per-warp OR / AND of the keys
  int warp_tot[NW];
  __device__ __forceinline__ float* scores() { return reinterpret_cast<float*>(nf); }
};

// Barrier scope of the selection: the whole CTA (one unit per CTA).
struct CtaSync {
  static __device__ __forceinline__ void sync() { __syncthreads(); }
  static __device__ __forceinline__ int tid() { return threadIdx.x; }
};

__device__ __forceinline__ uint32_t ord_score(float s) {
  s = (s != s) ? -INFINITY : s;  // NaN -> -inf
  s = (s == 0.f) ? 0.f : s;      // -0 -> +0
  uint32_t u = __float_as_uint(s);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ uint64_t make_key(uint32_t ord, int first) {
  return ((uint64_t)ord << kFirstBits) | (uint64_t)(kFirstMax - (uint32_t)first);
}

// Block-wide exclusive scan of one int per thread, ONE barrier: every warp scans itself, publishes
// its total, and after the barrier each thread adds the totals of the warps before it (and of all
// warps for *total).  The caller must separate two uses of warp_tot by a barrier.
template <int NT, class Sync>
__device__ __forceinline__ int block_excl_scan(int v, int* warp_tot, int& total) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = Sync::tid() >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  Sync::sync();
  int base = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int t = warp_tot[w];
    base += w < warp ? t : 0;
    tot += t;
  }
  total = tot;
  return base + x - v;
}

// Block-wide radix select over unique 64-bit keys, EC per thread (bit k of `valid` marks key[k]):
// on return exactly the `need` largest valid keys satisfy (key & mask) >= prefix.  Digits of 8 bits
// starting at the highest bit on which the keys differ; each pass histograms the keys that match
// the prefix so far (shared atomics), then EVERY warp scans the histogram for the digit where the
// count from the top reaches `need` (redundantly, so the result needs no second barrier), and the
// search stops as soon as that digit's whole bin is selected.  Three histograms rotate so one
// barrier per pass suffices: pass p fills H[p % 3] and clears H[(p + 2) % 3], whose last readers
// (pass p - 1's scans) are behind pass p's barrier.  Requires 1 <= need <= number of valid keys.
// Returns the number of histogram passes.
template <int NT, int EC, int NMAX, class Sync, int NW>
__device__ __forceinline__ int radix_top(const uint64_t (&key)[EC], uint32_t valid, int need, SelState<NMAX, NW>& st,
                                         uint64_t& prefix, uint64_t& mask) {
  const int tid = Sync::tid(), lane = tid & 31, warp = tid >> 5;
  static_assert(NW == NT / 32, "SelState sized for the team");
  // three histograms of 256 bins, two 16-bit counts per word (bin 2w low, 2w + 1 high): counts <=
  // 2 NMAX < 2^16
  uint32_t* hist = reinterpret_cast<uint32_t*>(st.rep);
  uint32_t olo = 0u, ohi = 0u, alo = ~0u, ahi = ~0u;
#pragma unroll
  for (int k = 0; k < EC; ++k)
    if (valid & (1u << k)) {
      olo |= (uint32_t)key[k];
      ohi |= (uint32_t)(key[k] >> 32);
      alo &= (uint32_t)key[k];
      ahi &= (uint32_t)(key[k] >> 32);
    }
  olo = __reduce_or_sync(0xffffffffu, olo);
  ohi = __reduce_or_sync(0xffffffffu, ohi);
  alo = __reduce_and_sync(0xffffffffu, alo);
  ahi = __reduce_and_sync(0xffffffffu, ahi);
  if (lane == 0) {
    st.red[warp] = ((uint64_t)ohi << 32) | olo;
    st.red[NW + warp] = ((uint64_t)ahi << 32) | alo;
  }
  for (int i = tid; i < 256; i += NT) hist[i] = 0u;  // H[0], H[1]
  Sync::sync();
  uint64_t o = 0ull, a = ~0ull;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    o |= st.red[w];
    a &= st.red[NW + w];
  }
  const uint64_t diff = o ^ a;
  if (diff == 0ull) {  // a single distinct key
    prefix = a;
    mask = ~0ull;
    return 0;
  }
  const int hb = 63 - __clzll((long long)diff);
  mask = hb == 63 ? 0ull : (~0ull << (hb + 1));
  prefix = a & mask;
  int top = hb;
  for (int pass = 0;; ++pass) {
    const int s = top >= 7 ? top - 7 : 0;
    const uint32_t dmask = (1u << (top - s + 1)) - 1u;
    uint32_t* h = hist + (pass % 3) * 128;
#pragma unroll
    for (int k = 0; k < EC; ++k)
      if ((valid & (1u << k)) && (key[k] & mask) == prefix) {
        const uint32_t bin = (uint32_t)((key[k] >> s) & dmask);
        atomicAdd(h + (bin >> 1), 1u << ((bin & 1u) * 16));
      }
    Sync::sync();
    {
      uint32_t* hz = hist + ((pass + 2) % 3) * 128;  // clear the histogram of pass + 2
      for (int i = tid; i < 128; i += NT) hz[i] = 0u;
    }
    // lane L owns bins [248 - 8L, 255 - 8L] (words [124 - 4L, 127 - 4L]), walked from the top
    // (every warp, same result)
    const int b0 = 248 - 8 * lane;
    const uint4 v = *reinterpret_cast<const uint4*>(h + (b0 >> 1));
    const int c[8] = {(int)(v.w >> 16), (int)(v.w & 0xffffu), (int)(v.z >> 16), (int)(v.z & 0xffffu),
                      (int)(v.y >> 16), (int)(v.y & 0xffffu), (int)(v.x >> 16), (int)(v.x & 0xffffu)};
    int sum = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) sum += c[i];
    int incl = sum;
#pragma unroll
    for (int w = 1; w < 32; w <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, w);
      if (lane >= w) incl += y;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, incl >= need);
    const int fl = __ffs(hit) - 1;
    int acc = incl - sum, d = -1, cb = 0, above = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (d < 0) {
        if (acc + c[i] >= need) {
          d = b0 + 7 - i;
          cb = c[i];
          above = acc;
        } else {
          acc += c[i];
        }
      }
    d = __shfl_sync(0xffffffffu, d, fl);
    cb = __shfl_sync(0xffffffffu, cb, fl);
    above = __shfl_sync(0xffffffffu, above, fl);
    prefix |= (uint64_t)d << s;
    mask |= (uint64_t)dmask << s;
    need -= above;
    if (cb == need || s == 0) return pass + 1;
    top = s - 1;
  }
}

// Ensemble sampling (reading G23): every split point moves by u uniform in [-R, R],
// m = clamp(floor((f + l + 1) / 2) + u, f + 1, l), u drawn from splitmix64 (Steele, Lea & Flood's
// published output function) keyed by (seed, unit, iteration, first block of the node).  R = 0 is
// the deterministic half-up split.
struct SplitJitter {
  int R = 0;
  uint64_t key = 0;
};
__device__ __forceinline__ uint64_t splitmix_out(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ SplitJitter make_jitter(int R, uint64_t seed, int64_t lin) {
  SplitJitter j;
  j.R = R;
  j.key = R > 0 ? splitmix_out(splitmix_out(seed + 0x9E3779B97F4A7C15ull) ^ (uint64_t)lin) : 0ull;
  return j;
}
__device__ __forceinline__ int jittered_split(const SplitJitter& jt, int iter, int f, int l) {
  int m = (f + l + 1) >> 1;
  if (jt.R > 0) {
    const uint64_t x = splitmix_out(jt.key ^ (((uint64_t)(uint32_t)iter << 32) | (uint64_t)(uint32_t)f));
    m += (int)(x % (uint64_t)(2 * jt.R + 1)) - jt.R;
    m = min(max(m, f + 1), l);
  }
  return m;
}

// Stridden partial top-k (reading G21): a launch runs units x S jobs; job (unit, s)
// searches chunk s = [a_s, a_{s+1}), a_s = floor((2 s B_q + S) / (2 S)), with n / S nodes and writes
// slots [s n / S, (s + 1) n / S) of the unit's output.  S = 1, or B_q <= n (exact case, chunk 0
// alone): the whole range with n nodes.  Returns false for a job with nothing to do.
__device__ __forceinline__ bool chunk_job(int Bq, int n, int S, int s, int& lo, int& len, int& nn, int& slot0) {
  if (S <= 1 || Bq <= n) {
    lo = 0; len = Bq; nn = n; slot0 = 0;
    return s == 0;
  }
  const int64_t a0 = (2 * (int64_t)s * Bq + S) / (2 * (int64_t)S);
  const int64_t a1 = (2 * (int64_t)(s + 1) * Bq + S) / (2 * (int64_t)S);
  lo = (int)a0; len = (int)(a1 - a0); nn = n / S; slot0 = s * nn;
  return true;
}

// Scorer::score_buf(st, iter) names the array the scores of iteration `iter` go to: st.scores() (the
// node arrays, dead while scoring) for the single-CTA scorers; a cluster scorer alternates two
// arrays of its own by iteration parity, so a peer CTA may already write the next iteration's scores
// while this CTA still reads this iteration's (one cluster barrier per iteration instead of two).
// Runs the tree search of one query block over the L key blocks [lo, lo + L) (lo = 0, L = B_q:
// Alg. 1; one chunk of the stridden partial top-k otherwise, reading G21) and writes the n
// selected blocks (ascending, -1 padded) to out_idx and, if out_cnt, the count.  All NT threads
// call it.  Scorer::score(rep, n_rep, rep_s) must fill rep_s[i] = tile score of key block rep[i] and
// end with a Sync::sync(); Scorer::mark(p) is a profiling hook (no-op in product builds).
template <int NMAX, int NT, class Scorer, class Sync = CtaSync, int NW = NT / 32>
__device__ void tree_search(SelState<NMAX, NW>& st, int n, int lo, int Bq, Scorer& scorer, int32_t* out_idx,
                            int32_t* out_cnt, const SplitJitter& jit = SplitJitter()) {
  static_assert(NMAX % NT == 0 || NT % NMAX == 0, "NMAX and NT must nest");
  constexpr int E = NMAX >= NT ? NMAX / NT : 1;  // nodes per thread (contiguous)
  constexpr int EC = 2 * E;                      // candidates per thread (their children)
  static_assert(EC <= 32, "valid mask");
  const int tid = Sync::tid();
  if (Bq <= n) {  // exact case (G1): every visible block
    for (int j = tid; j < n; j += NT) out_idx[j] = j < Bq ? lo + j : -1;
    if (tid == 0 && out_cnt) *out_cnt = Bq;
    return;
  }
  // Initial nodes (Alg. 1 line 4, readings G1-G3): f_j = lo + floor((2 j B_q + n) / (2 n)).
  for (int j = tid; j < n; j += NT) {
    const int64_t fj = lo + (2 * (int64_t)j * Bq + n) / (2 * (int64_t)n);
    const int64_t fj1 = lo + (2 * (int64_t)(j + 1) * Bq + n) / (2 * (int64_t)n);
    st.nf[j] = (int)fj;
    st.nl[j] = (int)fj1 - 1;
    st.ns[j] = 0u;
  }
  Sync::sync();
  bool first = true;
  // Lower bound of the next selection: the n inherited candidates (left children / unsplit nodes)
  // keep the keys selected last iteration, all >= that selection's radix prefix, so a key below it
  // can never be among the n best — excluding those keys narrows the radix range (fewer passes).
  uint64_t lb = 0ull;
  // Every iteration at least halves the largest node, so <= 31 iterations end the search; the cap
  // only guards against non-finite inputs.
  for (int iter = 0; iter < 40; ++iter) {
    // --- branching (Alg. 1 lines 6-9): place the children of every node by one scan of
    //     (children count | splits << 16)
    int f[E], l[E];
    uint32_t s[E];
    int packed = 0;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int j = E * tid + i;
      if (j < n) {
        f[i] = st.nf[j];
        l[i] = st.nl[j];
        s[i] = st.ns[j];
        packed += l[i] > f[i] ? 2 + (1 << 16) : 1;
      }
    }
    int tot;
    const int pre = block_excl_scan<NT, Sync>(packed, st.warp_tot, tot);
    const int C = tot & 0xffff, nB = tot >> 16;
    if (nB == 0) break;  // every node is a single block (G5/G6)
    // This thread's children stay in registers: candidate 2i = left child (or the unsplit node),
    // 2i + 1 = right child of node i.  Those needing a score get a unique slot r in the rep list:
    // the candidate position on the first iteration (all 2n scored), the split rank afterwards.
    int p = pre & 0xffff, S = pre >> 16;
    int kf[EC], kl[EC], kr[EC];  // first, last, rep slot (-1: inherited score in ks)
    uint32_t ks[EC];
    uint32_t valid = 0;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int j = E * tid + i;
      kf[2 * i] = kf[2 * i + 1] = 0;
      kl[2 * i] = kl[2 * i + 1] = 0;
      kr[2 * i] = kr[2 * i + 1] = -1;
      ks[2 * i] = ks[2 * i + 1] = 0u;
      if (j < n) {
        const bool split = l[i] > f[i];
        const int m = split ? jittered_split(jit, iter, f[i], l[i]) : f[i];
        kf[2 * i] = f[i];
        kl[2 * i] = split ? m - 1 : l[i];
        ks[2 * i] = s[i];
        valid |= 1u << (2 * i);
        if (first) {
          kr[2 * i] = p;
          st.rep[p] = f[i];
        }
        if (split) {
          const int r = first ? p + 1 : S;
          kf[2 * i + 1] = m;
          kl[2 * i + 1] = l[i];
          kr[2 * i + 1] = r;
          st.rep[r] = m;
          valid |= 1u << (2 * i + 1);
          ++S;
        }
        p += split ? 2 : 1;
      }
    }
    Sync::sync();
    scorer.mark(0);  // split + scan
    // --- representative scores (Alg. 1 lines 10-13)
    float* const sbuf = scorer.score_buf(st, iter);  // the scores array of this iteration
    scorer.score(st.rep, first ? C : nB, sbuf);
    // --- top-n (Alg. 1 lines 14-15)
    uint64_t key[EC];
#pragma unroll
    for (int k = 0; k < EC; ++k)
      key[k] = make_key(kr[k] >= 0 ? ord_score(sbuf[kr[k]]) : ks[k], kf[k]);
    uint64_t prefix, mask;
    scorer.mark(8);  // keys
    uint32_t live = valid;
#pragma unroll
    for (int k = 0; k < EC; ++k)
      if (key[k] < lb) live &= ~(1u << k);
    const int passes = radix_top<NT, EC, NMAX, Sync, NW>(key, live, n, st, prefix, mask);
    valid = live;
    lb = prefix;
    scorer.mark(4);  // radix select
#ifdef HIPATTN_PHASES
    if (tid == 0) {
      atomicAdd(&g_phase_cycles[9], (unsigned long long)passes);
      atomicAdd(&g_phase_cycles[10], 1ull);
    }
#else
    (void)passes;
#endif
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < EC; ++k) cnt += ((valid >> k) & 1u) && (key[k] & mask) >= prefix;
    int ctot;
    int pos = block_excl_scan<NT, Sync>(cnt, st.warp_tot, ctot);
#pragma unroll
    for (int k = 0; k < EC; ++k)
      if (((valid >> k) & 1u) && (key[k] & mask) >= prefix) {
        st.nf[pos] = kf[k];
        st.nl[pos] = kl[k];
        st.ns[pos] = (uint32_t)(key[k] >> kFirstBits);
        ++pos;
      }
    Sync::sync();
    scorer.mark(5);  // compaction
    first = false;
  }
  // --- output (Alg. 1 line 17): first blocks of the final single-block nodes, already ascending (G18)
  for (int j = tid; j < n; j += NT) out_idx[j] = st.nf[j];
  if (tid == 0 && out_cnt) *out_cnt = n;
  scorer.mark(6);  // output
}

}  // namespace hip
