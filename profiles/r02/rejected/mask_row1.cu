// mask_row1.cu — HiP mask estimation (Alg. 1) for single-row query blocks: the decode
// step (one query row per sequence and head against a paged KV cache, Alg. 2), bf16,
// d = 128, b_k <= 4.
//
// With one query row a branch score is a dot product per key row ("tensor units cannot
// help"); the kernel is bound by how many representative rows each unit has in flight while its
// serial chain (gather -> score -> select, ~log2(T/k) iterations) runs.  So, unlike the prefill mask
// (mask_tc, tcgen05), the scores come from the CUDA cores straight out of shared memory:
//   * the representative rows of one scoring call stream through a 5-slot ring of 8 KB items (32 key
//     rows x 256 B, 16-byte cp.async, one whole row per half-warp instruction); completion is tracked
//     on mbarriers (cp.async.mbarrier.arrive.noinc -> "full"; one arrival per warp once read ->
//     "empty"), so a slot is refilled as soon as its rows are scored — no tensor-core round trip and
//     no CTA barrier between items (40 KB in flight per unit against 32 KB in the tcgen05 ring);
//   * a half-warp scores one row: lane l runs the sequential fmaf chain over components 8l..8l+7 and
//     the 16 partials are combined by the xor tree o = 8, 4, 2, 1 — the "F32L" order of reading G9b,
//     so the bf16 decode mask is bit-identical to the oracle's F32L mode on ANY input (the tcgen05
//     path's accumulation order has no sequential counterpart);
//   * the block-table row of the sequence is staged in shared memory (uint16) and each scoring call
//     looks every representative's page up once before its rows are gathered.
// The tree control (position-ordered nodes, radix select, compaction) is select.cuh.
#include "kernels.h"
#include "select.cuh"

namespace hip {

constexpr int kM1Threads = 128;
constexpr int kM1Slots = 5;
constexpr uint32_t kM1Item = 8192;  // 32 rows x 256 B
constexpr int kM1NMax = 256;

struct MaskRow1Smem {
  static constexpr uint32_t ring = 0;
  static constexpr uint32_t sel = ring + kM1Slots * kM1Item;
  static constexpr uint32_t bt = sel + (uint32_t)align_up(sizeof(SelState<kM1NMax, 4>), 128);  // uint16 row
  static constexpr uint32_t bar = bt + (uint32_t)align_up(kBt16Max * 2, 16);                   // full[5], empty[5]
  static constexpr uint32_t jq = bar + 2 * kM1Slots * 8;
  static constexpr uint32_t total = jq + 16;
};

__device__ __forceinline__ void m1_arrive_noinc(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void m1_arrive(uint32_t bar) {
  asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(bar) : "memory");
}

template <bool kPaged>
struct Row1Scorer {
  float qv[32];          // q components of this lane's chunks p + 4 c (c < 4): qv[8 c + e] = q[8 (p + 4 c) + e]
  uint32_t ring, full0, empty0;
  const char* ring_p;    // the ring, generic address
  uint32_t* g;           // ring items issued so far by this CTA (slot g % 5, parity (g / 5) & 1)
  RowSrc ks;
  const char* kbh;       // row 0 of this (batch, kv head): key row r is kbh + r * row_bytes
  uint32_t row_bytes;
  int b, Tk, lbk, causal;
  int64_t tpos;          // the query row's key position (G7)
  const uint16_t* bt16 = nullptr;
  HIP_PT_MEMBER
  __device__ __forceinline__ void mark(int p) { HIP_MARK(p); (void)p; }

  // out[i] = max over the rows of key block rep[i] of q . k (F32L), for i < n_rep; ends with a barrier.
  __device__ void score(const int* rep, int n_rep, float* out) {
    const int tid = threadIdx.x, l16 = tid & 15, hw = tid >> 4, lane = tid & 31, warp = tid >> 5;
    const int rows = n_rep << lbk, bm = (1 << lbk) - 1;
    const int nit = (rows + 31) >> 5;
    // one lookup per representative block for the whole call: the row index of its first key row
    // (paged: page * page stride in rows + offset; a block never straddles a page).  rw[i] aliases
    // out[i]; it is read by the issue of the item holding block i, before that item's scores land.
    int* rw = reinterpret_cast<int*>(out);
    {
      const int32_t* btg = kPaged ? ks.block_table + (int64_t)b * ks.max_pages : nullptr;
      for (int i = tid; i < n_rep; i += kM1Threads) {
        const uint32_t s0 = (uint32_t)rep[i] << lbk;
        if constexpr (kPaged) {
          const uint32_t pi = ks.page_shift >= 0 ? (s0 >> ks.page_shift) : (s0 / (uint32_t)ks.page_size);
          const int page = bt16 ? (int)bt16[pi] : __ldg(btg + pi);
          rw[i] = (int)((int64_t)page * ks.sp_rows + (s0 - pi * (uint32_t)ks.page_size));
        } else {
          rw[i] = (int)s0;
        }
      }
      __syncthreads();
    }
    const uint32_t g0 = *g;
    // item i: rows 32 i .. 32 i + 31 of the call; thread t copies 16-byte chunk t % 16 of rows 8 j + t / 16
    // (one whole 256-byte row per half-warp instruction), stored at chunk (t % 16) ^ 4 (row & 1)
    auto issue = [&](int i) {
      const uint32_t gi = g0 + (uint32_t)i, slot = gi % kM1Slots;
      if (gi >= (uint32_t)kM1Slots) mbar_wait_u32(empty0 + 8 * slot, ((gi / kM1Slots) - 1) & 1u);
      const uint32_t dst0 = ring + slot * kM1Item + ((l16 ^ ((hw & 1) << 2)) << 4);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = 32 * i + 8 * j + hw;  // row of the call
        const int blk = r >> lbk;
        const bool ok = r < rows && (rep[blk] << lbk) + (r & bm) < Tk;
        const char* src = kbh + (uint64_t)(uint32_t)(ok ? rw[blk] + (r & bm) : 0) * row_bytes + l16 * 16;
        cp_async16_pf256(dst0 + (8 * j + hw) * 256, src, ok ? 16u : 0u);
      }
      m1_arrive_noinc(full0 + 8 * slot);
    };
    const int pre = min(nit, kM1Slots);
    for (int i = 0; i < pre; ++i) issue(i);
    // scoring: 4 lanes per row (row 8 warp + lane / 4 of the item); lane quarter p holds the F32L
    // segments p, p + 4, p + 8, p + 12 (8 components each, sequential fmaf), so the xor tree's o = 8
    // and o = 4 steps are local adds and o = 2, 1 are two shuffles (reading G9b, exactly)
    const int p = lane & 3, ir = 8 * warp + (lane >> 2);
    for (int i = 0; i < nit; ++i) {
      const uint32_t gi = g0 + (uint32_t)i, slot = gi % kM1Slots;
      mbar_wait_u32(full0 + 8 * slot, (gi / kM1Slots) & 1u);
      const char* rowp = ring_p + slot * kM1Item + ir * 256;
      float seg[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int ch = p + 4 * c;
        const uint4 kv = *reinterpret_cast<const uint4*>(rowp + ((ch ^ ((ir & 1) << 2)) << 4));
        const uint32_t w[4] = {kv.x, kv.y, kv.z, kv.w};
        float acc = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          acc = __fmaf_rn(qv[8 * c + 2 * e], bf16_lo(w[e]), acc);
          acc = __fmaf_rn(qv[8 * c + 2 * e + 1], bf16_hi(w[e]), acc);
        }
        seg[c] = acc;
      }
      // F32L tree: o = 8 (seg[p] + seg[p + 8], seg[p + 4] + seg[p + 12]), o = 4 (local), o = 2, 1 (shuffles)
      float v = (seg[0] + seg[2]) + (seg[1] + seg[3]);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      const int r = 32 * i + ir, blk = r >> lbk;
      const int s = r < rows ? (rep[blk] << lbk) + (r & bm) : Tk;
      float x = (s < Tk && (!causal || s <= tpos)) ? v : -INFINITY;
      for (int o = 4; o < (4 << lbk); o <<= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));  // block max
      if (p == 0 && (ir & bm) == 0 && r < rows) out[blk] = x;
      __syncwarp();
      if (lane == 0) m1_arrive(empty0 + 8 * slot);
      if (i + kM1Slots < nit) issue(i + kM1Slots);
    }
    *g = g0 + (uint32_t)nit;
    __syncthreads();
  }
};

template <bool kPaged>
__global__ void __launch_bounds__(kM1Threads, 4) mask_row1_kernel(Shape sh, QSrc qsrc, RowSrc ks,
                                                                   int32_t* __restrict__ idx,
                                                                   int32_t* __restrict__ cnt) {
  extern __shared__ __align__(16) char smem[];
  using L = MaskRow1Smem;
  SelState<kM1NMax, 4>& st = *reinterpret_cast<SelState<kM1NMax, 4>*>(smem + L::sel);
  const uint32_t sb = smem_u32(smem);
  const uint32_t full0 = sb + L::bar, empty0 = full0 + 8 * kM1Slots;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kM1Slots; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(full0 + 8 * s), "r"(kM1Threads) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(empty0 + 8 * s), "r"(4) : "memory");
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int lbk = 31 - __clz(sh.bk);
  uint32_t g = 0;
#ifdef HIPATTN_PHASES
  PhaseTimer ptimer;
#endif
  const int64_t units = (int64_t)sh.B * sh.Hq * sh.nqb;
  const int S = max(sh.chunks, 1);
  JobQueue jq(sh.sched, smem + L::jq);
  for (int64_t jb = blockIdx.x; jb < units * S; jb = jq.next(jb)) {
    jq.claim();
    const int64_t u = jb / S;
    const int cs = (int)(jb - u * S);
    int b, h, q;
    mask_unit_coords(sh, u, b, h, q);
    const int hk = h / (sh.Hq / sh.Hkv);
    const int Tk = seq_len(sh, b);
    const int Bq = visible_blocks(sh, q, Tk);
    const int64_t lin = ((int64_t)b * sh.Hq + h) * sh.nqb + q;
    int lo, len, nn, slot0;
    if (!chunk_job(Bq, sh.n, S, cs, lo, len, nn, slot0)) continue;
    Row1Scorer<kPaged> sc;
    {  // this lane's query components (chunks p + 4 c, fp32: exact widening of bf16)
      const char* qr = q_ptr(qsrc, b, h, (int64_t)q * sh.bq);
      const int p = tid & 3;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint4 qw = __ldg(reinterpret_cast<const uint4*>(qr + (p + 4 * c) * 16));
        const uint32_t w[4] = {qw.x, qw.y, qw.z, qw.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          sc.qv[8 * c + 2 * e] = bf16_lo(w[e]);
          sc.qv[8 * c + 2 * e + 1] = bf16_hi(w[e]);
        }
      }
    }
    sc.ring = sb + L::ring;
    sc.ring_p = smem + L::ring;
    sc.full0 = full0;
    sc.empty0 = empty0;
    sc.g = &g;
    sc.ks = ks;
    sc.kbh = ks.base + ((kPaged ? 0 : b * ks.sb) + hk * ks.sh) * (int64_t)ks.esize;
    sc.row_bytes = (uint32_t)(ks.st * ks.esize);
    sc.b = b; sc.Tk = Tk; sc.lbk = lbk; sc.causal = sh.causal;
    sc.tpos = (int64_t)q * sh.bq + (Tk - sh.Tq);
    if constexpr (kPaged) {
      if (ks.bt16 && Bq > sh.n) {  // stage this sequence's block-table row (uint16) for the lookups
        uint16_t* tb = reinterpret_cast<uint16_t*>(smem + L::bt);
        const int32_t* row = ks.block_table + (int64_t)b * ks.max_pages;
        const int np = min(ks.max_pages, (Tk + ks.page_size - 1) / ks.page_size);
        for (int i = tid; i < np; i += kM1Threads) tb[i] = (uint16_t)__ldg(row + i);
        sc.bt16 = tb;  // visible to the CTA after tree_search's first barrier
      }
    }
#ifdef HIPATTN_PHASES
    sc.pt = &ptimer;
    ptimer.mark(7);
#endif
    tree_search<kM1NMax, kM1Threads>(st, nn, lo, len, sc, idx + lin * sh.n + slot0, nullptr,
                                     make_jitter(sh.jitter, sh.seed, lin));
    if (cs == 0 && tid == 0) cnt[lin] = min(Bq, sh.n);
    __syncthreads();
  }
#ifdef HIPATTN_PHASES
  ptimer.flush();
#endif
}

// One query row per unit (decode), plain per-head masks, key rows addressable as 32-bit row indices (no GQA sharing, no top-r), bf16, d = 128,
// b_k in {1, 2, 4} (a block's rows inside one half-warp), n <= 256.
bool mask_row1_supported(const Shape& sh, const RowSrc& ks) {
  return ks.rows32 && sh.d == 128 && std::min(sh.bq, sh.Tq) == 1 && sh.group == 1 && sh.top_r == 0 && sh.bk <= 4 &&
         sh.n <= kM1NMax;
}

cudaError_t launch_mask_row1(const Shape& sh, const QSrc& qs, const RowSrc& ks, int32_t* idx, int32_t* cnt,
                             cudaStream_t stream, int num_sms) {
  auto kern = ks.paged ? mask_row1_kernel<true> : mask_row1_kernel<false>;
  int per_sm = 1;
  cudaError_t e = persistent_ctas(kern, kM1Threads, MaskRow1Smem::total, 0, &per_sm);
  if (e != cudaSuccess) return e;
  const int64_t jobs = (int64_t)sh.B * sh.Hq * sh.nqb * std::max(sh.chunks, 1);
  const int64_t grid = std::min<int64_t>(jobs, (int64_t)num_sms * per_sm);
  Shape s2 = sh;
  if ((e = setup_queue(s2, jobs, grid, stream)) != cudaSuccess) return e;
  kern<<<(unsigned)grid, kM1Threads, MaskRow1Smem::total, stream>>>(s2, qs, ks, idx, cnt);
  return cudaGetLastError();
}

}  // namespace hip

