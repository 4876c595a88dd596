// mask_tc.cu — HiP mask estimation (Alg. 1) with the branch scores on the 5th-gen
// tensor cores (tcgen05), bf16 inputs, fp32 accumulation in TMEM.
//
// Block approximation makes every representative score a small dense contraction:
// the b_q x d query block against the b_k x d rows of each representative key block.  Per iteration
// a CTA of 128 threads gathers the (up to 2n, then n) representative key blocks of its query block,
// 128 key rows per tile, straight from L2/HBM into 128-byte-swizzled K-major shared memory
// (coalesced 16-byte cp.async, 8 threads per 128-byte half row, so every warp instruction moves
// whole 32-byte sectors), and one elected lane of warp 0 issues
//     S^T_c [128 keys x 32 queries] = K_tile_c [128 x 128] . Q_block^T   (tcgen05.mma, M=128, N=32)
// into TMEM columns [32c, 32c+32) as two d-halves ("items", 4 x K16 each).  Items stream through a
// ring of SLOTS 16 KB shared slots: the MMA of an item is issued as soon as its bytes land and the
// slot is refilled as soon as that MMA completes, so SLOTS items are in flight.  After each round
// of up to TT tiles ONE epilogue pass reads the accumulators: each thread owns a TMEM lane (one key,
// 32 query columns), maxes over the valid query rows (a plain 32-way max unless the block touches
// the causal diagonal), then over the b_k lanes of a block with shuffles -> one fp32 score per
// representative block.  The selection (position-ordered split, radix select of the n best packed
// keys, tie toward the smaller block, stable compaction) is select.cuh.
//
// Why keys on M: b_q = 32 is below the smallest tcgen05 M (64), so the query block is the N=32
// operand and the gathered keys fill M = 128.  Gathers are 32 FLOP per byte, far below
// the tensor-core ridge; the kernel is bound by L2 gather latency (~1.2 us loaded, so ~128 KB must
// be in flight per SM for the ~15 TB/s L2 gather ceiling) and by the selection's serial chain.
//
// Launch shape: one unit (b, h, query block) per 128-thread CTA with a private 2-slot ring, 4 CTAs
// per SM, units claimed in order from a per-launch counter (common.cuh JobQueue).  When the units
// would leave SMs idle (decode at small batch, short prompts) a unit instead runs on a cluster of
// 2-8 CTAs on separate SMs (each scores a share of the tiles, scores exchanged through DSMEM) or on
// a deeper ring.  Measured and rejected (profiles/r01/notes.md, profiles/r02/notes.md): deeper rings
// with fewer units, rings shared between units (a lock in round 1, a slot allocator in round 2), five
// units per SM under a 96-register cap, one CTA per GQA group with collective scoring, TMA boxes
// ({64 x b_k} per block: ~half the cp.async rate).
#include "kernels.h"
#include "select.cuh"
#include "topr.cuh"

namespace hip {

constexpr int kMTNmax = 256;
constexpr uint32_t kQTileBytes = 2 * 32 * 128;   // two 64-column regions x 32 rows x 128 B
constexpr uint32_t kMTSlot = 128 * 128;          // one item: 128 rows x 64 bf16
constexpr uint32_t kIdescS = idesc_bf16(128, 32, 0, 0);

#ifdef HIPATTN_DEBUG_SCORES
// Debug builds only (libhipattn_debug.so; SURVEY 8(c) C-2 replay parity): every representative score
// of the units whose mask row `lin` has g_dbg_slot[lin] >= 0 is written to g_dbg_dump[slot * stride +
// block], so a test can feed the GPU's own scores to the oracle's selection steps.
__device__ const int32_t* g_dbg_slot = nullptr;
__device__ float* g_dbg_dump = nullptr;
__device__ int64_t g_dbg_stride = 0;
#define HIP_DBG_MEMBER float* dbg = nullptr;
#define HIP_DBG_STORE(blk, v) do { if (dbg) dbg[blk] = (v); } while (0)
#else
#define HIP_DBG_MEMBER
#define HIP_DBG_STORE(blk, v) do { } while (0)
#endif

template <int SLOTS, bool PAGED = false, bool CLU = false>
struct MaskTCSmemLayout {
  static constexpr uint32_t k0 = 0;                                        // ring (1024-aligned)
  static constexpr uint32_t q = k0 + SLOTS * kMTSlot;                      // Q tile
  static constexpr uint32_t sel = q + kQTileBytes;                         // SelState
  static constexpr uint32_t bt = sel + (uint32_t)align_up(sizeof(SelState<kMTNmax, 4>), 128);
  static constexpr uint32_t bt_bytes = PAGED ? (uint32_t)align_up(kBt16Max * 2, 128) : 0u;  // uint16 row
  static constexpr uint32_t misc = bt + bt_bytes;                          // mbarriers, TMEM address
  static constexpr uint32_t jq = misc + (uint32_t)align_up(8 * SLOTS + 4, 16); // JobQueue slots (2 x int64)
  static constexpr uint32_t dsc = jq + 16;                                  // CLU: 2 score arrays
  static constexpr uint32_t total = dsc + (CLU ? 2u * 4u * (uint32_t)SelState<kMTNmax, 4>::kRep : 0u);
};

template <int NT, int SLOTS, int TT, bool kPaged, class Sync, bool kGrp = false, bool kRow1 = false, bool kBk2 = false,
          int CL = 1>
struct TCScorer {
  static_assert(SLOTS >= 2 && SLOTS <= 8, "ring of 2..8 slots");
  static constexpr int RPP = NT / 8;        // rows per pass (8 threads per 128-byte half row)
  static constexpr int RJ = 128 / RPP;      // rows per thread per tile
  uint32_t q_s, k_s0;
  uint32_t mbar;      // shared address of [SLOTS] MMA-completion barriers, one per ring slot
  uint32_t phase;     // bit s: the parity to wait for on slot s's barrier (this thread's copy)
  uint32_t pend = 0;  // slots whose MMA has been committed but not yet waited
  uint32_t tmem;      // the CTA's first accumulator column
  RowSrc ks;
  const char* kh;        // contiguous: row 0 of this (b, kv head)
  uint32_t row_bytes;    // contiguous: bytes between key rows
  int b, hk, Tk, lbk, causal, rows_q, bpt;
  int rph = 32;          // kGrp: rows per query head (GQA-shared, G25): row j sits at tpos0 + j % rph
  int64_t tpos0;
  const int* pg;         // paged: page of each representative block (aliases the score output)
  const uint16_t* bt16 = nullptr;  // paged: the sequence's block-table row staged in shared memory
  float* dsc = nullptr;  // CL > 1: two score arrays, alternating by iteration (select.cuh score_buf)
  // this thread's source rows of the tile being issued (kBk2: the first row of each of its 4 blocks;
  // the second row is the first plus one row stride)
  const char* rp[kBk2 ? 4 : RJ];
  uint32_t rok;          // bit j: rp[j] is a real row (< T_k, block < n_rep)
  int crank = 0;         // CL > 1: this CTA's rank in the unit's cluster; it scores tiles crank + CL j
  uint32_t ckeep = 3u;   // top-r: bit h = this thread's chunk of d-half h has a kept component
                         // (else the chunk is zero-filled without a global read, topr.cuh)
  HIP_PT_MEMBER
  HIP_DBG_MEMBER
  __device__ __forceinline__ void mark(int p) { HIP_MARK(p); (void)p; }

  __device__ __forceinline__ const char* row(int s) const { return kh + (uint64_t)(uint32_t)s * row_bytes; }
  __device__ __forceinline__ int gtile(int lt) const { return CL == 1 ? lt : crank + lt * CL; }  // local -> call tile
  // Paged: key row s of a block whose page was looked up once per call (pg).
  __device__ __forceinline__ const char* paged_row(int page, int s) const {
    const uint32_t off = ks.page_shift >= 0 ? ((uint32_t)s & ((1u << ks.page_shift) - 1u))
                                            : ((uint32_t)s % (uint32_t)ks.page_size);
    return ks.base + ((int64_t)page * ks.sp + (int64_t)hk * ks.sh + (int64_t)off * ks.st) * ks.esize;
  }

  // Item i of a round = (tile c0 + i / 2, d-half i % 2) into slot i % SLOTS.  The row pointers are
  // computed once per tile (at its first half).
  __device__ __forceinline__ void issue(const int* rep, int n_rep, int c0, int i) {
    const int c = gtile(c0 + (i >> 1)), h = i & 1;
    const int tid = Sync::tid(), c8 = tid & 7, r0 = tid >> 3;
    if constexpr (kBk2) {  // b_k = 2 (the paper's setting): thread (c8, g) owns the 8 consecutive rows 8g..8g+7
      issue_bk2(rep, n_rep, c, h, c8, r0, i);
      return;
    } else {
    if (h == 0) {
      const int blk0 = c * bpt, nblk = min(bpt, n_rep - blk0);
      const int bmask = (1 << lbk) - 1;
      rok = 0;
#pragma unroll
      for (int j = 0; j < RJ; ++j) {
        const int r = r0 + RPP * j, lb = r >> lbk;
        const int s = lb < nblk ? (rep[blk0 + lb] << lbk) + (r & bmask) : Tk;
        const bool ok = s < Tk;
        if constexpr (kPaged) rp[j] = (ok ? paged_row(pg[blk0 + lb], s) : ks.base) + c8 * 16;
        else rp[j] = row(ok ? s : 0) + c8 * 16;
        rok |= (uint32_t)ok << j;
      }
    }
    const uint32_t dst = k_s0 + (i % SLOTS) * kMTSlot + sw128_off(r0, c8);
#pragma unroll
    for (int j = 0; j < RJ; ++j)  // rows r0 + RPP j share r0's swizzle phase (RPP % 8 == 0)
      cp_async16_pf256(dst + j * (RPP / 8) * 1024, rp[j] + h * 128, ((rok >> j) & (ckeep >> h) & 1u) ? 16u : 0u);
    }
  }

  // b_k = 2: rows 8g..8g+7 of the tile are the 4 blocks 4g..4g+3, so one 16-byte load brings their
  // representatives (and, paged, their pages) and the second row of a block is the first plus one
  // row stride (a block never straddles a page).  A warp instruction j still moves 4 whole 128-byte
  // half rows (rows 8g + j, g = 4w..4w+3).
  __device__ __forceinline__ void issue_bk2(const int* rep, int n_rep, int c, int h, int c8, int g, int i) {
    prep_bk2(rep, n_rep, c, h, g, c8);
    fire_bk2(h, c8, g, i);
  }
  // the row pointers of a tile, at its first half (before the slot it goes to is free)
  __device__ __forceinline__ void prep_bk2(const int* rep, int n_rep, int c, int h, int g, int c8) {
    if (h == 0) {
      const int blk0 = c * bpt, nblk = min(bpt, n_rep - blk0);
      const int4 rv = *reinterpret_cast<const int4*>(rep + blk0 + 4 * g);
      const int r4[4] = {rv.x, rv.y, rv.z, rv.w};
      int p4[4] = {0, 0, 0, 0};
      if constexpr (kPaged) {
        const int4 pv = *reinterpret_cast<const int4*>(pg + blk0 + 4 * g);
        p4[0] = pv.x; p4[1] = pv.y; p4[2] = pv.z; p4[3] = pv.w;
      }
      rok = 0;
#pragma unroll
      for (int b2 = 0; b2 < 4; ++b2) {
        const bool inb = 4 * g + b2 < nblk;
        const int s = inb ? r4[b2] << 1 : 0;
        const bool ok0 = inb && s < Tk, ok1 = inb && s + 1 < Tk;
        if constexpr (kPaged) rp[b2] = (ok0 ? paged_row(p4[b2], s) : ks.base) + c8 * 16;
        else rp[b2] = row(ok0 ? s : 0) + c8 * 16;
        rok |= ((uint32_t)ok0 << (2 * b2)) | ((uint32_t)ok1 << (2 * b2 + 1));
      }
    }
  }
  __device__ __forceinline__ void fire_bk2(int h, int c8, int g, int i) {
    const uint32_t dst = k_s0 + (uint32_t)(i % SLOTS) * kMTSlot + g * 1024;
    const uint32_t x = (uint32_t)c8;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      cp_async16_pf256(dst + j * 128 + ((x ^ j) << 4), rp[j >> 1] + ((j & 1) ? row_bytes : 0u) + h * 128,
                  ((rok >> j) & (ckeep >> h) & 1u) ? 16u : 0u);
  }

  template <class ST>
  __device__ __forceinline__ float* score_buf(ST& st, int iter) {
    if constexpr (CL > 1) return dsc + (iter & 1) * ST::kRep;
    else return st.scores();
  }

  __device__ __forceinline__ void wait_slot(int slot) {
    if (pend & (1u << slot)) {
      mbar_wait_u32(mbar + 8u * slot, (phase >> slot) & 1u);
      phase ^= 1u << slot;
      pend &= ~(1u << slot);
    }
  }

  __device__ void epilogue(const int* rep, int n_rep, int c0, int nt, float* out) {
    const int warp = Sync::tid() >> 5, lane = threadIdx.x & 31;
    const int r = 32 * warp + lane, bm = (1 << lbk) - 1;
    for (int cc = 0; cc < nt; ++cc) {
      const int c = gtile(c0 + cc);
      const int blk0 = c * bpt, nblk = min(bpt, n_rep - blk0);
      const int lb = r >> lbk;
      float best = -INFINITY;
      if constexpr (kRow1) {  // decode (rows_q == 1): one query row, one TMEM column per key
        const float v0 = tmem_ld_32x32b_x1(tmem + ((uint32_t)(32 * warp) << 16) + 32 * cc);
        if (lb < nblk) {
          const int s = (rep[blk0 + lb] << lbk) + (r & bm);
          if (s < Tk && (!causal || s <= tpos0)) best = v0;
        }
        for (int off = 1; off <= bm; off <<= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, off));
        if (lb < nblk && (r & bm) == 0) {
          HIP_DBG_STORE(rep[blk0 + lb], best);
          out[blk0 + lb] = best;
          if constexpr (CL > 1)  // every CTA of the cluster selects on all the scores
            for (int rr = 1; rr < CL; ++rr) st_cluster_f32(smem_u32(out + blk0 + lb), (crank + rr) % CL, best);
        }
        continue;
      }
      float v[32];
      tmem_ld_32x32b_x32(tmem + ((uint32_t)(32 * warp) << 16) + 32 * cc, v);
      if (lb < nblk) {
        const int s = (rep[blk0 + lb] << lbk) + (r & bm);
        if (s < Tk) {
          if (rows_q == 32 && (!causal || s <= tpos0)) {  // every query row sees this key
            float m0 = fmaxf(v[0], v[1]), m1 = fmaxf(v[2], v[3]), m2 = fmaxf(v[4], v[5]), m3 = fmaxf(v[6], v[7]);
#pragma unroll
            for (int j = 8; j < 32; j += 4) {
              m0 = fmaxf(m0, v[j]); m1 = fmaxf(m1, v[j + 1]); m2 = fmaxf(m2, v[j + 2]); m3 = fmaxf(m3, v[j + 3]);
            }
            best = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
          } else if constexpr (kGrp) {  // rows of G heads: row j sits at position tpos0 + j % rph
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < rows_q && (!causal || s <= tpos0 + j % rph)) best = fmaxf(best, v[j]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < rows_q && (!causal || s <= tpos0 + j)) best = fmaxf(best, v[j]);
          }
        }
      }
      for (int off = 1; off <= bm; off <<= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, off));
      if (lb < nblk && (r & bm) == 0) {
        HIP_DBG_STORE(rep[blk0 + lb], best);
        out[blk0 + lb] = best;
        if constexpr (CL > 1)
          for (int rr = 1; rr < CL; ++rr) st_cluster_f32(smem_u32(out + blk0 + lb), (crank + rr) % CL, best);
      }
    }
  }

  __device__ void score(const int* rep, int n_rep, float* out) {
    const int ntiles_all = (n_rep + bpt - 1) / bpt;
    // CL > 1: the cluster's CTAs hold identical search states; CTA `crank` gathers and scores tiles
    // crank, crank + CL, ... and stores each score into every CTA's score array of this iteration's
    // parity (DSMEM).  One cluster barrier at the end (every score everywhere before the
    // selections); a peer already writing the next iteration's scores uses the other array.
    const int ntiles = CL == 1 ? ntiles_all : (ntiles_all > crank ? (ntiles_all - crank + CL - 1) / CL : 0);
    if constexpr (kPaged) {
      // one block-table lookup per representative block for the whole call (a block never straddles
      // a page), so the gathers below carry no dependent global load.  pg[i] is read only before
      // the epilogue that overwrites out[i].
      int* pgw = reinterpret_cast<int*>(out);
      const int32_t* bt = ks.block_table + (int64_t)b * ks.max_pages;
      for (int i = Sync::tid(); i < n_rep; i += NT) {
        if (CL > 1 && ((i / bpt) % CL) != crank) continue;  // another CTA's tile (its score may land here)
        const uint32_t s0 = (uint32_t)rep[i] << lbk;
        const uint32_t pi = ks.page_shift >= 0 ? (s0 >> ks.page_shift) : (s0 / (uint32_t)ks.page_size);
        pgw[i] = bt16 ? (int)bt16[pi] : __ldg(bt + pi);  // staged row: no global round trip
      }
      Sync::sync();
      pg = pgw;
    }
    for (int c0 = 0; c0 < ntiles; c0 += TT) {  // rounds of up to TT tiles (TMEM columns)
      const int nt = min(TT, ntiles - c0), nitems = 2 * nt;
#pragma unroll
      for (int i = 0; i < SLOTS; ++i) {  // prologue: SLOTS items in flight
        if (i < nitems) issue(rep, n_rep, c0, i);
        cp_async_commit();
      }
      for (int i = 0; i < nitems; ++i) {
        cp_async_wait<SLOTS - 1>();  // item i landed
        fence_proxy_async_smem();
        Sync::sync();
        mark(11);  // (profiling builds) landing wait + barrier
        const int slot = i % SLOTS;
        // one elected lane of warp 0 issues the MMAs: a warp-uniform branch plus elect.sync lets the
        // compiler issue each tcgen05.mma once from uniform registers (behind `tid == 0` it wraps every
        // MMA in a per-lane waterfall loop of R2UR broadcasts: C4 mask 19.86 -> 18.84 ms without it)
        if ((Sync::tid() >> 5) == 0 && elect_one()) {
          tc_fence_after();
          const int cc = i >> 1, h = i & 1;
          const uint32_t kt = k_s0 + slot * kMTSlot;
#pragma unroll
          for (int s = 0; s < 4; ++s) {  // one d-half = 4 x K16
            uint64_t a = smem_desc(kt + s * 32, 16, 1024, kLayoutSw128);
            uint64_t bq = smem_desc(q_s + h * (32 * 128) + s * 32, 16, 1024, kLayoutSw128);
            umma_bf16(tmem + 32 * cc, a, bq, kIdescS, (h | s) ? 1u : 0u);
          }
          umma_commit_u32(mbar + 8u * slot);
        }
        pend |= 1u << slot;
        mark(12);  // MMA issue
        // refill this slot with item i + SLOTS as soon as MMA(i) has read it
        if (i + SLOTS < nitems) {
          if constexpr (kBk2) {  // the refill's addresses first, then wait for the slot
            const int ii = i + SLOTS, tid = Sync::tid();
            prep_bk2(rep, n_rep, gtile(c0 + (ii >> 1)), ii & 1, tid >> 3, tid & 7);
            wait_slot(slot);
            mark(13);  // MMA completion wait
            fire_bk2(ii & 1, tid & 7, tid >> 3, ii);
          } else {
          wait_slot(slot);
          mark(13);  // MMA completion wait
          issue(rep, n_rep, c0, i + SLOTS);
          }
        }
        cp_async_commit();
        mark(14);  // refill issue
      }
      mark(1);  // gathers + MMA issue
#pragma unroll
      for (int sl = 0; sl < SLOTS; ++sl) wait_slot(sl);  // drain the round's MMAs
      mark(2);  // MMA drain
      tc_fence_after();
      epilogue(rep, n_rep, c0, nt, out);
      tc_fence_before();
      Sync::sync();  // scores visible; TMEM reads done before the next round's MMAs
      mark(3);  // epilogue
    }
    if constexpr (CL > 1) cluster_sync();
  }
};

// One unit per 128-thread CTA (persistent: CTAs stride over the units).
// EXT: the mask options, each a separate instantiation so that the plain Alg. 1 kernel (EXT = 0)
// carries none of their code or registers: bit 0 ensemble split jitter (G23), bit 1 top-r (G22),
// bit 2 GQA-shared rows (G25); bit 3 = one query row per unit (decode), whose epilogue reads a single
// TMEM column per key; bit 4 = b_k = 2, the gather mapping with 4 blocks per thread.
template <int SLOTS, int TT, bool kPaged, int MINB, int EXT, int CL = 1>
__global__ void __launch_bounds__(128, MINB) mask_tc_kernel(Shape sh, QSrc qsrc, RowSrc ks,
                                                                   int32_t* __restrict__ idx,
                                                                   int32_t* __restrict__ cnt) {
  constexpr int NT = 128;
  constexpr bool kJit = (EXT & 1) != 0, kTopR = (EXT & 2) != 0, kGrp = (EXT & 4) != 0, kRow1 = (EXT & 8) != 0;
  constexpr bool kBk2 = (EXT & 16) != 0;  // b_k = 2 gather mapping (the caller checked b_k == 2)
  constexpr uint32_t kColsUsed = 32 * TT;
  constexpr uint32_t kCols = kColsUsed <= 32 ? 32 : kColsUsed <= 64 ? 64 : kColsUsed <= 128 ? 128
                             : kColsUsed <= 256 ? 256 : 512;  // allocation: a power of two
  static_assert(kColsUsed <= 512, "TMEM columns");
  using Sync = CtaSync;
  extern __shared__ __align__(16) char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t pad = ((raw + 1023u) & ~1023u) - raw;
  char* base = smem_raw + pad;
  const uint32_t sbase = raw + pad;
  using L = MaskTCSmemLayout<SLOTS, kPaged, (CL > 1)>;
  SelState<kMTNmax, 4>& st = *reinterpret_cast<SelState<kMTNmax, 4>*>(base + L::sel);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(base + L::misc);  // one MMA-completion barrier per slot
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + L::misc + 8 * SLOTS);
  const int warp = threadIdx.x >> 5;

  if (threadIdx.x == 0) {
    for (int s = 0; s < SLOTS; ++s) mbar_init(mbar + s, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<kCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  uint32_t phase = 0u;  // bit s: parity of ring slot s's barrier (carried across units)
  const int lbk = 31 - __clz(sh.bk);
#ifdef HIPATTN_PHASES
  PhaseTimer ptimer;
#endif

  const int64_t units = (int64_t)sh.B * (sh.group > 1 ? sh.Hkv : sh.Hq) * sh.nqb;
  const int S = max(sh.chunks, 1);
  // CL > 1: one unit per cluster of CL CTAs (grid = units x CL; the launcher guarantees a single wave)
  const int crank = CL > 1 ? (int)cluster_ctarank() : 0;
  JobQueue jq(sh.sched, base + L::jq);
  for (int64_t jb = CL > 1 ? blockIdx.x / CL : blockIdx.x; jb < units * S; jb = jq.next(jb)) {
    jq.claim();
    const int64_t u = jb / S;
    const int cs = (int)(jb - u * S);
    int b, h, q;  // h: mask head (the kv head when GQA-shared, G25)
    mask_unit_coords(sh, u, b, h, q);
    const int hk = sh.group > 1 ? h : h / (sh.Hq / sh.Hkv);
    const int Tk = seq_len(sh, b);
    const int Bq = visible_blocks(sh, q, Tk);
    const int64_t lin = ((int64_t)b * mask_heads(sh) + h) * sh.nqb + q;
    const int rph = min(sh.bq, sh.Tq - q * sh.bq);    // rows per query head
    const int rows_q = kGrp ? rph * sh.group : rph;   // rows scored together
    // query row r of the tile: head qhead(r), position q * b_q + r % rph
    auto qrow = [&](int r) -> const char* {
      if constexpr (kGrp) {
        if (sh.group > 1) return q_ptr(qsrc, b, h * sh.group + r / rph, (int64_t)q * sh.bq + r % rph);
      }
      return q_ptr(qsrc, b, h, (int64_t)q * sh.bq + r);
    };
    int lo, len, nn, slot0;
    if (!chunk_job(Bq, sh.n, S, cs, lo, len, nn, slot0)) continue;
    const uint32_t q_s = sbase + L::q;
    uint32_t ckeep = 3u;  // bit h: this thread's 16-byte key chunk of d-half h holds a kept component
    if (kTopR && Bq > sh.n && sh.top_r > 0 && sh.top_r < 128) {
      // top-r approximation (G22; topr.cuh): a_c = max_t |q_tc| (thread c), keep bits by
      // rank -> st.warp_tot[c / 32]; the query tile is stored with the dropped components zeroed
      float* a = reinterpret_cast<float*>(st.rep);
      {
        const int c = Sync::tid();
        float m = 0.f;
        for (int t = 0; t < rows_q; ++t) {
          const __nv_bfloat16 v = *reinterpret_cast<const __nv_bfloat16*>(qrow(t) + 2 * c);
          m = fmaxf(m, fabsf(__bfloat162float(v)));
        }
        a[c] = m;
      }
      Sync::sync();
      const unsigned kb = __ballot_sync(0xffffffffu, top_r_keep(a, 128, Sync::tid(), sh.top_r));
      if ((threadIdx.x & 31) == 0) st.warp_tot[Sync::tid() >> 5] = (int)kb;
      Sync::sync();
      const uint32_t* kw = reinterpret_cast<const uint32_t*>(st.warp_tot);  // 4 keep words (shared)
      for (int p = Sync::tid(); p < 32 * 16; p += NT) {
        const int r = p >> 4, c16 = p & 15;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (r < rows_q) v = *reinterpret_cast<const uint4*>(qrow(r) + c16 * 16);
        const uint32_t kbyte = (kw[c16 >> 2] >> ((c16 & 3) * 8)) & 0xffu;
        uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          w[e] &= (((kbyte >> (2 * e)) & 1u) ? 0x0000ffffu : 0u) | (((kbyte >> (2 * e + 1)) & 1u) ? 0xffff0000u : 0u);
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(q_s + (c16 >> 3) * (32 * 128) + sw128_off(r, c16 & 7)),
                     "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]) : "memory");
      }
      const int c8 = Sync::tid() & 7;  // the gather chunk of this thread: components 64 h + 8 c8 .. + 8
      ckeep = (((kw[c8 >> 2] >> ((c8 & 3) * 8)) & 0xffu) ? 1u : 0u) |
              (((kw[2 + (c8 >> 2)] >> ((c8 & 3) * 8)) & 0xffu) ? 2u : 0u);
      cp_async_commit();  // (empty group: keeps the ring's group accounting unchanged)
    } else if (Bq > sh.n) {
      // query block -> K-major SW128 tile (B operand, N = 32 rows, rows >= rows_q zero); waited for
      // together with the first item of the first round
      for (int p = Sync::tid(); p < 32 * 16; p += NT) {
        const int r = p >> 4, c16 = p & 15;
        const bool ok = r < rows_q;
        const char* src = qrow(ok ? r : 0) + c16 * 16;
        cp_async16(q_s + (c16 >> 3) * (32 * 128) + sw128_off(r, c16 & 7), src, ok ? 16u : 0u);
      }
      cp_async_commit();
    }
    TCScorer<NT, SLOTS, TT, kPaged, Sync, kGrp, kRow1, kBk2, CL> sc;
    sc.crank = crank;
    if constexpr (CL > 1) sc.dsc = reinterpret_cast<float*>(base + L::dsc);
    sc.q_s = q_s;
    sc.k_s0 = sbase + L::k0;
    sc.mbar = smem_u32(mbar);
    sc.phase = phase;
    sc.tmem = tmem;
    sc.ks = ks;
    sc.kh = ks.base + (b * ks.sb + hk * ks.sh) * (int64_t)ks.esize;
    sc.row_bytes = (uint32_t)(ks.st * ks.esize);
    sc.b = b; sc.hk = hk; sc.Tk = Tk; sc.lbk = lbk; sc.causal = sh.causal; sc.rows_q = rows_q;
    sc.bpt = 128 >> lbk;
    sc.tpos0 = (int64_t)q * sh.bq + (Tk - sh.Tq);
    sc.rph = rph;
    sc.ckeep = ckeep;
    if constexpr (kPaged) {
      if (ks.bt16 && Bq > sh.n) {  // stage this sequence's block-table row (uint16) for the lookups
        uint16_t* tb = reinterpret_cast<uint16_t*>(base + L::bt);
        const int32_t* row = ks.block_table + (int64_t)b * ks.max_pages;
        const int np = min(ks.max_pages, (Tk + ks.page_size - 1) / ks.page_size);
        for (int i = Sync::tid(); i < np; i += NT) tb[i] = (uint16_t)__ldg(row + i);
        sc.bt16 = tb;  // visible to the CTA after tree_search's first barrier
      }
    }
#ifdef HIPATTN_DEBUG_SCORES
    if (g_dbg_slot && g_dbg_slot[lin] >= 0) sc.dbg = g_dbg_dump + (int64_t)g_dbg_slot[lin] * g_dbg_stride;
#endif
#ifdef HIPATTN_PHASES
    sc.pt = &ptimer;
    ptimer.mark(7);  // unit setup / Q load / exact units
#endif
    tree_search<kMTNmax, NT, decltype(sc), Sync>(st, nn, lo, len, sc, idx + lin * sh.n + slot0, nullptr,
                                                 kJit ? make_jitter(sh.jitter, sh.seed, lin) : SplitJitter());
    phase = sc.phase;
    if (cs == 0 && Sync::tid() == 0 && crank == 0) cnt[lin] = min(Bq, sh.n);
    Sync::sync();
  }
  tc_fence_before();
  __syncthreads();
#ifdef HIPATTN_PHASES
  ptimer.flush();
#endif
  if (warp == 0) tmem_dealloc<kCols>(*tmem_slot);
}

// Any query block of <= 32 rows (the N = 32 operand is zero-padded): decode (b_q = 1) too — the
// tensor cores are idle in this gather-bound kernel, so padding costs nothing, and the ring of
// swizzled half tiles keeps more bytes in flight than the register-staged GEMV (C3: 229 vs 404 us).
// b_k must be a power of two <= 32 so that a block's rows sit in one warp's TMEM lanes.
bool mask_tc_supported(const Shape& sh) {
  return sh.d == 128 && sh.bq >= 1 && sh.bq * sh.group <= 32 && sh.bk >= 1 && sh.bk <= 32 && (32 % sh.bk) == 0 &&
         sh.n <= kMTNmax;
}

template <int SLOTS, int TT, int MINB, int EXT>
static cudaError_t launch_v(const Shape& sh, const QSrc& qs, const RowSrc& ks, int32_t* idx, int32_t* cnt,
                            cudaStream_t stream, int num_sms) {
  const size_t smem = (ks.paged ? MaskTCSmemLayout<SLOTS, true>::total : MaskTCSmemLayout<SLOTS, false>::total) + 1024;
  auto kern = ks.paged ? mask_tc_kernel<SLOTS, TT, true, MINB, EXT> : mask_tc_kernel<SLOTS, TT, false, MINB, EXT>;
  int per_sm = 1;
  cudaError_t e = persistent_ctas(kern, 128, smem, 32 * TT, &per_sm);
  if (e != cudaSuccess) return e;
  const int64_t units = (int64_t)sh.B * (sh.group > 1 ? sh.Hkv : sh.Hq) * sh.nqb;
  const int64_t jobs = units * std::max(sh.chunks, 1);
  const int64_t grid = std::min<int64_t>(jobs, (int64_t)num_sms * per_sm);
  Shape s2 = sh;
  if ((e = setup_queue(s2, jobs, grid, stream)) != cudaSuccess) return e;
  kern<<<(unsigned)grid, 128, smem, stream>>>(s2, qs, ks, idx, cnt);
  return cudaGetLastError();
}

// One unit per cluster of CL CTAs on CL SMs (small decode batches: the units would leave SMs idle,
// and one SM's memory-level parallelism bounds a unit's gathers).  Grid = units x CL, one wave.
template <int SLOTS, int TT, int EXT, int CL>
static cudaError_t launch_cluster(const Shape& sh, const QSrc& qs, const RowSrc& ks, int32_t* idx, int32_t* cnt,
                                  cudaStream_t stream) {
  const size_t smem = (ks.paged ? MaskTCSmemLayout<SLOTS, true, true>::total : MaskTCSmemLayout<SLOTS, false, true>::total) + 1024;
  auto kern = ks.paged ? mask_tc_kernel<SLOTS, TT, true, 1, EXT, CL> : mask_tc_kernel<SLOTS, TT, false, 1, EXT, CL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t units = (int64_t)sh.B * (sh.group > 1 ? sh.Hkv : sh.Hq) * sh.nqb * std::max(sh.chunks, 1);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(units * CL));
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  Shape s2 = sh;
  s2.sched = nullptr;  // one unit per cluster, no claiming
  e = cudaLaunchKernelEx(&cfg, kern, s2, qs, ks, idx, cnt);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// One instantiation per mask option (EXT bits above), so none inflates another's registers; the
// b_k = 2 gather mapping (bit 4) and the single-row decode epilogue (bit 3) are specialisations of
// Alg. 1 itself.  Dispatch depends on the arguments only.
cudaError_t launch_mask_tc(const Shape& sh, const QSrc& qs, const RowSrc& ks, int32_t* idx, int32_t* cnt,
                           cudaStream_t stream, int num_sms) {
  const int ext = (sh.jitter > 0 ? 1 : 0) | (sh.top_r > 0 ? 2 : 0) | (sh.group > 1 ? 4 : 0);
  const int64_t jobs = (int64_t)sh.B * (sh.group > 1 ? sh.Hkv : sh.Hq) * sh.nqb * std::max(sh.chunks, 1);
  switch (ext) {
    case 0:
      if (sh.bk == 2) {
        if (sh.bq == 1) {  // decode
          // Small batches leave SMs idle: spread each unit over a cluster of 4 or 2 CTAs (SMs) when the
          // units fit, else give each unit a deeper ring (one unit per SM: 8 slots, a whole
          // iteration's 8 items in flight; two per SM: 4 slots).  Same arithmetic.
          if (sh.chunks <= 1 && 4 * jobs <= num_sms)
            return launch_cluster<4, 4, 8 | 16, 4>(sh, qs, ks, idx, cnt, stream);
          if (sh.chunks <= 1 && 2 * jobs <= num_sms)
            return launch_cluster<4, 4, 8 | 16, 2>(sh, qs, ks, idx, cnt, stream);
          if (jobs <= num_sms) return launch_v<8, 4, 1, 8 | 16>(sh, qs, ks, idx, cnt, stream, num_sms);
          if (jobs <= 2 * (int64_t)num_sms) return launch_v<4, 4, 2, 8 | 16>(sh, qs, ks, idx, cnt, stream, num_sms);
          return launch_v<2, 4, 4, 8 | 16>(sh, qs, ks, idx, cnt, stream, num_sms);
        }
        // few units (short prompts, small batches): a cluster of CTAs per unit, as for decode
        if (sh.chunks <= 1 && 4 * jobs <= num_sms) return launch_cluster<4, 4, 16, 4>(sh, qs, ks, idx, cnt, stream);
        if (sh.chunks <= 1 && 2 * jobs <= num_sms) return launch_cluster<4, 4, 16, 2>(sh, qs, ks, idx, cnt, stream);
        return launch_v<2, 4, 4, 16>(sh, qs, ks, idx, cnt, stream, num_sms);
      }
      if (sh.bq == 1) return launch_v<2, 4, 4, 8>(sh, qs, ks, idx, cnt, stream, num_sms);
      return launch_v<2, 4, 4, 0>(sh, qs, ks, idx, cnt, stream, num_sms);
    case 1: return launch_v<2, 4, 4, 1>(sh, qs, ks, idx, cnt, stream, num_sms);
    case 2: return launch_v<2, 4, 4, 2>(sh, qs, ks, idx, cnt, stream, num_sms);
    case 4:  // GQA-shared masks: one unit per kv head, so few units at small batch -> clusters
      if (sh.chunks <= 1 && 8 * jobs <= num_sms) return launch_cluster<4, 4, 4, 8>(sh, qs, ks, idx, cnt, stream);
      if (sh.chunks <= 1 && 4 * jobs <= num_sms) return launch_cluster<4, 4, 4, 4>(sh, qs, ks, idx, cnt, stream);
      return launch_v<2, 4, 4, 4>(sh, qs, ks, idx, cnt, stream, num_sms);
    default: return launch_v<2, 4, 4, 7>(sh, qs, ks, idx, cnt, stream, num_sms);
  }
}

#ifdef HIPATTN_DEBUG_SCORES
// Debug builds only: slot_of_unit [units] (device, -1 = not dumped) and dump [slots, stride] (device);
// NULL slot_of_unit switches the dump off.
extern "C" int hip_debug_score_dump(const int32_t* slot_of_unit, float* dump, int64_t stride) {
  if (cudaMemcpyToSymbol(hip::g_dbg_slot, &slot_of_unit, sizeof(slot_of_unit)) != cudaSuccess) return 1;
  if (cudaMemcpyToSymbol(hip::g_dbg_dump, &dump, sizeof(dump)) != cudaSuccess) return 2;
  return cudaMemcpyToSymbol(hip::g_dbg_stride, &stride, sizeof(stride)) == cudaSuccess ? 0 : 3;
}
#endif

#ifdef HIPATTN_PHASES
// Profiling builds only (profiles/phase_timers.py): read and clear this translation unit's
// per-phase cycle counters.
extern "C" int hip_debug_phase_cycles(unsigned long long* out16) {
  if (cudaDeviceSynchronize() != cudaSuccess) return 1;
  if (cudaMemcpyFromSymbol(out16, hip::g_phase_cycles, 16 * sizeof(unsigned long long)) != cudaSuccess) return 2;
  unsigned long long z[16] = {0};
  return cudaMemcpyToSymbol(hip::g_phase_cycles, z, sizeof(z)) == cudaSuccess ? 0 : 3;
}
#endif

}  // namespace hip
