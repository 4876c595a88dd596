// attn_row1.cu — block-sparse attention for single-row query blocks (decode: T_q = 1, or b_q = 1),
// bf16, d = 128, contiguous or paged K/V (Eq. 2-3; paged decode P:451, Alg. 2 line
// "fused sparse attention" P:612).
//
// One query row against <= k selected keys is a vector-matrix product: "tensor units cannot help"
// (P:1053-1054), the kernel is HBM-bound, and what sets its speed is how many bytes each unit keeps
// in flight and how little else sits on its serial path.  So, unlike the prefill kernel (attn_tc,
// tcgen05), the math here runs on the CUDA cores straight from shared memory:
//   * items of 32 keys = 32 K rows + 32 V rows (16 KB) stream through a 3-slot ring of cp.async
//     gathers (16 lanes per 256-byte row: whole sectors, no L1); completion is tracked on mbarriers
//     (cp.async.mbarrier.arrive.noinc -> "full", one arrival per reading thread -> "empty"), so no CTA-wide
//     barrier sits between items and a slot is refilled as soon as the four warps have read it;
//   * warp w owns keys 8w..8w+7 of every item: 4 lanes per key each dot a quarter of d (q in
//     registers), two shuffles complete q.k; the warp keeps its own online softmax state (max, sum,
//     O[4 columns per lane]), so the per-item softmax needs shuffles only; PV reads V rows with
//     conflict-free 8-byte lanes; the four warp states are merged once per unit;
//   * probabilities stay fp32 (no bf16 rounding of P as in the tensor-core kernel).
// Rows are staged in shared memory with the 16-byte chunk index XOR 4 * (key & 1), which makes the
// QK reads (lanes of two keys x four quarters) bank-conflict-free per quarter warp.
// Split-K (when the units leave CTA slots idle): a unit runs on a thread-block cluster of S CTAs, CTA
// sp takes the unit's 128-key chunks [sp nch / S, (sp + 1) nch / S) and keeps their states in its
// shared memory; rank 0 merges all chunk states in chunk order through DSMEM (max-rescaled, like the
// warp states) — the unsplit kernel's operations, so the output does not depend on S.
#include "kernels.h"
#include "sinkwin.cuh"

namespace hip {

constexpr int kR1Threads = 128;
constexpr int kR1Slots = 3;
constexpr uint32_t kR1Item = 16384;            // 32 K rows + 32 V rows of 256 bytes
constexpr int kR1Tok = 768;                    // <= 512 selected keys + <= 256 sink / window tokens
constexpr int kR1MaxN = 512;                   // n = k / b_k <= kR1MaxN (the index row staged in the prologue)
constexpr int kR1BtStage = (int)(kR1Item / 4) - kR1MaxN;  // block-table entries staged with it (3584)
constexpr int kR1ChunkItems = 4;               // a softmax chunk: 4 items = 128 keys (<= 6 chunks per unit)
constexpr float kR1Log2e = 1.4426950408889634f;
constexpr float kR1Ln2 = 0.6931471805599453f;

struct Row1Smem {
  static constexpr uint32_t ring = 0;
  static constexpr uint32_t tok = ring + kR1Slots * kR1Item;      // [kR1Tok] row of each key slot (-1: none)
  static constexpr uint32_t xlist = tok + kR1Tok * 4;              // [kMaxExtra] sink / window tokens
  static constexpr uint32_t merge = xlist + kMaxExtra * 4;         // [4][128] O + [4] max + [4] sum, scan scratch
  static constexpr uint32_t bar = merge + (4 * 128 + 8 + 8) * 4;   // full[3], empty[3]
  static constexpr uint32_t jq = bar + 2 * kR1Slots * 8;           // JobQueue slots
  static constexpr uint32_t flag = jq + 16;                        // the unit's block count
  static constexpr uint32_t cstate = flag + 16;                    // cluster split: [3][132] chunk states
  static constexpr uint32_t total = cstate + 3 * kSplitStride * 4;
};


// acc <- acc (+) part: two softmax states over disjoint key sets merged at their common max.  The
// unit's result is the merge of its chunk states in chunk order, whichever jobs computed the chunks
// (one job, or split-K jobs whose chunk states pass through the workspace): the same operations in
// the same order, so the output does not depend on the split factor, i.e. on batch composition.
__device__ __forceinline__ void r1_merge(float& Ma, float& La, float& Oa, float Mc, float Lc, float Oc) {
  if (Mc == -INFINITY) return;  // no visible key in the part
  if (Ma == -INFINITY) {
    Ma = Mc; La = Lc; Oa = Oc;
    return;
  }
  const float Mn = fmaxf(Ma, Mc);
  const float fa = ex2_approx(Ma - Mn), fc = ex2_approx(Mc - Mn);
  Oa = fmaf(Oc, fc, Oa * fa);
  La = fmaf(Lc, fc, La * fa);
  Ma = Mn;
}

// kClu: split-K on a thread-block cluster (one unit per cluster, one split per CTA): the chunk states
// stay in each CTA's shared memory and rank 0 merges them in chunk order through DSMEM — the same
// operations as the unsplit kernel, with no workspace, atomics or global round trip.
template <bool kPaged, bool kSW, bool kClu>
__global__ void __launch_bounds__(kR1Threads, 4) attn_row1_kernel(Shape sh, QSrc qsrc, RowSrc ks, RowSrc vs,
                                                                   const int32_t* __restrict__ idx,
                                                                   const int32_t* __restrict__ cnt, float scale_log2,
                                                                   char* __restrict__ o, int64_t osb, int64_t osh,
                                                                   int64_t ost, float* __restrict__ lse) {
  extern __shared__ __align__(16) char smem[];
  using L = Row1Smem;
  const uint32_t sb = smem_u32(smem);
  int* tok = reinterpret_cast<int*>(smem + L::tok);
  int* xlist = reinterpret_cast<int*>(smem + L::xlist);
  float* mo = reinterpret_cast<float*>(smem + L::merge);          // [4][128]
  float* mm = mo + 4 * 128;                                        // [4] warp maxima
  float* ml = mm + 4;                                              // [4] warp sums
  int* scan = reinterpret_cast<int*>(ml + 4);                      // [8] build_extra scratch
  int* scnt = reinterpret_cast<int*>(smem + L::flag);             // the unit's block count
  const uint32_t full0 = sb + L::bar, empty0 = full0 + 8 * kR1Slots;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kR1Slots; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(full0 + 8 * s), "r"(kR1Threads) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(empty0 + 8 * s), "r"(kR1Threads) : "memory");
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int lbk = 31 - __clz(sh.bk);
  // QK lanes: key j = lane / 4 of the warp's 8, quarter p = lane % 4 (16-byte chunks p + 4 i, i < 4)
  const int kj = lane >> 2, kp = lane & 3;
  uint32_t g = 0;  // ring items issued / consumed by this CTA so far (slot g % 3, parity (g / 3) & 1)

  const int64_t units = (int64_t)sh.B * sh.Hq * sh.nqb;
  const int S = kClu ? sh.splits : 1;
  float* cst = reinterpret_cast<float*>(smem + L::cstate);         // kClu: this CTA's chunk states
  JobQueue jq(sh.sched, smem + L::jq);
  for (int64_t jb = blockIdx.x; jb < units * S; jb = jq.next(jb)) {
    jq.claim();
    const int64_t u = kClu ? jb / S : jb;
    const int sp = kClu ? (int)(jb - u * S) : 0;
    int b, h, q;
    unit_coords(sh, u, b, h, q);
    const int hk = h / (sh.Hq / sh.Hkv);
    const int Tk = seq_len(sh, b);
    const int64_t lin = mask_lin(sh, b, h, q);
    const int64_t tpos = (int64_t)q * sh.bq + (Tk - sh.Tq);  // the row's key position (G7)
    const int nkb = (Tk + sh.bk - 1) / sh.bk;
    // Prologue, one global round trip: the unit's count, its index row and (paged) the block-table
    // entries of its sequence are loaded together into ring slot 2 (free between jobs: every item of
    // the previous job has been consumed), then build_extra and the row staging work from shared
    // memory — no chain of dependent global loads (count -> indices -> pages) before the first gather.
    int* sblk = reinterpret_cast<int*>(smem + L::ring + 2 * kR1Item);       // [n] selected blocks
    int* sbt = sblk + kR1MaxN;                                              // [<= kR1BtStage] pages
    const int32_t* blk = idx + lin * sh.n;
    const int npg = kPaged ? (Tk + ks.page_size - 1) / ks.page_size : 0;
    const bool bt_staged = kPaged && npg <= kR1BtStage;
    for (int i = tid; i < sh.n; i += kR1Threads) sblk[i] = __ldg(blk + i);
    if (bt_staged) {
      const int32_t* btrow = ks.block_table + (int64_t)b * ks.max_pages;
      for (int i = tid; i < npg; i += kR1Threads) sbt[i] = __ldg(btrow + i);
    }
    if (tid == 0) *scnt = __ldg(cnt + lin);
    __syncthreads();
    const int c = min(max(*scnt, 0), sh.n);
    const int nkeys = c * sh.bk;
    const int ne = kSW ? build_extra<kR1Threads, true>(sblk, c, lbk, Tk, tpos, tpos, sh.causal, sh.sink, sh.window,
                                                       xlist, scan)
                       : 0;
    const int nall = nkeys + ne;
    const int nit_all = (nall + 31) >> 5;
    const int nch_all = (nit_all + kR1ChunkItems - 1) / kR1ChunkItems;
    // this job's chunks [c_lo, c_hi) and items [i_lo, i_lo + nit)
    const int c_lo = kClu ? sp * nch_all / S : 0;
    const int c_hi = kClu ? (sp + 1) * nch_all / S : nch_all;
    const int i_lo = c_lo * kR1ChunkItems;
    const int nit = max(0, min(c_hi * kR1ChunkItems, nit_all) - i_lo);
    const int k_lo = i_lo * 32, nk = max(0, min(nit * 32, nall - k_lo));

    // key slots of this job -> physical rows (-1: not a key, or not visible to the row)
    for (int kk = tid; kk < nit * 32; kk += kR1Threads) {
      const int k = k_lo + kk;
      int row = -1;
      if (kk < nk) {
        int s;
        bool ok;
        if (k < nkeys) {
          const int j = min(max(sblk[k >> lbk], 0), nkb - 1);
          s = (j << lbk) + (k & ((1 << lbk) - 1));
          ok = s < Tk && (!sh.causal || s <= tpos);
        } else {
          s = xlist[k - nkeys];
          ok = extra_visible(s, tpos, sh.causal, sh.sink, sh.window);
        }
        if (ok) {
          if constexpr (kPaged) {
            const uint32_t us = (uint32_t)s;
            const uint32_t pi = ks.page_shift >= 0 ? (us >> ks.page_shift) : (us / (uint32_t)ks.page_size);
            const uint32_t off = us - pi * (uint32_t)ks.page_size;
            const int64_t page = bt_staged ? (int64_t)sbt[pi] : __ldg(ks.block_table + (int64_t)b * ks.max_pages + pi);
            row = (int)(page * ks.sp_rows + off);
          } else {
            row = s;
          }
        }
      }
      tok[kk] = row;
    }
    // this lane's quarter of q: chunks kp + 4 i, as bf16 pairs
    uint32_t qv[16];
    {
      const char* qr = q_ptr(qsrc, b, h, (int64_t)q * sh.bq);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 t = __ldg(reinterpret_cast<const uint4*>(qr + (kp + 4 * i) * 16));
        qv[4 * i] = t.x; qv[4 * i + 1] = t.y; qv[4 * i + 2] = t.z; qv[4 * i + 3] = t.w;
      }
    }
    __syncthreads();  // tok visible

    const char* kbase = ks.base + ((kPaged ? 0 : b * ks.sb) + hk * ks.sh) * (int64_t)ks.esize;
    const char* vbase = vs.base + ((kPaged ? 0 : b * vs.sb) + hk * vs.sh) * (int64_t)vs.esize;
    const uint32_t krow = (uint32_t)(ks.st * ks.esize), vrow = (uint32_t)(vs.st * vs.esize);
    // item i of the job -> ring item g0 + i.  Thread t copies pieces p = 128 j + t (j < 8): row p / 16
    // of the item (< 32: K row of key p / 16, else V row of key p / 16 - 32), 16-byte chunk p % 16.
    const uint32_t g0 = g;
    auto issue = [&](int i) {
      const uint32_t gi = g0 + (uint32_t)i, slot = gi % kR1Slots;
      const int cc = tid & 15;
      // the thread's 4 keys (8 jj + tid / 16; K and V rows of each) and their source rows are read
      // and addressed before waiting for the slot, so its 8 copies go out as soon as it is free
      const char* ksrc[4];
      const char* vsrc[4];
      uint32_t okm = 0;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int row = tok[i * 32 + 8 * jj + (tid >> 4)];
        ksrc[jj] = kbase + (uint64_t)(uint32_t)max(row, 0) * krow + cc * 16;
        vsrc[jj] = vbase + (uint64_t)(uint32_t)max(row, 0) * vrow + cc * 16;
        okm |= (uint32_t)(row >= 0) << jj;
      }
      if (gi >= (uint32_t)kR1Slots) mbar_wait_u32(empty0 + 8 * slot, ((gi / kR1Slots) - 1) & 1u);
      const uint32_t dst0 = sb + L::ring + slot * kR1Item;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int jj = j & 3, key = 8 * jj + (tid >> 4);
        const bool isv = j >= 4;
        const uint32_t dst = dst0 + (isv ? 8192u : 0u) + key * 256 + ((cc ^ ((key & 1) << 2)) << 4);
        cp_async16(dst, isv ? vsrc[jj] : ksrc[jj], ((okm >> jj) & 1u) ? 16u : 0u);
      }
      cp_async_mbar_arrive_noinc(full0 + 8 * slot);
    };

    float m = -INFINITY, l = 0.f, ov[4] = {0.f, 0.f, 0.f, 0.f};  // this warp's state of the current chunk
    float Ma = -INFINITY, La = 0.f, Oa = 0.f;                     // thread d: merge of the chunks so far
    const int d = tid;
    const int pre = min(nit, kR1Slots);
    for (int i = 0; i < pre; ++i) issue(i);
    for (int i = 0; i < nit; ++i) {
      const uint32_t gi = g0 + (uint32_t)i, slot = gi % kR1Slots;
      mbar_wait_u32(full0 + 8 * slot, (gi / kR1Slots) & 1u);
      const char* it = smem + L::ring + slot * kR1Item;
      // q . k for key 8 warp + kj, quarter kp
      const int key = 8 * warp + kj;
      const char* kr = it + key * 256;
      float dot = 0.f;
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        const int ch = kp + 4 * c4;
        const uint4 kv = *reinterpret_cast<const uint4*>(kr + ((ch ^ ((key & 1) << 2)) << 4));
        const uint32_t kw[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          dot = fmaf(bf16_lo(qv[4 * c4 + e]), bf16_lo(kw[e]), dot);
          dot = fmaf(bf16_hi(qv[4 * c4 + e]), bf16_hi(kw[e]), dot);
        }
      }
      dot += __shfl_xor_sync(0xffffffffu, dot, 1);
      dot += __shfl_xor_sync(0xffffffffu, dot, 2);
      const bool valid = tok[i * 32 + key] >= 0;
      const float x = valid ? dot * scale_log2 : -INFINITY;
      // warp online softmax over its 8 keys
      float cm = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 4));
      cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 8));
      cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 16));
      const float mn = fmaxf(m, cm);
      if (mn != m) {  // warp-uniform
        const float cf = m == -INFINITY ? 0.f : ex2_approx(m - mn);
        l *= cf;
#pragma unroll
        for (int e = 0; e < 4; ++e) ov[e] *= cf;
        m = mn;
      }
      const float p = x == -INFINITY ? 0.f : ex2_approx(x - m);
      float ps = p + __shfl_xor_sync(0xffffffffu, p, 4);
      ps += __shfl_xor_sync(0xffffffffu, ps, 8);
      ps += __shfl_xor_sync(0xffffffffu, ps, 16);
      l += ps;
      // O[4 lane .. 4 lane + 3] += sum_j p_j V[8 warp + j]
      const char* vr0 = it + 8192;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float pj = __shfl_sync(0xffffffffu, p, 4 * j);
        const int vk = 8 * warp + j;
        const uint2 vv = *reinterpret_cast<const uint2*>(vr0 + vk * 256 + ((((lane >> 1) ^ ((vk & 1) << 2))) << 4) +
                                                         (lane & 1) * 8);
        ov[0] = fmaf(pj, bf16_lo(vv.x), ov[0]);
        ov[1] = fmaf(pj, bf16_hi(vv.x), ov[1]);
        ov[2] = fmaf(pj, bf16_lo(vv.y), ov[2]);
        ov[3] = fmaf(pj, bf16_hi(vv.y), ov[3]);
      }
      mbar_arrive(empty0 + 8 * slot);  // every reader releases its own reads of the slot
      if (i + kR1Slots < nit) issue(i + kR1Slots);
      if ((i + 1) % kR1ChunkItems == 0 || i == nit - 1) {
        // chunk end: merge the four warp states (fixed order) into the chunk state of column d
        *reinterpret_cast<float4*>(mo + warp * 128 + 4 * lane) = make_float4(ov[0], ov[1], ov[2], ov[3]);
        if (lane == 0) {
          mm[warp] = m;
          ml[warp] = l;
        }
        __syncthreads();
        const float Mc = fmaxf(fmaxf(mm[0], mm[1]), fmaxf(mm[2], mm[3]));
        float Oc = 0.f, Lc = 0.f;
        if (Mc != -INFINITY) {
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            if (mm[w] == -INFINITY) continue;
            const float f = ex2_approx(mm[w] - Mc);
            Oc = fmaf(f, mo[w * 128 + d], Oc);
            Lc = fmaf(f, ml[w], Lc);
          }
        }
        if constexpr (kClu) {  // the chunk state stays in shared memory for rank 0's merge
          float* my = cst + ((i_lo + i) / kR1ChunkItems - c_lo) * kSplitStride;
          my[d] = Oc;
          if (d == 0) {
            my[128] = Mc;
            my[129] = Lc;
          }
        } else {
          r1_merge(Ma, La, Oa, Mc, Lc, Oc);
        }
        m = -INFINITY;
        l = 0.f;
        ov[0] = ov[1] = ov[2] = ov[3] = 0.f;
        __syncthreads();  // mo / mm / ml are rewritten at the next chunk end
      }
    }
    g = g0 + (uint32_t)nit;

    if constexpr (kClu) {
      // every CTA's chunk states are in its shared memory; rank 0 merges them in chunk order (the
      // owner of chunk c is the split whose range [r nch / S, (r + 1) nch / S) holds it), then a second
      // cluster barrier keeps the other CTAs' shared memory alive until it has been read
      cluster_sync();
      if (sp == 0) {
        int r = 0;
        for (int c = 0; c < nch_all; ++c) {
          while ((r + 1) * nch_all / S <= c) ++r;
          const uint32_t a = smem_u32(cst + (c - r * nch_all / S) * kSplitStride);
          r1_merge(Ma, La, Oa, ld_cluster_f32(a + 128 * 4, r), ld_cluster_f32(a + 129 * 4, r),
                   ld_cluster_f32(a + d * 4, r));
        }
      }
      cluster_sync();
      if (sp != 0) continue;
    }
    const float M = Ma, Ls = La, O = Oa;
    __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(o + (b * osb + h * osh + (int64_t)q * sh.bq * ost) * 2);
    orow[d] = __float2bfloat16_rn(Ls > 0.f ? O / Ls : 0.f);  // a row with no visible key: O = 0 (G13)
    if (lse && d == 0)
      lse[((int64_t)b * sh.Hq + h) * sh.Tq + (int64_t)q * sh.bq] = Ls > 0.f ? M * kR1Ln2 + logf(Ls) : -INFINITY;
    __syncthreads();  // merge scratch and tok are rewritten by the next job
  }
}

// Single-row query blocks (every unit one row: b_q = 1 or T_q = 1), bf16, d = 128, up to 512
// selected keys + 256 sink / window tokens (wider union masks use attn_tc).
bool attn_row1_supported(const Shape& sh) {
  return sh.d == 128 && std::min(sh.bq, sh.Tq) == 1 && (int64_t)sh.n * sh.bk + kMaxExtra <= kR1Tok && sh.n <= kR1MaxN &&
         sh.sink + sh.window <= kMaxExtra;
}

template <bool kPaged, bool kSW>
static cudaError_t launch_r1_cluster(const Shape& s2, const QSrc& qs, const RowSrc& ks, const RowSrc& vs,
                                     const int32_t* idx, const int32_t* cnt, float sm_scale, char* o, int64_t osb,
                                     int64_t osh, int64_t ost, float* lse, cudaStream_t stream, int64_t grid) {
  auto kern = attn_row1_kernel<kPaged, kSW, true>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Row1Smem::total);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kR1Threads);
  cfg.dynamicSmemBytes = Row1Smem::total;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)s2.splits;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, s2, qs, ks, vs, idx, cnt, sm_scale * kR1Log2e, o, osb, osh, ost, lse);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <bool kPaged, bool kSW>
static cudaError_t launch_r1(const Shape& s2, const QSrc& qs, const RowSrc& ks, const RowSrc& vs, const int32_t* idx,
                             const int32_t* cnt, float sm_scale, char* o, int64_t osb, int64_t osh, int64_t ost,
                             float* lse, cudaStream_t stream, int64_t grid) {
  auto kern = attn_row1_kernel<kPaged, kSW, false>;
  int per_sm = 1;
  cudaError_t e = persistent_ctas(kern, kR1Threads, Row1Smem::total, 0, &per_sm);  // sets the smem attribute
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)grid, kR1Threads, Row1Smem::total, stream>>>(s2, qs, ks, vs, idx, cnt, sm_scale * kR1Log2e, o, osb,
                                                                osh, ost, lse);
  return cudaGetLastError();
}

cudaError_t launch_attn_row1(const Shape& sh, const QSrc& qs, const RowSrc& ks, const RowSrc& vs, const int32_t* idx,
                             const int32_t* cnt, float sm_scale, char* o, int64_t osb, int64_t osh, int64_t ost,
                             float* lse, cudaStream_t stream, int num_sms) {
  int per_sm = 1;
  cudaError_t e = persistent_ctas(attn_row1_kernel<false, false, false>, kR1Threads, Row1Smem::total, 0, &per_sm);
  if (e != cudaSuccess) return e;
  const int64_t units = (int64_t)sh.B * sh.Hq * sh.nqb;
  const int64_t slots = (int64_t)num_sms * per_sm;
  Shape s2 = sh;
  // split-K only to fill CTA slots the units leave idle (never a second wave), and never into more
  // jobs than a unit has 128-key chunks (the split granularity); a split unit runs on a cluster
  const int64_t max_keys = (int64_t)sh.n * sh.bk + ((sh.sink > 0 || sh.window > 0) ? sh.sink + sh.window : 0);
  const int64_t max_chunks = std::max<int64_t>(1, (max_keys + 32 * kR1ChunkItems - 1) / (32 * kR1ChunkItems));
  s2.splits = 1;
  if (units <= kSplitMaxUnits)
    s2.splits = (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(kSplitMax, max_chunks), slots / units));
#ifdef HIPATTN_TUNING
  if (const char* e2 = getenv("HIPATTN_SPLITS")) s2.splits = std::max(1, std::min(kSplitMax, atoi(e2)));
#endif
  const bool sw = sh.sink > 0 || sh.window > 0;
  if (s2.splits > 1) {  // one cluster of `splits` CTAs per unit, chunk states merged through DSMEM (one wave)
    s2.sched = nullptr;
    const int64_t grid = units * s2.splits;
    if (ks.paged) return sw ? launch_r1_cluster<true, true>(s2, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, grid)
                            : launch_r1_cluster<true, false>(s2, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, grid);
    return sw ? launch_r1_cluster<false, true>(s2, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, grid)
              : launch_r1_cluster<false, false>(s2, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, grid);
  }
  const int64_t grid = std::min<int64_t>(units, slots);
  if ((e = setup_queue(s2, units, grid, stream)) != cudaSuccess) return e;
  if (ks.paged) return sw ? launch_r1<true, true>(s2, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, grid)
                          : launch_r1<true, false>(s2, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, grid);
  return sw ? launch_r1<false, true>(s2, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, grid)
            : launch_r1<false, false>(s2, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, grid);
}

}  // namespace hip
