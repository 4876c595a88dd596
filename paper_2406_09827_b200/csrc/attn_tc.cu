// attn_tc.cu — block-sparse flash-style attention prefill on tcgen05 (Eq. 2-3, P:116-123;
// "Block Sparse Flash Attention"), bf16 in/out, fp32 scores / online softmax.
//
// Per query block (b_q <= 32 rows) the selected key blocks give <= k keys, processed in chunks of
// 128.  Each chunk streams four 16 KB items through a 2-slot shared ring (16-byte cp.async gathers
// into 128-byte-swizzled layouts; a slot is refilled as soon as the MMA that read it completes, so
// two items are in flight): the two d-halves of K_c and the two 64-key halves of V_c.  One
// thread issues
//     S^T_c [128 keys x 32 q]  = K_c . Q^T         (M=128, N=32, K=d; A, B K-major)
//     O^T   [128 d x 32 q]    += V_c^T . P_c^T     (M=128, N=32, K=keys; A, B MN-major)
// with S^T_c and O^T in 64 TMEM columns.  The softmax is online over chunks (flash style): each
// thread owns one key (a TMEM lane) and 32 query columns; the row max over keys is a 5-step shuffle
// reduce-scatter plus a 4-warp exchange.  The running max is updated lazily (only when a chunk's
// max exceeds it by more than 8 in log2 units, so P <= 2^8 stays exact in bf16 range), and O^T is
// rescaled in TMEM only then.  P is rounded to bf16 into a no-swizzle MN-major operand tile.
// Token-level causal masking and the ragged tails (short last query block, keys past T_k, fewer
// than n selected blocks) are applied to S before the max.  Small CTAs (128 threads, 64 TMEM
// columns, ~53 KB shared) keep 4 query blocks per SM in flight: the gathers are L2-bound
// (profiles/r01/gather_ceiling.json), and independent streams are what saturates L2.
#include "kernels.h"
#include "sinkwin.cuh"

namespace hip {

constexpr int kATThreads = 128;
constexpr uint32_t kATSlot = 128 * 128;               // one ring slot: 16 KB
constexpr uint32_t kATQTile = 2 * 32 * 128;
constexpr uint32_t kATPChunk = 128 * 32 * 2;          // 128 keys x 32 queries bf16
constexpr uint32_t kIdescQK = idesc_bf16(128, 32, 0, 0);
constexpr uint32_t kIdescPV = idesc_bf16(128, 32, 1, 1);
constexpr float kATLog2e = 1.4426950408889634f;
constexpr float kATLn2 = 0.6931471805599453f;
constexpr float kATRescale = 8.f;                     // lazy rescale threshold (log2 units)
// Ring slots of 16 KB items.  Two slots at 4 CTAs per SM beat three at 3 CTAs per SM (C4 attention
// 5.20 vs 6.57 ms, profiles/r02/notes.md): more concurrent units matter more than a deeper ring.
constexpr int kATRing = 2;

template <int kTokN>
struct AttnTCSmemT {
  static constexpr uint32_t q = 0;
  static constexpr uint32_t ring = kATQTile;                      // kATRing slots
  static constexpr uint32_t p = ring + kATRing * kATSlot;         // one P chunk
  static constexpr uint32_t red = p + kATPChunk;                  // floats, see below
  static constexpr int kRedFloats = 3 * 4 * 32 + 6 * 32 + 32;     // [3][4][32] + m, l, lu, corr, invl, pad + flag
  static constexpr int kTok = kTokN;                              // selected + extra (<= 256) key slots
  static constexpr uint32_t tok = red + kRedFloats * 4;           // [kTok] row of each key slot
  static constexpr uint32_t xlist = tok + kTok * 4;               // [kMaxExtra] sink / window tokens
  static constexpr uint32_t misc = (uint32_t)align_up(xlist + kMaxExtra * 4, 64);  // 2 mbarriers, TMEM address
  static constexpr uint32_t jq = misc + 32;                       // JobQueue slots (2 x int64)
  static constexpr uint32_t total = jq + 16;
};
// Default: <= 512 selected keys (k = 512) + <= 256 extra, 4 CTAs per SM.  Wide: the ensemble's
// union masks (hip_mask_vote with tau = 0, up to 16 x 256 blocks) — a longer staged key list, at
// the cost of shared memory (fewer CTAs per SM); the rest of the kernel is unchanged.
constexpr int kATTokDefault = 768, kATTokWide = 4096 + 256;
using AttnTCSmem = AttnTCSmemT<kATTokDefault>;

// Lane L ends with op-reduction over the 32 lanes of query L (values v[0..31] per lane = queries).
template <bool kMax>
__device__ __forceinline__ float reduce_scatter32(float (&v)[32], int lane) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const bool up = (lane & w) != 0;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      float send = up ? v[i] : v[i + w];
      float keep = up ? v[i + w] : v[i];
      float recv = __shfl_xor_sync(0xffffffffu, send, w);
      v[i] = kMax ? fmaxf(keep, recv) : keep + recv;
    }
  }
  return v[0];
}

// kSW: sink / sliding-window tokens enabled (a separate instantiation, so the plain path pays nothing).
template <bool kPaged, bool kSW, int TOK>
__global__ void __launch_bounds__(kATThreads, 4) attn_tc_kernel(Shape sh, QSrc qsrc, RowSrc ks, RowSrc vs,
                                                                const int32_t* __restrict__ idx,
                                                                const int32_t* __restrict__ cnt, float scale_log2,
                                                                char* __restrict__ o, int64_t osb, int64_t osh,
                                                                int64_t ost, float* __restrict__ lse) {
  extern __shared__ __align__(16) char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t pad = ((raw + 1023u) & ~1023u) - raw;
  char* base = smem_raw + pad;
  const uint32_t sb = raw + pad;
  using L = AttnTCSmemT<TOK>;
  float* red = reinterpret_cast<float*>(base + L::red);   // [0,384): per-warp max / sum / unrounded sum
  float* mrun = red + 384;                                 // running max per query (log2 units)
  float* lrun = red + 416;                                 // running sum of bf16-rounded p
  float* lurun = red + 448;                                // running sum of unrounded p (lse)
  float* corr = red + 480;                                 // rescale factor of this chunk
  float* invl = red + 512;
  float* thr = red + 544;                                  // mrun + kATRescale: the lazy-rescale thresholds
  int* flag = reinterpret_cast<int*>(red + 576);
  int* tok = reinterpret_cast<int*>(base + L::tok);
  int* xlist = reinterpret_cast<int*>(base + L::xlist);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(base + L::misc);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + L::misc + 8 * kATRing);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int r = 0; r < kATRing; ++r) mbar_init(mbar + r, 1);  // one MMA-completion barrier per ring slot
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<64>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S^T at columns [0, 32), O^T at [32, 64)
  const uint32_t tmem_lane = tmem + ((uint32_t)(32 * warp) << 16);
  uint32_t phase = 0u;                  // bit s: parity of ring slot s's MMA barrier
  const uint32_t mbar_a = smem_u32(mbar);  // shared address of the two barriers
  const int lbk = 31 - __clz(sh.bk);

  const int64_t units = (int64_t)sh.B * sh.Hq * sh.nqb;
  JobQueue jq(sh.sched, base + L::jq);
  for (int64_t u = blockIdx.x; u < units; u = jq.next(u)) {
    jq.claim();
    int b, h, q;
    unit_coords(sh, u, b, h, q);
    const int hk = h / (sh.Hq / sh.Hkv);
    const int Tk = seq_len(sh, b);
    const int64_t lin = mask_lin(sh, b, h, q);  // the unit's mask row (GQA-shared: its group's, G25)
    const int rows_q = min(sh.bq, sh.Tq - q * sh.bq);
    const int64_t tpos0 = (int64_t)q * sh.bq + (Tk - sh.Tq);
    const bool tail1 = rows_q == 1 && tpos0 >= Tk - 1;  // decode row at the end of its sequence
    const int nkb = (Tk + sh.bk - 1) / sh.bk;
    const int c = min(max(__ldg(cnt + lin), 0), sh.n);
    const int nkeys = c * sh.bk;
    // sink / sliding-window tokens not covered by the selected blocks (sinkwin.cuh)
    const int ne = kSW ? build_extra<kATThreads>(idx + lin * sh.n, c, lbk, Tk, tpos0, tpos0 + rows_q - 1, sh.causal,
                                                 sh.sink, sh.window, xlist, reinterpret_cast<int*>(red))
                       : 0;
    const int nall = nkeys + ne;
    const int nch = (nall + 127) / 128;
    const int32_t* blk = idx + lin * sh.n;

    if (nch == 0) {  // no selected block: O = 0, lse = -inf (G13)
      for (int i = threadIdx.x; i < rows_q * 16; i += kATThreads) {
        const int t = i >> 4, c16 = i & 15;
        *reinterpret_cast<uint4*>(o + (b * osb + h * osh + ((int64_t)q * sh.bq + t) * ost) * 2 + c16 * 16) =
            make_uint4(0u, 0u, 0u, 0u);
      }
      if (lse && threadIdx.x < rows_q) lse[((int64_t)b * sh.Hq + h) * sh.Tq + (int64_t)q * sh.bq + threadIdx.x] = -INFINITY;
      continue;
    }

    // Q tile (K-major SW128, 32 rows; rows >= rows_q zero)
    for (int p = threadIdx.x; p < 32 * 16; p += kATThreads) {
      const int r = p >> 4, c16 = p & 15;
      const bool ok = r < rows_q;
      const char* src = q_ptr(qsrc, b, h, (int64_t)q * sh.bq + (ok ? r : 0)) + c16 * 16;
      cp_async16(sb + L::q + (c16 >> 3) * (32 * 128) + sw128_off(r, c16 & 7), src, ok ? 16u : 0u);
    }
    // row of every selected key slot (or -1 past T_k / past cnt), staged once per unit: the token
    // index for contiguous K/V, the physical row page * (page stride in rows) + offset for a paged
    // cache (K and V share the block table and strides), so the gathers carry no dependent load
    for (int k = threadIdx.x; k < nch * 128; k += kATThreads) {
      int s = -1;
      if (k < nall) {
        if (k < nkeys) {
          const int j = min(max(__ldg(blk + (k >> lbk)), 0), nkb - 1);
          s = (j << lbk) + (k & ((1 << lbk) - 1));
          if (s >= Tk) s = -1;
        } else if constexpr (kSW) {
          s = xlist[k - nkeys];
        }
        if constexpr (kPaged) {
          if (s >= 0) {
            const uint32_t us = (uint32_t)s;
            const uint32_t pi = ks.page_shift >= 0 ? (us >> ks.page_shift) : (us / (uint32_t)ks.page_size);
            const uint32_t off = us - pi * (uint32_t)ks.page_size;
            const int64_t page = __ldg(ks.block_table + (int64_t)b * ks.max_pages + pi);
            s = (int)(page * ks.sp_rows + off);
          }
        } else if constexpr (kSW) {
          if (k >= nkeys && s >= 0) s |= kExtraBit;  // contiguous: the token itself, extras flagged
        }
      }
      tok[k] = s;
    }
    if (threadIdx.x < 32) {
      mrun[threadIdx.x] = -INFINITY;
      thr[threadIdx.x] = -INFINITY;
      lrun[threadIdx.x] = 0.f;
      lurun[threadIdx.x] = 0.f;
    }
    __syncthreads();
    const char* kbase = ks.base + ((kPaged ? 0 : b * ks.sb) + hk * ks.sh) * (int64_t)ks.esize;
    const char* vbase = vs.base + ((kPaged ? 0 : b * vs.sb) + hk * vs.sh) * (int64_t)vs.esize;
    const uint32_t krow = (uint32_t)(ks.st * ks.esize), vrow = (uint32_t)(vs.st * vs.esize);

    // item i: chunk ch = i >> 2; (i & 3) = 0, 1: K_ch d-half 0 / 1; 2, 3: V_ch keys [0,64) / [64,128)
    // Thread (c8, r0) moves 16-byte chunk c8 of the 8 keys r0 + 16 j (j = 0..7) of every chunk: for
    // K items those 8 rows (one d-half), for V items keys r0 + 16 j' + 64 (kind - 2) of both d-halves.
    // All eight keys share r0's swizzle phase, so the destinations are one base + immediates, and
    // the rows' tokens are read once per chunk (at its first item).
    const int c8 = threadIdx.x & 7, r0 = threadIdx.x >> 3;  // r0 < 16
    const uint32_t dbase = (uint32_t)((r0 >> 3) * 1024 + (r0 & 7) * 128 + ((c8 ^ (r0 & 7)) << 4));
    int srow[8];  // this thread's 8 key rows of the current chunk (-1: none)
    auto issue = [&](int i) {
      const int ch = i >> 2, kind = i & 3;
      const uint32_t dst = sb + L::ring + (i % kATRing) * kATSlot + dbase;
      if (kind == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int t = tok[ch * 128 + r0 + 16 * j];
          srow[j] = kSW ? (t & ~kExtraBit) : t;  // -1 stays negative
        }
      }
      if (kind < 2) {  // K: 128 keys x d-half `kind`
        const char* g = kbase + kind * 128 + c8 * 16;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          cp_async16_pf256(dst + 2048 * j, g + (uint64_t)(uint32_t)max(srow[j], 0) * krow, srow[j] >= 0 ? 16u : 0u);
      } else {         // V: 64 keys x both d-halves, d-half regions 8 KB apart
        const char* g = vbase + c8 * 16;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int sr = kind == 2 ? srow[j & 3] : srow[4 + (j & 3)];  // static indices (registers)
          cp_async16_pf256(dst + 2048 * (j & 3) + 8192 * (j >> 2), g + (uint64_t)(uint32_t)max(sr, 0) * vrow + (j >> 2) * 128,
                      sr >= 0 ? 16u : 0u);
        }
      }
    };
    uint32_t pend = 0u;  // bit s: slot s has an MMA committed but not yet waited
    auto wait_slot = [&](int sl) {
      if (pend & (1u << sl)) {
        mbar_wait_u32(mbar_a + 8u * sl, (phase >> sl) & 1u);
        phase ^= 1u << sl;
        pend &= ~(1u << sl);
      }
    };

    const int nitems = 4 * nch;
#pragma unroll
    for (int r = 0; r < kATRing; ++r) {  // nitems >= 4 >= kATRing
      issue(r);
      cp_async_commit();
    }
    for (int it = 0; it < nitems; ++it) {
      cp_async_wait<kATRing - 1>();  // item it landed (items it + 1 .. may still be in flight)
      fence_proxy_async_smem();
      __syncthreads();
      // Every MMA up to item it - 1 has completed here (each slot is refilled only after its MMA is
      // waited for, and tcgen05 MMAs of one thread complete in order): S of this chunk is final
      // before its softmax, and the previous chunk's PV is done before P is rewritten.
      const int ch = it >> 2, kind = it & 3;
      const uint32_t slot = sb + L::ring + (it % kATRing) * kATSlot;
      if (kATRing > 2 && kind == 2) wait_slot((it - 1) % kATRing);  // the tail does not refill: S, PV done
      if (kind == 2) {
        // ---- online softmax of chunk ch (S^T_ch complete: its last MMA was item it - 1)
        tc_fence_after();
        float v[32];
        tmem_ld_32x32b_x32(tmem_lane, v);
        int s;  // token position of this lane's key (-1: none)
        bool extra;  // a sink / window token: row-dependent visibility
        {
          const int k = ch * 128 + 32 * warp + lane;
          if constexpr (kPaged) {
            s = -1;
            extra = kSW && k >= nkeys;
            if (k < nkeys) {
              if (!kSW && tail1) {  // one row at the last position: every staged key is visible to it
                s = tok[k] >= 0 ? (int)tpos0 : -1;
              } else {
                const int j = min(max(__ldg(blk + (k >> lbk)), 0), nkb - 1);
                s = (j << lbk) + (k & ((1 << lbk) - 1));
                if (s >= Tk) s = -1;
              }
            } else if (kSW && k < nall) {
              s = xlist[k - nkeys];
            }
          } else {
            s = tok[k];
            extra = kSW && s >= 0 && (s & kExtraBit);
            if (extra) s &= ~kExtraBit;
          }
        }
        const bool all_vis = s >= 0 && rows_q == 32 && (!sh.causal || s <= tpos0) &&
                             (!extra || extra_visible(s, tpos0 + 31, sh.causal, sh.sink, sh.window));
        if (all_vis) {  // the common case: this key is visible to all 32 rows
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] *= scale_log2;
        } else if (rows_q == 1) {  // decode: query column 0 only
          const bool ok = s >= 0 && (!sh.causal || s <= tpos0) &&
                          (!extra || extra_visible(s, tpos0, sh.causal, sh.sink, sh.window));
          v[0] = ok ? v[0] * scale_log2 : -INFINITY;
#pragma unroll
          for (int j = 1; j < 32; ++j) v[j] = -INFINITY;
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const bool ok = s >= 0 && j < rows_q && (!sh.causal || s <= tpos0 + j) &&
                            (!extra || extra_visible(s, tpos0 + j, sh.causal, sh.sink, sh.window));
            v[j] = ok ? v[j] * scale_log2 : -INFINITY;
          }
        }
        float x[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) x[j] = v[j];
        // The running max moves only when some query's chunk max exceeds it by more than kATRescale
        // (lazy rule below).  Every thread first checks its own 32 scores against the thresholds
        // thr[j] = mrun[j] + kATRescale; only if any score in the CTA exceeds one (always on a unit's
        // first chunk) is the chunk max reduced and the running max updated — otherwise that whole
        // step would leave mrun, corr and the sums' scale unchanged, so skipping it is exact.
        bool grow = false;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 t = *reinterpret_cast<const float4*>(thr + j);
          grow |= (v[j] > t.x) | (v[j + 1] > t.y) | (v[j + 2] > t.z) | (v[j + 3] > t.w);
        }
        bool resc = false;
        if (__syncthreads_or(grow)) {
        red[warp * 32 + lane] = reduce_scatter32<true>(v, lane);
        __syncthreads();
        if (threadIdx.x < 32) {  // new running max per query (lazy), rescale factor, rescale flag
          const int j = threadIdx.x;
          const float mc = fmaxf(fmaxf(red[j], red[32 + j]), fmaxf(red[64 + j], red[96 + j]));
          const float mo = mrun[j];
          const float mn = (mc > mo + kATRescale || (mo == -INFINITY && mc != -INFINITY)) ? mc : mo;
          const float cf = (mn == mo) ? 1.f : (mo == -INFINITY ? 0.f : ex2_approx(mo - mn));
          corr[j] = cf;
          mrun[j] = mn;
          thr[j] = mn + kATRescale;
          lrun[j] *= cf;
          lurun[j] *= cf;
          const unsigned any = __ballot_sync(0xffffffffu, cf != 1.f);
          if (j == 0) *flag = (any != 0u) && ch > 0;
        }
        __syncthreads();
        resc = *flag;
        }
        float lq = 0.f, lu = 0.f;
        {
          uint32_t pk[16];
          float w[32];
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            float p2[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const float m = mrun[j + e];
              p2[e] = (x[j + e] == -INFINITY || m == -INFINITY) ? 0.f : ex2_approx(x[j + e] - m);
            }
            w[j] = p2[0];
            w[j + 1] = p2[1];
            __nv_bfloat162 pb = __floats2bfloat162_rn(p2[0], p2[1]);
            pk[j >> 1] = *reinterpret_cast<uint32_t*>(&pb);
            const float2 pr = __bfloat1622float2(pb);
            v[j] = pr.x;
            v[j + 1] = pr.y;
          }
          // P^T chunk: MN-major, no swizzle: 8-query piece cp at cp*2048, key group r/8 at (r/8)*128,
          // key r%8 at 16 B stride.
          const int r = 32 * warp + lane;
          char* pc = base + L::p + (r >> 3) * 128 + (r & 7) * 16;
#pragma unroll
          for (int cp = 0; cp < 4; ++cp)
            *reinterpret_cast<uint4*>(pc + cp * 2048) =
                make_uint4(pk[4 * cp], pk[4 * cp + 1], pk[4 * cp + 2], pk[4 * cp + 3]);
          lq = reduce_scatter32<false>(v, lane);
          if (lse) lu = reduce_scatter32<false>(w, lane);
        }
        red[128 + warp * 32 + lane] = lq;
        red[256 + warp * 32 + lane] = lu;
        if (resc) {  // rescale O^T columns (queries) whose running max moved; all PV MMAs retired
          float ov[32];
          tmem_ld_32x32b_x32(tmem_lane + 32, ov);
#pragma unroll
          for (int j = 0; j < 32; ++j) ov[j] *= corr[j];
          uint32_t* ou = reinterpret_cast<uint32_t*>(ov);
          asm volatile(
              "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
              "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
              "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(tmem_lane + 32),
              "r"(ou[0]), "r"(ou[1]), "r"(ou[2]), "r"(ou[3]), "r"(ou[4]), "r"(ou[5]), "r"(ou[6]), "r"(ou[7]),
              "r"(ou[8]), "r"(ou[9]), "r"(ou[10]), "r"(ou[11]), "r"(ou[12]), "r"(ou[13]), "r"(ou[14]), "r"(ou[15]),
              "r"(ou[16]), "r"(ou[17]), "r"(ou[18]), "r"(ou[19]), "r"(ou[20]), "r"(ou[21]), "r"(ou[22]), "r"(ou[23]),
              "r"(ou[24]), "r"(ou[25]), "r"(ou[26]), "r"(ou[27]), "r"(ou[28]), "r"(ou[29]), "r"(ou[30]), "r"(ou[31])
              : "memory");
          asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        }
        tc_fence_before();
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x < 32) {
          const int j = threadIdx.x;
          lrun[j] += red[128 + j] + red[160 + j] + red[192 + j] + red[224 + j];
          lurun[j] += red[256 + j] + red[288 + j] + red[320 + j] + red[352 + j];
        }
      }
      if (threadIdx.x == 0) {
        tc_fence_after();
        if (kind < 2) {  // S^T_ch (+)= K_ch(d-half) . Q^T(d-half)
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const uint64_t a = smem_desc(slot + s * 32, 16, 1024, kLayoutSw128);
            const uint64_t bq = smem_desc(sb + L::q + kind * (32 * 128) + s * 32, 16, 1024, kLayoutSw128);
            umma_bf16(tmem, a, bq, kIdescQK, (kind | s) ? 1u : 0u);
          }
        } else {         // O^T += V_ch(64 keys)^T . P_ch(those keys)^T
          const int hk2 = kind - 2;
#pragma unroll
          for (int s = 0; s < 4; ++s) {  // 64 keys = 4 x K16
            const uint64_t a = smem_desc(slot + s * 2048, 8192, 1024, kLayoutSw128);
            const uint64_t bp = smem_desc(sb + L::p + hk2 * 1024 + s * 256, 128, 2048, kLayoutNone);
            umma_bf16(tmem + 32, a, bp, kIdescPV, (ch > 0 || hk2 > 0 || s > 0) ? 1u : 0u);
          }
        }
        umma_commit_u32(mbar_a + 8u * (it % kATRing));
      }
      pend |= 1u << (it % kATRing);
      // refill this slot with item it + kATRing as soon as MMA(it) has read it
      if (it + kATRing < nitems) {
        wait_slot(it % kATRing);
        issue(it + kATRing);
      }
      cp_async_commit();
    }
#pragma unroll
    for (int r = 0; r < kATRing; ++r) wait_slot(r);  // the last MMAs (O^T complete)
    // ---- epilogue: O^T lanes = d, columns = queries -> normalise, stage [32 q][128 d] bf16 in the
    // (now free) ring, then 16-byte coalesced row stores
    if (threadIdx.x < 32) {
      const int j = threadIdx.x;
      invl[j] = lrun[j] > 0.f ? 1.f / lrun[j] : 0.f;
    }
    tc_fence_after();
    float v[32];
    tmem_ld_32x32b_x32(tmem_lane + 32, v);
    __syncthreads();
    const int d = 32 * warp + lane;
    __nv_bfloat16* ostage = reinterpret_cast<__nv_bfloat16*>(base + L::ring);
#pragma unroll
    for (int j = 0; j < 32; ++j) ostage[j * 128 + d] = __float2bfloat16_rn(v[j] * invl[j]);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int p = threadIdx.x + kATThreads * i, j = p >> 4, c16 = p & 15;
      if (j < rows_q) {
        char* dst = o + (b * osb + h * osh + ((int64_t)q * sh.bq + j) * ost) * 2 + c16 * 16;
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(base + L::ring + j * 256 + c16 * 16);
      }
    }
    if (lse && threadIdx.x < rows_q) {
      const int j = threadIdx.x;
      const float l = lurun[j], m = mrun[j];
      lse[((int64_t)b * sh.Hq + h) * sh.Tq + (int64_t)q * sh.bq + j] = l > 0.f ? m * kATLn2 + logf(l) : -INFINITY;
    }
    tc_fence_before();
    __syncthreads();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<64>(tmem);
}

// Any query block of <= 32 rows (decode included: the N = 32 operand is zero-padded, the tensor
// cores are idle anyway); up to 4096 selected keys plus <= 256 sink / window tokens (the staged list).
bool attn_tc_supported(const Shape& sh) {
  return sh.d == 128 && sh.bq >= 1 && sh.bq <= 32 && (128 % sh.bk) == 0 && (sh.bk & (sh.bk - 1)) == 0 &&
         (int64_t)sh.n * sh.bk <= 4096 && sh.sink + sh.window + sh.bq - 1 <= kMaxExtra;
}

template <int TOK>
static cudaError_t launch_attn_tc_t(const Shape& sh, const QSrc& qs, const RowSrc& ks, const RowSrc& vs,
                                    const int32_t* idx, const int32_t* cnt, float sm_scale, char* o, int64_t osb,
                                    int64_t osh, int64_t ost, float* lse, cudaStream_t stream, int num_sms) {
  const size_t smem = AttnTCSmemT<TOK>::total + 1024;
  const bool sw = sh.sink > 0 || sh.window > 0;
  auto kern = ks.paged ? (sw ? attn_tc_kernel<true, true, TOK> : attn_tc_kernel<true, false, TOK>)
                       : (sw ? attn_tc_kernel<false, true, TOK> : attn_tc_kernel<false, false, TOK>);
  int per_sm = 1;
  cudaError_t e = persistent_ctas(kern, kATThreads, smem, 64, &per_sm);
  if (e != cudaSuccess) return e;
  const int64_t units = (int64_t)sh.B * sh.Hq * sh.nqb;
  const int64_t grid = std::min<int64_t>(units, (int64_t)num_sms * per_sm);
  Shape s2 = sh;
  if ((e = setup_queue(s2, units, grid, stream)) != cudaSuccess) return e;
  kern<<<(unsigned)grid, kATThreads, smem, stream>>>(s2, qs, ks, vs, idx, cnt, sm_scale * kATLog2e, o, osb, osh, ost,
                                                     lse);
  return cudaGetLastError();
}

cudaError_t launch_attn_tc(const Shape& sh, const QSrc& qs, const RowSrc& ks, const RowSrc& vs, const int32_t* idx,
                           const int32_t* cnt, float sm_scale, char* o, int64_t osb, int64_t osh, int64_t ost,
                           float* lse, cudaStream_t stream, int num_sms) {
  if ((int64_t)sh.n * sh.bk + kMaxExtra <= kATTokDefault)
    return launch_attn_tc_t<kATTokDefault>(sh, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, num_sms);
  return launch_attn_tc_t<kATTokWide>(sh, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, num_sms);
}

}  // namespace hip
