// attn_tc.cu — block-sparse flash-style attention prefill on tcgen05 (Eq. 2-3, P:116-123;
// "Block Sparse Flash Attention"), bf16 in/out, fp32 scores/softmax in TMEM/registers.
//
// Per query block (b_q <= 32 rows) the selected key blocks give <= k = 512 keys (4 tiles of 128).
// The CTA streams K tiles then V tiles through a 2-slot shared ring (gathered with 16-byte
// cp.async into 128-byte-swizzled tiles: one key row = 256 B), and one thread issues
//     S^T_c [128 keys x 32 q] = K_c . Q^T          (M=128, N=32, K=d=128; A K-major, B K-major)
//     O^T  [128 d    x 32 q] += V_c^T . P_c^T       (M=128, N=32, K=128 keys; A, B MN-major)
// with all S tiles resident in TMEM (128 columns) and O^T in 32 more.  Softmax is exact two-pass
// over the on-chip S (the key count per query block is bounded by k, so no rescaling of O is ever
// needed): each thread owns one key (a TMEM lane) and 32 query columns; row max / row sum over keys
// are a 5-step shuffle reduce-scatter inside the warp plus a 4-warp exchange in shared memory.
// P is rounded to bf16 into a no-swizzle MN-major operand tile.  Token-level causal masking and
// the ragged tails (short last query block, keys past T_k, fewer than n selected blocks) are
// applied to S before the max.
#include "kernels.h"

namespace hip {

constexpr int kATThreads = 128;
constexpr uint32_t kATRegion = 128 * 128;              // 128 rows x 128 B
constexpr uint32_t kATTile = 2 * kATRegion;           // d = 128
constexpr uint32_t kATQTile = 2 * 32 * 128;
constexpr uint32_t kATPChunk = 128 * 32 * 2;          // 128 keys x 32 queries bf16
constexpr uint32_t kIdescQK = idesc_bf16(128, 32, 0, 0);
constexpr uint32_t kIdescPV = idesc_bf16(128, 32, 1, 1);
constexpr float kATLog2e = 1.4426950408889634f;
constexpr float kATLn2 = 0.6931471805599453f;

struct AttnTCSmem {
  static constexpr uint32_t q = 0;
  static constexpr uint32_t ring0 = kATQTile;
  static constexpr uint32_t ring1 = ring0 + kATTile;
  static constexpr uint32_t p = ring1 + kATTile;                 // 4 chunks
  static constexpr uint32_t red = p + 4 * kATPChunk;             // [3][4][32] floats
  static constexpr uint32_t tok = red + (3 * 4 * 32 + 32) * 4;   // [512] int token per key slot
  static constexpr uint32_t misc = tok + 512 * 4;
  static constexpr uint32_t total = misc + 64;
};

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

__global__ void __launch_bounds__(kATThreads) attn_tc_kernel(Shape sh, QSrc qsrc, RowSrc ks, RowSrc vs,
                                                             const int32_t* __restrict__ idx,
                                                             const int32_t* __restrict__ cnt, float scale_log2,
                                                             char* __restrict__ o, int64_t osb, int64_t osh,
                                                             int64_t ost, float* __restrict__ lse) {
  extern __shared__ __align__(16) char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t pad = ((raw + 1023u) & ~1023u) - raw;
  char* base = smem_raw + pad;
  const uint32_t sb = raw + pad;
  using L = AttnTCSmem;
  float* red = reinterpret_cast<float*>(base + L::red);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(base + L::misc);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + L::misc + 16);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(mbar, 1);  // one MMA-completion barrier per ring slot
    mbar_init(mbar + 1, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_lane = tmem + ((uint32_t)(32 * warp) << 16);
  uint32_t phase[2] = {0u, 0u};
  const int lbk = 31 - __clz(sh.bk);

  const int64_t units = (int64_t)sh.B * sh.Hq * sh.nqb;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    int b, h, q;
    unit_coords(sh, u, b, h, q);
    const int hk = h / (sh.Hq / sh.Hkv);
    const int Tk = seq_len(sh, b);
    const int64_t lin = ((int64_t)b * sh.Hq + h) * sh.nqb + q;
    const int rows_q = min(sh.bq, sh.Tq - q * sh.bq);
    const int64_t tpos0 = (int64_t)q * sh.bq + (Tk - sh.Tq);
    const int nkb = (Tk + sh.bk - 1) / sh.bk;
    const int c = min(max(__ldg(cnt + lin), 0), sh.n);
    const int nkeys = c * sh.bk;
    const int nch = (nkeys + 127) / 128;
    const int32_t* blk = idx + lin * sh.n;

    if (nch == 0) {  // no selected block: O = 0, lse = -inf (G13)
      for (int i = threadIdx.x; i < rows_q * 128; i += kATThreads) {
        int t = i >> 7, d = i & 127;
        reinterpret_cast<__nv_bfloat16*>(o)[b * osb + h * osh + ((int64_t)q * sh.bq + t) * ost + d] =
            __float2bfloat16_rn(0.f);
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
    // token of every selected key slot (or -1 past T_k / past cnt), staged once per unit
    int* tok = reinterpret_cast<int*>(base + L::tok);
    for (int k = threadIdx.x; k < nch * 128; k += kATThreads) {
      int s = -1;
      if (k < nkeys) {
        const int j = min(max(__ldg(blk + (k >> lbk)), 0), nkb - 1);
        s = (j << lbk) + (k & ((1 << lbk) - 1));
        if (s >= Tk) s = -1;
      }
      tok[k] = s;
    }
    __syncthreads();
    const char* kbase = ks.base + (b * ks.sb + hk * ks.sh) * (int64_t)ks.esize;
    const char* vbase = vs.base + (b * vs.sb + hk * vs.sh) * (int64_t)vs.esize;
    const uint32_t krow = (uint32_t)(ks.st * ks.esize), vrow = (uint32_t)(vs.st * vs.esize);
    // item i < nch: K tile i; item nch + i: V tile i; slot = i & 1.  16 threads per 256-B row.
    auto issue = [&](int item) {
      const bool isv = item >= nch;
      const int ch = isv ? item - nch : item;
      const char* g0 = isv ? vbase : kbase;
      const uint32_t rb = isv ? vrow : krow;
      const int c16 = threadIdx.x & 15, r0 = threadIdx.x >> 4;  // r0 < 8
      const uint32_t dst = ((item & 1) ? sb + L::ring1 : sb + L::ring0) + (c16 >> 3) * kATRegion + r0 * 128 +
                           (((c16 & 7) ^ r0) << 4);
      const int* tk = tok + ch * 128 + r0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int s = tk[8 * i];
        cp_async16(dst + i * 1024, g0 + (uint64_t)(uint32_t)(s >= 0 ? s : 0) * rb + c16 * 16, s >= 0 ? 16u : 0u);
      }
    };
    // token of this thread's key in chunk ch (or -1): used for masking
    auto key_token = [&](int ch) -> int64_t { return tok[ch * 128 + 32 * warp + lane]; };

    // Items stream through the 2-slot ring: item i < nch is K tile i, item nch + i is V tile i.  The
    // MMA of an item is issued as soon as its bytes land and waited only to refill its slot with
    // item + 2, so V0/V1 are already in flight while the softmax runs.
    const int nitems = 2 * nch;
    bool pend[2] = {false, false};
    auto wait_slot = [&](int sl) {
      if (pend[sl]) {
        mbar_wait(mbar + sl, phase[sl]);
        phase[sl] ^= 1u;
        pend[sl] = false;
      }
    };
    issue(0);
    cp_async_commit();
    if (nitems > 1) issue(1);
    cp_async_commit();
    for (int it = 0; it < nitems; ++it) {
      if (it + 1 < nitems) cp_async_wait<1>();
      else cp_async_wait<0>();
      fence_proxy_async_smem();
      __syncthreads();
      const uint32_t tile = (it & 1) ? sb + L::ring1 : sb + L::ring0;
      if (it < nch) {
        if (threadIdx.x == 0) {
          tc_fence_after();
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            uint64_t a = smem_desc(tile + (s >> 2) * kATRegion + (s & 3) * 32, 16, 1024, kLayoutSw128);
            uint64_t bq = smem_desc(sb + L::q + (s >> 2) * (32 * 128) + (s & 3) * 32, 16, 1024, kLayoutSw128);
            umma_bf16(tmem + 32 * it, a, bq, kIdescQK, s > 0 ? 1u : 0u);
          }
          umma_commit(mbar + (it & 1));
        }
        pend[it & 1] = true;
        if (it + 2 < nitems) {  // refill this slot (item it + 2) once its MMA has read it
          wait_slot(it & 1);
          issue(it + 2);
          cp_async_commit();
        }
        if (it == nch - 1) {
          // ---- softmax over all S tiles (two passes, S stays in TMEM)
          wait_slot(0);
          wait_slot(1);
          tc_fence_after();
          float mq;  // running max (log2 domain) of query `lane` over this warp's keys
          mq = -INFINITY;
          for (int ch = 0; ch < nch; ++ch) {
            float v[32];
            tmem_ld_32x32b_x32(tmem_lane + 32 * ch, v);
            const int64_t s = key_token(ch);
            if (s >= 0 && rows_q == 32 && (!sh.causal || s <= tpos0)) {  // visible to every row
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] *= scale_log2;
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const bool ok = s >= 0 && j < rows_q && (!sh.causal || s <= tpos0 + j);
                v[j] = ok ? v[j] * scale_log2 : -INFINITY;
              }
            }
            mq = fmaxf(mq, reduce_scatter32<true>(v, lane));
          }
          red[warp * 32 + lane] = mq;
          __syncthreads();
          float mrow[32];
#pragma unroll
          for (int j = 0; j < 32; ++j)
            mrow[j] = fmaxf(fmaxf(red[j], red[32 + j]), fmaxf(red[64 + j], red[96 + j]));
          float lq = 0.f, lu = 0.f;  // sums of the bf16-rounded p (normalises O) / unrounded p (lse)
          for (int ch = 0; ch < nch; ++ch) {
            float v[32], w[32];
            tmem_ld_32x32b_x32(tmem_lane + 32 * ch, v);
            const int64_t s = key_token(ch);
            const bool all_vis = s >= 0 && rows_q == 32 && (!sh.causal || s <= tpos0);  // => every m finite
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              float p2[2];
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int jj = j + e;
                const bool ok = all_vis || (s >= 0 && jj < rows_q && (!sh.causal || s <= tpos0 + jj) &&
                                            mrow[jj] != -INFINITY);
                p2[e] = ok ? ex2_approx(fmaf(v[jj], scale_log2, -mrow[jj])) : 0.f;
              }
              w[j] = p2[0];
              w[j + 1] = p2[1];
              __nv_bfloat162 pb = __floats2bfloat162_rn(p2[0], p2[1]);
              pk[j >> 1] = *reinterpret_cast<uint32_t*>(&pb);
              float2 pr = __bfloat1622float2(pb);
              v[j] = pr.x;
              v[j + 1] = pr.y;
            }
            // P^T chunk: MN-major, no swizzle: piece (8 queries) cp at cp*2048, key group r/8 at
            // (r/8)*128, key r%8 at 16 B stride.
            const int r = 32 * warp + lane;
            char* pc = base + L::p + ch * kATPChunk + (r >> 3) * 128 + (r & 7) * 16;
#pragma unroll
            for (int cp = 0; cp < 4; ++cp)
              *reinterpret_cast<uint4*>(pc + cp * 2048) = make_uint4(pk[4 * cp], pk[4 * cp + 1], pk[4 * cp + 2], pk[4 * cp + 3]);
            lq += reduce_scatter32<false>(v, lane);
            if (lse) lu += reduce_scatter32<false>(w, lane);
          }
          red[128 + warp * 32 + lane] = lq;
          red[256 + warp * 32 + lane] = lu;
          tc_fence_before();
          fence_proxy_async_smem();
          __syncthreads();
        }
      } else {
        const int ch = it - nch;
        if (threadIdx.x == 0) {
          tc_fence_after();
          const uint32_t pch = sb + L::p + ch * kATPChunk;
#pragma unroll
          for (int s = 0; s < 8; ++s) {  // 128 keys = 8 x K16
            uint64_t a = smem_desc(tile + s * 2048, kATRegion, 1024, kLayoutSw128);
            uint64_t bp = smem_desc(pch + s * 256, 128, 2048, kLayoutNone);
            umma_bf16(tmem + 128, a, bp, kIdescPV, (ch > 0 || s > 0) ? 1u : 0u);
          }
          umma_commit(mbar + (it & 1));
        }
        pend[it & 1] = true;
        if (it + 2 < nitems) {
          wait_slot(it & 1);
          issue(it + 2);
          cp_async_commit();
        }
      }
    }
    wait_slot(0);  // the last MMAs (O^T complete)
    wait_slot(1);
    // ---- epilogue: O^T lanes = d, columns = queries -> normalise, stage [32 q][128 d] bf16 in the
    // (now free) P buffer, then 16-byte coalesced row stores
    float* invl = red + 384;
    if (threadIdx.x < 32) {
      const int j = threadIdx.x;
      const float l = red[128 + j] + red[160 + j] + red[192 + j] + red[224 + j];
      invl[j] = l > 0.f ? 1.f / l : 0.f;
    }
    tc_fence_after();
    float v[32];
    tmem_ld_32x32b_x32(tmem_lane + 128, v);
    __syncthreads();
    const int d = 32 * warp + lane;
    __nv_bfloat16* ostage = reinterpret_cast<__nv_bfloat16*>(base + L::p);
#pragma unroll
    for (int j = 0; j < 32; ++j) ostage[j * 128 + d] = __float2bfloat16_rn(v[j] * invl[j]);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int p = threadIdx.x + kATThreads * i, j = p >> 4, c16 = p & 15;
      if (j < rows_q) {
        char* dst = o + (b * osb + h * osh + ((int64_t)q * sh.bq + j) * ost) * 2 + c16 * 16;
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(base + L::p + j * 256 + c16 * 16);
      }
    }
    if (lse && threadIdx.x < rows_q) {
      const int j = threadIdx.x;
      const float l = red[256 + j] + red[288 + j] + red[320 + j] + red[352 + j];
      const float m = fmaxf(fmaxf(red[j], red[32 + j]), fmaxf(red[64 + j], red[96 + j]));
      lse[((int64_t)b * sh.Hq + h) * sh.Tq + (int64_t)q * sh.bq + j] = l > 0.f ? m * kATLn2 + logf(l) : -INFINITY;
    }
    tc_fence_before();
    __syncthreads();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

bool attn_tc_supported(const Shape& sh) {
  return sh.d == 128 && sh.bq >= 8 && sh.bq <= 32 && (128 % sh.bk) == 0 && (sh.bk & (sh.bk - 1)) == 0 && (int64_t)sh.n * sh.bk <= 512;
}

cudaError_t launch_attn_tc(const Shape& sh, const QSrc& qs, const RowSrc& ks, const RowSrc& vs, const int32_t* idx,
                           const int32_t* cnt, float sm_scale, char* o, int64_t osb, int64_t osh, int64_t ost,
                           float* lse, cudaStream_t stream, int num_sms) {
  const size_t smem = AttnTCSmem::total + 1024;
  int per_sm = 1;
  cudaError_t e = persistent_ctas(attn_tc_kernel, kATThreads, smem, 256, &per_sm);
  if (e != cudaSuccess) return e;
  const int64_t units = (int64_t)sh.B * sh.Hq * sh.nqb;
  int64_t grid = std::min<int64_t>(units, (int64_t)num_sms * per_sm);
  attn_tc_kernel<<<(unsigned)grid, kATThreads, smem, stream>>>(sh, qs, ks, vs, idx, cnt, sm_scale * kATLog2e, o, osb,
                                                               osh, ost, lse);
  return cudaGetLastError();
}

}  // namespace hip
