// mask_decode.cu — HiP mask estimation for short query blocks (decode: one query row per sequence
// against a paged KV cache; also T_q <= 4 multi-query).  With b_q = 1 the tile
// score is a GEMV: nothing for tensor cores to do, and the kernel is bound by HBM
// (the cache of a 128k sequence is far larger than L2).
//
// Layout of the work: a half-warp (16 lanes) owns one representative key row at a time; lane l
// loads the row's 16-byte slice l (a coalesced 256-byte row per half-warp), keeps its slice of the
// query rows in registers, runs a sequential fmaf chain over its d/16 elements and the half-warp
// sums the 16 partials with a fixed xor tree (o = 8, 4, 2, 1).  That order is the canonical fp32
// order of this path, reading G9b ("F32L" in the oracle), so decode masks are bit-identical to the
// oracle.  Each half-warp takes U = 16 consecutive rows per batch (all 16 loads in flight), so the
// b_k <= 16 rows of a block stay in one half-warp and the block max needs no exchange.  Many small
// CTAs (128 threads) keep every (sequence, head) unit of a decode batch resident; the selection is
// select.cuh.
#include "kernels.h"
#include "select.cuh"
#include "topr.cuh"

namespace hip {

constexpr int kMDThreads = 128;
constexpr int kMDRows = 4;   // max query rows per block on this path
constexpr int kMDU = 16;     // rows per half-warp per batch (128 rows = 32 KB in flight per CTA)

template <typename T, int D, int RM, bool kPaged>
struct LaneScorer {
  template <class ST>
  __device__ __forceinline__ float* score_buf(ST& st, int) { return st.scores(); }
  static constexpr int E = D / 16;                 // elements per lane
  static constexpr int NV = (E * (int)sizeof(T) + 15) / 16;  // 16-byte vectors per lane (1 or 2)
  const float* qs;   // [rows_q][D] fp32 (smem)
  RowSrc ks;
  const char* kh;
  uint32_t row_bytes;
  int b, hk, Tk, lbk, causal, rows_q;
  int rph = 1;  // rows per query head (GQA-shared, G25): row t sits at position tpos0 + t % rph
  int64_t tpos0;
  HIP_PT_MEMBER
  __device__ __forceinline__ void mark(int p) { HIP_MARK(p); (void)p; }

  __device__ __forceinline__ const char* row(int s) const {
    if constexpr (kPaged) return row_ptr(ks, b, hk, s);
    else return kh + (uint64_t)(uint32_t)s * row_bytes;
  }

  __device__ void score(const int* rep, int n_rep, float* out) {
    const int lane16 = threadIdx.x & 15, hw = threadIdx.x >> 4;  // 8 half-warps
    const int bmask = (1 << lbk) - 1;
    const int rows_total = n_rep << lbk;
    // this lane's slice of every query row
    float qv[RM][E];
#pragma unroll
    for (int t = 0; t < RM; ++t)
#pragma unroll
      for (int e = 0; e < E; ++e) qv[t][e] = t < rows_q ? qs[t * D + lane16 * E + e] : 0.f;

    for (int base = 0; base < rows_total; base += 8 * kMDU) {
      const int r0 = base + hw * kMDU;
      uint4 buf[kMDU][NV];
      int sv[kMDU];
#pragma unroll
      for (int i = 0; i < kMDU; ++i) {
        const int r = r0 + i;
        int s = Tk;
        if (r < rows_total) s = (rep[r >> lbk] << lbk) + (r & bmask);
        sv[i] = s;
        if (s < Tk) {
          const char* p = row(s) + lane16 * (E * (int)sizeof(T));
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            if constexpr (E * sizeof(T) >= 16) buf[i][v] = __ldg(reinterpret_cast<const uint4*>(p) + v);
            else {
              const uint2 h = __ldg(reinterpret_cast<const uint2*>(p));
              buf[i][v] = make_uint4(h.x, h.y, 0u, 0u);
            }
          }
        } else {
#pragma unroll
          for (int v = 0; v < NV; ++v) buf[i][v] = make_uint4(0u, 0u, 0u, 0u);
        }
      }
      float blockbest = -INFINITY;
#pragma unroll
      for (int i = 0; i < kMDU; ++i) {
        float kvv[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint32_t* w = reinterpret_cast<const uint32_t*>(&buf[i][0]);
          if constexpr (sizeof(T) == 4) kvv[e] = __uint_as_float(w[e]);
          else kvv[e] = (e & 1) ? bf16_hi(w[e >> 1]) : bf16_lo(w[e >> 1]);
        }
        float best = -INFINITY;
#pragma unroll
        for (int t = 0; t < RM; ++t) {
          if (t < rows_q) {
            float acc = 0.f;
#pragma unroll
            for (int e = 0; e < E; ++e) acc = __fmaf_rn(qv[t][e], kvv[e], acc);
#pragma unroll
            for (int o = 8; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (sv[i] < Tk && (!causal || sv[i] <= tpos0 + t % rph) && acc > best) best = acc;
          }
        }
        // rows r0 + i of one block are consecutive inside this half-warp (b_k | U)
        blockbest = fmaxf(blockbest, best);
        const int r = r0 + i;
        if ((r & bmask) == bmask) {
          if (lane16 == 0 && r < rows_total) out[r >> lbk] = blockbest;
          blockbest = -INFINITY;
        }
      }
    }
    __syncthreads();
  }
};

template <typename T, int D, int NMAX, int RM, bool kPaged>
__global__ void __launch_bounds__(kMDThreads, 2) mask_decode_kernel(Shape sh, QSrc qsrc, RowSrc ks,
                                                                 int32_t* __restrict__ idx, int32_t* __restrict__ cnt) {
  extern __shared__ __align__(16) char smem[];
  SelState<NMAX, kMDThreads / 32>& st = *reinterpret_cast<SelState<NMAX, kMDThreads / 32>*>(smem);
  float* qs = reinterpret_cast<float*>(smem + align_up(sizeof(SelState<NMAX, kMDThreads / 32>), 128));
  const int lbk = 31 - __clz(sh.bk);
  const int64_t units = (int64_t)sh.B * mask_heads(sh) * sh.nqb;
  const int S = max(sh.chunks, 1);
  for (int64_t jb = blockIdx.x; jb < units * S; jb += gridDim.x) {
    const int64_t u = jb / S;
    const int cs = (int)(jb - u * S);
    int b, h, q;  // h: mask head (the kv head when GQA-shared, G25)
    mask_unit_coords(sh, u, b, h, q);
    const int hk = sh.group > 1 ? h : h / (sh.Hq / sh.Hkv);
    const int Tk = seq_len(sh, b);
    const int Bq = visible_blocks(sh, q, Tk);
    const int64_t lin = ((int64_t)b * mask_heads(sh) + h) * sh.nqb + q;
    const int rph = min(sh.bq, sh.Tq - q * sh.bq);  // rows per query head
    const int rows_q = rph * sh.group;               // rows scored together (G heads x rph)
    int lo, len, nn, slot0;
    if (!chunk_job(Bq, sh.n, S, cs, lo, len, nn, slot0)) continue;
    if (Bq > sh.n) {
      for (int i = threadIdx.x; i < rows_q * D; i += kMDThreads) {
        const int t = i / D, c = i - t * D;
        const T* src = reinterpret_cast<const T*>(q_ptr(qsrc, b, sh.group > 1 ? h * sh.group + t / rph : h, (int64_t)q * sh.bq + t % rph));
        float v;
        if constexpr (sizeof(T) == 4) v = src[c];
        else v = __bfloat162float(src[c]);
        qs[t * D + c] = v;
      }
      __syncthreads();
      if (sh.top_r > 0 && sh.top_r < D)  // top-r approximation (G22)
        top_r_zero_f32<kMDThreads>(qs, D, rows_q, D, sh.top_r, st.scores());
    }
    LaneScorer<T, D, RM, kPaged> sc;
    sc.qs = qs;
    sc.ks = ks;
    sc.kh = ks.base + (b * ks.sb + hk * ks.sh) * (int64_t)ks.esize;
    sc.row_bytes = (uint32_t)(ks.st * ks.esize);
    sc.b = b; sc.hk = hk; sc.Tk = Tk; sc.lbk = lbk; sc.causal = sh.causal; sc.rows_q = rows_q;
    sc.tpos0 = (int64_t)q * sh.bq + (Tk - sh.Tq);
    sc.rph = rph;
    tree_search<NMAX, kMDThreads>(st, nn, lo, len, sc, idx + lin * sh.n + slot0, nullptr,
                            make_jitter(sh.jitter, sh.seed, lin));
    if (cs == 0 && threadIdx.x == 0) cnt[lin] = min(Bq, sh.n);
    __syncthreads();
  }
}

// <= 4 query rows per block, b_k a power of two <= 16 (a block inside one half-warp batch).
bool mask_decode_supported(const Shape& sh) {
  return std::min(sh.bq, sh.Tq) * sh.group <= kMDRows && sh.bk <= kMDU && (sh.bk & (sh.bk - 1)) == 0 &&
         (sh.d == 64 || sh.d == 128);
}

template <typename T, int D, int NMAX, int RM>
static cudaError_t launch_md(const Shape& sh, const QSrc& qs, const RowSrc& ks, int32_t* idx, int32_t* cnt,
                             cudaStream_t stream, int num_sms) {
  const size_t smem = align_up(sizeof(SelState<NMAX, kMDThreads / 32>), 128) + kMDRows * D * 4;
  auto kern = ks.paged ? mask_decode_kernel<T, D, NMAX, RM, true> : mask_decode_kernel<T, D, NMAX, RM, false>;
  int per_sm = 1;
  cudaError_t e = persistent_ctas(kern, kMDThreads, smem, 0, &per_sm);
  if (e != cudaSuccess) return e;
  const int64_t units = (int64_t)sh.B * (sh.group > 1 ? sh.Hkv : sh.Hq) * sh.nqb;
  const int64_t grid = std::min<int64_t>(units * std::max(sh.chunks, 1), (int64_t)num_sms * per_sm);
  kern<<<(unsigned)grid, kMDThreads, smem, stream>>>(sh, qs, ks, idx, cnt);
  return cudaGetLastError();
}

template <typename T, int D>
static cudaError_t launch_md_n(const Shape& sh, const QSrc& qs, const RowSrc& ks, int32_t* idx, int32_t* cnt,
                               cudaStream_t stream, int num_sms) {
  const bool one = std::min(sh.bq, sh.Tq) * sh.group == 1;  // plain decode: one query row
  if (sh.n <= 256)
    return one ? launch_md<T, D, 256, 1>(sh, qs, ks, idx, cnt, stream, num_sms)
               : launch_md<T, D, 256, kMDRows>(sh, qs, ks, idx, cnt, stream, num_sms);
  return one ? launch_md<T, D, 1024, 1>(sh, qs, ks, idx, cnt, stream, num_sms)
             : launch_md<T, D, 1024, kMDRows>(sh, qs, ks, idx, cnt, stream, num_sms);
}

cudaError_t launch_mask_decode(const Shape& sh, const QSrc& qs, const RowSrc& ks, bool bf16, int32_t* idx,
                               int32_t* cnt, cudaStream_t stream, int num_sms) {
  if (bf16) {
    if (sh.d == 128) return launch_md_n<__nv_bfloat16, 128>(sh, qs, ks, idx, cnt, stream, num_sms);
    return launch_md_n<__nv_bfloat16, 64>(sh, qs, ks, idx, cnt, stream, num_sms);
  }
  if (sh.d == 128) return launch_md_n<float, 128>(sh, qs, ks, idx, cnt, stream, num_sms);
  return launch_md_n<float, 64>(sh, qs, ks, idx, cnt, stream, num_sms);
}

}  // namespace hip
