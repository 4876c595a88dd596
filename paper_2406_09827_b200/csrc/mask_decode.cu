// mask_decode.cu — HiP mask estimation for short query blocks (decode: one query row per sequence
// against a paged KV cache; also T_q <= 4 multi-query).  With b_q = 1 the tile
// score is a GEMV: there is nothing for tensor cores to do, and the kernel is bound by
// HBM (the cache of a 128k sequence is far larger than L2).  Each thread owns one representative
// key row per round, loads its 256 bytes straight from HBM with 16 independent 16-byte loads (the
// whole round of a CTA, 32 KB, is in flight at once), and runs the canonical sequential fp32 chain
// acc = fmaf(q[c], k[c], acc), c = 0..d-1 (reading G9) — so decode masks are bit-identical to the
// oracle's F32C mode.  The max over the b_k rows of a block is a shuffle across adjacent lanes.
// Many small CTAs (128 threads, ~15 KB of shared memory) keep every (sequence, head) unit of a
// decode batch resident at once; the selection is select.cuh.
#include "kernels.h"
#include "select.cuh"

namespace hip {

constexpr int kMDThreads = 128;
constexpr int kMDRows = 4;  // max query rows per block on this path

template <typename T, int D, bool kPaged>
struct DirectScorer {
  const float* qs;   // [rows_q][D] fp32 (smem, broadcast reads)
  RowSrc ks;
  const char* kh;
  int64_t row_bytes;
  int b, hk, Tk, lbk, causal, rows_q;
  int64_t tpos0;

  __device__ __forceinline__ const char* row(int64_t s) const {
    if constexpr (kPaged) return row_ptr(ks, b, hk, s);
    else return kh + s * row_bytes;
  }

  __device__ void score(const int* rep, int n_rep, float* out) {
    constexpr int EPP = 16 / sizeof(T);          // elements per 16-byte piece
    constexpr int NPIECE = D / EPP;              // pieces per row
    constexpr int G = NPIECE < 16 ? NPIECE : 16; // pieces held in registers at once
    const int bmask = (1 << lbk) - 1;
    const int rows_total = n_rep << lbk;
    for (int base = 0; base < rows_total; base += kMDThreads) {
      const int r = base + threadIdx.x;
      float best = -INFINITY;
      int64_t s = Tk;
      if (r < rows_total) s = (int64_t)rep[r >> lbk] * (1 << lbk) + (r & bmask);
      if (s < Tk) {
        const uint4* src = reinterpret_cast<const uint4*>(row(s));
        float acc[kMDRows];
#pragma unroll
        for (int t = 0; t < kMDRows; ++t) acc[t] = 0.f;
#pragma unroll
        for (int g0 = 0; g0 < NPIECE; g0 += G) {
          uint4 buf[G];
#pragma unroll
          for (int i = 0; i < G; ++i) buf[i] = __ldg(src + g0 + i);
#pragma unroll
          for (int i = 0; i < G; ++i) {
            float kv[EPP];
            if constexpr (sizeof(T) == 4) {
              kv[0] = __uint_as_float(buf[i].x); kv[1] = __uint_as_float(buf[i].y);
              kv[2] = __uint_as_float(buf[i].z); kv[3] = __uint_as_float(buf[i].w);
            } else {
              kv[0] = bf16_lo(buf[i].x); kv[1] = bf16_hi(buf[i].x); kv[2] = bf16_lo(buf[i].y); kv[3] = bf16_hi(buf[i].y);
              kv[4] = bf16_lo(buf[i].z); kv[5] = bf16_hi(buf[i].z); kv[6] = bf16_lo(buf[i].w); kv[7] = bf16_hi(buf[i].w);
            }
            const int c0 = (g0 + i) * EPP;
#pragma unroll
            for (int t = 0; t < kMDRows; ++t) {
              if (t < rows_q) {
                const float4* qv = reinterpret_cast<const float4*>(qs + t * D + c0);
#pragma unroll
                for (int e4 = 0; e4 < EPP / 4; ++e4) {
                  const float4 qq = qv[e4];
                  acc[t] = __fmaf_rn(qq.x, kv[4 * e4 + 0], acc[t]);
                  acc[t] = __fmaf_rn(qq.y, kv[4 * e4 + 1], acc[t]);
                  acc[t] = __fmaf_rn(qq.z, kv[4 * e4 + 2], acc[t]);
                  acc[t] = __fmaf_rn(qq.w, kv[4 * e4 + 3], acc[t]);
                }
              }
            }
          }
        }
#pragma unroll
        for (int t = 0; t < kMDRows; ++t)
          if (t < rows_q && (!causal || s <= tpos0 + t) && acc[t] > best) best = acc[t];
      }
      for (int off = 1; off <= bmask; off <<= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, off));
      if (r < rows_total && (r & bmask) == 0) out[r >> lbk] = best;
    }
    __syncthreads();
  }
};

template <typename T, int D, int NMAX, bool kPaged>
__global__ void __launch_bounds__(kMDThreads) mask_decode_kernel(Shape sh, QSrc qsrc, RowSrc ks,
                                                                 int32_t* __restrict__ idx, int32_t* __restrict__ cnt) {
  extern __shared__ __align__(16) char smem[];
  SelState<NMAX>& st = *reinterpret_cast<SelState<NMAX>*>(smem);
  float* qs = reinterpret_cast<float*>(smem + align_up(sizeof(SelState<NMAX>), 128));
  const int lbk = 31 - __clz(sh.bk);
  const int64_t units = (int64_t)sh.B * sh.Hq * sh.nqb;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    int b, h, q;
    unit_coords(sh, u, b, h, q);
    const int hk = h / (sh.Hq / sh.Hkv);
    const int Tk = seq_len(sh, b);
    const int Bq = visible_blocks(sh, q, Tk);
    const int64_t lin = ((int64_t)b * sh.Hq + h) * sh.nqb + q;
    const int rows_q = min(sh.bq, sh.Tq - q * sh.bq);
    if (Bq > sh.n) {
      for (int i = threadIdx.x; i < rows_q * D; i += kMDThreads) {
        const int t = i / D, c = i - t * D;
        const T* src = reinterpret_cast<const T*>(q_ptr(qsrc, b, h, (int64_t)q * sh.bq + t));
        float v;
        if constexpr (sizeof(T) == 4) v = src[c];
        else v = __bfloat162float(src[c]);
        qs[t * D + c] = v;
      }
      __syncthreads();
    }
    DirectScorer<T, D, kPaged> sc;
    sc.qs = qs;
    sc.ks = ks;
    sc.kh = ks.base + (b * ks.sb + hk * ks.sh) * (int64_t)ks.esize;
    sc.row_bytes = ks.st * (int64_t)ks.esize;
    sc.b = b; sc.hk = hk; sc.Tk = Tk; sc.lbk = lbk; sc.causal = sh.causal; sc.rows_q = rows_q;
    sc.tpos0 = (int64_t)q * sh.bq + (Tk - sh.Tq);
    tree_search<NMAX, kMDThreads>(st, sh.n, Bq, sc, idx + lin * sh.n, cnt + lin);
    __syncthreads();
  }
}

bool mask_decode_supported(const Shape& sh) {
  return std::min(sh.bq, sh.Tq) <= kMDRows && sh.bk <= 32 && (sh.bk & (sh.bk - 1)) == 0 && (sh.d == 64 || sh.d == 128);
}

template <typename T, int D, int NMAX>
static cudaError_t launch_md(const Shape& sh, const QSrc& qs, const RowSrc& ks, int32_t* idx, int32_t* cnt,
                             cudaStream_t stream, int num_sms) {
  const size_t smem = align_up(sizeof(SelState<NMAX>), 128) + kMDRows * D * 4;
  auto kern = ks.paged ? mask_decode_kernel<T, D, NMAX, true> : mask_decode_kernel<T, D, NMAX, false>;
  int per_sm = 1;
  cudaError_t e = persistent_ctas(kern, kMDThreads, smem, 0, &per_sm);
  if (e != cudaSuccess) return e;
  const int64_t units = (int64_t)sh.B * sh.Hq * sh.nqb;
  const int64_t grid = std::min<int64_t>(units, (int64_t)num_sms * per_sm);
  kern<<<(unsigned)grid, kMDThreads, smem, stream>>>(sh, qs, ks, idx, cnt);
  return cudaGetLastError();
}

template <typename T, int D>
static cudaError_t launch_md_n(const Shape& sh, const QSrc& qs, const RowSrc& ks, int32_t* idx, int32_t* cnt,
                               cudaStream_t stream, int num_sms) {
  if (sh.n <= 256) return launch_md<T, D, 256>(sh, qs, ks, idx, cnt, stream, num_sms);
  return launch_md<T, D, 1024>(sh, qs, ks, idx, cnt, stream, num_sms);
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
