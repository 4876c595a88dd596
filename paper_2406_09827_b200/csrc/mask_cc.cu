// mask_cc.cu — HiP mask estimation with CUDA-core scoring (Alg. 1; block approximation
// P:172-186).  Every dot product is the canonical sequential chain acc = fmaf(q[c], k[c], acc),
// c = 0..d-1, in fp32 (reading G9), so the selected blocks are bit-identical to the oracle's F32C
// mode on any input.  Used for fp32 inputs (BASELINE config C1), for bf16 with
// HIP_FLAG_EXACT_SCORES, for shapes the tcgen05 kernel does not cover, and for decode (T_q rows
// against a paged KV cache), where scoring is a GEMV and the kernel is HBM-bound.
//
// One CTA (256 threads) per (b, h, query block) at a time, persistent over units.  Per iteration the
// representative key blocks are gathered with coalesced 16-byte cp.async into a padded shared
// stage (double-buffered chunks), each thread computes whole dot products for (query row, key row)
// pairs, and one thread per block takes the tile max over the valid (causal) pairs.
#include "kernels.h"
#include "select.cuh"
#include "topr.cuh"

namespace hip {

constexpr int kCCThreads = 256;

constexpr int kCCStages = 4;  // cp.async ring depth: 3 chunks in flight while one is scored

template <typename T>
struct CCScorer {
  template <class ST>
  __device__ __forceinline__ float* score_buf(ST& st, int) { return st.scores(); }
  const float* qs;   // [rows_q][qpitch] fp32
  int qpitch;        // floats
  char* stage0;      // kCCStages staged chunks of key rows
  int stage_bytes;
  int kpitch;        // bytes
  float* pairs;      // [rows_per_chunk][rows_q]
  RowSrc ks;
  int b, hk, Tk, d, bk, causal, rows_q, ch;  // ch = key blocks per chunk
  int rph = 1;       // rows per query head: row t sits at position tpos0 + t % rph (GQA-shared, G25)
  int64_t tpos0;     // key position of query row 0 of the block: q*bq + Tk - Tq
  HIP_PT_MEMBER
  __device__ __forceinline__ void mark(int p) { HIP_MARK(p); (void)p; }

  __device__ void issue(const int* rep, int n_rep, int c) {
    const int blk0 = c * ch, nblk = min(ch, n_rep - blk0);
    if (nblk <= 0) return;
    const int rows = nblk * bk, pieces = (d * (int)sizeof(T)) / 16;
    const uint32_t dst0 = smem_u32(stage0 + (c % kCCStages) * stage_bytes);
    for (int p = threadIdx.x; p < rows * pieces; p += kCCThreads) {
      int r = p / pieces, c16 = p - r * pieces;
      int64_t s = (int64_t)rep[blk0 + r / bk] * bk + (r % bk);
      bool ok = s < Tk;
      const char* src = row_ptr(ks, b, hk, ok ? s : 0) + c16 * 16;
      cp_async16(dst0 + r * kpitch + c16 * 16, src, ok ? 16u : 0u);
    }
  }

  __device__ void score(const int* rep, int n_rep, float* out) {
    const int nch = (n_rep + ch - 1) / ch;
#pragma unroll
    for (int c = 0; c < kCCStages - 1; ++c) {
      issue(rep, n_rep, c);
      cp_async_commit();
    }
    for (int c = 0; c < nch; ++c) {
      issue(rep, n_rep, c + kCCStages - 1);  // slot of chunk c - 1, freed by the last barrier
      cp_async_commit();
      cp_async_wait<kCCStages - 1>();
      __syncthreads();
      const int blk0 = c * ch, nblk = min(ch, n_rep - blk0), rows = nblk * bk;
      const char* kst = stage0 + (c % kCCStages) * stage_bytes;
      for (int p = threadIdx.x; p < rows * rows_q; p += kCCThreads) {
        int t = p % rows_q, r = p / rows_q;
        int64_t s = (int64_t)rep[blk0 + r / bk] * bk + (r % bk);
        bool valid = s < Tk && (!causal || s <= tpos0 + t % rph);
        float acc = -INFINITY;
        if (valid) {
          const float4* qr = reinterpret_cast<const float4*>(qs + t * qpitch);
          acc = 0.f;
          if constexpr (sizeof(T) == 4) {
            const float4* kr = reinterpret_cast<const float4*>(kst + r * kpitch);
            for (int i = 0; i < d / 4; ++i) {
              float4 kv = kr[i], qv = qr[i];
              acc = __fmaf_rn(qv.x, kv.x, acc);
              acc = __fmaf_rn(qv.y, kv.y, acc);
              acc = __fmaf_rn(qv.z, kv.z, acc);
              acc = __fmaf_rn(qv.w, kv.w, acc);
            }
          } else {
            const uint4* kr = reinterpret_cast<const uint4*>(kst + r * kpitch);
            for (int i = 0; i < d / 8; ++i) {
              uint4 kv = kr[i];
              float4 qa = qr[2 * i], qb = qr[2 * i + 1];
              acc = __fmaf_rn(qa.x, bf16_lo(kv.x), acc);
              acc = __fmaf_rn(qa.y, bf16_hi(kv.x), acc);
              acc = __fmaf_rn(qa.z, bf16_lo(kv.y), acc);
              acc = __fmaf_rn(qa.w, bf16_hi(kv.y), acc);
              acc = __fmaf_rn(qb.x, bf16_lo(kv.z), acc);
              acc = __fmaf_rn(qb.y, bf16_hi(kv.z), acc);
              acc = __fmaf_rn(qb.z, bf16_lo(kv.w), acc);
              acc = __fmaf_rn(qb.w, bf16_hi(kv.w), acc);
            }
          }
        }
        pairs[r * rows_q + t] = acc;
      }
      __syncthreads();
      for (int lb = threadIdx.x; lb < nblk; lb += kCCThreads) {
        float best = -INFINITY;
        for (int r = lb * bk; r < lb * bk + bk; ++r)
          for (int t = 0; t < rows_q; ++t) {
            float v = pairs[r * rows_q + t];
            if (v > best) best = v;
          }
        out[blk0 + lb] = best;
      }
      __syncthreads();  // the stage of chunk c and pairs are reused
    }
    cp_async_wait<0>();
  }
};

template <typename T, int NMAX>
__global__ void __launch_bounds__(kCCThreads, 2) mask_cc_kernel(Shape sh, QSrc qsrc, RowSrc ks, int32_t* __restrict__ idx,
                                                                int32_t* __restrict__ cnt, int ch, int kpitch,
                                                                int stage_bytes) {
  extern __shared__ __align__(16) char smem[];
  SelState<NMAX, kCCThreads / 32>& st = *reinterpret_cast<SelState<NMAX, kCCThreads / 32>*>(smem);
  const int rows_max = min(sh.bq, sh.Tq) * sh.group;
  const int qpitch = sh.d + 4;
  float* qs = reinterpret_cast<float*>(smem + align_up(sizeof(SelState<NMAX, kCCThreads / 32>), 128));
  char* stage0 = reinterpret_cast<char*>(qs + rows_max * qpitch);  // qpitch*4 is a multiple of 16
  float* pairs = reinterpret_cast<float*>(stage0 + kCCStages * stage_bytes);

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
      for (int i = threadIdx.x; i < rows_q * sh.d; i += kCCThreads) {
        int t = i / sh.d, c = i - t * sh.d;
        const T* src = reinterpret_cast<const T*>(q_ptr(qsrc, b, sh.group > 1 ? h * sh.group + t / rph : h, (int64_t)q * sh.bq + t % rph));
        float v;
        if constexpr (sizeof(T) == 4) v = src[c];
        else v = __bfloat162float(src[c]);
        qs[t * qpitch + c] = v;
      }
      __syncthreads();
      if (sh.top_r > 0 && sh.top_r < sh.d)  // top-r approximation (G22)
        top_r_zero_f32<kCCThreads>(qs, qpitch, rows_q, sh.d, sh.top_r, st.scores());
    }
    CCScorer<T> sc;
    sc.qs = qs; sc.qpitch = qpitch; sc.stage0 = stage0; sc.stage_bytes = stage_bytes; sc.kpitch = kpitch;
    sc.pairs = pairs; sc.ks = ks; sc.b = b; sc.hk = hk; sc.Tk = Tk; sc.d = sh.d; sc.bk = sh.bk;
    sc.causal = sh.causal; sc.rows_q = rows_q; sc.ch = ch;
    sc.tpos0 = (int64_t)q * sh.bq + (Tk - sh.Tq);
    sc.rph = rph;
    tree_search<NMAX, kCCThreads>(st, nn, lo, len, sc, idx + lin * sh.n + slot0, nullptr,
                            make_jitter(sh.jitter, sh.seed, lin));
    if (cs == 0 && threadIdx.x == 0) cnt[lin] = min(Bq, sh.n);
    __syncthreads();
  }
}

// Host launcher.  Returns a cudaError_t.
template <typename T, int NMAX>
static cudaError_t launch_cc(const Shape& sh, const QSrc& qs, const RowSrc& ks, int32_t* idx, int32_t* cnt,
                             cudaStream_t stream, int num_sms) {
  const int esize = sizeof(T);
  const int kpitch = sh.d * esize + 16;
  const int rows_max = std::min(sh.bq, sh.Tq) * sh.group;
  // decode (a single query row) is HBM-latency-bound: small chunks, many in flight; prefill rows
  // amortise bigger chunks.
  const int target = rows_max <= 4 ? 10 * 1024 : 16 * 1024;
  const int ch = std::max(1, target / (sh.bk * kpitch));
  const int stage_bytes = (int)align_up((size_t)ch * sh.bk * kpitch, 128);
  size_t smem = align_up(sizeof(SelState<NMAX, kCCThreads / 32>), 128) + (size_t)rows_max * (sh.d + 4) * 4 +
                (size_t)kCCStages * stage_bytes + (size_t)ch * sh.bk * rows_max * 4;
  smem = align_up(smem, 16);
  auto kern = mask_cc_kernel<T, NMAX>;
  int per_sm = 1;
  cudaError_t e = persistent_ctas(kern, kCCThreads, smem, 0, &per_sm);
  if (e != cudaSuccess) return e;
  const int64_t units = (int64_t)sh.B * (sh.group > 1 ? sh.Hkv : sh.Hq) * sh.nqb;
  int64_t grid = std::min<int64_t>(units * std::max(sh.chunks, 1), (int64_t)num_sms * per_sm);
  kern<<<(unsigned)grid, kCCThreads, smem, stream>>>(sh, qs, ks, idx, cnt, ch, kpitch, stage_bytes);
  return cudaGetLastError();
}

cudaError_t launch_mask_cc(const Shape& sh, const QSrc& qs, const RowSrc& ks, bool bf16, int32_t* idx, int32_t* cnt,
                           cudaStream_t stream, int num_sms) {
  if (bf16) {
    if (sh.n <= 256) return launch_cc<__nv_bfloat16, 256>(sh, qs, ks, idx, cnt, stream, num_sms);
    return launch_cc<__nv_bfloat16, 1024>(sh, qs, ks, idx, cnt, stream, num_sms);
  }
  if (sh.n <= 256) return launch_cc<float, 256>(sh, qs, ks, idx, cnt, stream, num_sms);
  return launch_cc<float, 1024>(sh, qs, ks, idx, cnt, stream, num_sms);
}

}  // namespace hip
