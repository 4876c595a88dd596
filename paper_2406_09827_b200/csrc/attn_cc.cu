// attn_cc.cu — block-sparse attention on CUDA cores (Eq. 2-3; "Block Sparse Flash
// Attention"): softmax over the tokens of the selected key blocks only, flash-style
// (online softmax over staged key chunks, no T x T matrix).  fp32 for BASELINE config C1 and the
// paged decode path (T_q rows per sequence against a paged cache), where attention is
// a GEMV and HBM-bound.  bf16 prefill with d = 128 runs on tcgen05 (attn_tc.cu).
//
// One CTA (8 warps) per (b, h, query block), persistent.  Selected K/V rows are gathered with
// 16-byte cp.async into double-buffered shared chunks of KC keys.  Warps form a WR x WK grid:
// WR row groups (prefill: one row per warp at a time) x WK key groups (decode: the keys of the
// single row are split over warps), and the WK partial softmax states are merged at the end.
#include "kernels.h"
#include "sinkwin.cuh"

namespace hip {

constexpr int kACThreads = 256;
constexpr int kKC = 32;  // keys per staged chunk
constexpr int kACStages = 3;  // cp.async ring depth (2 chunks in flight while one is consumed)
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

template <typename T, int D, int RPWM>
__global__ void __launch_bounds__(kACThreads, RPWM <= 2 ? 4 : 1) attn_cc_kernel(Shape sh, QSrc qsrc, RowSrc ks, RowSrc vs,
                                                             const int32_t* __restrict__ idx,
                                                             const int32_t* __restrict__ cnt, float scale_log2,
                                                             char* __restrict__ o, int64_t osb, int64_t osh,
                                                             int64_t ost, float* __restrict__ lse, int WR) {
  extern __shared__ __align__(16) char smem[];
  constexpr int E = D / 32;  // output elements per lane
  constexpr int KP = D * sizeof(T) + 16;  // padded staged row pitch (bytes)
  const int R = min(sh.bq, sh.Tq);
  const int QP = D + 4;
  float* qs = reinterpret_cast<float*>(smem);                 // [R][QP]
  float* S = qs + R * QP;                                      // [R][kKC + 1]
  int* tok = reinterpret_cast<int*>(S + R * (kKC + 1));        // [S][kKC] token of each staged key (-1 none)
  int* xlist = tok + kACStages * kKC;                          // [kMaxExtra] sink / window tokens
  int* wtot = xlist + kMaxExtra;                               // [32] scan scratch
  char* kst = smem + align_up((size_t)((char*)(wtot + 32) - smem), 128);  // [S][kKC][KP]
  char* vst = kst + kACStages * kKC * KP;                      // [S][kKC][KP]
  float* part = reinterpret_cast<float*>(kst);                 // reused for the WK merge

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int WK = 8 / WR;
  const int wr = warp % WR, wk = warp / WR;
  const int RPW = (R + WR - 1) / WR;  // rows per warp (<= 8)

  const int64_t units = (int64_t)sh.B * sh.Hq * sh.nqb;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    int b, h, q;
    unit_coords(sh, u, b, h, q);
    const int hk = h / (sh.Hq / sh.Hkv);
    const int Tk = seq_len(sh, b);
    const int64_t lin = mask_lin(sh, b, h, q);  // the unit's mask row (GQA-shared: its group's, G25)
    const int rows_q = min(sh.bq, sh.Tq - q * sh.bq);
    const int64_t tpos0 = (int64_t)q * sh.bq + (Tk - sh.Tq);
    const int nkb = (Tk + sh.bk - 1) / sh.bk;
    const int c = min(max(__ldg(cnt + lin), 0), sh.n);
    const int nkeys = c * sh.bk;
    const int32_t* blk = idx + lin * sh.n;
    const int lbk = 31 - __clz(sh.bk);
    const int ne = (sh.sink > 0 || sh.window > 0)
                       ? build_extra<kACThreads>(blk, c, lbk, Tk, tpos0, tpos0 + rows_q - 1, sh.causal, sh.sink,
                                                 sh.window, xlist, wtot)
                       : 0;
    const int nall = nkeys + ne;

    for (int i = threadIdx.x; i < rows_q * D; i += kACThreads) {
      int t = i / D, cc = i - t * D;
      const T* src = reinterpret_cast<const T*>(q_ptr(qsrc, b, h, (int64_t)q * sh.bq + t));
      float v;
      if constexpr (sizeof(T) == 4) v = src[cc];
      else v = __bfloat162float(src[cc]);
      qs[t * QP + cc] = v;
    }

    float m[RPWM], l[RPWM], acc[RPWM][E];
#pragma unroll
    for (int i = 0; i < RPWM; ++i) {
      m[i] = -INFINITY;
      l[i] = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) acc[i][e] = 0.f;
    }

    const int nch = (nall + kKC - 1) / kKC;
    auto issue = [&](int ch) {
      if (ch >= nch) return;
      const int k0 = ch * kKC, kc = min(kKC, nall - k0);
      constexpr int pieces = D * sizeof(T) / 16;
      const int slot = ch % kACStages;
      int* tk = tok + slot * kKC;
      for (int p = threadIdx.x; p < kKC * pieces * 2; p += kACThreads) {
        int which = p / (kKC * pieces);  // 0 = K, 1 = V
        int rem = p - which * kKC * pieces;
        int r = rem / pieces, c16 = rem - r * pieces;
        int64_t s = -1;
        bool extra = false;
        if (r < kc) {
          if (k0 + r < nkeys) {
            int j = min(max(__ldg(blk + (k0 + r) / sh.bk), 0), nkb - 1);
            s = (int64_t)j * sh.bk + (k0 + r) % sh.bk;
            if (s >= Tk) s = -1;
          } else {
            s = xlist[k0 + r - nkeys];
            extra = true;
          }
        }
        if (which == 0 && c16 == 0) tk[r] = s >= 0 && extra ? (int)s | kExtraBit : (int)s;
        const RowSrc& src = which ? vs : ks;
        char* dst = (which ? vst : kst) + (slot * kKC + r) * KP + c16 * 16;
        const char* g = row_ptr(src, b, hk, s >= 0 ? s : 0) + c16 * 16;
        cp_async16(smem_u32(dst), g, s >= 0 ? 16u : 0u);
      }
    };
    __syncthreads();
#pragma unroll
    for (int ch = 0; ch < kACStages - 1; ++ch) {
      issue(ch);
      cp_async_commit();
    }
    for (int ch = 0; ch < nch; ++ch) {
      issue(ch + kACStages - 1);  // slot of chunk ch - 1, freed by the last barrier
      cp_async_commit();
      cp_async_wait<kACStages - 1>();
      __syncthreads();
      const int buf = ch % kACStages;
      const int* tk = tok + buf * kKC;
      // scores x * log2(e), x = sm_scale q.k (G11); invalid -> -inf
      for (int p = threadIdx.x; p < rows_q * kKC; p += kACThreads) {
        int t = p % rows_q, r = p / rows_q;
        int s = tk[r];
        const bool extra = s >= 0 && (s & kExtraBit);
        if (extra) s &= ~kExtraBit;
        float x = -INFINITY;
        if (s >= 0 && (!sh.causal || s <= tpos0 + t) &&
            (!extra || extra_visible(s, tpos0 + t, sh.causal, sh.sink, sh.window))) {
          const float4* qr = reinterpret_cast<const float4*>(qs + t * QP);
          float a = 0.f;
          if constexpr (sizeof(T) == 4) {
            const float4* kr = reinterpret_cast<const float4*>(kst + (buf * kKC + r) * KP);
#pragma unroll 8
            for (int i = 0; i < D / 4; ++i) {
              float4 kv = kr[i], qv = qr[i];
              a = fmaf(qv.x, kv.x, a); a = fmaf(qv.y, kv.y, a); a = fmaf(qv.z, kv.z, a); a = fmaf(qv.w, kv.w, a);
            }
          } else {
            const uint4* kr = reinterpret_cast<const uint4*>(kst + (buf * kKC + r) * KP);
#pragma unroll 4
            for (int i = 0; i < D / 8; ++i) {
              uint4 kv = kr[i];
              float4 qa = qr[2 * i], qb = qr[2 * i + 1];
              a = fmaf(qa.x, bf16_lo(kv.x), a); a = fmaf(qa.y, bf16_hi(kv.x), a);
              a = fmaf(qa.z, bf16_lo(kv.y), a); a = fmaf(qa.w, bf16_hi(kv.y), a);
              a = fmaf(qb.x, bf16_lo(kv.z), a); a = fmaf(qb.y, bf16_hi(kv.z), a);
              a = fmaf(qb.z, bf16_lo(kv.w), a); a = fmaf(qb.w, bf16_hi(kv.w), a);
            }
          }
          x = a * scale_log2;
        }
        S[t * (kKC + 1) + r] = x;
      }
      __syncthreads();
      // online softmax + PV: this warp's rows x this warp's keys (k = wk + WK * j)
#pragma unroll
      for (int i = 0; i < RPWM; ++i) {
        const int t = wr + i * WR;
        if (i >= RPW || t >= rows_q) continue;
        const int k = wk + WK * lane;
        float x = k < kKC ? S[t * (kKC + 1) + k] : -INFINITY;
        float mx = x;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        const float mn = fmaxf(m[i], mx);
        if (mn == -INFINITY) continue;
        const float corr = exp2f(m[i] - mn);
        m[i] = mn;
        float p = exp2f(x - mn);
        float ps = p;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
        l[i] = l[i] * corr + ps;
#pragma unroll
        for (int e = 0; e < E; ++e) acc[i][e] *= corr;
        const int nk = (kKC - wk + WK - 1) / WK;
        for (int jj = 0; jj < nk; ++jj) {
          float pj = __shfl_sync(0xffffffffu, p, jj);
          if (pj == 0.f) continue;
          const char* vr = vst + (buf * kKC + wk + WK * jj) * KP;
          if constexpr (sizeof(T) == 4) {
            const float* vv = reinterpret_cast<const float*>(vr) + lane * E;
#pragma unroll
            for (int e = 0; e < E; ++e) acc[i][e] = fmaf(pj, vv[e], acc[i][e]);
          } else {
            const __nv_bfloat16* vv = reinterpret_cast<const __nv_bfloat16*>(vr) + lane * E;
#pragma unroll
            for (int e = 0; e < E; ++e) acc[i][e] = fmaf(pj, __bfloat162float(vv[e]), acc[i][e]);
          }
        }
      }
      __syncthreads();
    }
    // merge the WK key-group partial states of each row, then normalise and write
    if (WK > 1) {
      const int stride = D + 2;
#pragma unroll
      for (int i = 0; i < RPWM; ++i) {
        const int t = wr + i * WR;
        if (i >= RPW || t >= rows_q) continue;
        float* pp = part + ((size_t)wk * R + t) * stride;
#pragma unroll
        for (int e = 0; e < E; ++e) pp[lane * E + e] = acc[i][e];
        if (lane == 0) { pp[D] = m[i]; pp[D + 1] = l[i]; }
      }
      __syncthreads();
      if (wk == 0) {
#pragma unroll
        for (int i = 0; i < RPWM; ++i) {
          const int t = wr + i * WR;
          if (i >= RPW || t >= rows_q) continue;
          float mm = -INFINITY;
          for (int g = 0; g < WK; ++g) mm = fmaxf(mm, part[((size_t)g * R + t) * stride + D]);
          float ll = 0.f, a2[E];
#pragma unroll
          for (int e = 0; e < E; ++e) a2[e] = 0.f;
          if (mm != -INFINITY) {
            for (int g = 0; g < WK; ++g) {
              const float* pp = part + ((size_t)g * R + t) * stride;
              float w = exp2f(pp[D] - mm);  // partial with m = -inf contributes 0
              ll = fmaf(pp[D + 1], w, ll);
#pragma unroll
              for (int e = 0; e < E; ++e) a2[e] = fmaf(pp[lane * E + e], w, a2[e]);
            }
          }
          m[i] = mm;
          l[i] = ll;
#pragma unroll
          for (int e = 0; e < E; ++e) acc[i][e] = a2[e];
        }
      }
    }
    if (wk == 0) {
#pragma unroll
      for (int i = 0; i < RPWM; ++i) {
        const int t = wr + i * WR;
        if (i >= RPW || t >= rows_q) continue;
        const bool empty = !(l[i] > 0.f);
        const float inv = empty ? 0.f : 1.f / l[i];
        char* orow = o + (b * osb + h * osh + ((int64_t)q * sh.bq + t) * ost) * (int64_t)sizeof(T);
#pragma unroll
        for (int e = 0; e < E; ++e) {
          float v = empty ? 0.f : acc[i][e] * inv;
          if constexpr (sizeof(T) == 4) reinterpret_cast<float*>(orow)[lane * E + e] = v;
          else reinterpret_cast<__nv_bfloat16*>(orow)[lane * E + e] = __float2bfloat16_rn(v);
        }
        if (lse && lane == 0)
          lse[((int64_t)b * sh.Hq + h) * sh.Tq + (int64_t)q * sh.bq + t] =
              empty ? -INFINITY : m[i] * kLn2 + logf(l[i]);
      }
    }
    __syncthreads();
  }
}

template <typename T, int D, int RPWM>
static cudaError_t launch_acc(const Shape& sh, const QSrc& qs, const RowSrc& ks, const RowSrc& vs, const int32_t* idx,
                              const int32_t* cnt, float sm_scale, char* o, int64_t osb, int64_t osh, int64_t ost,
                              float* lse, cudaStream_t stream, int num_sms) {
  const int R = std::min(sh.bq, sh.Tq);
  if (R > 64) return cudaErrorInvalidValue;
  int WR = R >= 8 ? 8 : (R >= 4 ? 4 : (R >= 2 ? 2 : 1));
  constexpr int KP = D * sizeof(T) + 16;
  const size_t stages = 2 * (size_t)kACStages * kKC * KP;
  size_t smem = align_up((size_t)R * (D + 4) * 4 + (size_t)R * (kKC + 1) * 4 + kACStages * kKC * 4 +
                              (kMaxExtra + 32) * 4, 128) + stages;
  size_t merge = (size_t)(8 / WR) * R * (D + 2) * 4;
  if (merge > stages) smem += merge - stages;
  smem = align_up(smem, 16);
  auto kern = attn_cc_kernel<T, D, RPWM>;
  int per_sm = 1;
  cudaError_t e = persistent_ctas(kern, kACThreads, smem, 0, &per_sm);
  if (e != cudaSuccess) return e;
  const int64_t units = (int64_t)sh.B * sh.Hq * sh.nqb;
  int64_t grid = std::min<int64_t>(units, (int64_t)num_sms * std::max(per_sm, 1));
  kern<<<(unsigned)grid, kACThreads, smem, stream>>>(sh, qs, ks, vs, idx, cnt, sm_scale * kLog2e, o, osb, osh, ost,
                                                     lse, WR);
  return cudaGetLastError();
}

template <typename T, int D>
static cudaError_t launch_acc_r(const Shape& sh, const QSrc& qs, const RowSrc& ks, const RowSrc& vs, const int32_t* idx,
                                const int32_t* cnt, float sm_scale, char* o, int64_t osb, int64_t osh, int64_t ost,
                                float* lse, cudaStream_t stream, int num_sms) {
  // rows per warp = ceil(R / WR) <= 2 whenever R <= 8 (decode / multi-query): fewer registers,
  // 4 CTAs per SM
  if (std::min(sh.bq, sh.Tq) <= 8)
    return launch_acc<T, D, 2>(sh, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, num_sms);
  return launch_acc<T, D, 8>(sh, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, num_sms);
}

cudaError_t launch_attn_cc(const Shape& sh, const QSrc& qs, const RowSrc& ks, const RowSrc& vs, bool bf16,
                           const int32_t* idx, const int32_t* cnt, float sm_scale, char* o, int64_t osb, int64_t osh,
                           int64_t ost, float* lse, cudaStream_t stream, int num_sms) {
  if (bf16) {
    if (sh.d == 128)
      return launch_acc_r<__nv_bfloat16, 128>(sh, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, num_sms);
    return launch_acc_r<__nv_bfloat16, 64>(sh, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, num_sms);
  }
  if (sh.d == 128)
    return launch_acc_r<float, 128>(sh, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, num_sms);
  return launch_acc_r<float, 64>(sh, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, num_sms);
}

}  // namespace hip
