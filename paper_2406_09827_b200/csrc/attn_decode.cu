// attn_decode.cu — block-sparse attention for short query blocks (decode against a paged KV cache,
// P:451, Alg. 2 "fused sparse attention"; T_q <= 4).  With one query row the contraction is
// a GEMV: HBM-bound, no tensor-core work.
//
// Each half-warp (16 lanes) streams selected keys U = 8 at a time: lane l loads the 16-byte slice l
// of the key row and of the value row (coalesced 256-byte rows, 16 loads in flight per lane), the
// score is a 16-lane fmaf + xor-tree dot product, and the half-warp keeps an online-softmax state
// (running max, running sum, and its lane's d/16 slice of the output accumulator) per query row.
// The 8 half-warps of the CTA split the unit's keys and merge their states through shared memory
// at the end; rows are normalised and stored coalesced.
#include "kernels.h"
#include "sinkwin.cuh"

namespace hip {

constexpr int kADThreads = 128;
constexpr int kADRows = 4;
constexpr int kADU = 8;
constexpr float kADLog2e = 1.4426950408889634f;
constexpr float kADLn2 = 0.6931471805599453f;

template <typename T, int D, int RM, bool kPaged>
__global__ void __launch_bounds__(kADThreads, 4) attn_decode_kernel(Shape sh, QSrc qsrc, RowSrc ks, RowSrc vs,
                                                                 const int32_t* __restrict__ idx,
                                                                 const int32_t* __restrict__ cnt, float scale_log2,
                                                                 char* __restrict__ o, int64_t osb, int64_t osh,
                                                                 int64_t ost, float* __restrict__ lse) {
  constexpr int E = D / 16;
  constexpr int NV = (E * (int)sizeof(T) + 15) / 16;
  constexpr int HW = kADThreads / 16;
  __shared__ float part[HW][RM][D + 2];
  __shared__ int xlist[kMaxExtra];  // sink / window tokens of the unit (sinkwin.cuh)
  __shared__ int wtot[32];
  const int lane16 = threadIdx.x & 15, hw = threadIdx.x >> 4;
  const int lbk = 31 - __clz(sh.bk), bmask = sh.bk - 1;

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
    const int nkeys = c << lbk;
    const int32_t* blk = idx + lin * sh.n;
    const int ne = (sh.sink > 0 || sh.window > 0)
                       ? build_extra<kADThreads>(blk, c, lbk, Tk, tpos0, tpos0 + rows_q - 1, sh.causal, sh.sink,
                                                 sh.window, xlist, wtot)
                       : 0;
    const int nall = nkeys + ne;
    const char* kbase = ks.base + (b * ks.sb + hk * ks.sh) * (int64_t)ks.esize;
    const char* vbase = vs.base + (b * vs.sb + hk * vs.sh) * (int64_t)vs.esize;
    const uint32_t krow = (uint32_t)(ks.st * ks.esize), vrow = (uint32_t)(vs.st * vs.esize);

    float qv[RM][E];
#pragma unroll
    for (int t = 0; t < RM; ++t) {
      const T* src = reinterpret_cast<const T*>(q_ptr(qsrc, b, h, (int64_t)q * sh.bq + min(t, rows_q - 1)));
#pragma unroll
      for (int e = 0; e < E; ++e) {
        float x;
        if constexpr (sizeof(T) == 4) x = src[lane16 * E + e];
        else x = __bfloat162float(src[lane16 * E + e]);
        qv[t][e] = t < rows_q ? x : 0.f;
      }
    }
    float m[RM], l[RM], acc[RM][E];
#pragma unroll
    for (int t = 0; t < RM; ++t) {
      m[t] = -INFINITY;
      l[t] = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) acc[t][e] = 0.f;
    }

    // uniform trip count for every half-warp (the xor shuffles below span the full warp)
    const int nbatch = (nall + HW * kADU - 1) / (HW * kADU);
    for (int bt = 0; bt < nbatch; ++bt) {
      const int k0 = bt * HW * kADU + hw * kADU;
      uint4 kb[kADU][NV], vb[kADU][NV];
      int sv[kADU];
#pragma unroll
      for (int i = 0; i < kADU; ++i) {
        const int k = k0 + i;
        int s = -1;
        bool extra = false;
        if (k < nkeys) {
          const int j = min(max(__ldg(blk + (k >> lbk)), 0), nkb - 1);
          s = (j << lbk) + (k & bmask);
          if (s >= Tk) s = -1;
        } else if (k < nall) {
          s = xlist[k - nkeys];
          extra = true;
        }
        sv[i] = extra ? (s | kExtraBit) : s;
        const int ss = s >= 0 ? s : 0;
        const char* kp;
        const char* vp;
        if constexpr (kPaged) {
          kp = row_ptr(ks, b, hk, ss);
          vp = row_ptr(vs, b, hk, ss);
        } else {
          kp = kbase + (uint64_t)(uint32_t)ss * krow;
          vp = vbase + (uint64_t)(uint32_t)ss * vrow;
        }
        kp += lane16 * (E * (int)sizeof(T));
        vp += lane16 * (E * (int)sizeof(T));
#pragma unroll
        for (int w = 0; w < NV; ++w) {
          if constexpr (E * sizeof(T) >= 16) {
            kb[i][w] = __ldg(reinterpret_cast<const uint4*>(kp) + w);
            vb[i][w] = __ldg(reinterpret_cast<const uint4*>(vp) + w);
          } else {
            const uint2 a = __ldg(reinterpret_cast<const uint2*>(kp)), bb = __ldg(reinterpret_cast<const uint2*>(vp));
            kb[i][w] = make_uint4(a.x, a.y, 0u, 0u);
            vb[i][w] = make_uint4(bb.x, bb.y, 0u, 0u);
          }
        }
      }
#pragma unroll
      for (int t = 0; t < RM; ++t) {
        if (t >= rows_q) continue;
        float x[kADU];
        float bm = -INFINITY;
#pragma unroll
        for (int i = 0; i < kADU; ++i) {
          const uint32_t* w = reinterpret_cast<const uint32_t*>(&kb[i][0]);
          float a = 0.f;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            float kv;
            if constexpr (sizeof(T) == 4) kv = __uint_as_float(w[e]);
            else kv = (e & 1) ? bf16_hi(w[e >> 1]) : bf16_lo(w[e >> 1]);
            a = fmaf(qv[t][e], kv, a);
          }
#pragma unroll
          for (int off = 8; off >= 1; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
          const int si = sv[i] & ~kExtraBit;
          const bool ok = sv[i] >= 0 && (!sh.causal || si <= tpos0 + t) &&
                          (!(sv[i] & kExtraBit) || extra_visible(si, tpos0 + t, sh.causal, sh.sink, sh.window));
          x[i] = ok ? a * scale_log2 : -INFINITY;
          bm = fmaxf(bm, x[i]);
        }
        const float mn = fmaxf(m[t], bm);
        if (mn == -INFINITY) continue;
        const float corr = ex2_approx(m[t] - mn);
        m[t] = mn;
        l[t] *= corr;
#pragma unroll
        for (int e = 0; e < E; ++e) acc[t][e] *= corr;
#pragma unroll
        for (int i = 0; i < kADU; ++i) {
          const float p = ex2_approx(x[i] - mn);
          l[t] += p;
          const uint32_t* w = reinterpret_cast<const uint32_t*>(&vb[i][0]);
#pragma unroll
          for (int e = 0; e < E; ++e) {
            float vv;
            if constexpr (sizeof(T) == 4) vv = __uint_as_float(w[e]);
            else vv = (e & 1) ? bf16_hi(w[e >> 1]) : bf16_lo(w[e >> 1]);
            acc[t][e] = fmaf(p, vv, acc[t][e]);
          }
        }
      }
    }
    // merge the half-warp states of each row
#pragma unroll
    for (int t = 0; t < RM; ++t) {
      if (t >= rows_q) continue;
#pragma unroll
      for (int e = 0; e < E; ++e) part[hw][t][lane16 * E + e] = acc[t][e];
      if (lane16 == 0) {
        part[hw][t][D] = m[t];
        part[hw][t][D + 1] = l[t];
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < rows_q * D; i += kADThreads) {
      const int t = i / D, dd = i - t * D;
      float mm = -INFINITY;
#pragma unroll
      for (int g = 0; g < HW; ++g) mm = fmaxf(mm, part[g][t][D]);
      float ll = 0.f, a = 0.f;
      if (mm != -INFINITY) {
#pragma unroll
        for (int g = 0; g < HW; ++g) {
          const float w = ex2_approx(part[g][t][D] - mm);
          ll = fmaf(part[g][t][D + 1], w, ll);
          a = fmaf(part[g][t][dd], w, a);
        }
      }
      const float val = ll > 0.f ? a / ll : 0.f;
      char* orow = o + (b * osb + h * osh + ((int64_t)q * sh.bq + t) * ost) * (int64_t)sizeof(T);
      if constexpr (sizeof(T) == 4) reinterpret_cast<float*>(orow)[dd] = val;
      else reinterpret_cast<__nv_bfloat16*>(orow)[dd] = __float2bfloat16_rn(val);
      if (lse && dd == 0)
        lse[((int64_t)b * sh.Hq + h) * sh.Tq + (int64_t)q * sh.bq + t] = ll > 0.f ? mm * kADLn2 + logf(ll) : -INFINITY;
    }
    __syncthreads();
  }
}

bool attn_decode_supported(const Shape& sh) {
  return std::min(sh.bq, sh.Tq) <= kADRows && (sh.bk & (sh.bk - 1)) == 0 && (sh.d == 64 || sh.d == 128);
}

template <typename T, int D, int RM>
static cudaError_t launch_ad(const Shape& sh, const QSrc& qs, const RowSrc& ks, const RowSrc& vs, const int32_t* idx,
                             const int32_t* cnt, float sm_scale, char* o, int64_t osb, int64_t osh, int64_t ost,
                             float* lse, cudaStream_t stream, int num_sms) {
  auto kern = ks.paged ? attn_decode_kernel<T, D, RM, true> : attn_decode_kernel<T, D, RM, false>;
  int per_sm = 1;
  cudaError_t e = persistent_ctas(kern, kADThreads, 0, 0, &per_sm);
  if (e != cudaSuccess) return e;
  const int64_t units = (int64_t)sh.B * sh.Hq * sh.nqb;
  const int64_t grid = std::min<int64_t>(units, (int64_t)num_sms * per_sm);
  kern<<<(unsigned)grid, kADThreads, 0, stream>>>(sh, qs, ks, vs, idx, cnt, sm_scale * kADLog2e, o, osb, osh, ost,
                                                   lse);
  return cudaGetLastError();
}

template <typename T, int D>
static cudaError_t launch_ad_r(const Shape& sh, const QSrc& qs, const RowSrc& ks, const RowSrc& vs, const int32_t* idx,
                               const int32_t* cnt, float sm_scale, char* o, int64_t osb, int64_t osh, int64_t ost,
                               float* lse, cudaStream_t stream, int num_sms) {
  if (std::min(sh.bq, sh.Tq) == 1)
    return launch_ad<T, D, 1>(sh, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, num_sms);
  return launch_ad<T, D, kADRows>(sh, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, num_sms);
}

cudaError_t launch_attn_decode(const Shape& sh, const QSrc& qs, const RowSrc& ks, const RowSrc& vs, bool bf16,
                               const int32_t* idx, const int32_t* cnt, float sm_scale, char* o, int64_t osb,
                               int64_t osh, int64_t ost, float* lse, cudaStream_t stream, int num_sms) {
  if (bf16) {
    if (sh.d == 128)
      return launch_ad_r<__nv_bfloat16, 128>(sh, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, num_sms);
    return launch_ad_r<__nv_bfloat16, 64>(sh, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, num_sms);
  }
  if (sh.d == 128)
    return launch_ad_r<float, 128>(sh, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, num_sms);
  return launch_ad_r<float, 64>(sh, qs, ks, vs, idx, cnt, sm_scale, o, osb, osh, ost, lse, stream, num_sms);
}

}  // namespace hip
