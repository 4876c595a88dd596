// mask_tc.cu — HiP mask estimation (Alg. 1) with the branch scores on the 5th-gen
// tensor cores (tcgen05), bf16 inputs, fp32 accumulation in TMEM.
//
// Block approximation makes every representative score a small dense contraction:
// the b_q x d query block against the b_k x d rows of each representative key block.  Per iteration
// the CTA gathers the (up to 2n, then n) representative key blocks of its query block, 128 key rows
// per tile, straight from HBM/L2 into a 128-byte-swizzled K-major shared tile (coalesced 16-byte
// cp.async; one key row = 256 B), and one thread issues
//     S^T[128 keys x 32 queries] = K_tile[128 x 128] . Q_block^T      (tcgen05.mma, M=128, N=32)
// into 32 TMEM columns.  The epilogue warps read their 32 TMEM lanes (one key per thread, 32 query
// columns), take the max over the valid (causal) query rows, then the max over the b_k lanes of a
// block with shuffles -> one fp32 score per representative block, in shared memory.  The
// selection (split, rank-merge top-n, tie toward the smaller block) is select.cuh.
//
// Why keys on M: b_q = 32 is below the smallest tcgen05 M (64), so the query block is the N=32
// operand and the gathered keys fill M = 128.  The kernel is bound by the L2->SM
// gather of representative rows (32 FLOP per gathered byte, far below the tensor-core ridge).
#include "kernels.h"
#include "select.cuh"

namespace hip {

constexpr int kMTThreads = 128;
constexpr int kMTNmax = 256;
constexpr uint32_t kQTileBytes = 2 * 32 * 128;   // two 64-column regions x 32 rows x 128 B
constexpr uint32_t kKRegion = 128 * 128;         // 128 rows x 128 B
constexpr uint32_t kKTileBytes = 2 * kKRegion;   // d = 128 -> two regions
constexpr uint32_t kIdescS = idesc_bf16(128, 32, 0, 0);

struct MaskTCSmemLayout {
  static constexpr uint32_t q = 0;
  static constexpr uint32_t k0 = kQTileBytes;
  static constexpr uint32_t k1 = k0 + kKTileBytes;
  static constexpr uint32_t sel = k1 + kKTileBytes;
  static constexpr uint32_t misc = (uint32_t)align_up(sel + sizeof(SelState<kMTNmax>), 128);  // mbarrier: 8B
  static constexpr uint32_t total = misc + 64;
};

struct TCScorer {
  uint32_t q_s, k_s[2];
  uint64_t* mbar;
  uint32_t* phase;
  uint32_t tmem;
  RowSrc ks;
  int b, hk, Tk, bk, causal, rows_q, bpt;
  int64_t tpos0;

  __device__ void issue(const int* rep, int n_rep, int c) {
    const int blk0 = c * bpt, nblk = min(bpt, n_rep - blk0);
    const uint32_t dst = k_s[c & 1];
#pragma unroll 4
    for (int p = threadIdx.x; p < 128 * 16; p += kMTThreads) {
      const int r = p >> 4, c16 = p & 15;
      const int lb = r / bk;
      int64_t s = -1;
      if (lb < nblk) s = (int64_t)rep[blk0 + lb] * bk + (r - lb * bk);
      const bool ok = s >= 0 && s < Tk;
      const char* src = row_ptr(ks, b, hk, ok ? s : 0) + c16 * 16;
      cp_async16(dst + (c16 >> 3) * kKRegion + sw128_off(r, c16 & 7), src, ok ? 16u : 0u);
    }
  }

  __device__ void score(const int* rep, int n_rep, float* out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = (n_rep + bpt - 1) / bpt;
    issue(rep, n_rep, 0);
    cp_async_commit();
    for (int c = 0; c < ntiles; ++c) {
      if (c + 1 < ntiles) issue(rep, n_rep, c + 1);
      cp_async_commit();
      cp_async_wait<1>();
      fence_proxy_async_smem();
      __syncthreads();
      if (threadIdx.x == 0) {
        tc_fence_after();
        const uint32_t kt = k_s[c & 1];
#pragma unroll
        for (int s = 0; s < 8; ++s) {  // d = 128 = 8 x K16
          uint64_t a = smem_desc(kt + (s >> 2) * kKRegion + (s & 3) * 32, 16, 1024, kLayoutSw128);
          uint64_t bq = smem_desc(q_s + (s >> 2) * (32 * 128) + (s & 3) * 32, 16, 1024, kLayoutSw128);
          umma_bf16(tmem, a, bq, kIdescS, s > 0 ? 1u : 0u);
        }
        umma_commit(mbar);
      }
      mbar_wait(mbar, *phase);
      *phase ^= 1u;
      tc_fence_after();
      float v[32];
      tmem_ld_32x32b_x32(tmem + ((uint32_t)(32 * warp) << 16), v);
      const int blk0 = c * bpt, nblk = min(bpt, n_rep - blk0);
      const int r = 32 * warp + lane, lb = r / bk;
      float best = -INFINITY;
      if (lb < nblk) {
        const int64_t s = (int64_t)rep[blk0 + lb] * bk + (r - lb * bk);
        if (s < Tk) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < rows_q && (!causal || s <= tpos0 + j)) best = fmaxf(best, v[j]);
        }
      }
      for (int off = 1; off < bk; off <<= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, off));
      if (lb < nblk && (r - lb * bk) == 0) out[blk0 + lb] = best;
      tc_fence_before();
      __syncthreads();  // TMEM read before the next MMA; tile c consumed before issue(c + 2)
    }
  }
};

__global__ void __launch_bounds__(kMTThreads) mask_tc_kernel(Shape sh, QSrc qsrc, RowSrc ks, int32_t* __restrict__ idx,
                                                             int32_t* __restrict__ cnt) {
  extern __shared__ __align__(16) char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t pad = ((raw + 1023u) & ~1023u) - raw;
  char* base = smem_raw + pad;
  const uint32_t sbase = raw + pad;
  using L = MaskTCSmemLayout;
  SelState<kMTNmax>& st = *reinterpret_cast<SelState<kMTNmax>*>(base + L::sel);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(base + L::misc);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + L::misc + 8);
  const int warp = threadIdx.x >> 5;

  if (threadIdx.x == 0) {
    mbar_init(mbar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<32>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  uint32_t phase = 0;

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
      // query block -> K-major SW128 tile (B operand, N = 32 rows, rows >= rows_q zero)
      for (int p = threadIdx.x; p < 32 * 16; p += kMTThreads) {
        const int r = p >> 4, c16 = p & 15;
        const bool ok = r < rows_q;
        const char* src = q_ptr(qsrc, b, h, (int64_t)q * sh.bq + (ok ? r : 0)) + c16 * 16;
        cp_async16(sbase + L::q + (c16 >> 3) * (32 * 128) + sw128_off(r, c16 & 7), src, ok ? 16u : 0u);
      }
      cp_async_commit();
    }
    TCScorer sc;
    sc.q_s = sbase + L::q;
    sc.k_s[0] = sbase + L::k0;
    sc.k_s[1] = sbase + L::k1;
    sc.mbar = mbar;
    sc.phase = &phase;
    sc.tmem = tmem;
    sc.ks = ks;
    sc.b = b; sc.hk = hk; sc.Tk = Tk; sc.bk = sh.bk; sc.causal = sh.causal; sc.rows_q = rows_q;
    sc.bpt = 128 / sh.bk;
    sc.tpos0 = (int64_t)q * sh.bq + (Tk - sh.Tq);
    tree_search<kMTNmax, kMTThreads>(st, sh.n, Bq, sc, idx + lin * sh.n, cnt + lin);
    __syncthreads();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<32>(tmem);
}

// The tensor-core path needs a real query block on N (>= 8 rows); single-row decode scoring is a
// GEMV and runs on CUDA cores (mask_cc.cu, HBM-bound).
bool mask_tc_supported(const Shape& sh) {
  return sh.d == 128 && sh.bq >= 8 && sh.bq <= 32 && sh.bk <= 32 && (32 % sh.bk) == 0 && sh.n <= kMTNmax;
}

cudaError_t launch_mask_tc(const Shape& sh, const QSrc& qs, const RowSrc& ks, int32_t* idx, int32_t* cnt,
                           cudaStream_t stream, int num_sms) {
  const size_t smem = MaskTCSmemLayout::total + 1024;
  cudaError_t e = cudaFuncSetAttribute(mask_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mask_tc_kernel, kMTThreads, smem);
  if (e != cudaSuccess) return e;
  per_sm = std::min(std::max(per_sm, 1), 16);  // TMEM: 32 columns per CTA, 512 per SM
  const int64_t units = (int64_t)sh.B * sh.Hq * sh.nqb;
  int64_t grid = std::min<int64_t>(units, (int64_t)num_sms * per_sm);
  mask_tc_kernel<<<(unsigned)grid, kMTThreads, smem, stream>>>(sh, qs, ks, idx, cnt);
  return cudaGetLastError();
}

}  // namespace hip
