// common.cuh — device helpers shared by the HiP kernels (sm_100a only).
//
// PTX wrappers for cp.async (LDGSTS), mbarrier, tcgen05 (TMEM alloc / MMA / commit / ld) and the
// UMMA shared-memory + instruction descriptors, plus the problem descriptors passed to kernels.
// Nothing here is shared with the CPU oracle (oracle/), by design.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef __CUDACC__
#error "CUDA only"
#endif

namespace hip {

// ----------------------------------------------------------------------------------------------
// Problem descriptors
// ----------------------------------------------------------------------------------------------
// Where key (or value) row s of (batch b, kv head hk) lives: contiguous [B,Hkv,T,d] or paged
// [num_pages, Hkv, page_size, d] through a block table.  Strides are in elements.
struct RowSrc {
  const char* base;          // bytes
  int64_t sb, sh, st;        // contiguous strides (elements); paged: sh, st used + sp
  int64_t sp;                // paged: page stride (elements)
  const int32_t* block_table;
  int32_t page_size, max_pages;
  int32_t page_shift;        // paged: log2(page_size) if a power of two, else -1
  int64_t sp_rows;           // paged: sp / st when integral (page stride in rows), else 0
  int32_t paged;
  int32_t esize;             // bytes per element
  int32_t bt16;              // paged: physical page ids fit 16 bits and a sequence's block-table row
                             // fits kBt16Max entries (kernels may stage it in shared memory)
};
constexpr int kBt16Max = 3072;

__device__ __forceinline__ const char* row_ptr(const RowSrc& r, int b, int hk, int64_t s) {
  if (!r.paged) return r.base + (b * r.sb + hk * r.sh + s * r.st) * r.esize;
  const uint32_t us = (uint32_t)s;  // token index < 2^31
  uint32_t pi, off;
  if (r.page_shift >= 0) {
    pi = us >> r.page_shift;
    off = us & ((1u << r.page_shift) - 1u);
  } else {
    pi = us / (uint32_t)r.page_size;
    off = us - pi * (uint32_t)r.page_size;
  }
  const int64_t page = __ldg(r.block_table + (int64_t)b * r.max_pages + pi);
  return r.base + (page * r.sp + hk * r.sh + (int64_t)off * r.st) * r.esize;
}

struct QSrc {
  const char* base;
  int64_t sb, sh, st;
  int32_t esize;
};

__device__ __forceinline__ const char* q_ptr(const QSrc& q, int b, int h, int64_t t) {
  return q.base + (b * q.sb + h * q.sh + t * q.st) * q.esize;
}

// Shape of one launch.  Tk is uniform unless seq_lens != nullptr (paged decode).
struct Shape {
  int B, Hq, Hkv, Tq, Tk, d;
  int n, bq, bk, causal;
  int nqb;
  int sink, window;  // attention: sink / sliding-window tokens (sinkwin.cuh), 0 = off
  int chunks;        // mask: stridden partial top-k chunks S (select.cuh chunk_job), 1 = Alg. 1
  int top_r;         // mask: top-r approximation (topr.cuh), 0 = all d components
  int jitter;        // mask: ensemble split jitter R (select.cuh SplitJitter), 0 = half-up split
  uint64_t seed;     // mask: ensemble sample seed
  int group;         // query heads per mask: H_q / H_kv for GQA-shared masks (reading G25), else 1
  const int32_t* seq_lens;
  unsigned int* sched;  // dynamic job counter (JobQueue), zeroed before the launch; nullptr = static
  int splits;           // single-row attention: split-K factor S (a cluster of S CTAs per unit), 1 = off
};

__device__ __forceinline__ int seq_len(const Shape& sh, int b) {
  return sh.seq_lens ? __ldg(sh.seq_lens + b) : sh.Tk;
}

// Unit u -> (b, h, q): head-major (all query blocks of one head adjacent, so K of that head stays
// in L2 while they run); within a head the heavier (later) query blocks first.
__device__ __forceinline__ void unit_coords(const Shape& sh, int64_t u, int& b, int& h, int& q) {
  int64_t bh = u / sh.nqb;
  q = sh.nqb - 1 - (int)(u - bh * sh.nqb);
  b = (int)(bh / sh.Hq);
  h = (int)(bh - (int64_t)b * sh.Hq);
}

// Persistent-CTA job distribution.  Static (sched == nullptr): CTA i takes jobs i, i + grid, ...
// Dynamic (sched = a counter the launcher zeroed on the launch stream): after its first job
// (blockIdx.x) a CTA claims grid + atomicAdd(sched, 1).  Thread 0 claims at the START of the current
// job (the atomic's latency is hidden behind the job) and publishes the index through a
// double-buffered shared slot that every thread reads after a CTA barrier in next(): the slot
// written during job j is rewritten only during job j + 2, after barriers every thread has passed.
// Claiming in order keeps the concurrently running jobs a window of consecutive indices (one or
// two heads' K stay L2-resident; with static striding the CTAs drift apart) and balances uneven
// job costs (C4: mask 21.9 -> 20.0 ms, attention 5.9 -> 5.35 ms).
struct JobQueue {
  unsigned int* sched;
  volatile int64_t* slot;  // [2] in shared memory
  int par;
  __device__ __forceinline__ JobQueue(unsigned int* s, void* smem_slot)
      : sched(s), slot(reinterpret_cast<volatile int64_t*>(smem_slot)), par(0) {}
  __device__ __forceinline__ void claim() {
    if (sched && threadIdx.x == 0) slot[par] = (int64_t)gridDim.x + (int64_t)atomicAdd(sched, 1u);
  }
  __device__ __forceinline__ int64_t next(int64_t j) {
    if (!sched) return j + gridDim.x;
    __syncthreads();
    const int64_t v = slot[par];
    par ^= 1;
    return v;
  }
};

// Mask heads: one mask per kv head when GQA-shared (G25), else one per query head.
__device__ __forceinline__ int mask_heads(const Shape& sh) { return sh.group > 1 ? sh.Hkv : sh.Hq; }

// Mask unit u -> (b, mask head hm, q), in unit_coords' order.
__device__ __forceinline__ void mask_unit_coords(const Shape& sh, int64_t u, int& b, int& hm, int& q) {
  const int Hm = mask_heads(sh);
  int64_t bh = u / sh.nqb;
  q = sh.nqb - 1 - (int)(u - bh * sh.nqb);
  b = (int)(bh / Hm);
  hm = (int)(bh - (int64_t)b * Hm);
}

// Row of block_idx / block_cnt that query head h of batch b reads at query block q.
__device__ __forceinline__ int64_t mask_lin(const Shape& sh, int b, int h, int q) {
  return sh.group > 1 ? ((int64_t)b * sh.Hkv + h / sh.group) * sh.nqb + q : ((int64_t)b * sh.Hq + h) * sh.nqb + q;
}

// Visible key blocks of query block q (a1; reading G7): all blocks if not causal, else the blocks
// that start at or before the key position of the block's last row.
__device__ __forceinline__ int visible_blocks(const Shape& sh, int q, int Tk) {
  int nkb = (Tk + sh.bk - 1) / sh.bk;
  if (!sh.causal) return nkb;
  int64_t tlast = min((int64_t)(q + 1) * sh.bq, (int64_t)sh.Tq) - 1;
  int64_t v = (tlast + (Tk - sh.Tq)) / sh.bk + 1;
  return (int)min(v, (int64_t)nkb);
}

// ----------------------------------------------------------------------------------------------
// Small utilities
// ----------------------------------------------------------------------------------------------
__host__ __device__ constexpr size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Phase timers (profiling builds only: -DHIPATTN_PHASES, see profiles/phase_timers.py).  Thread 0
// of each CTA accumulates clock64() deltas per phase into g_phase_cycles.
#ifdef HIPATTN_PHASES
__device__ unsigned long long g_phase_cycles[16];
struct PhaseTimer {
  unsigned long long acc[16];
  long long t0;
  __device__ PhaseTimer() { for (int i = 0; i < 16; ++i) acc[i] = 0; t0 = clock64(); }
  __device__ __forceinline__ void mark(int p) {
    long long t = clock64();
    acc[p] += (unsigned long long)(t - t0);
    t0 = t;
  }
  __device__ void flush() {
    if (threadIdx.x == 0)
      for (int i = 0; i < 16; ++i) atomicAdd(&g_phase_cycles[i], acc[i]);
  }
};
#define HIP_PT_MEMBER PhaseTimer* pt = nullptr;
#define HIP_MARK(p) do { if (pt) pt->mark(p); } while (0)
#else
#define HIP_PT_MEMBER
#define HIP_MARK(p) do { } while (0)
#endif

// 2^x with the SFU (relative error ~2^-22; the probabilities it feeds are rounded to bf16).
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// ----------------------------------------------------------------------------------------------
// cp.async (LDGSTS): 16-byte global -> shared copy; src_bytes < 16 zero-fills the remainder.
// ----------------------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes)
               : "memory");
}
// Same with an L2 prefetch-size hint of 256 bytes: the L2 fetches the whole 256-byte line pair
// around the address from DRAM, so the other half of a 256-byte bf16 key row (the second d-half
// item, gathered a moment later) is already in L2.  Pays where the gathered rows come from DRAM
// (paged decode: C3 mask 136 -> 123 us); neutral where they are L2-resident (prefill).
__device__ __forceinline__ void cp_async16_pf256(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
// Make generic-proxy shared-memory writes (cp.async / st.shared) visible to the async proxy
// (tcgen05.mma operand reads).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// ----------------------------------------------------------------------------------------------
// mbarrier
// ----------------------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// mbarrier wait on a shared-memory address (no generic-to-shared conversion in the spin loop)
__device__ __forceinline__ void mbar_wait_u32(uint32_t addr, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(phase)
      : "memory");
}
// Arrive on `bar` once all of this thread's earlier cp.async copies have landed (no pending-count
// increment: the barrier's expected count includes this arrival).
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void umma_commit_u32(uint32_t addr) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(addr)
               : "memory");
}
// ----------------------------------------------------------------------------------------------
// Thread-block clusters: rank, barrier, stores into a peer CTA's shared memory (DSMEM)
// ----------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {  // every thread of every CTA of the cluster
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ float ld_cluster_f32(uint32_t local_saddr, uint32_t rank) {
  uint32_t ra;
  float v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(local_saddr), "r"(rank));
  asm volatile("ld.shared::cluster.f32 %0, [%1];\n" : "=f"(v) : "r"(ra) : "memory");
  return v;
}
__device__ __forceinline__ void st_cluster_f32(uint32_t local_saddr, uint32_t rank, float v) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(local_saddr), "r"(rank));
  asm volatile("st.shared::cluster.f32 [%0], %1;\n" ::"r"(ra), "f"(v) : "memory");
}

// ----------------------------------------------------------------------------------------------
// tcgen05: TMEM allocation, MMA, commit, loads
// ----------------------------------------------------------------------------------------------
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {  // one full warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst_smem)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {  // the same warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(kCols) : "memory");
}
// One lane of the (converged) warp returns true (elect.sync).
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.b32 %0, 1, 0, P;\n}\n"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem], kind::f16 (bf16 inputs, fp32 accumulate), issued by ONE thread.
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: thread i of the warp gets lane (base + i), columns
// [col, col + 32).  The warp must be the one allowed to access that lane quadrant (warp % 4).
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Same, one column.
__device__ __forceinline__ float tmem_ld_32x32b_x1(uint32_t taddr) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(r) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  return __uint_as_float(r);
}
// ----------------------------------------------------------------------------------------------
// UMMA descriptors (sm_100 tcgen05)
// ----------------------------------------------------------------------------------------------
// Shared-memory matrix descriptor: start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46), version 1 at
// [46,48), base offset 0, layout type at [61,64) (0 none/interleave, 2 = 128B swizzle,
// 4 = 64B swizzle, 6 = 32B swizzle).
enum : uint32_t { kLayoutNone = 0, kLayoutSw128 = 2, kLayoutSw64 = 4, kLayoutSw32 = 6 };

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}

// Instruction descriptor, kind::f16: D fp32 (bits 4-5 = 1), A bf16 (7-9 = 1), B bf16 (10-12 = 1),
// A major (15), B major (16) (0 = K-major, 1 = MN-major), N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t M, uint32_t N, uint32_t a_mn_major, uint32_t b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (a_mn_major << 15) | (b_mn_major << 16) | ((N >> 3) << 17) |
         ((M >> 4) << 24);
}

// Byte offset of 16-byte chunk `c` (0..7) of row `r` inside a K-major / MN-major 128-byte-swizzled
// region whose rows are 128 bytes (8-row atoms of 1024 bytes; chunk XOR (row % 8)).
__device__ __forceinline__ uint32_t sw128_off(uint32_t r, uint32_t c) {
  return (r >> 3) * 1024u + (r & 7u) * 128u + ((c ^ (r & 7u)) << 4);
}

}  // namespace hip
