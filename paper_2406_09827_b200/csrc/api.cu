// api.cu — the C ABI declared in include/hip_attn.h: host-side validation (before any launch),
// dispatch to the sm_100a kernels, thread-local error strings.  No exception crosses the ABI.
#include <stdarg.h>
#include <stdio.h>

#include <atomic>

#include "hip_attn.h"
#include "kernels.h"

namespace {

thread_local char g_err[512] = "";

hip_status_t fail(hip_status_t s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

hip_status_t cuda_fail(cudaError_t e, const char* where) {
  return fail(HIP_ERROR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

constexpr int kMaxDev = 64;
std::atomic<int> g_sms[kMaxDev];     // 0 = unknown, -1 = unsupported arch
std::atomic<int> g_arch_ok[kMaxDev];

// SM count of the current device; NOT_SUPPORTED unless it is an sm_100 part (B200).
hip_status_t device_info(int* num_sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (dev < 0 || dev >= kMaxDev) return fail(HIP_ERROR_NOT_SUPPORTED, "device ordinal %d", dev);
  int s = g_sms[dev].load(std::memory_order_relaxed);
  if (s == 0) {
    int major = 0, minor = 0, n = 0;
    if ((e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev)) != cudaSuccess ||
        (e = cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev)) != cudaSuccess ||
        (e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
      return cuda_fail(e, "cudaDeviceGetAttribute");
    s = (major == 10 && minor == 0) ? n : -1;
    g_sms[dev].store(s, std::memory_order_relaxed);
    g_arch_ok[dev].store(major * 10 + minor, std::memory_order_relaxed);
  }
  if (s < 0)
    return fail(HIP_ERROR_NOT_SUPPORTED, "device %d is sm_%d, this library is built for sm_100a only", dev,
                g_arch_ok[dev].load());
  *num_sms = s;
  return HIP_SUCCESS;
}

int esize_of(hip_dtype_t dt) { return dt == HIP_DTYPE_F32 ? 4 : 2; }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

hip_status_t check_tensor(const char* name, const hip_tensor_t& t, int esz) {
  if (!t.ptr) return fail(HIP_ERROR_INVALID_VALUE, "%s: NULL pointer", name);
  if (!aligned16(t.ptr)) return fail(HIP_ERROR_INVALID_VALUE, "%s: base pointer not 16-byte aligned", name);
  const int64_t v = 16 / esz;
  if (t.stride_b % v || t.stride_h % v || t.stride_t % v || t.stride_b < 0 || t.stride_h < 0 || t.stride_t < 0)
    return fail(HIP_ERROR_INVALID_VALUE, "%s: strides must be non-negative multiples of %lld elements", name,
                (long long)v);
  return HIP_SUCCESS;
}

hip_status_t check_common(hip_dtype_t dt, int32_t B, int32_t Hq, int32_t Hkv, int32_t Tq, int32_t Tk, int32_t d,
                          const hip_params_t* p) {
  if (!p) return fail(HIP_ERROR_INVALID_VALUE, "params is NULL");
  if (dt != HIP_DTYPE_F32 && dt != HIP_DTYPE_BF16) return fail(HIP_ERROR_NOT_SUPPORTED, "dtype %d", (int)dt);
  if (B < 1 || Hq < 1 || Hkv < 1 || Tq < 1 || d < 1)
    return fail(HIP_ERROR_INVALID_VALUE, "dims must be >= 1 (B=%d H_q=%d H_kv=%d T_q=%d d=%d)", B, Hq, Hkv, Tq, d);
  if (Tk < 1) return fail(HIP_ERROR_INVALID_VALUE, "empty K: T_k=%d (S:209)", Tk);
  if (Hq % Hkv) return fail(HIP_ERROR_INVALID_VALUE, "H_q=%d not a multiple of H_kv=%d", Hq, Hkv);
  if (d != 64 && d != 128) return fail(HIP_ERROR_NOT_SUPPORTED, "head dim d=%d (supported: 64, 128)", d);
  if (p->b_q < 1 || p->b_k < 1) return fail(HIP_ERROR_INVALID_VALUE, "b_q=%d b_k=%d must be >= 1", p->b_q, p->b_k);
  if (p->k < p->b_k || p->k % p->b_k)
    return fail(HIP_ERROR_INVALID_VALUE, "k=%d must be a positive multiple of b_k=%d (reading G12)", p->k, p->b_k);
  if (p->k / p->b_k > 1024) return fail(HIP_ERROR_INVALID_VALUE, "n = k/b_k = %d > 1024", p->k / p->b_k);
  if (p->causal != 0 && p->causal != 1) return fail(HIP_ERROR_INVALID_VALUE, "causal must be 0 or 1");
  if (p->causal && Tq > Tk) return fail(HIP_ERROR_INVALID_VALUE, "causal with T_q=%d > T_k=%d", Tq, Tk);
  if (((int64_t)Tk + p->b_k - 1) / p->b_k >= (1 << 22))
    return fail(HIP_ERROR_NOT_SUPPORTED, "ceil(T_k / b_k) >= 2^22 key blocks (T_k=%d, b_k=%d)", Tk, p->b_k);
  if (std::min(p->b_q, Tq) > 64) return fail(HIP_ERROR_NOT_SUPPORTED, "query block of %d rows > 64", std::min(p->b_q, Tq));
  if ((p->flags & HIP_FLAG_GQA_SHARED_MASK) && (int64_t)std::min(p->b_q, Tq) * (Hq / Hkv) > 64)
    return fail(HIP_ERROR_NOT_SUPPORTED, "GQA-shared mask: (H_q / H_kv) x b_q = %d x %d rows > 64", Hq / Hkv,
                std::min(p->b_q, Tq));
  if (p->chunks < 0 || (p->chunks > 1 && (p->k / p->b_k) % p->chunks))
    return fail(HIP_ERROR_INVALID_VALUE, "chunks=%d must be >= 0 and divide n = k/b_k = %d", p->chunks,
                p->k / p->b_k);
  if (p->top_r < 0) return fail(HIP_ERROR_INVALID_VALUE, "top_r=%d must be >= 0", p->top_r);
  if (p->split_jitter < 0 || p->split_jitter > 65535)
    return fail(HIP_ERROR_INVALID_VALUE, "split_jitter=%d must be in [0, 65535]", p->split_jitter);
  if (p->sink_tokens < 0 || p->window_tokens < 0)
    return fail(HIP_ERROR_INVALID_VALUE, "sink_tokens=%d window_tokens=%d must be >= 0", p->sink_tokens,
                p->window_tokens);
  if ((int64_t)p->sink_tokens + p->window_tokens + std::min(p->b_q, Tq) - 1 > 256 &&
      (p->sink_tokens > 0 || p->window_tokens > 0))
    return fail(HIP_ERROR_NOT_SUPPORTED, "sink + window + b_q - 1 = %lld > 256",
                (long long)p->sink_tokens + p->window_tokens + std::min(p->b_q, Tq) - 1);
  (void)dt;
  return HIP_SUCCESS;
}

hip_status_t check_paged(const hip_paged_kv_t* pg, int esz, bool need_v, int bk) {
  if (!pg->k_pages || (need_v && !pg->v_pages) || !pg->block_table || !pg->seq_lens)
    return fail(HIP_ERROR_INVALID_VALUE, "paged: NULL pointer");
  if (!aligned16(pg->k_pages) || (need_v && !aligned16(pg->v_pages)))
    return fail(HIP_ERROR_INVALID_VALUE, "paged: pages not 16-byte aligned");
  const int64_t v = 16 / esz;
  if (pg->stride_page % v || pg->stride_h % v || pg->stride_t % v || pg->stride_page < 0 || pg->stride_h < 0 ||
      pg->stride_t < 0)
    return fail(HIP_ERROR_INVALID_VALUE, "paged: strides must be non-negative multiples of %lld", (long long)v);
  if (pg->page_size < 1 || pg->page_size % bk)
    return fail(HIP_ERROR_INVALID_VALUE, "paged: page_size=%d must be a positive multiple of b_k=%d", pg->page_size,
                bk);
  if (pg->max_pages_per_seq < 1 || pg->max_seq_len < 1 ||
      (int64_t)pg->max_pages_per_seq * pg->page_size < pg->max_seq_len)
    return fail(HIP_ERROR_INVALID_VALUE, "paged: max_pages_per_seq * page_size < max_seq_len");
  return HIP_SUCCESS;
}

// Workspace layout (bytes): [0, 256) the JobQueue counter of the launch.  (Split single-row
// attention units merge their chunk states through a thread-block cluster's shared memory, so no
// call needs more.)
constexpr size_t kWsQueue = 256;

size_t workspace_bytes_for(hip_op_t, int32_t, int32_t, int32_t, int32_t, const hip_params_t*) { return kWsQueue; }

hip_status_t check_workspace(void* ws, size_t have, size_t need) {
  if (need == 0) return HIP_SUCCESS;
  if (!ws) return fail(HIP_ERROR_WORKSPACE, "workspace is NULL; hip_workspace_bytes() = %zu", need);
  if (have < need) return fail(HIP_ERROR_WORKSPACE, "workspace of %zu bytes < hip_workspace_bytes() = %zu", have, need);
  if (!aligned16(ws)) return fail(HIP_ERROR_WORKSPACE, "workspace not 16-byte aligned");
  return HIP_SUCCESS;
}

// Point the launch's job counter at the caller's workspace.
void bind_workspace(hip::Shape& sh, void* ws, bool, int32_t, int32_t, int32_t, int32_t, const hip_params_t*) {
  sh.sched = reinterpret_cast<unsigned int*>(ws);
}

hip::Shape make_shape(int32_t B, int32_t Hq, int32_t Hkv, int32_t Tq, int32_t Tk, int32_t d, const hip_params_t* p,
                      const int32_t* seq_lens) {
  hip::Shape s{};
  s.B = B; s.Hq = Hq; s.Hkv = Hkv; s.Tq = Tq; s.Tk = Tk; s.d = d;
  s.n = p->k / p->b_k; s.bq = std::min(p->b_q, Tq); s.bk = p->b_k; s.causal = p->causal;
  s.nqb = (Tq + s.bq - 1) / s.bq;
  s.sink = p->sink_tokens; s.window = p->window_tokens;
  s.chunks = p->chunks > 1 ? p->chunks : 1;
  s.top_r = p->top_r > 0 && p->top_r < d ? p->top_r : 0;
  s.jitter = p->split_jitter;
  s.group = (p->flags & HIP_FLAG_GQA_SHARED_MASK) ? Hq / Hkv : 1;
  s.seed = p->sample_seed;
  s.seq_lens = seq_lens;
  s.sched = nullptr;
  s.splits = 1;
  return s;
}

hip::QSrc make_q(const hip_tensor_t& t, int esz) {
  hip::QSrc q;
  q.base = static_cast<const char*>(t.ptr);
  q.sb = t.stride_b; q.sh = t.stride_h; q.st = t.stride_t; q.esize = esz;
  return q;
}

hip::RowSrc make_rows(const hip_tensor_t& t, int esz) {
  hip::RowSrc r{};
  r.base = static_cast<const char*>(t.ptr);
  r.sb = t.stride_b; r.sh = t.stride_h; r.st = t.stride_t; r.esize = esz; r.paged = 0;
  return r;
}

hip::RowSrc make_paged(const hip_paged_kv_t& pg, const void* pages, int esz) {
  hip::RowSrc r{};
  r.base = static_cast<const char*>(pages);
  r.sp = pg.stride_page; r.sh = pg.stride_h; r.st = pg.stride_t; r.esize = esz; r.paged = 1;
  r.block_table = pg.block_table; r.page_size = pg.page_size; r.max_pages = pg.max_pages_per_seq;
  r.page_shift = -1;
  r.sp_rows = (pg.stride_t > 0 && pg.stride_page % pg.stride_t == 0) ? pg.stride_page / pg.stride_t : 0;
  for (int sh = 0; sh < 31; ++sh)
    if ((1 << sh) == pg.page_size) r.page_shift = sh;
  r.bt16 = pg.num_pages > 0 && pg.num_pages <= 65536 && pg.max_pages_per_seq <= hip::kBt16Max;
  return r;
}

}  // namespace

extern "C" {

int32_t hip_version(void) { return HIP_ATTN_VERSION; }

const char* hip_last_error(void) { return g_err; }

int32_t hip_num_blocks(const hip_params_t* p) {
  if (!p || p->b_k < 1 || p->k < p->b_k || p->k % p->b_k) return 0;
  return p->k / p->b_k;
}

size_t hip_workspace_bytes(hip_op_t op, hip_dtype_t dtype, int32_t B, int32_t H_q, int32_t H_kv, int32_t T_q,
                           int32_t T_k, int32_t d, const hip_params_t* params) {
  (void)dtype; (void)H_kv; (void)T_k;
  if (!params || B < 1 || H_q < 1 || T_q < 1 || params->b_q < 1) return 0;
  if (op != HIP_OP_MASK && op != HIP_OP_PREFILL && op != HIP_OP_DECODE) return 0;
  return workspace_bytes_for(op, B, H_q, T_q, d, params);
}

hip_status_t hip_mask_estimate(hip_dtype_t dtype, int32_t B, int32_t H_q, int32_t H_kv, int32_t T_q, int32_t T_k,
                               int32_t d, hip_tensor_t q, hip_tensor_t k, const hip_paged_kv_t* paged,
                               const hip_params_t* params, int32_t* block_idx, int32_t* block_cnt, void* workspace,
                               size_t workspace_bytes, void* stream) {
  hip_status_t s = check_common(dtype, B, H_q, H_kv, T_q, T_k, d, params);
  if (s) return s;
  const int esz = esize_of(dtype);
  if ((s = check_tensor("q", q, esz))) return s;
  if (!block_idx || !block_cnt) return fail(HIP_ERROR_INVALID_VALUE, "block_idx / block_cnt is NULL");
  if (paged) {
    if ((s = check_paged(paged, esz, false, params->b_k))) return s;
    if (T_k != paged->max_seq_len)
      return fail(HIP_ERROR_INVALID_VALUE, "paged: T_k=%d must equal max_seq_len=%d", T_k, paged->max_seq_len);
  } else if ((s = check_tensor("k", k, esz))) {
    return s;
  }
  if ((s = check_workspace(workspace, workspace_bytes, workspace_bytes_for(HIP_OP_MASK, B, H_q, T_q, d, params))))
    return s;
  int sms = 0;
  if ((s = device_info(&sms))) return s;
  hip::Shape sh = make_shape(B, H_q, H_kv, T_q, T_k, d, params, paged ? paged->seq_lens : nullptr);
  bind_workspace(sh, workspace, false, B, H_q, T_q, d, params);
  hip::QSrc qs = make_q(q, esz);
  hip::RowSrc ks = paged ? make_paged(*paged, paged->k_pages, esz) : make_rows(k, esz);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  const bool exact = (params->flags & HIP_FLAG_EXACT_SCORES) != 0;
  if (dtype == HIP_DTYPE_BF16 && !exact && hip::mask_tc_supported(sh))
    e = hip::launch_mask_tc(sh, qs, ks, block_idx, block_cnt, st, sms);
  else if (!exact && hip::mask_decode_supported(sh))
    e = hip::launch_mask_decode(sh, qs, ks, dtype == HIP_DTYPE_BF16, block_idx, block_cnt, st, sms);
  else
    e = hip::launch_mask_cc(sh, qs, ks, dtype == HIP_DTYPE_BF16, block_idx, block_cnt, st, sms);
  if (e != cudaSuccess) return cuda_fail(e, "hip_mask_estimate launch");
  return HIP_SUCCESS;
}

hip_status_t hip_mask_vote(int32_t n_e, int64_t units, int32_t n_in, const int32_t* block_idx_samples,
                           const int32_t* block_cnt_samples, int32_t theta, int32_t tau, int32_t n_out,
                           int32_t* block_idx, int32_t* block_cnt, void* stream) {
  if (!block_idx_samples || !block_cnt_samples || !block_idx || !block_cnt)
    return fail(HIP_ERROR_INVALID_VALUE, "hip_mask_vote: NULL pointer");
  if (n_e < 1 || n_e > 16) return fail(HIP_ERROR_INVALID_VALUE, "n_e=%d must be in [1, 16]", n_e);
  if (units < 0) return fail(HIP_ERROR_INVALID_VALUE, "units=%lld < 0", (long long)units);
  if (n_in < 1 || (int64_t)n_e * n_in > 4096)
    return fail(HIP_ERROR_INVALID_VALUE, "n_in=%d: need 1 <= n_in and n_e * n_in <= 4096", n_in);
  if (theta < 1 || theta > n_e) return fail(HIP_ERROR_INVALID_VALUE, "theta=%d must be in [1, n_e=%d]", theta, n_e);
  if (tau != 0 && tau != 1) return fail(HIP_ERROR_INVALID_VALUE, "tau=%d must be 0 or 1", tau);
  if (n_out < (tau ? n_in : n_e * n_in))
    return fail(HIP_ERROR_INVALID_VALUE, "n_out=%d < %d", n_out, tau ? n_in : n_e * n_in);
  int sms = 0;
  hip_status_t s;
  if ((s = device_info(&sms))) return s;
  cudaError_t e = hip::launch_vote(n_e, units, n_in, block_idx_samples, block_cnt_samples, theta, tau, n_out,
                                   block_idx, block_cnt, static_cast<cudaStream_t>(stream), sms);
  if (e != cudaSuccess) return cuda_fail(e, "hip_mask_vote launch");
  return HIP_SUCCESS;
}

hip_status_t hip_sparse_attention_prefill(hip_dtype_t dtype, int32_t B, int32_t H_q, int32_t H_kv, int32_t T_q,
                                          int32_t T_k, int32_t d, hip_tensor_t q, hip_tensor_t k, hip_tensor_t v,
                                          const hip_params_t* params, const int32_t* block_idx,
                                          const int32_t* block_cnt, hip_tensor_t o, float* lse, void* workspace,
                                          size_t workspace_bytes, void* stream) {
  hip_status_t s = check_common(dtype, B, H_q, H_kv, T_q, T_k, d, params);
  if (s) return s;
  const int esz = esize_of(dtype);
  if ((s = check_tensor("q", q, esz)) || (s = check_tensor("k", k, esz)) || (s = check_tensor("v", v, esz)) ||
      (s = check_tensor("o", o, esz)))
    return s;
  if (!block_idx || !block_cnt) return fail(HIP_ERROR_INVALID_VALUE, "block_idx / block_cnt is NULL");
  if ((s = check_workspace(workspace, workspace_bytes, workspace_bytes_for(HIP_OP_PREFILL, B, H_q, T_q, d, params))))
    return s;
  int sms = 0;
  if ((s = device_info(&sms))) return s;
  hip::Shape sh = make_shape(B, H_q, H_kv, T_q, T_k, d, params, nullptr);
  bind_workspace(sh, workspace, true, B, H_q, T_q, d, params);
  const float scale = params->sm_scale > 0.f ? params->sm_scale : 1.0f / sqrtf((float)d);
  hip::QSrc qs = make_q(q, esz);
  hip::RowSrc ks = make_rows(k, esz), vs = make_rows(v, esz);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* op = static_cast<char*>(const_cast<void*>(o.ptr));
  cudaError_t e;
  if (dtype == HIP_DTYPE_BF16 && hip::attn_row1_supported(sh))
    e = hip::launch_attn_row1(sh, qs, ks, vs, block_idx, block_cnt, scale, op, o.stride_b, o.stride_h, o.stride_t, lse,
                              st, sms);
  else if (dtype == HIP_DTYPE_BF16 && hip::attn_tc_supported(sh))
    e = hip::launch_attn_tc(sh, qs, ks, vs, block_idx, block_cnt, scale, op, o.stride_b, o.stride_h, o.stride_t, lse,
                            st, sms);
  else if (hip::attn_decode_supported(sh))
    e = hip::launch_attn_decode(sh, qs, ks, vs, dtype == HIP_DTYPE_BF16, block_idx, block_cnt, scale, op, o.stride_b,
                                o.stride_h, o.stride_t, lse, st, sms);
  else
    e = hip::launch_attn_cc(sh, qs, ks, vs, dtype == HIP_DTYPE_BF16, block_idx, block_cnt, scale, op, o.stride_b,
                            o.stride_h, o.stride_t, lse, st, sms);
  if (e != cudaSuccess) return cuda_fail(e, "hip_sparse_attention_prefill launch");
  return HIP_SUCCESS;
}

hip_status_t hip_sparse_attention_decode(hip_dtype_t dtype, int32_t B, int32_t H_q, int32_t H_kv, int32_t T_q,
                                         int32_t d, hip_tensor_t q, const hip_paged_kv_t* paged,
                                         const hip_params_t* params, const int32_t* block_idx,
                                         const int32_t* block_cnt, hip_tensor_t o, float* lse, void* workspace,
                                         size_t workspace_bytes, void* stream) {
  if (!paged) return fail(HIP_ERROR_INVALID_VALUE, "paged is NULL");
  hip_status_t s = check_common(dtype, B, H_q, H_kv, T_q, paged->max_seq_len, d, params);
  if (s) return s;
  const int esz = esize_of(dtype);
  if ((s = check_tensor("q", q, esz)) || (s = check_tensor("o", o, esz))) return s;
  if ((s = check_paged(paged, esz, true, params->b_k))) return s;
  if (!block_idx || !block_cnt) return fail(HIP_ERROR_INVALID_VALUE, "block_idx / block_cnt is NULL");
  if ((s = check_workspace(workspace, workspace_bytes, workspace_bytes_for(HIP_OP_DECODE, B, H_q, T_q, d, params))))
    return s;
  int sms = 0;
  if ((s = device_info(&sms))) return s;
  hip::Shape sh = make_shape(B, H_q, H_kv, T_q, paged->max_seq_len, d, params, paged->seq_lens);
  bind_workspace(sh, workspace, true, B, H_q, T_q, d, params);
  const float scale = params->sm_scale > 0.f ? params->sm_scale : 1.0f / sqrtf((float)d);
  hip::QSrc qs = make_q(q, esz);
  hip::RowSrc ks = make_paged(*paged, paged->k_pages, esz), vs = make_paged(*paged, paged->v_pages, esz);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* op = static_cast<char*>(const_cast<void*>(o.ptr));
  cudaError_t e;
  // tcgen05 path: physical row index page * (page stride in rows) + offset must fit in int32
  const bool tc_rows = ks.sp_rows > 0 && paged->num_pages > 0 &&
                       (int64_t)paged->num_pages * ks.sp_rows < ((int64_t)1 << 31);
  if (dtype == HIP_DTYPE_BF16 && tc_rows && hip::attn_row1_supported(sh))
    e = hip::launch_attn_row1(sh, qs, ks, vs, block_idx, block_cnt, scale, op, o.stride_b, o.stride_h, o.stride_t, lse,
                              st, sms);
  else if (dtype == HIP_DTYPE_BF16 && tc_rows && hip::attn_tc_supported(sh))
    e = hip::launch_attn_tc(sh, qs, ks, vs, block_idx, block_cnt, scale, op, o.stride_b, o.stride_h, o.stride_t, lse,
                            st, sms);
  else if (hip::attn_decode_supported(sh))
    e = hip::launch_attn_decode(sh, qs, ks, vs, dtype == HIP_DTYPE_BF16, block_idx, block_cnt, scale, op, o.stride_b,
                                o.stride_h, o.stride_t, lse, st, sms);
  else
    e = hip::launch_attn_cc(sh, qs, ks, vs, dtype == HIP_DTYPE_BF16, block_idx, block_cnt, scale, op, o.stride_b,
                            o.stride_h, o.stride_t, lse, st, sms);
  if (e != cudaSuccess) return cuda_fail(e, "hip_sparse_attention_decode launch");
  return HIP_SUCCESS;
}

}  // extern "C"

