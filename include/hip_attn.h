/*
 * hip_attn.h — C ABI of the B200 (sm_100a) hot path of HiP, Hierarchically Pruned Attention
 * (arXiv 2406.09827).  Library: paper_2406_09827_b200/libhipattn.so.
 *
 * Citation key: P:n = /root/reference/PAPER.md line n (LaTeX source of the paper), S:n = SPEC.md
 * line n.  "Gn" = reading n of the paper listed in DESIGN.md ("Readings of the paper").
 *
 * The hot path has two stages (Alg. 1; Eq. 1-3):
 *   1. hip_mask_estimate: per query block of b_q rows, a greedy tree search over key blocks of b_k
 *      keys keeps n = k / b_k nodes, splits each into two branches, scores each branch by the
 *      max of the b_q x b_k score tile of its FIRST key block, keeps the n best branches, and
 *      repeats until every node is a single key block.  Output: the n selected key-block indices.
 *   2. hip_sparse_attention_prefill / _decode: softmax(mask(Q K^T) * sm_scale) V over the tokens of
 *      the selected key blocks only (Eq. 2-3), prefill on contiguous K/V, decode on a paged cache.
 *
 * Conventions (all entry points)
 *   - Tensors are [B, H, T, d] with d contiguous (stride 1) and arbitrary B/H/T strides given in
 *     ELEMENTS; rows must be 16-byte aligned (d * elem_size % 16 == 0 and 16-byte aligned base).
 *   - Queries are bottom-right aligned: query row t sits at key position t + T_k - T_q (reading G7).
 *     Causal: row t sees key s iff s <= t + T_k - T_q.
 *   - GQA: query head h reads kv head h / (H_q / H_kv).  One mask per query head (G15).
 *   - All pointers are DEVICE pointers owned by the caller; the library allocates nothing on the
 *     device and never frees caller memory.  Work is enqueued on `stream` (a cudaStream_t passed as
 *     void*, NULL = legacy default stream) and is asynchronous; device faults surface as
 *     HIP_ERROR_CUDA on a later call or at the caller's synchronisation.
 *   - Arguments are validated on the host BEFORE any launch; an invalid call launches nothing and
 *     leaves outputs untouched.  hip_last_error() returns a thread-local message for the last
 *     non-success status.  No C++ exception crosses the ABI; functions are thread-safe.
 *   - Results are deterministic: the same inputs give the same bits regardless of batch
 *     composition, stream or the number of GPUs the caller shards over.
 *   - The `hip_` prefix is the north-star name (BASELINE.json); it is unrelated to AMD HIP.
 */
#ifndef HIP_ATTN_H_
#define HIP_ATTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HIP_ATTN_VERSION 201 /* 2.0.1: hip_workspace_bytes is 256 for every call (split single-row
                                 attention merges on thread-block clusters; 2.0 callers unaffected);
                                 2.0.0: every compute call takes a workspace (prefill gained the two
                                 arguments); 1.2.0: + HIP_FLAG_GQA_SHARED_MASK (1.1.0: top_r,
                                 split_jitter, sample_seed, hip_mask_vote) */

typedef enum {
    HIP_SUCCESS = 0,
    HIP_ERROR_INVALID_VALUE = 1, /* bad shape, pointer, stride or parameter (see each call)      */
    HIP_ERROR_NOT_SUPPORTED = 2, /* valid but not implemented here (dtype, d, device arch)       */
    HIP_ERROR_WORKSPACE = 3,     /* workspace missing or smaller than hip_workspace_bytes()      */
    HIP_ERROR_CUDA = 4           /* a CUDA runtime error (message in hip_last_error())           */
} hip_status_t;

typedef enum {
    HIP_DTYPE_F32 = 0, /* fp32 in, fp32 out; mask scores on CUDA cores, sequential fmaf (G9)      */
    HIP_DTYPE_BF16 = 1 /* bf16 in, bf16 out; fp32 accumulation; tcgen05 tensor cores where shaped */
} hip_dtype_t;

/* Flags (hip_params_t.flags). */
#define HIP_FLAG_EXACT_SCORES 1u /* mask: score every branch with the canonical sequential fp32 fmaf
                                    chain on CUDA cores even for bf16 (bit-exact with the oracle's
                                    F32C mode on any input; slower)                                 */
#define HIP_FLAG_GQA_SHARED_MASK 2u /* GQA-shared masks (reading G25): ONE mask per
                                    (b, kv head, query block), its branch scores the max of the tile
                                    over the b_q rows of ALL H_q / H_kv query heads of the group.
                                    hip_mask_estimate then writes block_idx [B, H_kv, N_qb, n] and
                                    block_cnt [B, H_kv, N_qb]; the attention calls given the same
                                    flag read query head h's selection from kv head h / (H_q/H_kv).
                                    Requires (H_q / H_kv) x min(b_q, T_q) <= 64 rows.               */

typedef struct {
    int32_t k;        /* token budget per query block; n = k / b_k key blocks are kept (G1)    */
    int32_t b_q;      /* query block size; >= 1                                             */
    int32_t b_k;      /* key block size; >= 1, k % b_k == 0 (G12)                             */
    int32_t causal;   /* 0 / 1 (reading G7/G8)                                               */
    float sm_scale;   /* attention softmax scale; <= 0 means 1/sqrt(d) (G11).  The mask uses raw
                         q.k and ignores it.                                         */
    uint32_t flags;   /* HIP_FLAG_*                                                                  */
    int32_t sink_tokens;   /* attention only (0 = off): every row also attends to keys [0, sink)    */
    int32_t window_tokens; /* attention only (0 = off): row at position p also attends to keys
                              (p - window, p].  StreamingLLM sink + sliding window, fused into the
                              sparse kernels (the paper uses (window, sink) = (128, 32);
                              the union of S:285-301, each token once; reading G14).  Both >= 0,
                              sink + window + b_q - 1 <= 256.  hip_mask_estimate ignores them.     */
    int32_t chunks;        /* mask only: stridden partial top-k (reading G21).  0 or 1 =
                              Alg. 1.  S > 1 (S | n): when B_q > n the visible key blocks are split
                              into S contiguous chunks [a_s, a_{s+1}), a_s = floor((2 s B_q + S)/(2 S)),
                              each searched with n / S nodes by its own job (S x more parallel jobs);
                              the output concatenates the chunks (still ascending, cnt = n).        */
    int32_t top_r;         /* mask only: top-r approximation (reading G22).  0 (or >= d) =
                              exact branch scores.  0 < r < d: a branch score sums q_c k_c over the r
                              components with the largest max-over-rows |q_c| of the query block
                              (ties -> smaller c) only; key chunks holding no kept component are not
                              fetched.                                                              */
    int32_t split_jitter;  /* mask only: ensemble sampling (reading G23).  0 = Alg. 1's
                              half-up split.  R > 0 (<= 65535): every split point moves by u uniform in
                              [-R, R] (splitmix64 keyed by sample_seed, the unit (b*H_q + h)*N_qb + q,
                              the iteration and the node's first block), clamped so both branches stay
                              non-empty.  Combine samples with hip_mask_vote.                       */
    uint64_t sample_seed;  /* mask only: seed of the ensemble sample (ignored when split_jitter = 0) */
} hip_params_t;

typedef struct {
    const void* ptr;  /* element [b, h, t, c] at ptr + (b*stride_b + h*stride_h + t*stride_t + c) */
    int64_t stride_b, stride_h, stride_t; /* in elements                                           */
} hip_tensor_t;

/* Paged KV cache (decode; layout [num_pages, H_kv, page_size, d] through strides).
 * Token s of sequence b is slot s % page_size of physical page block_table[b*max_pages_per_seq +
 * s / page_size].  page_size % b_k == 0 so a key block never straddles two pages. */
typedef struct {
    const void* k_pages;
    const void* v_pages;              /* may be NULL for hip_mask_estimate                     */
    int64_t stride_page, stride_h, stride_t; /* in elements, shared by k_pages and v_pages       */
    const int32_t* block_table;       /* [B, max_pages_per_seq] device, physical page ids        */
    const int32_t* seq_lens;          /* [B] device, T_k of each sequence, 1 <= T_k <= max_seq_len */
    int32_t page_size;
    int32_t max_pages_per_seq;
    int32_t num_pages;                /* physical pages; 0 = unknown (the decode attention then  */
                                      /* avoids the tcgen05 path, which indexes rows in int32)   */
    int32_t max_seq_len;              /* host-side upper bound of seq_lens (sizes the launch)    */
} hip_paged_kv_t;

typedef enum { HIP_OP_MASK = 0, HIP_OP_PREFILL = 1, HIP_OP_DECODE = 2 } hip_op_t;

/* Library version (HIP_ATTN_VERSION of the build). */
int32_t hip_version(void);

/* Thread-local, NUL-terminated message describing the last non-success status of this thread. */
const char* hip_last_error(void);

/* Number of key blocks kept per query block, n = k / b_k (0 if the params are invalid). */
int32_t hip_num_blocks(const hip_params_t* params);

/* Device workspace (bytes) a call with these arguments needs: scratch owned by the caller, at
 * least 16-byte aligned, passed as (workspace, workspace_bytes).  A call returns
 * HIP_ERROR_WORKSPACE (before any launch) if it is NULL or smaller.  Contents need no
 * initialisation and are meaningless after the call; the library (re)initialises what it uses on
 * `stream` (cudaMemsetAsync) before each launch.  One workspace must not serve two calls that may
 * run concurrently (different streams without ordering), exactly like the outputs.
 *   - every op: 256 bytes for the launch's job counter (persistent CTAs claim (b, h, query block)
 *     jobs in order, which balances uneven query blocks and keeps the running jobs within one or
 *     two heads, so that head's K stays L2-resident).
 *   (Single-row attention units split over idle CTA slots run each unit on a thread-block cluster
 *   and merge the partial softmax states in shared memory, so they need nothing more; ABI 2.0
 *   callers that size the workspace with this function are unaffected.)
 * Returns 0 for invalid arguments. */
size_t hip_workspace_bytes(hip_op_t op, hip_dtype_t dtype, int32_t B, int32_t H_q, int32_t H_kv, int32_t T_q,
                           int32_t T_k, int32_t d, const hip_params_t* params);

/*
 * hip_mask_estimate — Alg. 1 with block approximation.
 *
 *   q            [B, H_q, T_q, d] queries (dtype)
 *   k            [B, H_kv, T_k, d] keys (dtype); ignored when `paged` != NULL
 *   paged        NULL for contiguous K; else the paged cache (then T_k is per sequence =
 *                seq_lens[b] and the T_k argument must equal paged->max_seq_len)
 *   block_idx    OUT int32 [B, H_q, N_qb, n], N_qb = ceil(T_q / b_q), n = k / b_k: the selected key
 *                blocks of every query block in ascending order, -1 after the first block_cnt
 *   block_cnt    OUT int32 [B, H_q, N_qb]: min(n, B_q) where B_q is the number of visible key blocks
 *                (all of them if causal == 0)
 *   workspace    device scratch of at least hip_workspace_bytes(HIP_OP_MASK, ...) bytes (see there)
 *   Semantics per query block (G1-G10): if B_q <= n all visible blocks are selected; else n initial
 *   nodes f_j = floor((2 j B_q + n) / 2n), split at m = floor((f + l + 1) / 2), branch score = max of
 *   q_t . k_s over the tile of the branch's first block (causal pairs only), keep the n best by
 *   (score desc, first block asc), until all nodes are single blocks.  Scores are fp32; the
 *   summation order of each dot product depends on the path (readings G9/G9b):
 *     - bf16, b_q <= 32 (decode included), d = 128, b_k | 32, n <= 256: tcgen05 fp32 accumulation,
 *       whose rounding can flip near-tied selections (reported as a fraction by the tests,
 *       DESIGN.md "Parity");
 *     - other query blocks of <= 4 rows (fp32 or d = 64 decode), b_k a power of two <= 16: 16
 *       sequential fmaf segments of d/16 terms combined by the xor tree o = 8, 4, 2, 1 ("F32L");
 *     - otherwise, and always with HIP_FLAG_EXACT_SCORES: the sequential chain c = 0..d-1 ("F32C").
 *   Errors: INVALID_VALUE for NULL pointers, dims < 1, T_k = 0 ("empty K"), k < b_k or
 *   k % b_k != 0, H_q % H_kv != 0, causal with T_q > T_k, page_size % b_k != 0, n > 1024,
 *   misaligned rows; WORKSPACE for a NULL, short or misaligned workspace; NOT_SUPPORTED for d not in
 *   {64, 128} or a device that is not sm_100.
 *   b_q > T_q or b_k > T_k is NOT an error (one ragged block).
 */
hip_status_t hip_mask_estimate(hip_dtype_t dtype, int32_t B, int32_t H_q, int32_t H_kv, int32_t T_q, int32_t T_k,
                               int32_t d, hip_tensor_t q, hip_tensor_t k, const hip_paged_kv_t* paged,
                               const hip_params_t* params, int32_t* block_idx, int32_t* block_cnt,
                               void* workspace, size_t workspace_bytes, void* stream);

/*
 * hip_sparse_attention_prefill — Eq. 2-3 over contiguous K/V, block-sparse
 * flash-style.
 *
 *   q, k, v      [B, H_q, T_q, d], [B, H_kv, T_k, d], [B, H_kv, T_k, d] (dtype)
 *   block_idx    [B, H_q, N_qb, n] ascending selected key blocks, block_cnt [B, H_q, N_qb]
 *                (normally the output of hip_mask_estimate with the same params; any ascending
 *                set of distinct blocks in [0, ceil(T_k / b_k)) is accepted)
 *   o            OUT [B, H_q, T_q, d] (dtype): row t = sum_s softmax_s(sm_scale q_t . k_s) v_s over
 *                the tokens s of the selected blocks with s < T_k and (causal) s <= t + T_k - T_q,
 *                united with [0, params->sink_tokens) and (p - params->window_tokens, p] for the
 *                row's position p = t + T_k - T_q when those are > 0 (each token once; G14)
 *   lse          OUT optional fp32 [B, H_q, T_q] contiguous (natural log-sum-exp of the scaled
 *                scores), NULL to skip.  A row with no visible token gets o = 0 and
 *                lse = -inf (G13).
 *   workspace    device scratch of at least hip_workspace_bytes(HIP_OP_PREFILL, ...) bytes
 *   Arithmetic: fp32 scores and softmax; bf16 probabilities into the PV contraction (bf16 path).
 *   Single-row units that do not fill the GPU are split over the keys (split-K) and merged in the
 *   kernel by rescaling each split's partial softmax state to the common max (same result up to
 *   fp32 rounding).
 *   Errors: as hip_mask_estimate; block indices are NOT range-checked on the device (garbage in,
 *   garbage out, never an out-of-bounds read: indices are clamped to [0, ceil(T_k/b_k)) ).
 */
hip_status_t hip_sparse_attention_prefill(hip_dtype_t dtype, int32_t B, int32_t H_q, int32_t H_kv, int32_t T_q,
                                          int32_t T_k, int32_t d, hip_tensor_t q, hip_tensor_t k, hip_tensor_t v,
                                          const hip_params_t* params, const int32_t* block_idx,
                                          const int32_t* block_cnt, hip_tensor_t o, float* lse, void* workspace,
                                          size_t workspace_bytes, void* stream);

/*
 * hip_sparse_attention_decode — Eq. 2-3 for T_q query rows per sequence (T_q = 1 for plain decode)
 * against a paged KV cache (Alg. 2 line "Perform fused sparse attention").
 *
 *   q            [B, H_q, T_q, d]; the rows sit at positions seq_lens[b] - T_q + t
 *   paged        the cache (k_pages and v_pages required)
 *   block_idx / block_cnt / o / lse as for prefill, with N_qb = ceil(T_q / b_q)
 *   workspace    device scratch of at least hip_workspace_bytes(HIP_OP_DECODE, ...) bytes
 *   Errors: as hip_mask_estimate.
 */
hip_status_t hip_sparse_attention_decode(hip_dtype_t dtype, int32_t B, int32_t H_q, int32_t H_kv, int32_t T_q,
                                         int32_t d, hip_tensor_t q, const hip_paged_kv_t* paged,
                                         const hip_params_t* params, const int32_t* block_idx,
                                         const int32_t* block_cnt, hip_tensor_t o, float* lse, void* workspace,
                                         size_t workspace_bytes, void* stream);

/*
 * hip_mask_vote — the HiP ensemble vote (Appendix D; reading G24).
 *
 *   n_e          number of sample masks, 1 <= n_e <= 16 (typically hip_mask_estimate outputs with
 *                split_jitter > 0 and different sample_seed)
 *   units        number of query blocks per sample (B * H_q * N_qb)
 *   n_in         index row length of the samples (n = k / b_k); n_e * n_in <= 4096
 *   block_idx_samples  [n_e, units, n_in] int32 device, each row ascending distinct, -1 padded
 *   block_cnt_samples  [n_e, units] int32 device
 *   theta        agreement threshold, 1 <= theta <= n_e (1 = union, n_e = intersection)
 *   tau          0: keep every index with >= theta votes (a row may exceed n_in — dynamic sparsity);
 *                1: keep at most n_in of them, by (votes desc, block asc)
 *   n_out        OUT row length: >= n_in if tau = 1, >= n_e * n_in if tau = 0
 *   block_idx    OUT [units, n_out] ascending, -1 padded; block_cnt OUT [units]
 *   The outputs feed hip_sparse_attention_* with a params whose k = n_out * b_k.
 *   Errors: INVALID_VALUE for NULL pointers or out-of-range n_e / n_in / theta / tau / n_out;
 *   NOT_SUPPORTED on a device that is not sm_100.  Sample rows must be ascending and distinct (not
 *   checked on the device; other input gives an unspecified but in-bounds result).
 */
hip_status_t hip_mask_vote(int32_t n_e, int64_t units, int32_t n_in, const int32_t* block_idx_samples,
                           const int32_t* block_cnt_samples, int32_t theta, int32_t tau, int32_t n_out,
                           int32_t* block_idx, int32_t* block_cnt, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HIP_ATTN_H_ */
