/*
 * hip_oracle.c — CPU ORACLE for HiP (Hierarchically Pruned Attention, arXiv 2406.09827).
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the plain, slow, obviously-correct reference that the
 * CUDA path is checked against.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  It shares NO code, header, table or constant with the CUDA
 * path (paper_2406_09827_b200/csrc); neither includes the other.
 *
 * Citation key: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n; G<n> = reading n in
 * DESIGN.md §"Readings of the paper" (the same numbering as SURVEY.md §8c).
 *
 * What it computes (per batch b, query head h, query block q; kv head = h*Hkv/Hq):
 *   - oracle_mask             Alg. 1 with block approximation, step by step:
 *                             initial n = k/b_k nodes (G1), half-up rounding (G3), split into two
 *                             branches, representative = FIRST block of each branch
 *                             (G4), branch score = max of the b_q x b_k tile
 *                             (P:178-180), keep the top-n branches with
 *                             ties toward the smaller block (G10), until every node is one block
 *                             (G5, G6).  Causal reading G7/G8.
 *   - oracle_sparse_attention Eq. 2-3: softmax over the selected tokens only, fp64;
 *                             *_sw adds the StreamingLLM sink and sliding-window tokens (P:641-645,
 *                             the EffectiveMask union of S:285-301; reading G14).
 *   - oracle_dense_attention  S = QK^T, P = softmax(S), O = PV, fp64, causal optional.
 *   - oracle_exact_block_topn top-n of the exact block-max scores (the textbook top-k of P:116 at
 *                             block granularity) — used for pins and recall.
 *   - oracle_mask_ext         + the appendix extensions: top-r approximation (readings
 *                             G22) and the ensemble's jittered splits (G23), with the
 *                             stridden partial top-k (G21).
 *                             gqa_shared: one mask per GQA group scored over all its query
 *                             heads' rows (reading G25).
 *   - oracle_vote             the ensemble vote (G24).
 *   - *_paged                 the same on a paged KV cache (decode): token s of
 *                             sequence b lives at page block_table[b][s / page_size], slot
 *                             s % page_size; gathered with plain loops.
 *
 * Arithmetic.  Inputs are float32 arrays (bf16 inputs are widened exactly by the caller).  Mask
 * scores come in three modes: ORC_F32C — `acc = fmaf(q[c], k[c], acc)` for c = 0..d-1 (the canonical
 * fp32 order, reading G9); ORC_F32L — 16 sequential fmaf segments of d/16 terms combined by the
 * xor tree o = 8, 4, 2, 1 (the decode GEMV's order, reading G9b); and ORC_F64 — the dot product in
 * double.  Both fp32 orders are pinned by exact rational recomputation in the pin suite (one
 * rounding per fmaf / tree addition).  Attention is fp64 throughout.
 * Compile with -ffp-contract=off and without -ffast-math so that the written order is the order run.
 *
 * Pins (tests/test_oracle_pins.py): PIN-1 k >= T => dense causal attention (vs torch SDPA fp64);
 * PIN-2 n < B_q <= 2n => exact top-n of block maxima (brute-force sort); PIN-3 monotone scores;
 * PIN-4 worked examples; PIN-5 invariants;
 * PIN-6 scale invariance; PIN-7 complexity counter; PIN-8 attention special cases.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ENOMEM 2
#define ORC_ERANGE 3
#define ORC_EREPLAY 4 /* replay: the search asked for a block score that was not supplied */

#define ORC_F32C 0
#define ORC_F64 1
#define ORC_F32L 2 /* reading G9b: 16 sequential segments + pairwise tree (d % 16 == 0) */

typedef struct {
    int64_t f, l; /* first / last key-block index of the range, inclusive */
    double s;     /* score of the representative (= first) block         */
} orc_node;

static int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

/* Extensions of Alg. 1 from the paper's appendix (all off = Alg. 1 itself):
 *   top-r approximation: a branch score sums q_c k_c over the r components c with the
 *     largest |q_c| only; for a query block |q_c| is reduced by the max over its rows and ties go to
 *     the smaller component (reading G22, SPEC D5); the terms are summed in ascending c (G22).
 *   ensemble sampling: every split point is moved by a random integer offset,
 *     m = clamp(round_half_up((f+l)/2) + u, f+1, l) with u uniform in [-R, R], R = r_e (reading G23),
 *     drawn from the counter-based generator below keyed by (seed, unit, iteration, node first). */
typedef struct {
    const int *comp; /* top-r components, ascending; NULL = all d components */
    int ncomp;
    int R;           /* split jitter magnitude (0 = the deterministic half-up split) */
    uint64_t key;    /* per-unit generator key (orc_unit_key) */
    int G;           /* query heads scored together (GQA-shared mask, G25); 1 = one head */
    int64_t hstride; /* floats between the Q rows of consecutive heads of the group */
    int replay;      /* 1: scores come only from the caller-filled memo (oracle_mask_replay) */
} orc_ext;

/* splitmix64 output function (Steele, Lea & Flood 2014): the counter-based generator of the
 * ensemble.  The CUDA path implements the same published function independently. */
static uint64_t orc_mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
#define ORC_GOLDEN 0x9E3779B97F4A7C15ULL

/* first output of a splitmix64 stream seeded with `state` (pinned against the published vector) */
uint64_t oracle_splitmix64(uint64_t state) { return orc_mix64(state + ORC_GOLDEN); }

/* key of unit lin = (b*Hq + h)*N_qb + q for sample seed `seed` */
static uint64_t orc_unit_key(uint64_t seed, int64_t lin) { return orc_mix64(orc_mix64(seed + ORC_GOLDEN) ^ (uint64_t)lin); }

/* split offset u in [-R, R] of the node whose first block is f, at iteration it (0 = first split) */
static int64_t orc_jitter(uint64_t key, int it, int64_t f, int R)
{
    uint64_t x = orc_mix64(key ^ (((uint64_t)(uint32_t)it << 32) | (uint64_t)(uint32_t)f));
    return (int64_t)(x % (uint64_t)(2 * R + 1)) - R;
}

/* argtop_r(|q|) of a query block (reading G22): a_c = max over the rows of |q_c|, the r
 * largest a_c with ties toward the smaller c, returned in ascending order.  r >= d: all. */
static void top_r_components(const float *Qh, int64_t t0, int64_t t1, int G, int64_t hstride, int d, int r,
                             int *out)
{
    double *a = (double *)malloc(sizeof(double) * (size_t)d);
    char *taken = (char *)calloc((size_t)d, 1);
    for (int c = 0; c < d; ++c) {
        a[c] = 0.0;
        for (int g = 0; g < G; ++g)
            for (int64_t t = t0; t < t1; ++t) {
                double v = fabs((double)Qh[g * hstride + t * d + c]);
                if (v > a[c]) a[c] = v;
            }
    }
    /* r rounds of "take the largest remaining, smallest index on ties" */
    for (int i = 0; i < r; ++i) {
        int best = -1;
        for (int c = 0; c < d; ++c)
            if (!taken[c] && (best < 0 || a[c] > a[best])) best = c;
        taken[best] = 1;
    }
    int w = 0;
    for (int c = 0; c < d; ++c)
        if (taken[c]) out[w++] = c;
    free(a);
    free(taken);
}

/* Validation shared by every entry point. */
static int check_dims(int B, int Hq, int Hkv, int Tq, int Tk, int d, int k, int bq, int bk, int causal)
{
    if (B < 1 || Hq < 1 || Hkv < 1 || Tq < 1 || Tk < 1 || d < 1) return ORC_EINVAL;
    if (Hq % Hkv != 0) return ORC_EINVAL;
    if (bq < 1 || bk < 1 || k < bk || k % bk != 0) return ORC_EINVAL; /* G12 */
    if (causal && Tq > Tk) return ORC_EINVAL;                          /* G7  */
    return ORC_OK;
}

/* Number of visible key blocks B_q of query block q (a1; causal reading G7:
 * query row t sits at key position t + Tk - Tq, a block is visible if it starts at or before the
 * position of the block's last row). */
static int64_t visible_blocks(int64_t q, int bq, int bk, int Tq, int Tk, int causal)
{
    int64_t nkb = ((int64_t)Tk + bk - 1) / bk;
    if (!causal) return nkb;
    int64_t tlast = imin64((q + 1) * (int64_t)bq, Tq) - 1;
    int64_t v = (tlast + (Tk - Tq)) / bk + 1;
    return imin64(v, nkb);
}

/* Branch score: max over the b_q x b_k tile of q_t . k_s for the representative
 * block j, restricted to valid pairs (s < Tk; causal: s <= t + Tk - Tq, reading G8).  No softmax
 * scale (G11).  `emax` (optional) receives max over the pairs of sum_c |q_c k_c|, used
 * to bound the rounding error of any fp32 evaluation order. */
static double block_score_c(const float *Qh, const float *Kh, int64_t t0, int64_t t1, int64_t j, int bk,
                            int Tq, int Tk, int d, int causal, int mode, const int *comp, int ncomp, int G,
                            int64_t hstride, double *emax);
static double block_score(const float *Qh, const float *Kh, int64_t t0, int64_t t1, int64_t j, int bk,
                          int Tq, int Tk, int d, int causal, int mode, double *emax)
{
    return block_score_c(Qh, Kh, t0, t1, j, bk, Tq, Tk, d, causal, mode, NULL, d, 1, 0, emax);
}

/* The same over the component list comp[0..ncomp) (top-r: sum_{l=1..r} q_{p_l} k_{p_l}, in
 * ascending component order; comp = NULL: c = 0..d-1), and over the query rows of G heads
 * (GQA-shared mask, reading G25: head g's rows start at Qh + g * hstride; G = 1: one head). */
static double block_score_c(const float *Qh, const float *Kh, int64_t t0, int64_t t1, int64_t j, int bk,
                            int Tq, int Tk, int d, int causal, int mode, const int *comp, int ncomp, int G,
                            int64_t hstride, double *emax)
{
    int64_t delta = (int64_t)Tk - Tq;
    int64_t s0 = j * bk, s1 = imin64((j + 1) * (int64_t)bk, Tk);
    double best = -INFINITY, e_best = 0.0;
    for (int64_t gt = 0; gt < (int64_t)G * (t1 - t0); ++gt) {
        int64_t t = t0 + gt % (t1 - t0); /* row t of head gt / (t1 - t0) of the group */
        const float *q = Qh + (gt / (t1 - t0)) * hstride + t * d;
        for (int64_t s = s0; s < s1; ++s) {
            if (causal && s > t + delta) continue;
            const float *kk = Kh + s * d;
            double v, e = 0.0;
            if (mode == ORC_F32C) {
                float acc = 0.0f;
                for (int i = 0; i < ncomp; ++i) {
                    int c = comp ? comp[i] : i;
                    acc = fmaf(q[c], kk[c], acc);
                }
                v = (double)acc;
                for (int i = 0; i < ncomp; ++i) {
                    int c = comp ? comp[i] : i;
                    e += fabs((double)q[c] * (double)kk[c]);
                }
            } else if (mode == ORC_F32L) {
                /* reading G9b: 16 segments of d/16 consecutive components, each a sequential fmaf
                 * chain (over the segment's selected components), combined by the pairwise tree
                 * v[l] <- v[l] + v[l ^ o], o = 8, 4, 2, 1 */
                float seg[16], nxt[16];
                int w = d / 16;
                for (int l = 0; l < 16; ++l) seg[l] = 0.0f;
                for (int i = 0; i < ncomp; ++i) {
                    int c = comp ? comp[i] : i;
                    seg[c / w] = fmaf(q[c], kk[c], seg[c / w]);
                }
                for (int o = 8; o >= 1; o >>= 1) {
                    for (int l = 0; l < 16; ++l) nxt[l] = seg[l] + seg[l ^ o];
                    for (int l = 0; l < 16; ++l) seg[l] = nxt[l];
                }
                v = (double)seg[0];
                for (int i = 0; i < ncomp; ++i) {
                    int c = comp ? comp[i] : i;
                    e += fabs((double)q[c] * (double)kk[c]);
                }
            } else {
                double acc = 0.0;
                for (int i = 0; i < ncomp; ++i) {
                    int c = comp ? comp[i] : i;
                    double p = (double)q[c] * (double)kk[c]; /* exact: 24+24 bit mantissas */
                    acc += p;
                    e += fabs(p);
                }
                v = acc;
            }
            if (v > best) best = v;
            if (e > e_best) e_best = e;
        }
    }
    if (emax) *emax = e_best;
    return best;
}

/* Ranking of branches: larger score first; equal scores -> smaller first block (G10). */
static int node_cmp(const void *pa, const void *pb)
{
    const orc_node *a = (const orc_node *)pa, *b = (const orc_node *)pb;
    if (a->s > b->s) return -1;
    if (a->s < b->s) return 1;
    if (a->f < b->f) return -1;
    if (a->f > b->f) return 1;
    return 0;
}

static int i64_cmp(const void *pa, const void *pb)
{
    int64_t a = *(const int64_t *)pa, b = *(const int64_t *)pb;
    return (a > b) - (a < b);
}

/* Per-unit diagnostics (all optional). */
typedef struct {
    double margin_min;   /* min over iterations of score(C[n-1]) - score(C[n]) (selection gap)   */
    double emax;         /* max over all scored pairs of sum_c |q_c k_c|                          */
    int64_t n_scored;    /* distinct representative blocks scored (PIN-7 counter)                 */
    int32_t n_iter;      /* iterations run                                                        */
} orc_diag;

/*
 * Alg. 1 for ONE query block, followed exactly:
 *   line 4   initial nodes: n = k/b_k equal ranges over the visible blocks [0, B_q) (G1, G2),
 *            f_j = round_half_up(j*B_q/n) = floor((2 j B_q + n) / (2n)) (G3), l_j = f_{j+1} - 1;
 *   line 7-8 split every node at m = round_half_up((f+l)/2) = floor((f+l+1)/2) into (f, m-1) and
 *            (m, l); a one-block node passes through unchanged (G5);
 *   line 10-13 score each branch by its first block (G4) with the tile max;
 *   line 14-15 keep the n best branches (G10 tie rule);
 *   repeat until every node is a single block (G6); line 17: I = first blocks, ascending.
 * Exact case (G1): B_q <= n selects every visible block.
 * trace_nodes (optional) receives the node ranges after every iteration: [max_trace+1][n][2]
 * (row 0 = initial partition); trace_scores [max_trace][n] the kept scores.
 */
/* Alg. 1 lines 4-17 over the key blocks [lo, lo + L) with n nodes (L > n): initial nodes
 * f_j = lo + floor((2 j L + n) / (2 n)), split / score / keep the n best until all are single
 * blocks; writes the n selected blocks ascending to out_idx.  memo is indexed by absolute block. */
static int search_range(const float *Qh, const float *Kh, int Tq, int Tk, int d, int64_t t0, int64_t t1,
                        int64_t lo, int64_t L, int n, int bk, int causal, int mode, double *memo,
                        int32_t *out_idx, orc_diag *dg, int32_t *trace_nodes, double *trace_scores,
                        int max_trace, const orc_ext *ex)
{
    int it = 0; /* iteration of this search (0 = first split), keys the ensemble jitter */
    orc_node *nodes = (orc_node *)malloc(sizeof(orc_node) * (size_t)n);
    orc_node *cand = (orc_node *)malloc(sizeof(orc_node) * 2 * (size_t)n);
    int64_t *firsts = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    if (!nodes || !cand || !firsts) {
        free(nodes); free(cand); free(firsts);
        return ORC_ENOMEM;
    }
    for (int j = 0; j < n; ++j) {
        int64_t fj = lo + (2 * (int64_t)j * L + n) / (2 * (int64_t)n);
        int64_t fj1 = lo + (2 * (int64_t)(j + 1) * L + n) / (2 * (int64_t)n);
        nodes[j].f = fj;
        nodes[j].l = fj1 - 1;
        nodes[j].s = NAN;
    }
    if (trace_nodes)
        for (int j = 0; j < n; ++j) {
            trace_nodes[2 * j] = (int32_t)nodes[j].f;
            trace_nodes[2 * j + 1] = (int32_t)nodes[j].l;
        }

    for (;;) {
        int any_split = 0;
        for (int j = 0; j < n; ++j) any_split |= nodes[j].l > nodes[j].f;
        if (!any_split) break;

        int nc = 0;
        for (int j = 0; j < n; ++j) {
            int64_t f = nodes[j].f, l = nodes[j].l;
            if (l == f) {
                cand[nc].f = f; cand[nc].l = f; ++nc;
            } else {
                int64_t m = (f + l + 1) / 2;
                if (ex->R > 0) { /* ensemble: split "around the center" (G23) */
                    m += orc_jitter(ex->key, it, f, ex->R);
                    if (m < f + 1) m = f + 1;
                    if (m > l) m = l;
                }
                cand[nc].f = f; cand[nc].l = m - 1; ++nc;
                cand[nc].f = m; cand[nc].l = l; ++nc;
            }
        }
        for (int c = 0; c < nc; ++c) {
            int64_t r = cand[c].f; /* representative = first block of the branch */
            if (isnan(memo[r])) {
                if (ex->replay) { /* replay: every score must have been supplied */
                    free(nodes); free(cand); free(firsts);
                    return ORC_EREPLAY;
                }
                double e = 0.0;
                memo[r] = block_score_c(Qh, Kh, t0, t1, r, bk, Tq, Tk, d, causal, mode, ex->comp, ex->ncomp, ex->G,
                                        ex->hstride, &e);
                if (e > dg->emax) dg->emax = e;
                dg->n_scored++;
            }
            cand[c].s = memo[r];
        }
        qsort(cand, (size_t)nc, sizeof(orc_node), node_cmp);
        if (nc > n) {
            double gap = cand[n - 1].s - cand[n].s;
            if (gap < dg->margin_min) dg->margin_min = gap;
        }
        memcpy(nodes, cand, sizeof(orc_node) * (size_t)n);
        if (trace_nodes && dg->n_iter < max_trace) {
            int32_t *tn = trace_nodes + (size_t)(dg->n_iter + 1) * 2 * n;
            for (int j = 0; j < n; ++j) {
                tn[2 * j] = (int32_t)nodes[j].f;
                tn[2 * j + 1] = (int32_t)nodes[j].l;
                if (trace_scores) trace_scores[(size_t)dg->n_iter * n + j] = nodes[j].s;
            }
        }
        dg->n_iter++;
        it++;
    }

    for (int j = 0; j < n; ++j) firsts[j] = nodes[j].f;
    qsort(firsts, (size_t)n, sizeof(int64_t), i64_cmp);
    for (int j = 0; j < n; ++j) out_idx[j] = (int32_t)firsts[j];
    free(nodes); free(cand); free(firsts);
    return ORC_OK;
}

/* One query block.  chunks = S >= 1 (stridden partial top-k; reading G21): when
 * B_q > n the visible blocks are split into S contiguous chunks [a_s, a_{s+1}),
 * a_s = floor((2 s B_q + S) / (2 S)), and Alg. 1 runs on each with n / S nodes; the chunks' selections
 * are concatenated (ascending).  S = 1 is Alg. 1 itself. */
static int mask_unit_chunked(const float *Qh, const float *Kh, int Tq, int Tk, int d, int64_t q, int n, int bq,
                             int bk, int causal, int mode, int chunks, int32_t *out_idx, int32_t *out_cnt,
                             orc_diag *diag, int32_t *trace_nodes, double *trace_scores, int max_trace,
                             int top_r, int R, uint64_t seed, int64_t lin, int G)
{
    int64_t Bq = visible_blocks(q, bq, bk, Tq, Tk, causal);
    int64_t t0 = q * (int64_t)bq, t1 = imin64(t0 + bq, Tq);
    orc_diag dg = {INFINITY, 0.0, 0, 0};
    if (mode == ORC_F32L && d % 16) return ORC_EINVAL;
    if (chunks < 1 || n % chunks) return ORC_EINVAL;

    if (Bq <= n) { /* exact case */
        for (int64_t j = 0; j < n; ++j) out_idx[j] = j < Bq ? (int32_t)j : -1;
        *out_cnt = (int32_t)Bq;
        if (diag) *diag = dg;
        return ORC_OK;
    }

    double *memo = (double *)malloc(sizeof(double) * (size_t)Bq);
    if (!memo) return ORC_ENOMEM;
    int comp[1024];
    orc_ext ex = {NULL, d, R > 0 ? R : 0, 0, G, (int64_t)Tq * d, 0};
    if (top_r > 0 && top_r < d) { /* top-r approximation */
        if (d > 1024) { free(memo); return ORC_EINVAL; }
        top_r_components(Qh, t0, t1, G, (int64_t)Tq * d, d, top_r, comp);
        ex.comp = comp;
        ex.ncomp = top_r;
    }
    if (ex.R > 0) ex.key = orc_unit_key(seed, lin);
    for (int64_t j = 0; j < Bq; ++j) memo[j] = NAN;
    int ns = n / chunks, rc = ORC_OK;
    for (int c = 0; c < chunks && rc == ORC_OK; ++c) {
        int64_t a0 = (2 * (int64_t)c * Bq + chunks) / (2 * (int64_t)chunks);
        int64_t a1 = (2 * (int64_t)(c + 1) * Bq + chunks) / (2 * (int64_t)chunks);
        rc = search_range(Qh, Kh, Tq, Tk, d, t0, t1, a0, a1 - a0, ns, bk, causal, mode, memo, out_idx + c * ns,
                          &dg, chunks == 1 ? trace_nodes : NULL, trace_scores, max_trace, &ex);
    }
    *out_cnt = n;
    if (diag) *diag = dg;
    free(memo);
    return rc;
}

static int mask_unit(const float *Qh, const float *Kh, int Tq, int Tk, int d, int64_t q, int n, int bq,
                     int bk, int causal, int mode, int32_t *out_idx, int32_t *out_cnt, orc_diag *diag,
                     int32_t *trace_nodes, double *trace_scores, int max_trace)
{
    return mask_unit_chunked(Qh, Kh, Tq, Tk, d, q, n, bq, bk, causal, mode, 1, out_idx, out_cnt, diag,
                             trace_nodes, trace_scores, max_trace, 0, 0, 0, 0, 1);
}

/* Replay (test infrastructure): Alg. 1's split / rank / keep steps (search_range,
 * unchanged) driven by SUPPLIED branch scores instead of computed ones — scores[u][j] is the score of
 * key block j for the u-th listed query block q_of_unit[u] (NaN = not supplied; asking for one is
 * ORC_EREPLAY).  Fed the GPU's own fp32 scores, it checks the GPU's splitting, inheritance, top-n and
 * tie rule independently of how the scores were rounded.  Plain Alg. 1 only (no chunks / options).
 * trace_nodes (optional, [nunits][max_trace + 1][n][2]) receives every unit's node ranges per
 * iteration (row 0 = initial partition), as oracle_mask_trace does. */
int oracle_mask_replay(int Tq, int Tk, int k, int bq, int bk, int causal, int64_t nunits, const int64_t *q_of_unit,
                       const float *scores, int64_t nkb, int32_t *idx, int32_t *cnt, int32_t *trace_nodes,
                       int max_trace)
{
    if (Tq < 1 || Tk < 1 || bq < 1 || bk < 1 || k < bk || k % bk || (causal && Tq > Tk)) return ORC_EINVAL;
    int n = k / bk;
    int64_t nqb = ((int64_t)Tq + bq - 1) / bq;
    int err = ORC_OK;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t u = 0; u < nunits; ++u) {
        int64_t q = q_of_unit[u];
        int r = ORC_OK;
        if (q < 0 || q >= nqb) {
            r = ORC_ERANGE;
        } else {
            int64_t Bq = visible_blocks(q, bq, bk, Tq, Tk, causal);
            if (Bq > nkb) {
                r = ORC_ERANGE;
            } else if (Bq <= n) { /* exact case: no score involved */
                for (int64_t j = 0; j < n; ++j) idx[u * n + j] = j < Bq ? (int32_t)j : -1;
                cnt[u] = (int32_t)Bq;
            } else {
                double *memo = (double *)malloc(sizeof(double) * (size_t)Bq);
                if (!memo) {
                    r = ORC_ENOMEM;
                } else {
                    for (int64_t j = 0; j < Bq; ++j) memo[j] = (double)scores[u * nkb + j];
                    orc_ext ex = {NULL, 0, 0, 0, 1, 0, 1};
                    orc_diag dg = {INFINITY, 0.0, 0, 0};
                    int32_t *tn = trace_nodes ? trace_nodes + (size_t)u * (size_t)(max_trace + 1) * 2 * n : NULL;
                    r = search_range(NULL, NULL, Tq, Tk, 0, q * (int64_t)bq, imin64((q + 1) * (int64_t)bq, Tq), 0, Bq,
                                     n, bk, causal, ORC_F32C, memo, idx + u * n, &dg, tn, NULL, max_trace, &ex);
                    cnt[u] = (int32_t)n;
                    free(memo);
                }
            }
        }
        if (r) {
#pragma omp critical
            err = r;
        }
    }
    return err;
}

/* -------------------------------------------------------------------------------------------- */
/* Contiguous layout: Q [B, Hq, Tq, d], K/V [B, Hkv, Tk, d], all row-major float32.               */
/* idx [B, Hq, Nqb, n] int32 ascending, -1 padded; cnt [B, Hq, Nqb].                              */
/* Optional per-unit outputs (NULL to skip): margin_min, emax (double), n_scored (int64), n_iter. */
/* -------------------------------------------------------------------------------------------- */
int oracle_mask(const float *Q, const float *K, int B, int Hq, int Hkv, int Tq, int Tk, int d, int k,
                int bq, int bk, int causal, int mode, int32_t *idx, int32_t *cnt, double *margin_min,
                double *emax, int64_t *n_scored, int32_t *n_iter)
{
    int rc = check_dims(B, Hq, Hkv, Tq, Tk, d, k, bq, bk, causal);
    if (rc) return rc;
    int n = k / bk;
    int64_t nqb = ((int64_t)Tq + bq - 1) / bq;
    int64_t units = (int64_t)B * Hq * nqb;
    int err = ORC_OK;
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t u = 0; u < units; ++u) {
        int64_t q = u % nqb, bh = u / nqb;
        int64_t b = bh / Hq, h = bh % Hq, hk = h / (Hq / Hkv);
        const float *Qh = Q + ((b * Hq + h) * (int64_t)Tq) * d;
        const float *Kh = K + ((b * Hkv + hk) * (int64_t)Tk) * d;
        orc_diag dg;
        int r = mask_unit(Qh, Kh, Tq, Tk, d, q, n, bq, bk, causal, mode, idx + u * n, cnt + u, &dg, NULL,
                          NULL, 0);
        if (r) {
#pragma omp critical
            err = r;
        }
        if (margin_min) margin_min[u] = dg.margin_min;
        if (emax) emax[u] = dg.emax;
        if (n_scored) n_scored[u] = dg.n_scored;
        if (n_iter) n_iter[u] = dg.n_iter;
    }
    return err;
}

/* oracle_mask with stridden partial top-k over S = chunks contiguous chunks (G21). */
/* gqa_shared = 1 (reading G25): one mask per (b, kv head, query block), scored over the query rows
 * of all H_q / H_kv heads of the group; idx [B, Hkv, Nqb, n], cnt [B, Hkv, Nqb]. */
int oracle_mask_ext(const float *Q, const float *K, int B, int Hq, int Hkv, int Tq, int Tk, int d, int k,
                    int bq, int bk, int causal, int mode, int chunks, int top_r, int jitter, uint64_t seed,
                    int gqa_shared, int32_t *idx, int32_t *cnt, double *margin_min, double *emax)
{
    if (top_r < 0 || jitter < 0) return ORC_EINVAL;
    int rc = check_dims(B, Hq, Hkv, Tq, Tk, d, k, bq, bk, causal);
    if (rc) return rc;
    int n = k / bk;
    if (chunks < 1 || n % chunks) return ORC_EINVAL;
    int64_t nqb = ((int64_t)Tq + bq - 1) / bq;
    int G = gqa_shared ? Hq / Hkv : 1, Hm = gqa_shared ? Hkv : Hq; /* heads scored together, mask heads */
    int64_t units = (int64_t)B * Hm * nqb;
    int err = ORC_OK;
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t u = 0; u < units; ++u) {
        int64_t q = u % nqb, bh = u / nqb;
        int64_t b = bh / Hm, h = bh % Hm, hk = gqa_shared ? h : h / (Hq / Hkv);
        const float *Qh = Q + ((b * Hq + h * G) * (int64_t)Tq) * d; /* first query head of the group */
        const float *Kh = K + ((b * Hkv + hk) * (int64_t)Tk) * d;
        orc_diag dg;
        int r = mask_unit_chunked(Qh, Kh, Tq, Tk, d, q, n, bq, bk, causal, mode, chunks, idx + u * n, cnt + u,
                                  &dg, NULL, NULL, 0, top_r, jitter, seed, u, G);
        if (r) {
#pragma omp critical
            err = r;
        }
        if (margin_min) margin_min[u] = dg.margin_min;
        if (emax) emax[u] = dg.emax;
    }
    return err;
}

int oracle_mask_chunked(const float *Q, const float *K, int B, int Hq, int Hkv, int Tq, int Tk, int d, int k,
                        int bq, int bk, int causal, int mode, int chunks, int32_t *idx, int32_t *cnt,
                        double *margin_min, double *emax)
{
    return oracle_mask_ext(Q, K, B, Hq, Hkv, Tq, Tk, d, k, bq, bk, causal, mode, chunks, 0, 0, 0, 0, idx, cnt,
                           margin_min, emax);
}

/* Node trace of one unit (for the invariant pins, PIN-5).  trace_nodes: [(max_trace+1) * n * 2],
 * trace_scores: [max_trace * n]; *n_iter receives the iteration count. */
int oracle_mask_trace_ext(const float *Q, const float *K, int B, int Hq, int Hkv, int Tq, int Tk, int d, int k,
                          int bq, int bk, int causal, int mode, int b, int h, int q, int32_t *idx_out,
                          int32_t *cnt_out, int32_t *trace_nodes, double *trace_scores, int max_trace,
                          int32_t *n_iter, int64_t *n_scored, int top_r, int jitter, uint64_t seed)
{
    int rc = check_dims(B, Hq, Hkv, Tq, Tk, d, k, bq, bk, causal);
    if (rc) return rc;
    if (top_r < 0 || jitter < 0) return ORC_EINVAL;
    int hk = h / (Hq / Hkv);
    int64_t nqb = ((int64_t)Tq + bq - 1) / bq;
    const float *Qh = Q + (((int64_t)b * Hq + h) * (int64_t)Tq) * d;
    const float *Kh = K + (((int64_t)b * Hkv + hk) * (int64_t)Tk) * d;
    orc_diag dg;
    rc = mask_unit_chunked(Qh, Kh, Tq, Tk, d, q, k / bk, bq, bk, causal, mode, 1, idx_out, cnt_out, &dg,
                           trace_nodes, trace_scores, max_trace, top_r, jitter, seed,
                           ((int64_t)b * Hq + h) * nqb + q, 1);
    if (n_iter) *n_iter = dg.n_iter;
    if (n_scored) *n_scored = dg.n_scored;
    return rc;
}

int oracle_mask_trace(const float *Q, const float *K, int B, int Hq, int Hkv, int Tq, int Tk, int d, int k,
                      int bq, int bk, int causal, int mode, int b, int h, int q, int32_t *idx_out,
                      int32_t *cnt_out, int32_t *trace_nodes, double *trace_scores, int max_trace,
                      int32_t *n_iter, int64_t *n_scored)
{
    return oracle_mask_trace_ext(Q, K, B, Hq, Hkv, Tq, Tk, d, k, bq, bk, causal, mode, b, h, q, idx_out, cnt_out,
                                 trace_nodes, trace_scores, max_trace, n_iter, n_scored, 0, 0, 0);
}

/* argtop_r(|q|) of one query block (rows [0, nrows) of Qb [nrows, d]) -> out[r], ascending (G22). */
int oracle_top_r_components(const float *Qb, int nrows, int d, int r, int32_t *out)
{
    if (nrows < 1 || d < 1 || r < 1 || r > d) return ORC_EINVAL;
    int *tmp = (int *)malloc(sizeof(int) * (size_t)d);
    if (!tmp) return ORC_ENOMEM;
    top_r_components(Qb, 0, nrows, 1, 0, d, r, tmp);
    for (int i = 0; i < r; ++i) out[i] = tmp[i];
    free(tmp);
    return ORC_OK;
}

/* Split offset of the ensemble generator (for the generator pins). */
int64_t oracle_jitter(uint64_t seed, int64_t lin, int it, int64_t f, int R)
{
    return R > 0 ? orc_jitter(orc_unit_key(seed, lin), it, f, R) : 0;
}

/* -------------------------------------------------------------------------------------------- */
/* Ensemble vote: per unit, an index survives iff at least theta of the n_e sample   */
/* masks contain it; tau = 1 truncates the survivors to n, preferring more votes, then the smaller */
/* block (reading G24, SPEC vote ordering); the output is ascending, -1 padded to n_out.           */
/* idx [n_e][units][n_in] with cnt [n_e][units]; out_idx [units][n_out], out_cnt [units].          */
/* -------------------------------------------------------------------------------------------- */
typedef struct { int32_t j, v; } orc_vote;

static int vote_cmp(const void *pa, const void *pb) /* votes desc, block asc */
{
    const orc_vote *a = (const orc_vote *)pa, *b = (const orc_vote *)pb;
    if (a->v != b->v) return a->v > b->v ? -1 : 1;
    return (a->j > b->j) - (a->j < b->j);
}

static int i32_cmp(const void *pa, const void *pb)
{
    int32_t a = *(const int32_t *)pa, b = *(const int32_t *)pb;
    return (a > b) - (a < b);
}

int oracle_vote(int n_e, int64_t units, int n_in, const int32_t *idx, const int32_t *cnt, int theta, int tau,
                int n_out, int32_t *out_idx, int32_t *out_cnt)
{
    if (n_e < 1 || units < 0 || n_in < 1 || theta < 1 || theta > n_e || (tau != 0 && tau != 1) || n_out < 1)
        return ORC_EINVAL;
    if (!tau && n_out < n_e * n_in) return ORC_EINVAL;
    int err = ORC_OK;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t u = 0; u < units; ++u) {
        int32_t *all = (int32_t *)malloc(sizeof(int32_t) * (size_t)n_e * n_in);
        orc_vote *sv = (orc_vote *)malloc(sizeof(orc_vote) * (size_t)n_e * n_in);
        int m = 0, ns = 0, bad = 0;
        for (int e = 0; e < n_e; ++e) {
            int c = cnt[(int64_t)e * units + u];
            if (c < 0 || c > n_in) { bad = 1; break; }
            for (int i = 0; i < c; ++i) all[m++] = idx[((int64_t)e * units + u) * n_in + i];
        }
        if (!bad) {
            /* count the agreements per index: sort, then runs of equal values */
            qsort(all, (size_t)m, sizeof(int32_t), i32_cmp);
            for (int i = 0; i < m;) {
                int j = i;
                while (j < m && all[j] == all[i]) ++j;
                if (j - i >= theta) { sv[ns].j = all[i]; sv[ns].v = j - i; ++ns; }
                i = j;
            }
            if (tau && ns > n_in) { /* truncate by votes, then block (G24) */
                qsort(sv, (size_t)ns, sizeof(orc_vote), vote_cmp);
                ns = n_in;
            }
            if (ns > n_out) bad = 1;
        }
        if (bad) {
#pragma omp critical
            err = ORC_ERANGE;
        } else {
            for (int i = 0; i < ns; ++i) all[i] = sv[i].j;
            qsort(all, (size_t)ns, sizeof(int32_t), i32_cmp);
            for (int i = 0; i < n_out; ++i) out_idx[u * n_out + i] = i < ns ? all[i] : -1;
            out_cnt[u] = ns;
        }
        free(all);
        free(sv);
    }
    return err;
}

/* Exact block-level top-n (textbook top-k, at key-block granularity with the same tile
 * score and tie rule): used by PIN-2 and for mask recall. */
int oracle_exact_block_topn(const float *Q, const float *K, int B, int Hq, int Hkv, int Tq, int Tk, int d,
                            int k, int bq, int bk, int causal, int mode, int32_t *idx, int32_t *cnt)
{
    int rc = check_dims(B, Hq, Hkv, Tq, Tk, d, k, bq, bk, causal);
    if (rc) return rc;
    if (mode == ORC_F32L && d % 16) return ORC_EINVAL;
    int n = k / bk;
    int64_t nqb = ((int64_t)Tq + bq - 1) / bq;
    int64_t units = (int64_t)B * Hq * nqb;
    int err = ORC_OK;
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t u = 0; u < units; ++u) {
        int64_t q = u % nqb, bh = u / nqb;
        int64_t b = bh / Hq, h = bh % Hq, hk = h / (Hq / Hkv);
        const float *Qh = Q + ((b * Hq + h) * (int64_t)Tq) * d;
        const float *Kh = K + ((b * Hkv + hk) * (int64_t)Tk) * d;
        int64_t Bq = visible_blocks(q, bq, bk, Tq, Tk, causal);
        int64_t t0 = q * (int64_t)bq, t1 = imin64(t0 + bq, Tq);
        orc_node *all = (orc_node *)malloc(sizeof(orc_node) * (size_t)Bq);
        int64_t *firsts = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
        if (!all || !firsts) {
            free(all); free(firsts);
#pragma omp critical
            err = ORC_ENOMEM;
            continue;
        }
        for (int64_t j = 0; j < Bq; ++j) {
            all[j].f = all[j].l = j;
            all[j].s = block_score(Qh, Kh, t0, t1, j, bk, Tq, Tk, d, causal, mode, NULL);
        }
        qsort(all, (size_t)Bq, sizeof(orc_node), node_cmp);
        int64_t m = imin64(Bq, n);
        for (int64_t j = 0; j < m; ++j) firsts[j] = all[j].f;
        qsort(firsts, (size_t)m, sizeof(int64_t), i64_cmp);
        for (int64_t j = 0; j < n; ++j) idx[u * n + j] = j < m ? (int32_t)firsts[j] : -1;
        cnt[u] = (int32_t)m;
        free(all); free(firsts);
    }
    return err;
}

/* Representative-block scores for a list of (b, h, q, j) tuples (certification of near-ties):
 * scores[i] = tile max (mode), emax[i] = max_pairs sum_c |q_c k_c|. */
int oracle_block_scores(const float *Q, const float *K, int B, int Hq, int Hkv, int Tq, int Tk, int d,
                        int bq, int bk, int causal, int mode, const int32_t *tuples, int64_t m,
                        double *scores, double *emax)
{
    if (check_dims(B, Hq, Hkv, Tq, Tk, d, bk, bq, bk, causal)) return ORC_EINVAL;
    if (mode == ORC_F32L && d % 16) return ORC_EINVAL;
    int err = ORC_OK;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        int64_t b = tuples[4 * i], h = tuples[4 * i + 1], q = tuples[4 * i + 2], j = tuples[4 * i + 3];
        int64_t nkb = ((int64_t)Tk + bk - 1) / bk, nqb = ((int64_t)Tq + bq - 1) / bq;
        if (b < 0 || b >= B || h < 0 || h >= Hq || q < 0 || q >= nqb || j < 0 || j >= nkb) {
#pragma omp critical
            err = ORC_ERANGE;
            continue;
        }
        int64_t hk = h / (Hq / Hkv);
        const float *Qh = Q + ((b * Hq + h) * (int64_t)Tq) * d;
        const float *Kh = K + ((b * Hkv + hk) * (int64_t)Tk) * d;
        int64_t t0 = q * (int64_t)bq, t1 = imin64(t0 + bq, Tq);
        double e = 0.0;
        scores[i] = block_score(Qh, Kh, t0, t1, j, bk, Tq, Tk, d, causal, mode, &e);
        if (emax) emax[i] = e;
    }
    return err;
}

/* -------------------------------------------------------------------------------------------- */
/* Attention (Eq. 2-3), fp64.  Row t of query block q attends to the tokens of the     */
/* selected key blocks that are < Tk and (causal) <= t + Tk - Tq, visited in ascending order.     */
/* Softmax scale sm_scale (G11; <= 0 means 1/sqrt(d)).  Empty row: O = 0, lse = -inf (G13).       */
/* O [B, Hq, Tq, d] double, lse [B, Hq, Tq] double (optional).                                    */
/* -------------------------------------------------------------------------------------------- */
static void attend_row(const float *q, const float *Kh, const float *Vh, int Tk, int d, const int64_t *tok,
                       int64_t ntok, double sm_scale, double *o, double *lse)
{
    if (ntok == 0) {
        for (int c = 0; c < d; ++c) o[c] = 0.0;
        if (lse) *lse = -INFINITY;
        return;
    }
    double *x = (double *)malloc(sizeof(double) * (size_t)ntok);
    double M = -INFINITY;
    for (int64_t i = 0; i < ntok; ++i) {
        const float *kk = Kh + tok[i] * d;
        double acc = 0.0;
        for (int c = 0; c < d; ++c) acc += (double)q[c] * (double)kk[c];
        x[i] = sm_scale * acc;
        if (x[i] > M) M = x[i];
    }
    double Z = 0.0;
    for (int c = 0; c < d; ++c) o[c] = 0.0;
    for (int64_t i = 0; i < ntok; ++i) {
        double p = exp(x[i] - M);
        Z += p;
        const float *vv = Vh + tok[i] * d;
        for (int c = 0; c < d; ++c) o[c] += p * (double)vv[c];
    }
    for (int c = 0; c < d; ++c) o[c] /= Z;
    if (lse) *lse = M + log(Z);
    (void)Tk;
    free(x);
}

/* Shared driver: dense = 1 attends to every visible key; else the idx/cnt selection,  */
/* optionally united with StreamingLLM sink and sliding-window tokens ("local sliding window and    */
/* global sink attention are also added during block sparse flash attention"; the       */
/* EffectiveMask of S:285-301): row t at position p = t + Tk - Tq attends to                         */
/*     (selected block tokens) U [0, sink) U (p - window, p],  intersected with [0, Tk) and, if       */
/* causal, with s <= p; each token once (sorted, duplicates removed), visited in ascending order.    */
static int attention_impl(const float *Q, const float *K, const float *V, int B, int Hq, int Hkv, int Tq,
                          int Tk, int d, int n, int bq, int bk, int causal, double sm_scale,
                          const int32_t *idx, const int32_t *cnt, int dense, int sink, int window, double *O,
                          double *lse)
{
    if (sink < 0 || window < 0) return ORC_EINVAL;
    if (sm_scale <= 0.0) sm_scale = 1.0 / sqrt((double)d);
    int64_t nqb = ((int64_t)Tq + bq - 1) / bq;
    int64_t nkb = ((int64_t)Tk + bk - 1) / bk;
    int64_t delta = (int64_t)Tk - Tq;
    int64_t rows = (int64_t)B * Hq * Tq;
    int err = ORC_OK;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < rows; ++r) {
        int64_t t = r % Tq, bh = r / Tq;
        int64_t b = bh / Hq, h = bh % Hq, hk = h / (Hq / Hkv);
        int64_t q = t / bq, u = bh * nqb + q;
        const float *Kh = K + ((b * Hkv + hk) * (int64_t)Tk) * d;
        const float *Vh = V + ((b * Hkv + hk) * (int64_t)Tk) * d;
        int64_t cap = dense ? (int64_t)Tk : (int64_t)n * bk + sink + window;
        int64_t *tok = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
        int64_t ntok = 0;
        int bad = 0;
        if (dense) {
            for (int64_t s = 0; s < Tk; ++s)
                if (!causal || s <= t + delta) tok[ntok++] = s;
        } else {
            int32_t c = cnt[u];
            if (c < 0 || c > n) bad = 1;
            int64_t prev = -1;
            for (int32_t i = 0; !bad && i < c; ++i) {
                int64_t j = idx[u * n + i];
                if (j < 0 || j >= nkb || j <= prev) { bad = 1; break; } /* S:309 index out of range */
                prev = j;
                for (int64_t s = j * bk; s < imin64((j + 1) * (int64_t)bk, Tk); ++s)
                    if (!causal || s <= t + delta) tok[ntok++] = s;
            }
            if (!bad && (sink > 0 || window > 0)) {
                int64_t p = t + delta;
                for (int64_t s = 0; s < imin64(sink, Tk); ++s)
                    if (!causal || s <= p) tok[ntok++] = s;
                for (int64_t s = p - window + 1; s <= p; ++s)
                    if (s >= 0 && s < Tk) tok[ntok++] = s;
                qsort(tok, (size_t)ntok, sizeof(int64_t), i64_cmp);
                int64_t w = 0;
                for (int64_t i = 0; i < ntok; ++i)
                    if (w == 0 || tok[i] != tok[w - 1]) tok[w++] = tok[i];
                ntok = w;
            }
        }
        if (bad) {
#pragma omp critical
            err = ORC_ERANGE;
        } else {
            attend_row(Q + r * d, Kh, Vh, Tk, d, tok, ntok, sm_scale, O + r * d, lse ? lse + r : NULL);
        }
        free(tok);
    }
    return err;
}

int oracle_sparse_attention(const float *Q, const float *K, const float *V, int B, int Hq, int Hkv, int Tq,
                            int Tk, int d, int k, int bq, int bk, int causal, double sm_scale,
                            const int32_t *idx, const int32_t *cnt, double *O, double *lse)
{
    int rc = check_dims(B, Hq, Hkv, Tq, Tk, d, k, bq, bk, causal);
    if (rc) return rc;
    return attention_impl(Q, K, V, B, Hq, Hkv, Tq, Tk, d, k / bk, bq, bk, causal, sm_scale, idx, cnt, 0, 0, 0,
                          O, lse);
}

/* The same with sink and sliding-window tokens. */
int oracle_sparse_attention_sw(const float *Q, const float *K, const float *V, int B, int Hq, int Hkv, int Tq,
                               int Tk, int d, int k, int bq, int bk, int causal, double sm_scale,
                               const int32_t *idx, const int32_t *cnt, int sink, int window, double *O,
                               double *lse)
{
    int rc = check_dims(B, Hq, Hkv, Tq, Tk, d, k, bq, bk, causal);
    if (rc) return rc;
    return attention_impl(Q, K, V, B, Hq, Hkv, Tq, Tk, d, k / bk, bq, bk, causal, sm_scale, idx, cnt, 0, sink,
                          window, O, lse);
}

int oracle_dense_attention(const float *Q, const float *K, const float *V, int B, int Hq, int Hkv, int Tq,
                           int Tk, int d, int causal, double sm_scale, double *O, double *lse)
{
    int rc = check_dims(B, Hq, Hkv, Tq, Tk, d, 1, 1, 1, causal);
    if (rc) return rc;
    return attention_impl(Q, K, V, B, Hq, Hkv, Tq, Tk, d, 1, 1, 1, causal, sm_scale, NULL, NULL, 1, 0, 0, O,
                          lse);
}

/* -------------------------------------------------------------------------------------------- */
/* Paged KV cache (decode).  pages: [num_pages, Hkv, page_size, d] float32 row-major.       */
/* Sequence b has Tk = seq_lens[b] tokens; token s is at page block_table[b*max_pages + s/ps],     */
/* slot s % ps.  Q [B, Hq, Tq, d] with the same Tq for every sequence (Tq = 1 for plain decode).   */
/* The oracle gathers each (b, kv-head) into a contiguous [Tk, d] buffer with plain loops and runs  */
/* the contiguous routines on it.                                                                  */
/* -------------------------------------------------------------------------------------------- */
static float *gather_paged(const float *pages, int num_pages, int Hkv, int ps, int d,
                           const int32_t *block_table, int max_pages, int b, int hk, int Tk, int *err)
{
    float *out = (float *)malloc(sizeof(float) * (size_t)Tk * d);
    if (!out) { *err = ORC_ENOMEM; return NULL; }
    for (int64_t s = 0; s < Tk; ++s) {
        int64_t pi = s / ps;
        if (pi >= max_pages) { *err = ORC_ERANGE; free(out); return NULL; }
        int64_t page = block_table[(int64_t)b * max_pages + pi];
        if (page < 0 || page >= num_pages) { *err = ORC_ERANGE; free(out); return NULL; }
        const float *src = pages + (((page * Hkv + hk) * (int64_t)ps) + s % ps) * d;
        memcpy(out + s * d, src, sizeof(float) * (size_t)d);
    }
    return out;
}

int oracle_mask_paged_ext(const float *Q, const float *Kpages, int num_pages, int page_size,
                      const int32_t *block_table, int max_pages, const int32_t *seq_lens, int B, int Hq,
                      int Hkv, int Tq, int d, int k, int bq, int bk, int causal, int mode, int32_t *idx,
                      int32_t *cnt, double *margin_min, double *emax, int64_t *n_scored, int32_t *n_iter,
                          int chunks, int top_r, int jitter, uint64_t seed, int gqa_shared)
{
    if (top_r < 0 || jitter < 0 || chunks < 1 || bk < 1 || (k / bk) % chunks) return ORC_EINVAL;
    if (page_size < 1 || page_size % bk != 0 || num_pages < 1) return ORC_EINVAL;
    int n = k / bk;
    int64_t nqb = ((int64_t)Tq + bq - 1) / bq;
    int err = ORC_OK;
    for (int b = 0; b < B && !err; ++b) {
        int Tk = seq_lens[b];
        int rc = check_dims(1, Hq, Hkv, Tq, Tk, d, k, bq, bk, causal);
        if (rc) return rc;
        for (int hk = 0; hk < Hkv && !err; ++hk) {
            float *Kh = gather_paged(Kpages, num_pages, Hkv, page_size, d, block_table, max_pages, b, hk, Tk,
                                     &err);
            if (!Kh) break;
            int g = Hq / Hkv;
            int gm = gqa_shared ? 1 : g; /* masks of this kv head: one shared (G25) or one per q head */
#pragma omp parallel for schedule(dynamic, 1)
            for (int64_t w = 0; w < (int64_t)gm * nqb; ++w) {
                int64_t h = (int64_t)hk * gm + w / nqb, q = w % nqb; /* mask head */
                int64_t u = ((int64_t)b * (gqa_shared ? Hkv : Hq) + h) * nqb + q;
                const float *Qh = Q + (((int64_t)b * Hq + (gqa_shared ? h * g : h)) * (int64_t)Tq) * d;
                orc_diag dg;
                int r = mask_unit_chunked(Qh, Kh, Tq, Tk, d, q, n, bq, bk, causal, mode, chunks, idx + u * n,
                                          cnt + u, &dg, NULL, NULL, 0, top_r, jitter, seed, u,
                                          gqa_shared ? g : 1);
                if (r) {
#pragma omp critical
                    err = r;
                }
                if (margin_min) margin_min[u] = dg.margin_min;
                if (emax) emax[u] = dg.emax;
                if (n_scored) n_scored[u] = dg.n_scored;
                if (n_iter) n_iter[u] = dg.n_iter;
            }
            free(Kh);
        }
    }
    return err;
}

int oracle_mask_paged(const float *Q, const float *Kpages, int num_pages, int page_size,
                      const int32_t *block_table, int max_pages, const int32_t *seq_lens, int B, int Hq,
                      int Hkv, int Tq, int d, int k, int bq, int bk, int causal, int mode, int32_t *idx,
                      int32_t *cnt, double *margin_min, double *emax, int64_t *n_scored, int32_t *n_iter)
{
    return oracle_mask_paged_ext(Q, Kpages, num_pages, page_size, block_table, max_pages, seq_lens, B, Hq, Hkv, Tq,
                                 d, k, bq, bk, causal, mode, idx, cnt, margin_min, emax, n_scored, n_iter, 1, 0, 0,
                                 0, 0);
}

int oracle_sparse_attention_paged_sw(const float *Q, const float *Kpages, const float *Vpages, int num_pages,
                                     int page_size, const int32_t *block_table, int max_pages,
                                     const int32_t *seq_lens, int B, int Hq, int Hkv, int Tq, int d, int k,
                                     int bq, int bk, int causal, double sm_scale, const int32_t *idx,
                                     const int32_t *cnt, int sink, int window, double *O, double *lse)
{
    if (page_size < 1 || page_size % bk != 0 || num_pages < 1) return ORC_EINVAL;
    int n = k / bk;
    int64_t nqb = ((int64_t)Tq + bq - 1) / bq;
    int err = ORC_OK;
    for (int b = 0; b < B && !err; ++b) {
        int Tk = seq_lens[b];
        int rc = check_dims(1, Hq, Hkv, Tq, Tk, d, k, bq, bk, causal);
        if (rc) return rc;
        for (int hk = 0; hk < Hkv && !err; ++hk) {
            float *Kh = gather_paged(Kpages, num_pages, Hkv, page_size, d, block_table, max_pages, b, hk, Tk,
                                     &err);
            if (!Kh) break;
            float *Vh = gather_paged(Vpages, num_pages, Hkv, page_size, d, block_table, max_pages, b, hk, Tk,
                                     &err);
            if (!Vh) { free(Kh); break; }
            int g = Hq / Hkv;
            for (int hh = 0; hh < g && !err; ++hh) {
                int64_t h = (int64_t)hk * g + hh;
                int64_t off = ((int64_t)b * Hq + h);
                /* one (b, h) slice as a B=Hq=Hkv=1 problem */
                rc = attention_impl(Q + off * Tq * d, Kh, Vh, 1, 1, 1, Tq, Tk, d, n, bq, bk, causal, sm_scale,
                                    idx + off * nqb * n, cnt + off * nqb, 0, sink, window, O + off * Tq * d,
                                    lse ? lse + off * Tq : NULL);
                if (rc) err = rc;
            }
            free(Kh);
            free(Vh);
        }
    }
    return err;
}

int oracle_sparse_attention_paged(const float *Q, const float *Kpages, const float *Vpages, int num_pages,
                                  int page_size, const int32_t *block_table, int max_pages,
                                  const int32_t *seq_lens, int B, int Hq, int Hkv, int Tq, int d, int k, int bq,
                                  int bk, int causal, double sm_scale, const int32_t *idx, const int32_t *cnt,
                                  double *O, double *lse)
{
    return oracle_sparse_attention_paged_sw(Q, Kpages, Vpages, num_pages, page_size, block_table, max_pages,
                                            seq_lens, B, Hq, Hkv, Tq, d, k, bq, bk, causal, sm_scale, idx, cnt, 0,
                                            0, O, lse);
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int t)
{
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}
