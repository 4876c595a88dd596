"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each test names the pin and the passage it follows.  Library routines used as
independent references: torch SDPA (fp64) for dense attention, numpy matmul + sort for brute-force
top-n.  Integer-valued inputs make every score exact, so ties and tie-breaks are tested bit-exactly.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

from paper_2406_09827_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")


def _qk_from_scores(scores):
    """q = (1, 0), key s = (score_s, 0): q . k_s = score_s exactly."""
    T = len(scores)
    Q = np.zeros((1, 1, 1, 2), np.float32)
    Q[..., 0] = 1.0
    K = np.zeros((1, 1, T, 2), np.float32)
    K[0, 0, :, 0] = np.asarray(scores, np.float32)
    return Q, K


def _brute_block_scores(Q, K, bq, bk, causal):
    """[B,Hq,Nqb,Nkb] tile maxima by full matmul (library primitive) + masking; -inf = invisible."""
    Q = np.asarray(Q, np.float64)
    K = np.asarray(K, np.float64)
    B, Hq, Tq, d = Q.shape
    Hkv, Tk = K.shape[1], K.shape[2]
    g = Hq // Hkv
    nqb, nkb = -(-Tq // bq), -(-Tk // bk)
    out = np.full((B, Hq, nqb, nkb), -np.inf)
    t = np.arange(Tq)[:, None]
    s = np.arange(Tk)[None, :]
    valid = (s <= t + (Tk - Tq)) if causal else np.ones((Tq, Tk), bool)
    for b in range(B):
        for h in range(Hq):
            S = Q[b, h] @ K[b, h // g].T
            S = np.where(valid, S, -np.inf)
            for q in range(nqb):
                rows = S[q * bq:(q + 1) * bq]
                for j in range(nkb):
                    out[b, h, q, j] = rows[:, j * bk:(j + 1) * bk].max()
    return out


def _visible(q, bq, bk, Tq, Tk, causal):
    nkb = -(-Tk // bk)
    if not causal:
        return nkb
    tlast = min((q + 1) * bq, Tq) - 1
    return min((tlast + Tk - Tq) // bk + 1, nkb)


def _topn_sorted(scores_row, n):
    """Exact top-n of a score vector, ties -> smaller index (np.lexsort), returned ascending."""
    idx = np.arange(len(scores_row))
    order = np.lexsort((idx, -scores_row))
    return np.sort(order[:n])


# --------------------------------------------------------------------------------------------
# PIN-4: worked examples (paper P:902-904)
# --------------------------------------------------------------------------------------------
def test_pin4_token_traces(orc):
    gold = json.load(open(GOLD))
    for case in gold["token_traces"]:
        Q, K = _qk_from_scores(case["scores"])
        idx, cnt = orc.mask(Q, K, case["k"], case["b_q"], case["b_k"], case["causal"], mode=orc.F32C)
        got = idx[0, 0, 0, : cnt[0, 0, 0]].tolist()
        assert got == case["expect"], case["name"]
        idx64, _ = orc.mask(Q, K, case["k"], case["b_q"], case["b_k"], case["causal"], mode=orc.F64)
        assert idx64[0, 0, 0, : cnt[0, 0, 0]].tolist() == case["expect"]
        if "exact_top" in case:  # the greedy miss really is a miss
            ex, ecnt = orc.exact_block_topn(Q, K, case["k"], case["b_q"], case["b_k"], case["causal"])
            assert ex[0, 0, 0, : ecnt[0, 0, 0]].tolist() == case["exact_top"]


def test_pin4_block_trace(orc):
    gold = json.load(open(GOLD))
    for case in gold["block_traces"]:
        T, bq, bk = case["T"], case["b_q"], case["b_k"]
        Q = np.zeros((1, 1, T, 2), np.float32)
        Q[..., 0] = 1.0
        K = np.zeros((1, 1, T, 2), np.float32)
        for j, m in enumerate(case["block_max"]):
            K[0, 0, j * bk, 0] = m
            K[0, 0, j * bk + 1, 0] = m - 0.5
        idx, cnt = orc.mask(Q, K, case["k"], bq, bk, case["causal"])
        for q in range(T // bq):
            assert idx[0, 0, q, : cnt[0, 0, q]].tolist() == case["expect"], case["name"]


def _split_observed(orc, node, favour_right):
    """Observe the branches of a node through the first iteration of a unit whose single node is
    `node` (n = 1) or, for the pass-through case, n = 2 over 3 blocks."""
    f, l = node
    if f == l:
        nblocks, k = 3, 2
    else:
        assert f == 0
        nblocks, k = l + 1, 1
    scores = np.full(nblocks, 0.0, np.float32)
    if f == l:
        scores[l] = 9.0
    else:
        m = (f + l + 1) // 2 if favour_right else f
        scores[m if favour_right else f] = 9.0
    Q, K = _qk_from_scores(scores)
    tr = orc.mask_trace(Q, K, k, 1, 1, False, 0, 0, 0)
    return [tuple(r) for r in tr["nodes"][1].tolist()]


def test_pin4_splits(orc):
    gold = json.load(open(GOLD))
    for case in gold["splits"]:
        node, br = case["node"], [tuple(b) for b in case["branches"]]
        if len(br) == 1:
            kept = _split_observed(orc, node, True)
            assert br[0] in kept, case["name"]
        else:
            assert _split_observed(orc, node, True) == [br[1]], case["name"]
            assert _split_observed(orc, node, False) == [br[0]], case["name"]
            # both branches non-empty and equal-sized up to one block
            (a0, a1), (b0, b1) = br
            assert a0 <= a1 and b0 <= b1 and abs((a1 - a0) - (b1 - b0)) <= 1


def test_pin4_paper_configuration(orc):
    """T=4k, k=512, b_q=32, b_k=2 -> initial groups of 8 blocks, final mask at iteration 3."""
    cfg = json.load(open(GOLD))["paper_configuration"]
    T = cfg["T"]
    Q, K, _ = synth.gen_qkv(1, 1, 1, T, T, 128, "iid", seed=3, dtype=torch.float32, make_v=False)
    last = T // cfg["b_q"] - 1
    tr = orc.mask_trace(Q, K, cfg["k"], cfg["b_q"], cfg["b_k"], cfg["causal"], 0, 0, last)
    sizes = tr["nodes"][0][:, 1] - tr["nodes"][0][:, 0] + 1
    assert (sizes == cfg["initial_node_blocks"]).all()
    assert tr["n_iter"] == cfg["last_query_block_iterations"]


# --------------------------------------------------------------------------------------------
# PIN-1: k >= T  =>  HiP == dense (causal) attention (Eq. 1-3 with M = all ones)
# --------------------------------------------------------------------------------------------
def _sdpa64(Q, K, V, causal, scale):
    Q, K, V = (torch.as_tensor(np.asarray(x, np.float32)).double() for x in (Q, K, V))
    Tq, Tk = Q.shape[2], K.shape[2]
    g = Q.shape[1] // K.shape[1]
    K = K.repeat_interleave(g, dim=1)
    V = V.repeat_interleave(g, dim=1)
    mask = None
    if causal:
        mask = torch.ones(Tq, Tk, dtype=torch.bool).tril(diagonal=Tk - Tq)
    return torch.nn.functional.scaled_dot_product_attention(Q, K, V, attn_mask=mask, scale=scale).numpy()


@pytest.mark.parametrize("Tq,Tk,Hq,Hkv,causal", [(256, 256, 2, 2, True), (96, 300, 4, 2, True),
                                                 (200, 200, 1, 1, False), (1, 333, 2, 1, True)])
def test_pin1_exact_case_is_dense(orc, Tq, Tk, Hq, Hkv, causal):
    d, k, bq, bk = 64, 512, 32, 2
    Q, K, V = synth.gen_qkv(1, Hq, Hkv, Tq, Tk, d, "iid", seed=11, dtype=torch.float32)
    idx, cnt = orc.mask(Q, K, k, bq, bk, causal)
    nqb = idx.shape[2]
    for q in range(nqb):
        vis = _visible(q, bq, bk, Tq, Tk, causal)
        assert (cnt[:, :, q] == vis).all()
        assert (idx[:, :, q, :vis] == np.arange(vis)).all() and (idx[:, :, q, vis:] == -1).all()
    O, lse = orc.sparse_attention(Q, K, V, k, bq, bk, causal, idx, cnt)
    Od, lsed = orc.dense_attention(Q, K, V, causal)
    assert np.array_equal(O, Od) and np.array_equal(lse, lsed)  # shared loop: bit-identical
    ref = _sdpa64(Q, K, V, causal, 1.0 / math.sqrt(d))
    assert np.abs(O - ref).max() < 1e-12


# --------------------------------------------------------------------------------------------
# PIN-2: n < B_q <= 2n  =>  one iteration, every visible block is a candidate once => the mask is
# the exact top-n of the block maxima (P:150-153 with the tile score of P:178-180).
# --------------------------------------------------------------------------------------------
@pytest.mark.parametrize("dist,mode", [("int", 0), ("int", 1), ("iid", 1)])
def test_pin2_one_level_is_exact_topn(orc, dist, mode):
    T, d, k, bq, bk = 1024, 32, 128, 16, 2  # n = 64; causal blocks with 64 < B_q <= 128: q in [8, 16)
    Q, K, _ = synth.gen_qkv(1, 2, 1, T, T, d, dist, seed=5, dtype=torch.float32, make_v=False)
    n = k // bk
    idx, cnt = orc.mask(Q, K, k, bq, bk, True, mode=mode)
    bs = _brute_block_scores(Q, K, bq, bk, True)
    checked = 0
    for h in range(2):
        for q in range(idx.shape[2]):
            vis = _visible(q, bq, bk, T, T, True)
            if not (n < vis <= 2 * n):
                continue
            want = _topn_sorted(bs[0, h, q, :vis], n)
            assert cnt[0, h, q] == n
            assert np.array_equal(idx[0, h, q], want), (h, q)
            checked += 1
    assert checked == 16
    # non-causal with N_kb in (n, 2n]
    Tk = 200
    Q2, K2, _ = synth.gen_qkv(1, 1, 1, 40, Tk, d, dist, seed=6, dtype=torch.float32, make_v=False)
    idx2, _ = orc.mask(Q2, K2, k, bq, bk, False, mode=mode)
    bs2 = _brute_block_scores(Q2, K2, bq, bk, False)
    for q in range(idx2.shape[2]):
        assert np.array_equal(idx2[0, 0, q], _topn_sorted(bs2[0, 0, q], n))


def test_pin2_exact_topn_routine(orc):
    """oracle_exact_block_topn (used for recall) against the brute-force sort at every query block."""
    T, d, k, bq, bk = 512, 16, 64, 8, 4
    Q, K, _ = synth.gen_qkv(1, 2, 2, T, T, d, "int", seed=9, dtype=torch.float32, make_v=False)
    idx, cnt = orc.exact_block_topn(Q, K, k, bq, bk, True)
    bs = _brute_block_scores(Q, K, bq, bk, True)
    n = k // bk
    for h in range(2):
        for q in range(idx.shape[2]):
            vis = _visible(q, bq, bk, T, T, True)
            want = _topn_sorted(bs[0, h, q, :vis], n)
            assert cnt[0, h, q] == len(want)
            assert np.array_equal(idx[0, h, q, : len(want)], want)


# --------------------------------------------------------------------------------------------
# PIN-3: strictly monotone block scores => greedy = exact top-n (last n / first n visible blocks)
# --------------------------------------------------------------------------------------------
@pytest.mark.parametrize("T,k,bq,bk", [(2048, 128, 32, 2), (1000, 64, 8, 1), (3000, 96, 16, 4), (777, 40, 4, 8)])
@pytest.mark.parametrize("sign", [1, -1])
def test_pin3_monotone(orc, T, k, bq, bk, sign):
    Q = np.zeros((1, 1, T, 4), np.float32)
    Q[..., 0] = 1.0
    K = np.zeros((1, 1, T, 4), np.float32)
    K[0, 0, :, 0] = sign * (np.arange(T, dtype=np.float32) / np.float32(T))
    n = k // bk
    for causal in (True, False):
        idx, cnt = orc.mask(Q, K, k, bq, bk, causal)
        for q in range(idx.shape[2]):
            vis = _visible(q, bq, bk, T, T, causal)
            m = min(n, vis)
            want = np.arange(vis - m, vis) if sign > 0 else np.arange(m)
            assert cnt[0, 0, q] == m
            assert np.array_equal(idx[0, 0, q, :m], want), (q, vis)


# --------------------------------------------------------------------------------------------
# PIN-5: invariants: per iteration n disjoint non-empty nodes nested in the previous
# ones and inside [0, B_q); final: min(n, B_q) distinct ascending blocks; leaf exactness.
# --------------------------------------------------------------------------------------------
@pytest.mark.parametrize("dist", ["iid", "int", "llm"])
def test_pin5_invariants(orc, dist):
    T, d, k, bq, bk = 3000, 32, 96, 16, 2
    Q, K, _ = synth.gen_qkv(1, 1, 1, T, T, d, dist, seed=21, dtype=torch.float32, make_v=False)
    n = k // bk
    nqb = -(-T // bq)
    for q in [0, 2, 3, 5, 6, 7, 50, 101, 150, nqb - 1]:
        vis = _visible(q, bq, bk, T, T, True)
        tr = orc.mask_trace(Q, K, k, bq, bk, True, 0, 0, q)
        final = tr["idx"][: tr["cnt"]]
        assert tr["cnt"] == min(n, vis)
        assert np.all(np.diff(final) > 0) and final.min() >= 0 and final.max() < vis
        if vis <= n:
            assert tr["n_iter"] == 0
            continue
        assert tr["n_iter"] == math.ceil(math.log2(math.ceil(vis / n))) or tr["n_iter"] < math.ceil(
            math.log2(math.ceil(vis / n))) + 1
        prev = None
        for it, nodes in enumerate(tr["nodes"]):
            f, l = nodes[:, 0], nodes[:, 1]
            assert len(nodes) == n and (f <= l).all() and f.min() >= 0 and l.max() < vis
            o = np.argsort(f)
            assert (f[o][1:] > l[o][:-1]).all()  # disjoint
            if it == 0:
                assert f[o][0] == 0 and l[o][-1] == vis - 1  # initial partition covers [0, B_q)
                sz = l - f + 1
                assert sz.max() - sz.min() <= 1          # "k equal-sized ranges"
            else:
                pf, pl = prev[:, 0], prev[:, 1]
                for a, b in zip(f, l):                   # nesting
                    assert ((pf <= a) & (b <= pl)).any()
            prev = nodes
        assert (tr["nodes"][-1][:, 0] == tr["nodes"][-1][:, 1]).all()  # leaves are single blocks
        # leaf exactness: the kept scores of the last iteration are the exact tile maxima
        last = tr["nodes"][-1]
        tuples = [(0, 0, q, int(j)) for j in last[:, 0]]
        sc, _ = orc.block_scores(Q, K, bq, bk, True, tuples, mode=orc.F32C)
        assert np.array_equal(sc, tr["scores"][-1])


def test_pin5_causal_budget(orc):
    """Row t_last of an aligned query block keeps exactly min(k, visible) tokens."""
    T, d, k, bq, bk = 2048, 16, 128, 32, 2
    Q, K, _ = synth.gen_qkv(1, 1, 1, T, T, d, "iid", seed=4, dtype=torch.float32, make_v=False)
    idx, cnt = orc.mask(Q, K, k, bq, bk, True)
    for q in range(idx.shape[2]):
        tlast = (q + 1) * bq - 1
        toks = [s for j in idx[0, 0, q, : cnt[0, 0, q]] for s in range(j * bk, (j + 1) * bk) if s <= tlast]
        assert len(toks) == min(k, tlast + 1)


# --------------------------------------------------------------------------------------------
# PIN-6: scale / permutation invariance
# --------------------------------------------------------------------------------------------
def test_pin6_power_of_two_scaling(orc):
    T, d = 1500, 64
    Q, K, _ = synth.gen_qkv(1, 2, 2, T, T, d, "llm", seed=8, dtype=torch.float32, make_v=False)
    base = orc.mask(Q, K, 64, 16, 2, True)[0]
    for j in (-3, 1, 5):
        Qs = Q * (2.0 ** j)
        for mode in (orc.F32C, orc.F64):
            assert np.array_equal(orc.mask(Qs, K, 64, 16, 2, True, mode=mode)[0],
                                  orc.mask(Q, K, 64, 16, 2, True, mode=mode)[0])
    assert base.shape[-1] == 32


def test_pin6_row_permutation_integer(orc):
    T, d, bq = 1024, 32, 16
    Q, K, _ = synth.gen_qkv(1, 1, 1, T, T, d, "int", seed=12, dtype=torch.float32, make_v=False)
    Qn = Q.numpy().copy()
    rng = np.random.default_rng(0)
    for q in range(T // bq):
        rows = np.arange(q * bq, (q + 1) * bq)
        Qn[0, 0, rows] = Qn[0, 0, rng.permutation(rows)]
    a = orc.mask(Q, K, 64, bq, 2, False)[0]
    b = orc.mask(Qn, K, 64, bq, 2, False)[0]
    assert np.array_equal(a, b)


# --------------------------------------------------------------------------------------------
# PIN-7: complexity counter: distinct representative blocks scored per query block
# = 2n + (n_it - 1) n when every node has the same power-of-two size, <= that bound otherwise.
# --------------------------------------------------------------------------------------------
def test_pin7_counter(orc):
    T, d, k, bq, bk = 8192, 16, 64, 16, 2
    n = k // bk
    Q, K, _ = synth.gen_qkv(1, 1, 1, T, T, d, "iid", seed=2, dtype=torch.float32, make_v=False)
    _, _, dg = orc.mask(Q, K, k, bq, bk, True, diag=True)
    exact = 0
    for q in range(T // bq):
        vis = _visible(q, bq, bk, T, T, True)
        ns, nit = int(dg["n_scored"][0, 0, q]), int(dg["n_iter"][0, 0, q])
        if vis <= n:
            assert ns == 0 and nit == 0
            continue
        full_it = math.ceil(math.log2(math.ceil(vis / n)))
        bound = 2 * n + (full_it - 1) * n
        ratio = vis / n
        if ratio == int(ratio) and (int(ratio) & (int(ratio) - 1)) == 0:
            assert nit == full_it and ns == bound
            exact += 1
        else:
            assert ns <= bound and nit <= full_it
    assert exact >= 5


# --------------------------------------------------------------------------------------------
# PIN-8: attention special cases
# --------------------------------------------------------------------------------------------
def test_pin8_attention_special_cases(orc):
    T, d, k, bq, bk = 64, 8, 16, 4, 2
    Q, K, V = synth.gen_qkv(1, 1, 1, T, T, d, "iid", seed=1, dtype=torch.float32)
    nqb, n = T // bq, k // bk
    # a single selected block whose first token is the only visible one for row 0 -> O = V[0]
    idx = np.full((1, 1, nqb, n), -1, np.int32)
    cnt = np.zeros((1, 1, nqb), np.int32)
    idx[0, 0, 0, 0] = 0
    cnt[0, 0, 0] = 1
    O, lse = orc.sparse_attention(Q, K, V, k, bq, bk, True, idx, cnt)
    assert np.array_equal(O[0, 0, 0], V[0, 0, 0].double().numpy())
    assert np.isfinite(lse[0, 0, 0])
    # empty rows -> zeros, -inf (G13)
    assert (O[0, 0, bq:] == 0).all() and np.isneginf(lse[0, 0, bq:]).all()
    # convexity: each output coordinate within [min, max] of the selected (visible) V rows
    rng = np.random.default_rng(3)
    for q in range(nqb):
        c = rng.integers(1, n + 1)
        sel = np.sort(rng.choice(nqb * bq // bk, size=c, replace=False))
        idx[0, 0, q] = -1
        idx[0, 0, q, :c] = sel
        cnt[0, 0, q] = c
    O, lse = orc.sparse_attention(Q, K, V, k, bq, bk, False, idx, cnt)
    Vn = V[0, 0].double().numpy()
    for t in range(T):
        q = t // bq
        toks = [s for j in idx[0, 0, q, : cnt[0, 0, q]] for s in range(j * bk, (j + 1) * bk)]
        lo, hi = Vn[toks].min(0), Vn[toks].max(0)
        assert (O[0, 0, t] >= lo - 1e-12).all() and (O[0, 0, t] <= hi + 1e-12).all()
    # out-of-range index is an error
    idx[0, 0, 0, 0] = 10_000
    with pytest.raises(ValueError):
        orc.sparse_attention(Q, K, V, k, bq, bk, False, idx, cnt)


def test_pin8_dense_vs_sdpa_gqa(orc):
    Q, K, V = synth.gen_qkv(2, 4, 2, 50, 70, 16, "llm", seed=7, dtype=torch.float32)
    for causal in (True, False):
        O, _ = orc.dense_attention(Q, K, V, causal, sm_scale=0.3)
        ref = _sdpa64(Q, K, V, causal, 0.3)
        assert np.abs(O - ref).max() < 1e-12


# --------------------------------------------------------------------------------------------
# Decode / paged: the paged routines see exactly the contiguous problem (reading G16)
# --------------------------------------------------------------------------------------------
def test_paged_equals_contiguous_and_bq_irrelevant(orc):
    B, Hq, Hkv, d, ps = 3, 4, 2, 32, 8
    seq = [700, 64, 1031]
    Tmax = max(seq)
    Q = synth.gen_decode_q(B, Hq, d, seed=1, dtype=torch.float32)
    _, K, V = synth.gen_qkv(B, Hkv, Hkv, 1, Tmax, d, "iid", seed=2, dtype=torch.float32)
    kp, vp, bt, sl = synth.to_paged(K, V, seq, ps, seed=2)
    k, bk = 128, 2
    idx_p, cnt_p = orc.mask_paged(Q, kp, bt, sl, k, 32, bk, True)
    idx_p1, _ = orc.mask_paged(Q, kp, bt, sl, k, 1, bk, True)
    assert np.array_equal(idx_p, idx_p1)
    O_p, lse_p = orc.sparse_attention_paged(Q, kp, vp, bt, sl, k, 1, bk, True, idx_p, cnt_p)
    for b in range(B):
        Tk = seq[b]
        idx_c, cnt_c = orc.mask(Q[b:b + 1], K[b:b + 1, :, :Tk], k, 1, bk, True)
        assert np.array_equal(idx_c, idx_p[b:b + 1]) and np.array_equal(cnt_c, cnt_p[b:b + 1])
        O_c, lse_c = orc.sparse_attention(Q[b:b + 1], K[b:b + 1, :, :Tk], V[b:b + 1, :, :Tk], k, 1, bk, True,
                                          idx_c, cnt_c)
        assert np.array_equal(O_c, O_p[b:b + 1]) and np.array_equal(lse_c, lse_p[b:b + 1])


def test_iteration_count_reading_g6(orc):
    """Any number of extra iterations is a no-op (G5/G6): the loop stops when all nodes are single
    blocks, and the mask of a query block whose nodes are already singletons never changes."""
    T, d = 4096, 32
    Q, K, _ = synth.gen_qkv(1, 1, 1, T, T, d, "iid", seed=31, dtype=torch.float32, make_v=False)
    _, _, dg = orc.mask(Q, K, 512, 32, 2, True, diag=True)
    vis = np.array([_visible(q, 32, 2, T, T, True) for q in range(T // 32)])
    need = np.array([0 if v <= 256 else math.ceil(math.log2(math.ceil(v / 256))) for v in vis])
    assert (dg["n_iter"][0, 0] <= need).all()
    assert (dg["n_iter"][0, 0][vis > 256] >= 1).all()


# --------------------------------------------------------------------------------------------
# F32L (reading G9b, the decode GEMV's fp32 order): exact on integer inputs, reduces to F32C when a
# single segment is non-zero, and stays within the fp32 error bound of the exact (fp64) score.
# --------------------------------------------------------------------------------------------
def test_f32l_mode_pins(orc):
    T, d, k, bq, bk = 1200, 128, 64, 1, 2
    Qi, Ki, _ = synth.gen_qkv(1, 2, 1, T, T, d, "int", seed=13, dtype=torch.float32, make_v=False)
    a = orc.mask(Qi, Ki, k, bq, bk, True, mode=orc.F32L)[0]
    b = orc.mask(Qi, Ki, k, bq, bk, True, mode=orc.F64)[0]
    assert np.array_equal(a, b)
    Q, K, _ = synth.gen_qkv(1, 1, 1, 64, 64, d, "iid", seed=14, dtype=torch.float32, make_v=False)
    Q1 = Q.clone()
    Q1[..., 8:] = 0  # only segment 0 (elements 0..7) contributes: F32L == F32C bit-for-bit
    tup = [(0, 0, q, j) for q in range(64) for j in range(0, 32, 3) if j <= q // 2]
    s_l, _ = orc.block_scores(Q1, K, 1, 2, True, tup, mode=orc.F32L)
    s_c, _ = orc.block_scores(Q1, K, 1, 2, True, tup, mode=orc.F32C)
    assert np.array_equal(s_l, s_c)
    s_l, em = orc.block_scores(Q, K, 1, 2, True, tup, mode=orc.F32L)
    s_64, _ = orc.block_scores(Q, K, 1, 2, True, tup, mode=orc.F64)
    gamma = (d // 16 + 4) * 2.0 ** -24 * 1.01
    assert (np.abs(s_l - s_64) <= gamma * em).all()
    with pytest.raises(ValueError):
        orc.mask(Q[..., :24], K[..., :24], k, bq, bk, True, mode=orc.F32L)


# --------------------------------------------------------------------------------------------
# Replay entry (C-2): the split / rank / keep steps on supplied scores.  Supplied the exact block
# maxima (computed here by brute force, independently of the oracle), it must give the oracle's own
# F64 mask; a missing score is an error; and in the one-level regime it is the exact top-n of the
# supplied scores (PIN-2 again, now for the replay path).
# --------------------------------------------------------------------------------------------
def _brute_block_max(Q, K, bq, bk, q):
    Qn, Kn = Q[0, 0].double().numpy(), K[0, 0].double().numpy()
    Tq, Tk = Qn.shape[0], Kn.shape[0]
    t0, t1 = q * bq, min((q + 1) * bq, Tq)
    S = Qn[t0:t1] @ Kn.T
    S[np.arange(t0, t1)[:, None] + (Tk - Tq) < np.arange(Tk)[None, :]] = -np.inf
    nkb = -(-Tk // bk)
    Sp = np.full((t1 - t0, nkb * bk), -np.inf)
    Sp[:, :Tk] = S
    return Sp.reshape(t1 - t0, nkb, bk).max(axis=(0, 2)).astype(np.float32)


def test_replay_reproduces_mask_from_supplied_scores(orc):
    Tq, Tk, d, k, bq, bk = 1000, 1200, 32, 64, 16, 2
    Q, K, _ = synth.gen_qkv(1, 1, 1, Tq, Tk, d, "int", seed=21, dtype=torch.float32, make_v=False)
    qs = [0, 3, 10, 30, 45, 50, 62]
    nkb = -(-Tk // bk)
    sc = np.stack([_brute_block_max(Q, K, bq, bk, q) for q in qs])  # integer inputs: exact in fp32
    ri, rc, tr = orc.mask_replay(Tq, Tk, k, bq, bk, True, qs, sc, trace=True)
    oi, oc = orc.mask(Q, K, k, bq, bk, True, mode=orc.F64)
    assert np.array_equal(ri, oi[0, 0, qs]) and np.array_equal(rc, oc[0, 0, qs])
    for u, q in enumerate(qs):  # the replay's per-iteration node sets are the oracle's own trace
        t = orc.mask_trace(Q, K, k, bq, bk, True, 0, 0, q, mode=orc.F64)
        assert len(tr[u]) == len(t["nodes"]) and all(np.array_equal(a, b) for a, b in zip(tr[u], t["nodes"]))
    # a score the search needs but nobody supplied: an error, not a silent choice
    holey = sc.copy()
    holey[-1, 0] = np.nan  # block 0 is always a first-iteration representative (f_0 = 0)
    with pytest.raises(ValueError):
        orc.mask_replay(Tq, Tk, k, bq, bk, True, qs, holey)
    # one-level regime (n < B_q <= 2n): the replayed mask is the exact top-n of the supplied scores
    n = k // bk
    rng = np.random.default_rng(2)
    for q in range(Tq // bq):
        Bq = min(((q + 1) * bq - 1 + Tk - Tq) // bk + 1, nkb)
        if not n < Bq <= 2 * n:
            continue
        s = rng.integers(-3, 4, size=(1, nkb)).astype(np.float32)  # many ties: tie rule matters
        ri, _ = orc.mask_replay(Tq, Tk, k, bq, bk, True, [q], s)
        order = np.lexsort((np.arange(Bq), -s[0, :Bq]))[:n]
        assert np.array_equal(ri[0], np.sort(order))


# --------------------------------------------------------------------------------------------
# F32C / F32L pinned by exact rational arithmetic: the two fp32 orders of
# readings G9 / G9b restated from their DEFINITIONS with fractions.Fraction — fmaf(a, b, c) is ONE
# rounding of the exact a*b + c to binary32 (round to nearest, ties to even), an fp32 add one
# rounding of the exact sum — and compared bit-for-bit with the oracle's C arithmetic on iid inputs
# (where every partial sum rounds).  A reversed tree or strided segments fail here.
# --------------------------------------------------------------------------------------------
from fractions import Fraction


def _round_f32(x: Fraction) -> Fraction:
    """Exact value of binary32 round-to-nearest-even of the rational x (normal and subnormal)."""
    if x == 0:
        return Fraction(0)
    sgn, a = (1, x) if x > 0 else (-1, -x)
    e = a.numerator.bit_length() - a.denominator.bit_length()  # 2^e <= a < 2^(e+2)
    if Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    q = Fraction(2) ** (max(e, -126) - 23)  # spacing of binary32 around a
    m = a / q
    fl = m.numerator // m.denominator
    rem = m - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    assert fl * q < Fraction(2) ** 128, "overflow"
    return sgn * fl * q


def _fmaf(a, b, c):
    return _round_f32(Fraction(a) * Fraction(b) + Fraction(c))


def _f32c_dot(q, k):
    acc = Fraction(0)
    for c in range(len(q)):
        acc = _fmaf(float(q[c]), float(k[c]), acc)
    return acc


def _f32l_dot(q, k):
    """G9b: 16 segments of d/16 consecutive components, each a sequential fmaf chain, then the
    pairwise tree v[l] <- v[l] + v[l xor o] for o = 8, 4, 2, 1 (all l at once), result v[0]."""
    d = len(q)
    w = d // 16
    seg = []
    for l in range(16):
        acc = Fraction(0)
        for c in range(l * w, (l + 1) * w):
            acc = _fmaf(float(q[c]), float(k[c]), acc)
        seg.append(acc)
    for o in (8, 4, 2, 1):
        seg = [_round_f32(seg[l] + seg[l ^ o]) for l in range(16)]
    return seg[0]


@pytest.mark.parametrize("mode_name", ["F32C", "F32L"])
def test_fp32_orders_pinned_by_exact_rationals(orc, mode_name):
    d, T = 128, 48
    Q, K, _ = synth.gen_qkv(1, 1, 1, T, T, d, "iid", seed=77, dtype=torch.float32, make_v=False)
    Q = Q * 3.0  # larger partial sums: more of them round
    qn, kn = Q[0, 0].numpy(), K[0, 0].numpy()
    mode = getattr(orc, mode_name)
    ref = _f32c_dot if mode_name == "F32C" else _f32l_dot
    # b_q = 1, b_k = 1: a tile is one (row, key) pair, so the oracle's block score IS one dot product
    tup = [(0, 0, t, s) for t in range(T) for s in range(0, t + 1, 5)]
    got, _ = orc.block_scores(Q, K, 1, 1, True, tup, mode=mode)
    want = np.array([float(ref(qn[t], kn[s])) for _, _, t, s in tup])
    assert np.array_equal(got, want), np.flatnonzero(got != want)[:10]
    # the two orders really differ on these inputs (the test can tell them apart)
    other = _f32l_dot if mode_name == "F32C" else _f32c_dot
    assert any(float(other(qn[t], kn[s])) != g for (_, _, t, s), g in zip(tup, got))


def test_round_f32_matches_numpy():
    rng = np.random.default_rng(5)
    for x in rng.standard_normal(2000) * 10.0 ** rng.integers(-40, 38, 2000):
        assert float(_round_f32(Fraction(float(x)))) == float(np.float32(x))
    for x in (1 + 2 ** -24, 1 + 3 * 2 ** -24, 2 ** -149 * 0.5, 2 ** -149 * 1.5, -(2 ** -126) * (1 - 2 ** -24)):
        assert float(_round_f32(Fraction(x))) == float(np.float32(x))


# --------------------------------------------------------------------------------------------
# Sink + sliding window (f1; "local sliding window and global sink attention are also
# added", sizes (128, 32); the EffectiveMask of S:285-301: per row the union of the selected block
# tokens, [0, sink) and (p - window, p], intersected with the causal bound, each token once).
# --------------------------------------------------------------------------------------------
def _brute_effective_attention(Q, K, V, bq, bk, causal, idx, cnt, sink, window, scale):
    """Plain-Python sets -> explicit boolean mask -> fp64 softmax (independent of the oracle)."""
    Q, K, V = (np.asarray(x, np.float64) for x in (Q, K, V))
    B, Hq, Tq, d = Q.shape
    Hkv, Tk = K.shape[1], K.shape[2]
    O = np.zeros_like(Q)
    for b in range(B):
        for h in range(Hq):
            hk = h // (Hq // Hkv)
            for t in range(Tq):
                p = t + Tk - Tq
                q = t // bq
                keys = set()
                for i in range(int(cnt[b, h, q])):
                    j = int(idx[b, h, q, i])
                    keys |= set(range(j * bk, min((j + 1) * bk, Tk)))
                keys |= set(range(min(sink, Tk)))
                keys |= {s for s in range(p - window + 1, p + 1) if 0 <= s < Tk}
                if causal:
                    keys = {s for s in keys if s <= p}
                ks = sorted(keys)
                if not ks:
                    continue
                x = scale * (K[b, hk, ks] @ Q[b, h, t])
                w = np.exp(x - x.max())
                O[b, h, t] = (w[:, None] * V[b, hk, ks]).sum(0) / w.sum()
    return O


def test_sinkwin_spec_example(orc):
    """empty BlockMask, sink = 1, window = 1, causal, row at position 5 -> tokens {0, 5}."""
    T, d = 8, 16
    Q, K, V = synth.gen_qkv(1, 1, 1, T, T, d, "iid", seed=40, dtype=torch.float32)
    idx = np.full((1, 1, T, 1), -1, np.int32)
    cnt = np.zeros((1, 1, T), np.int32)
    O, lse = orc.sparse_attention(Q, K, V, 1, 1, 1, True, idx, cnt, sink=1, window=1)
    q, Kn, Vn = (x.double().numpy() for x in (Q[0, 0, 5], K[0, 0], V[0, 0]))
    x = np.array([q @ Kn[0], q @ Kn[5]]) / math.sqrt(d)
    w = np.exp(x - x.max())
    ref = (w[0] * Vn[0] + w[1] * Vn[5]) / w.sum()
    assert np.abs(O[0, 0, 5] - ref).max() < 1e-12
    assert abs(lse[0, 0, 5] - (x.max() + math.log(w.sum()))) < 1e-12


def test_sinkwin_zero_is_plain_and_full_window_is_dense(orc):
    T, d, k, bq, bk = 300, 32, 64, 16, 2
    Q, K, V = synth.gen_qkv(1, 2, 1, T, T, d, "llm", seed=41, dtype=torch.float32)
    idx, cnt = orc.mask(Q, K, k, bq, bk, True)
    a = orc.sparse_attention(Q, K, V, k, bq, bk, True, idx, cnt)
    b = orc.sparse_attention(Q, K, V, k, bq, bk, True, idx, cnt, sink=0, window=0)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    # window >= T: every causal key of every row -> dense causal attention (library routine)
    O, _ = orc.sparse_attention(Q, K, V, k, bq, bk, True, idx, cnt, sink=3, window=T)
    assert np.abs(O - _sdpa64(Q, K, V, True, 1.0 / math.sqrt(d))).max() < 1e-12
    # defaults (window 128, sink 32) at position 40 cover {0..40}: the row is dense causal
    O, _ = orc.sparse_attention(Q, K, V, k, bq, bk, True, idx, cnt, sink=32, window=128)
    assert np.abs(O[:, :, 40] - _sdpa64(Q, K, V, True, 1.0 / math.sqrt(d))[:, :, 40]).max() < 1e-12


@pytest.mark.parametrize("Tq,Tk,bq,bk,k,causal,sink,window", [
    (200, 200, 16, 2, 32, True, 4, 16),     # overlaps between blocks, sink and window (dedup)
    (70, 250, 8, 4, 40, True, 32, 128),     # T_q < T_k (bottom-right), paper sizes
    (120, 120, 32, 1, 16, False, 5, 9),     # non-causal
    (33, 33, 32, 2, 2, True, 0, 3),         # ragged last block, window only
])
def test_sinkwin_union_brute_force(orc, Tq, Tk, bq, bk, k, causal, sink, window):
    d = 16
    Q, K, V = synth.gen_qkv(2, 2, 1, Tq, Tk, d, "iid", seed=42, dtype=torch.float32)
    nqb = -(-Tq // bq)
    hi = torch.tensor([[[_visible(q, bq, bk, Tq, Tk, causal) for q in range(nqb)]] * 2] * 2)
    idx, cnt = synth.gen_block_indices(2, 2, nqb, k // bk, hi, seed=42)
    O, _ = orc.sparse_attention(Q, K, V, k, bq, bk, causal, idx, cnt, sink=sink, window=window)
    ref = _brute_effective_attention(Q, K, V, bq, bk, causal, idx.numpy(), cnt.numpy(), sink, window,
                                     1.0 / math.sqrt(d))
    assert np.abs(O - ref).max() < 1e-12


def test_sinkwin_paged_equals_contiguous(orc):
    B, Hq, Hkv, d, k, bk = 2, 4, 2, 32, 64, 2
    seq = [300, 129]
    T = max(seq)
    Q = synth.gen_decode_q(B, Hq, d, seed=43, dtype=torch.float32)
    _, Kc, Vc = synth.gen_qkv(B, Hkv, Hkv, 1, T, d, "iid", seed=43, dtype=torch.float32)
    kp, vp, bt, sl = synth.to_paged(Kc, Vc, seq, 16, seed=1)
    idx, cnt = orc.mask_paged(Q, kp, bt, sl, k, 1, bk, True)
    O, lse = orc.sparse_attention_paged(Q, kp, vp, bt, sl, k, 1, bk, True, idx, cnt, sink=32, window=128)
    for b in range(B):
        Ob, lb = orc.sparse_attention(Q[b:b + 1], Kc[b:b + 1, :, : seq[b]], Vc[b:b + 1, :, : seq[b]], k, 1, bk, True,
                                      idx[b:b + 1], cnt[b:b + 1], sink=32, window=128)
        assert np.array_equal(O[b:b + 1], Ob) and np.array_equal(lse[b:b + 1], lb)


# --------------------------------------------------------------------------------------------
# Stridden partial top-k (f3; "splits the key-value sequence into S chunks"; reading
# G21: S contiguous chunks a_s = floor((2 s B_q + S) / (2 S)), Alg. 1 with n / S nodes on each).
# --------------------------------------------------------------------------------------------
def test_chunks_one_is_plain(orc):
    Q, K, _ = synth.gen_qkv(1, 2, 1, 2048, 2048, 64, "llm", seed=50, dtype=torch.float32, make_v=False)
    a = orc.mask(Q, K, 128, 32, 2, True)
    b = orc.mask(Q, K, 128, 32, 2, True, chunks=1)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("S", [2, 4])
def test_chunks_one_level_is_exact_topn_per_chunk(orc, S):
    """n_s < chunk <= 2 n_s: one iteration per chunk scores every block of the chunk once, so each
    chunk keeps the exact top-n_s of its block maxima (brute force, integer inputs with ties)."""
    Tq, Tk, d, bq, bk, k = 500, 523, 32, 24, 2, 64  # n = 32; B_q of every parity (boundary rounding)
    Q, K, _ = synth.gen_qkv(1, 1, 1, Tq, Tk, d, "int", seed=51, dtype=torch.float32, make_v=False)
    idx, cnt = orc.mask(Q, K, k, bq, bk, True, chunks=S)
    n, ns = k // bk, k // bk // S
    scores = _brute_block_scores(Q.double().numpy(), K.double().numpy(), bq, bk, True)[0, 0]
    checked = 0
    for q in range(-(-Tq // bq)):
        Bq = _visible(q, bq, bk, Tq, Tk, True)
        if Bq <= n:
            assert cnt[0, 0, q] == Bq
            continue
        for s in range(S):
            a0 = (2 * s * Bq + S) // (2 * S)
            a1 = (2 * (s + 1) * Bq + S) // (2 * S)
            got = idx[0, 0, q, s * ns:(s + 1) * ns]
            assert (got >= a0).all() and (got < a1).all() and (np.diff(got) > 0).all()
            if a1 - a0 <= 2 * ns:
                row = np.full(scores.shape[1], -np.inf)
                row[a0:a1] = scores[q, a0:a1]
                assert np.array_equal(got, _topn_sorted(row, ns))
                checked += 1
        assert cnt[0, 0, q] == n
    assert checked > 0


# --------------------------------------------------------------------------------------------
# f4a: top-r approximation: q.k ~ sum over the r components with the largest |q_c|;
# reading G22: a query block reduces |q_c| by the max over its rows, ties -> smaller component,
# terms summed in ascending component order.
# --------------------------------------------------------------------------------------------
def _brute_top_r(Qb, r):
    a = np.abs(np.asarray(Qb, np.float64)).max(axis=0)
    order = np.lexsort((np.arange(len(a)), -a))
    return np.sort(order[:r])


def test_topr_spec_examples(orc):
    """SPEC top_r_select examples and the tie rule."""
    assert orc.top_r_components([[3, -5, 1]], 2).tolist() == [0, 1]
    assert orc.top_r_components([[3, -5, 1]], 3).tolist() == [0, 1, 2]
    assert orc.top_r_components([[1, 0], [0, 2]], 1).tolist() == [1]  # componentwise max |q| = [1, 2]
    assert orc.top_r_components([[2, -2, 1]], 1).tolist() == [0]      # tie -> smaller component
    assert orc.top_r_components([[0, 1, -1, 1]], 2).tolist() == [1, 2]


def test_topr_components_brute_force(orc):
    rng = np.random.default_rng(70)
    for _ in range(200):
        rows, d = int(rng.integers(1, 9)), int(rng.integers(2, 40))
        r = int(rng.integers(1, d + 1))
        Qb = rng.integers(-3, 4, size=(rows, d)).astype(np.float32)  # many ties
        assert np.array_equal(orc.top_r_components(Qb, r), _brute_top_r(Qb, r))


def test_topr_r_equals_d_is_plain(orc):
    Q, K, _ = synth.gen_qkv(1, 2, 1, 1500, 1500, 32, "llm", seed=71, dtype=torch.float32, make_v=False)
    a = orc.mask(Q, K, 64, 16, 2, True)
    for r in (32, 0):
        b = orc.mask(Q, K, 64, 16, 2, True, top_r=r)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_topr_fixed_components_equal_sliced_problem(orc):
    """If every query block's top-r set is the same P, the top-r mask is the plain mask of the problem
    restricted to the components P (Q[..., P], K[..., P]) — bit-identical, since both sum q_c k_c
    over P in ascending order."""
    T, d, r = 2000, 32, 8
    Q, K, _ = synth.gen_qkv(1, 2, 1, T, T, d, "int", seed=72, dtype=torch.float32, make_v=False)
    Q = Q.clone()
    P = np.array([1, 4, 5, 11, 17, 20, 26, 31])
    sign = torch.where(Q[..., P] >= 0, 1.0, -1.0)
    Q[..., P] = sign * (8.0 + Q[..., P].abs())  # |q_c| >= 8 > 4 >= the others
    for mode in (orc.F32C, orc.F64):
        a = orc.mask(Q, K, 64, 16, 2, True, mode=mode, top_r=r)
        b = orc.mask(Q[..., P].contiguous(), K[..., P].contiguous(), 64, 16, 2, True, mode=mode)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        c = orc.mask(Q, K, 64, 16, 2, True, mode=mode)
        assert not np.array_equal(a[0], c[0])  # the approximation really changes the mask


def test_topr_one_level_is_exact_topn_of_approximate_scores(orc):
    """n < B_q <= 2n: the mask is the exact top-n of the block maxima of the APPROXIMATE scores
    sum_{c in P_q} q_c k_c, P_q = argtop_r of the block (numpy brute force, per query block)."""
    T, d, k, bq, bk, r = 1024, 32, 128, 16, 2, 6
    Q, K, _ = synth.gen_qkv(1, 1, 1, T, T, d, "int", seed=73, dtype=torch.float32, make_v=False)
    n = k // bk
    idx, _ = orc.mask(Q, K, k, bq, bk, True, top_r=r)
    Qn, Kn = Q.double().numpy()[0, 0], K.double().numpy()[0, 0]
    checked = 0
    for q in range(T // bq):
        vis = _visible(q, bq, bk, T, T, True)
        if not (n < vis <= 2 * n):
            continue
        P = _brute_top_r(Qn[q * bq:(q + 1) * bq], r)
        Qz = np.zeros_like(Qn)
        Qz[q * bq:(q + 1) * bq, P] = Qn[q * bq:(q + 1) * bq, P]
        bs = _brute_block_scores(Qz[None, None], Kn[None, None], bq, bk, True)[0, 0, q, :vis]
        assert np.array_equal(idx[0, 0, q], _topn_sorted(bs, n)), q
        checked += 1
    assert checked == 8


# --------------------------------------------------------------------------------------------
# f4b: HiP ensemble.  Samples: every split is moved "around the center" by a random
# integer in [-R, R] (reading G23), clamped so both branches stay non-empty, drawn from splitmix64
# keyed by (seed, unit, iteration, node).  Vote: an index survives with >= theta votes; tau = 1
# truncates to n by (votes desc, block asc) (reading G24).
# --------------------------------------------------------------------------------------------
def test_splitmix64_published_vectors(orc):
    """splitmix64 seeded with 0: the published first outputs (Vigna's reference implementation)."""
    g = 0x9E3779B97F4A7C15
    assert orc.splitmix64(0) == 0xE220A8397B1DCDAF
    assert orc.splitmix64(g) == 0x6E789E6AA1B965F4
    assert orc.splitmix64((2 * g) % 2**64) == 0x06C45D188009454F


def test_jitter_offsets_uniform(orc):
    """u is uniform on the 2R+1 integers [-R, R] (chi-square, loose) for any key."""
    for R in (1, 3, 5):
        u = np.array([orc.jitter_offset(7, lin, it, f, R) for lin in range(20) for it in range(5)
                      for f in range(0, 600, 7)])
        assert u.min() == -R and u.max() == R
        cnt = np.bincount(u + R, minlength=2 * R + 1)
        exp = len(u) / (2 * R + 1)
        assert ((cnt - exp) ** 2 / exp).sum() < 4 * (2 * R + 1)
    assert orc.jitter_offset(7, 3, 1, 40, 0) == 0


def test_jitter_zero_is_plain_and_deterministic(orc):
    Q, K, _ = synth.gen_qkv(1, 2, 1, 3000, 3000, 32, "llm", seed=74, dtype=torch.float32, make_v=False)
    a = orc.mask(Q, K, 64, 16, 2, True)
    b = orc.mask(Q, K, 64, 16, 2, True, jitter=0, seed=123)
    assert np.array_equal(a[0], b[0])
    c1 = orc.mask(Q, K, 64, 16, 2, True, jitter=5, seed=9)
    c2 = orc.mask(Q, K, 64, 16, 2, True, jitter=5, seed=9)
    c3 = orc.mask(Q, K, 64, 16, 2, True, jitter=5, seed=10)
    assert np.array_equal(c1[0], c2[0])
    assert not np.array_equal(c1[0], a[0]) and not np.array_equal(c1[0], c3[0])


def test_jitter_one_level_unchanged(orc):
    """B_q <= 2n: every initial node has <= 2 blocks, whose only split is (f, f)(l, l) — the jitter
    cannot move it, so the sample equals the deterministic mask."""
    T, d, k, bq, bk = 1024, 32, 128, 16, 2
    Q, K, _ = synth.gen_qkv(1, 1, 1, T, T, d, "iid", seed=75, dtype=torch.float32, make_v=False)
    a = orc.mask(Q, K, k, bq, bk, True)
    b = orc.mask(Q, K, k, bq, bk, True, jitter=4, seed=3)
    n = k // bk
    for q in range(T // bq):
        if _visible(q, bq, bk, T, T, True) <= 2 * n:
            assert np.array_equal(a[0][0, 0, q], b[0][0, 0, q])


def test_jitter_trace_invariants(orc):
    """Jittered samples keep PIN-5's invariants: n disjoint non-empty nested nodes per iteration,
    each split point within R of the half-up midpoint; final: n distinct ascending visible blocks."""
    T, d, k, bq, bk, R = 3000, 32, 96, 16, 2, 3
    Q, K, _ = synth.gen_qkv(1, 1, 1, T, T, d, "llm", seed=76, dtype=torch.float32, make_v=False)
    n = k // bk
    moved = 0
    for q in [7, 50, 101, 150, -(-T // bq) - 1]:
        vis = _visible(q, bq, bk, T, T, True)
        tr = orc.mask_trace(Q, K, k, bq, bk, True, 0, 0, q, jitter=R, seed=5)
        prev = None
        for nodes in tr["nodes"]:
            f, l = nodes[:, 0], nodes[:, 1]
            assert (l >= f).all() and (f >= 0).all() and (l < vis).all()
            o = np.argsort(f)
            assert (f[o][1:] > l[o][:-1]).all()  # disjoint
            if prev is not None:
                pf, pl = prev
                for a, b in zip(f, l):  # nested in a parent; a split child starts at f or at m
                    j = np.nonzero((pf <= a) & (b <= pl))[0]
                    assert len(j) == 1
                    pa, pb = pf[j[0]], pl[j[0]]
                    mid = (pa + pb + 1) // 2
                    if (a, b) != (pa, pb):
                        m = a if a > pa else b + 1
                        assert pa + 1 <= m <= pb and abs(m - mid) <= R
                        moved += m != mid
            prev = (f, l)
        final = tr["idx"][: tr["cnt"]]
        assert tr["cnt"] == n and (np.diff(final) > 0).all() and final[-1] < vis
    assert moved > 0


def test_vote_spec_examples(orc):
    A, B, C = 3, 7, 9
    def v(samples, theta, tau, n):
        I = np.full((len(samples), 1, n), -1, np.int32)
        Cn = np.zeros((len(samples), 1), np.int32)
        for e, s in enumerate(samples):
            I[e, 0, :len(s)] = sorted(s)
            Cn[e, 0] = len(s)
        idx, cnt = orc.vote(I, Cn, theta, tau)
        return idx[0, :cnt[0]].tolist()
    assert v([[A], [A, B]], 2, 0, 2) == [A]
    assert v([[A], [B]], 1, 0, 2) == [A, B]
    assert v([[A], [A, B], [B, C]], 1, 1, 2) == [A, B]
    assert v([[A, B]], 1, 0, 2) == [A, B]


def test_vote_brute_force(orc):
    """Counter-based brute force: survivors, truncation order, ascending output; monotone in theta;
    theta = n_e is the intersection, theta = 1 (tau = 0) the union."""
    from collections import Counter
    rng = np.random.default_rng(77)
    for _ in range(60):
        n_e, n, units = int(rng.integers(1, 6)), int(rng.integers(1, 12)), 5
        hi = int(rng.integers(n, 3 * n + 2))
        I = np.full((n_e, units, n), -1, np.int32)
        Cn = np.zeros((n_e, units), np.int32)
        for e in range(n_e):
            for u in range(units):
                c = int(rng.integers(0, n + 1))
                I[e, u, :c] = np.sort(rng.choice(hi, c, replace=False))
                Cn[e, u] = c
        prev = None
        for theta in range(1, n_e + 1):
            for tau in (0, 1):
                idx, cnt = orc.vote(I, Cn, theta, tau)
                for u in range(units):
                    votes = Counter(x for e in range(n_e) for x in I[e, u, :Cn[e, u]].tolist())
                    surv = sorted(x for x, c in votes.items() if c >= theta)
                    if tau and len(surv) > n:
                        surv = sorted(sorted(surv, key=lambda x: (-votes[x], x))[:n])
                    got = idx[u, :cnt[u]].tolist()
                    assert got == surv
                    assert (idx[u, cnt[u]:] == -1).all()
                    if theta == n_e and not tau:
                        inter = set.intersection(*[set(I[e, u, :Cn[e, u]].tolist()) for e in range(n_e)])
                        assert set(got) == inter
                    if theta == 1 and not tau:
                        assert set(got) == set(votes)
            cur = orc.vote(I, Cn, theta, 0)
            if prev is not None:
                for u in range(units):
                    assert set(cur[0][u, :cur[1][u]].tolist()) <= set(prev[0][u, :prev[1][u]].tolist())
            prev = cur


def test_ensemble_single_sample_is_plain(orc):
    """(n_e = 1, R = 0, theta = 1): the pipeline output equals the deterministic mask (SPEC)."""
    Q, K, _ = synth.gen_qkv(1, 2, 1, 2000, 2000, 32, "llm", seed=78, dtype=torch.float32, make_v=False)
    a = orc.mask(Q, K, 64, 16, 2, True)
    s = orc.mask(Q, K, 64, 16, 2, True, jitter=0, seed=4)
    idx, cnt = orc.vote(s[0][None], s[1][None], 1, 1)
    assert np.array_equal(idx, a[0]) and np.array_equal(cnt, a[1])


# --------------------------------------------------------------------------------------------
# f3b: GQA-shared masks (reading G25): one mask per (b, kv head, query block), the
# representative score being the max of the tile over the query rows of ALL H_q / H_kv heads of
# the group.  Pinned by reduction to the plain mask on a stacked-row input and by brute force.
# --------------------------------------------------------------------------------------------
def test_gqa_shared_group_of_one_is_plain(orc):
    Q, K, _ = synth.gen_qkv(1, 2, 2, 1500, 1500, 32, "llm", seed=90, dtype=torch.float32, make_v=False)
    a = orc.mask(Q, K, 64, 16, 2, True)
    b = orc.mask(Q, K, 64, 16, 2, True, gqa_shared=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("mode", [0, 1])
def test_gqa_shared_equals_stacked_rows_noncausal(orc, mode):
    """Non-causal: the shared mask of group g at query block q is the plain mask of ONE query block
    holding the G heads' rows of block q (a stacked [Nqb * G * b_q, d] query, b_q' = G * b_q)."""
    B, Hq, Hkv, Tq, Tk, d, bq, k, bk = 2, 6, 2, 200, 1800, 32, 8, 64, 2
    G = Hq // Hkv
    Q, K, _ = synth.gen_qkv(B, Hq, Hkv, Tq, Tk, d, "iid", seed=91, dtype=torch.float32, make_v=False)
    si, sc = orc.mask(Q, K, k, bq, bk, False, mode=mode, gqa_shared=True)
    nqb = Tq // bq
    for b in range(B):
        for g in range(Hkv):
            rows = Q[b, g * G:(g + 1) * G].reshape(G, nqb, bq, d).permute(1, 0, 2, 3).reshape(1, 1, nqb * G * bq, d)
            pi, pc = orc.mask(rows, K[b:b + 1, g:g + 1], k, G * bq, bk, False, mode=mode)
            assert np.array_equal(si[b, g], pi[0, 0]) and np.array_equal(sc[b, g], pc[0, 0])


def test_gqa_shared_decode_equals_stacked_rows(orc):
    """Paged decode (T_q = 1, causal: every key visible): the shared mask = the plain non-causal mask
    of the G query rows of the group as one block, on the sequence's keys."""
    B, Hq, Hkv, d, ps, k, bk = 3, 8, 2, 32, 16, 64, 2
    seq = [900, 40, 2001]
    G = Hq // Hkv
    Q = synth.gen_decode_q(B, Hq, d, seed=92, dtype=torch.float32)
    _, K, V = synth.gen_qkv(B, Hkv, Hkv, 1, max(seq), d, "iid", seed=92, dtype=torch.float32)
    kp, vp, bt, sl = synth.to_paged(K, V, seq, ps, seed=92)
    si, sc = orc.mask_paged(Q, kp, bt, sl, k, 1, bk, True, gqa_shared=True)
    assert si.shape[1] == Hkv
    for b in range(B):
        for g in range(Hkv):
            rows = Q[b, g * G:(g + 1) * G].reshape(1, 1, G, d)
            pi, pc = orc.mask(rows, K[b:b + 1, g:g + 1, :seq[b]], k, G, bk, False)
            assert np.array_equal(si[b, g, 0], pi[0, 0, 0]) and sc[b, g, 0] == pc[0, 0, 0]


def test_gqa_shared_one_level_is_exact_topn(orc):
    """Causal, n < B_q <= 2n: exact top-n of the block maxima over the whole group's rows (brute force)."""
    T, d, k, bq, bk, Hq, Hkv = 1024, 16, 128, 16, 2, 4, 1
    Q, K, _ = synth.gen_qkv(1, Hq, Hkv, T, T, d, "int", seed=93, dtype=torch.float32, make_v=False)
    si, _ = orc.mask(Q, K, k, bq, bk, True, gqa_shared=True)
    bs = _brute_block_scores(Q, K, bq, bk, True).max(axis=1)  # max over the group's heads
    n, checked = k // bk, 0
    for q in range(T // bq):
        vis = _visible(q, bq, bk, T, T, True)
        if n < vis <= 2 * n:
            assert np.array_equal(si[0, 0, q], _topn_sorted(bs[0, q, :vis], n))
            checked += 1
    assert checked == 8
