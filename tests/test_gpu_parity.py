"""GPU (sm_100a) vs CPU oracle parity, through the C ABI (paper_2406_09827_b200.hipattn).

Bars (BASELINE.json north_star):
  * mask indices: bit-exact wherever both sides take the selection decisions in the same fp32
    arithmetic — the fp32 / HIP_FLAG_EXACT_SCORES kernels (sequential fmaf = oracle F32C), the
    decode GEMV kernel (16-segment fmaf + xor tree = oracle F32L, reading G9b; fp32 / d=64 decode)
    on every input, and the tcgen05 kernel (prefill and bf16 decode) on integer-valued inputs (every
    sum exact).  For the tcgen05 kernel on Gaussian inputs the mismatching query blocks are reported
    as a fraction and every one must be certified as a near-tie by the oracle's fp64 selection
    margins.
  * attention outputs: max-abs <= 1e-4 (fp32) / 2e-2 (bf16) against the fp64 oracle on the same
    selection (seeded synthetic selections from synth.py, or the oracle's own mask).
"""
import math

import numpy as np
import pytest
import torch

from paper_2406_09827_b200 import hipattn as H
from paper_2406_09827_b200 import synth

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-4, torch.bfloat16: 2e-2}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    H.load()
    torch.cuda.init()


def _visible(q, bq, bk, Tq, Tk, causal):
    nkb = -(-Tk // bk)
    if not causal:
        return nkb
    tlast = min((q + 1) * bq, Tq) - 1
    return min((tlast + Tk - Tq) // bk + 1, nkb)


def _gpu_mask(Q, K, k, bq, bk, causal, exact=False):
    idx, cnt = H.mask_estimate(Q.cuda(), K.cuda(), k_budget=k, b_q=bq, b_k=bk, causal=causal, exact=exact)
    torch.cuda.synchronize()
    return idx.cpu().numpy(), cnt.cpu().numpy()


def _assert_mask_equal(gi, gc, oi, oc):
    assert np.array_equal(gc, oc), f"cnt mismatch at {np.argwhere(gc != oc)[:5]}"
    bad = np.argwhere((gi != oi).any(-1))
    assert len(bad) == 0, f"{len(bad)} query blocks differ, first {bad[:5].tolist()}"


# ------------------------------------------------------------------------------------------------
# Mask: bit-exact tiers
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("dist", ["iid", "int", "llm"])
def test_mask_fp32_c1_bitexact(orc, dist):
    """BASELINE config C1: single head, T=4096, d=128, k=512, b_q=32, b_k=2, fp32 causal."""
    Q, K, _ = synth.gen_qkv(1, 1, 1, 4096, 4096, 128, dist, seed=0, dtype=torch.float32, make_v=False)
    gi, gc = _gpu_mask(Q, K, 512, 32, 2, True)
    oi, oc = orc.mask(Q, K, 512, 32, 2, True, mode=orc.F32C)
    _assert_mask_equal(gi, gc, oi, oc)


@pytest.mark.parametrize("B,Hq,Hkv,Tq,Tk,d,k,bq,bk,causal,dist", [
    (1, 4, 2, 3000, 3000, 128, 256, 32, 2, True, "iid"),     # ragged tails, GQA
    (2, 2, 1, 700, 2100, 64, 128, 16, 4, True, "llm"),       # T_q < T_k, d=64
    (1, 2, 2, 1000, 1500, 128, 64, 32, 1, False, "iid"),     # non-causal, b_k=1
    (1, 1, 1, 50, 4000, 128, 512, 64, 8, True, "llm"),       # b_q=64 > 32 (CUDA-core path)
    (1, 1, 1, 5, 3, 128, 16, 64, 8, False, "iid"),           # b_q > T_q and b_k > T_k
    (1, 1, 1, 5, 700, 128, 16, 64, 8, False, "iid"),         # one ragged query block, 88 key blocks
    (1, 1, 1, 300, 300, 128, 2, 32, 2, True, "iid"),         # n = 1
])
def test_mask_exact_scores_bitexact(orc, B, Hq, Hkv, Tq, Tk, d, k, bq, bk, causal, dist):
    for dt in (torch.bfloat16, torch.float32):
        Q, K, _ = synth.gen_qkv(B, Hq, Hkv, Tq, Tk, d, dist, seed=1, dtype=dt, make_v=False)
        gi, gc = _gpu_mask(Q, K, k, bq, bk, causal, exact=True)
        oi, oc = orc.mask(Q, K, k, min(bq, Tq), bk, causal, mode=orc.F32C)
        _assert_mask_equal(gi, gc, oi, oc)


@pytest.mark.parametrize("Tq,Tk,Hq,Hkv,bk,k,causal", [
    (4096, 4096, 2, 1, 2, 512, True),
    (3001, 3333, 4, 2, 2, 256, True),
    (2048, 2048, 1, 1, 4, 512, False),
    (1024, 5000, 2, 2, 1, 128, True),
    (96, 96, 1, 1, 32, 64, True),
])
def test_mask_tcgen05_integer_bitexact(orc, Tq, Tk, Hq, Hkv, bk, k, causal):
    """Integer-valued bf16 inputs: every fp32 partial sum is exact, so the tensor-core scores equal
    the oracle's exactly and the masks must match bit-for-bit, ties and tie-breaks included."""
    Q, K, _ = synth.gen_qkv(1, Hq, Hkv, Tq, Tk, 128, "int", seed=2, dtype=torch.bfloat16, make_v=False)
    gi, gc = _gpu_mask(Q, K, k, 32, bk, causal)
    oi, oc = orc.mask(Q, K, k, 32, bk, causal, mode=orc.F32C)
    _assert_mask_equal(gi, gc, oi, oc)


def _slot_map(lins, units):
    slot = torch.full((units,), -1, dtype=torch.int32, device="cuda")
    slot[torch.as_tensor(lins, dtype=torch.long, device="cuda")] = torch.arange(len(lins), dtype=torch.int32,
                                                                                 device="cuda")
    return slot


@pytest.mark.parametrize("dist", ["iid", "llm"])
def test_mask_tcgen05_gaussian_certified(orc, dist):
    """tcgen05 masks on Gaussian inputs: every unit's scores within the fp32 bound, the GPU's selection
    replayed bit-exactly from its own scores, and every mismatch vs F64 certified at its first
    divergent iteration (tests/test_gpu_replay.py check_unit)."""
    from test_gpu_replay import check_unit
    Hq, Hkv, T, d = 4, 2, 4096, 128
    Q, K, _ = synth.gen_qkv(1, Hq, Hkv, T, T, d, dist, seed=3, dtype=torch.bfloat16, make_v=False)
    nqb, nkb = T // 32, T // 2
    dump = torch.full((Hq * nqb, nkb), float("nan"), dtype=torch.float32, device="cuda")
    with H.debug_score_dump(_slot_map(list(range(Hq * nqb)), Hq * nqb), dump):
        idx, cnt = H.mask_estimate(Q.cuda(), K.cuda(), k_budget=512, b_q=32, b_k=2)
    gi, gs = idx.cpu().numpy(), dump.cpu().numpy()
    st = dict(units=0, scores=0, replayed=0, mismatch=0, certified=0, unexplained=0)
    for h in range(Hq):
        for q in range(nqb):
            check_unit(orc, Q[:, h:h + 1], K[:, h // 2:h // 2 + 1], 512, 32, 2, True, q, gi[0, h, q],
                       gs[h * nqb + q], d, st)
    print(f"\n[parity] tcgen05 mask vs F64 oracle ({dist}): {st}")
    assert st["unexplained"] == 0
    assert st["mismatch"] <= 0.10 * st["units"]


# ------------------------------------------------------------------------------------------------
# Attention on seeded synthetic selections (no mask involved)
# ------------------------------------------------------------------------------------------------
def _synthetic_selection(B, Hq, Tq, Tk, k, bq, bk, causal, seed):
    nqb = -(-Tq // bq)
    hi = torch.tensor([[[_visible(q, bq, bk, Tq, Tk, causal) for q in range(nqb)]] * Hq] * B)
    return synth.gen_block_indices(B, Hq, nqb, k // bk, hi, seed=seed)


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("B,Hq,Hkv,Tq,Tk,d,k,bq,bk,causal", [
    (1, 2, 1, 1000, 1000, 128, 512, 32, 2, True),
    (2, 4, 2, 333, 900, 128, 256, 32, 4, True),
    (1, 2, 2, 257, 257, 64, 128, 16, 2, False),
    (1, 1, 1, 100, 100, 128, 64, 64, 8, True),
    (1, 2, 1, 130, 4000, 128, 512, 32, 1, True),
])
def test_attention_prefill_parity(orc, dt, B, Hq, Hkv, Tq, Tk, d, k, bq, bk, causal):
    Q, K, V = synth.gen_qkv(B, Hq, Hkv, Tq, Tk, d, "llm", seed=4, dtype=dt)
    idx, cnt = _synthetic_selection(B, Hq, Tq, Tk, k, bq, bk, causal, seed=4)
    o, lse = H.sparse_attention_prefill(Q.cuda(), K.cuda(), V.cuda(), idx.cuda(), cnt.cuda(), k_budget=k, b_q=bq,
                                        b_k=bk, causal=causal, return_lse=True)
    torch.cuda.synchronize()
    Oo, lo = orc.sparse_attention(Q, K, V, k, bq, bk, causal, idx, cnt)
    err = np.abs(o.float().cpu().numpy() - Oo).max()
    assert err <= TOL[dt], err
    lg = lse.cpu().numpy()
    fin = np.isfinite(lo)
    assert np.array_equal(np.isfinite(lg), fin)
    assert np.abs(lg[fin] - lo[fin]).max() <= 1e-3


def test_attention_empty_rows(orc):
    """k = b_k: one block per query block; rows before the block's first token see nothing:
    O = 0, lse = -inf (G13)."""
    for dt in (torch.bfloat16, torch.float32):
        Q, K, V = synth.gen_qkv(1, 1, 1, 256, 256, 128, "iid", seed=5, dtype=dt)
        idx, cnt = orc.mask(Q, K, 2, 32, 2, True)
        o, lse = H.sparse_attention_prefill(Q.cuda(), K.cuda(), V.cuda(), torch.from_numpy(idx).cuda(),
                                            torch.from_numpy(cnt).cuda(), k_budget=2, b_q=32, b_k=2, causal=True,
                                            return_lse=True)
        Oo, lo = orc.sparse_attention(Q, K, V, 2, 32, 2, True, idx, cnt)
        assert np.isneginf(lo).any()
        lg = lse.cpu().numpy()
        assert np.array_equal(np.isneginf(lg), np.isneginf(lo))
        assert (o.float().cpu().numpy()[np.isneginf(lo)] == 0).all()
        assert np.abs(o.float().cpu().numpy() - Oo).max() <= TOL[dt]


def test_exact_case_equals_dense(orc):
    """PIN-1 on the GPU: k >= T -> HiP attention == dense causal attention."""
    for dt in (torch.bfloat16, torch.float32):
        Q, K, V = synth.gen_qkv(1, 2, 1, 384, 384, 128, "llm", seed=6, dtype=dt)
        o = H.hip_attention(Q.cuda(), K.cuda(), V.cuda(), k_budget=512, b_q=32, b_k=2, causal=True)
        Od, _ = orc.dense_attention(Q, K, V, True)
        assert np.abs(o.float().cpu().numpy() - Od).max() <= TOL[dt]


# ------------------------------------------------------------------------------------------------
# Decode on a paged KV cache
# ------------------------------------------------------------------------------------------------
def _paged_to_contiguous(kp, bt, sl, b):
    """K rows of sequence b, [1, H_kv, seq_len, d], gathered through the block table (host side)."""
    ps = kp.shape[2]
    pages = [int(bt[b, i]) for i in range(-(-int(sl[b]) // ps))]
    return torch.cat([kp[p] for p in pages], dim=1)[:, : int(sl[b])].unsqueeze(0)


@pytest.mark.parametrize("dt,dist", [(torch.bfloat16, "iid"), (torch.bfloat16, "int"), (torch.float32, "iid")])
@pytest.mark.parametrize("ps", [16, 64])
def test_decode_paged_parity(orc, dt, dist, ps):
    B, Hq, Hkv, d, k, bk = 4, 8, 2, 128, 512, 2
    seq = [5000, 1, 777, 4096]
    Q = synth.gen_decode_q(B, Hq, d, seed=7, dtype=dt, dist=dist)
    kp, vp, bt, sl = synth.gen_paged_direct(B, Hkv, seq, d, ps, seed=7, dtype=dt, dist=dist)
    T = max(seq)
    dump = torch.full((B * Hq, -(-T // bk)), float("nan"), dtype=torch.float32, device="cuda")
    with H.debug_score_dump(_slot_map(list(range(B * Hq)), B * Hq), dump):
        idx, cnt = H.mask_estimate_paged(Q.cuda(), kp.cuda(), bt.cuda(), sl.cuda(), T, k_budget=k, b_q=1, b_k=bk,
                                         causal=True)
    torch.cuda.synchronize()
    gi, gc, gs = idx.cpu().numpy(), cnt.cpu().numpy(), dump.cpu().numpy()
    if dt == torch.float32:  # decode GEMV kernel: oracle F32L order (G9b), bit-exact
        oi, oc = orc.mask_paged(Q, kp, bt, sl, k, 1, bk, True, mode=orc.F32L)
        _assert_mask_equal(gi, gc, oi, oc)
    elif dist == "int":  # tcgen05 scoring on integer inputs: every sum exact
        oi, oc = orc.mask_paged(Q, kp, bt, sl, k, 1, bk, True, mode=orc.F32C)
        _assert_mask_equal(gi, gc, oi, oc)
    else:  # tcgen05 scoring on Gaussian inputs: scores bounded, replay exact, mismatches certified
        from test_gpu_replay import check_unit
        oi, oc = orc.mask_paged(Q, kp, bt, sl, k, 1, bk, True, mode=orc.F64)
        assert np.array_equal(gc, oc)
        st = dict(units=0, scores=0, replayed=0, mismatch=0, certified=0, unexplained=0)
        for b in range(B):
            Kb = _paged_to_contiguous(kp, bt, sl, b)
            for h in range(Hq):
                hk = h // (Hq // Hkv)
                check_unit(orc, Q[b:b + 1, h:h + 1], Kb[:, hk:hk + 1], k, 1, bk, True, 0, gi[b, h, 0],
                           gs[b * Hq + h], d, st)
        print(f"\n[parity] tcgen05 decode mask vs F64 oracle: {st}")
        assert st["unexplained"] == 0
    # attention on the ORACLE's selection (never feed GPU output to the oracle)
    o, lse = H.sparse_attention_decode(Q.cuda(), kp.cuda(), vp.cuda(), bt.cuda(), sl.cuda(), T,
                                       torch.from_numpy(oi).cuda(), torch.from_numpy(oc).cuda(), k_budget=k,
                                       b_q=1, b_k=bk, causal=True, return_lse=True)
    torch.cuda.synchronize()
    # HIP_FLAG_EXACT_SCORES: the sequential chain, == oracle F32C
    ie, ce = H.mask_estimate_paged(Q.cuda(), kp.cuda(), bt.cuda(), sl.cuda(), T, k_budget=k, b_q=1, b_k=bk,
                                   causal=True, exact=True)
    oi2, oc2 = orc.mask_paged(Q, kp, bt, sl, k, 1, bk, True, mode=orc.F32C)
    _assert_mask_equal(ie.cpu().numpy(), ce.cpu().numpy(), oi2, oc2)
    Oo, lo = orc.sparse_attention_paged(Q, kp, vp, bt, sl, k, 1, bk, True, oi, oc)
    assert np.abs(o.float().cpu().numpy() - Oo).max() <= TOL[dt]
    assert np.abs(lse.cpu().numpy() - lo).max() <= 1e-3


def test_paged_equals_contiguous_and_page_permutation():
    """PIN-9: the paged path sees exactly the contiguous problem (bit-identical), for any page order."""
    B, Hq, Hkv, d, k, bk = 2, 4, 2, 128, 256, 2
    seq = [3000, 2048]
    T = max(seq)
    Q = synth.gen_decode_q(B, Hq, d, seed=8).cuda()
    _, Kc, Vc = synth.gen_qkv(B, Hkv, Hkv, 1, T, d, "iid", seed=8)
    outs = []
    for perm_seed in (0, 1):
        kp, vp, bt, sl = synth.to_paged(Kc, Vc, seq, 64, seed=perm_seed)
        idx, cnt = H.mask_estimate_paged(Q, kp.cuda(), bt.cuda(), sl.cuda(), T, k_budget=k, b_q=1, b_k=bk)
        o = H.sparse_attention_decode(Q, kp.cuda(), vp.cuda(), bt.cuda(), sl.cuda(), T, idx, cnt, k_budget=k, b_q=1,
                                      b_k=bk)
        outs.append((idx.cpu(), o.cpu()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    for b in range(B):
        Kb, Vb = Kc[b:b + 1, :, : seq[b]].cuda(), Vc[b:b + 1, :, : seq[b]].cuda()
        idx_c, cnt_c = H.mask_estimate(Q[b:b + 1], Kb, k_budget=k, b_q=1, b_k=bk)
        assert torch.equal(idx_c.cpu(), outs[0][0][b:b + 1])


def test_batch_invariance():
    """A sequence's result does not depend on the other sequences in the batch (PIN-9)."""
    Q, K, V = synth.gen_qkv(3, 2, 2, 600, 600, 128, "llm", seed=9)
    Q, K, V = Q.cuda(), K.cuda(), V.cuda()
    o_all = H.hip_attention(Q, K, V, k_budget=128, b_q=32, b_k=2)
    o_one = H.hip_attention(Q[1:2].contiguous(), K[1:2].contiguous(), V[1:2].contiguous(), k_budget=128, b_q=32, b_k=2)
    assert torch.equal(o_all[1:2], o_one)


def test_strided_views():
    """Non-contiguous [B,H,T,d] views (e.g. a fused QKV buffer) give the same bits."""
    B, Hq, T, d = 1, 2, 500, 128
    base = torch.randn(B, T, 3, Hq, d, generator=torch.Generator().manual_seed(0)).to(torch.bfloat16).cuda()
    q, k, v = (base[:, :, i].permute(0, 2, 1, 3) for i in range(3))
    o1 = H.hip_attention(q, k, v, k_budget=128, b_q=32, b_k=2)
    o2 = H.hip_attention(q.contiguous(), k.contiguous(), v.contiguous(), k_budget=128, b_q=32, b_k=2)
    assert torch.equal(o1, o2)


# ------------------------------------------------------------------------------------------------
# End to end (mask -> attention) vs oracle (mask -> attention)
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("dt,dist", [(torch.float32, "llm"), (torch.bfloat16, "int"), (torch.bfloat16, "llm")])
def test_hip_layer_end_to_end(orc, dt, dist):
    B, Hq, Hkv, T, d, k, bq, bk = 1, 2, 1, 2048, 128, 256, 32, 2
    Q, K, V = synth.gen_qkv(B, Hq, Hkv, T, T, d, dist, seed=10, dtype=dt)
    gi, gc = _gpu_mask(Q, K, k, bq, bk, True)
    o = H.sparse_attention_prefill(Q.cuda(), K.cuda(), V.cuda(), torch.from_numpy(gi).cuda(),
                                   torch.from_numpy(gc).cuda(), k_budget=k, b_q=bq, b_k=bk).float().cpu().numpy()
    oi, oc = orc.mask(Q, K, k, bq, bk, True, mode=orc.F32C if dt == torch.float32 or dist == "int" else orc.F64)
    Oo, _ = orc.sparse_attention(Q, K, V, k, bq, bk, True, oi, oc)
    same = ~(gi != oi).any(-1)  # [B,Hq,nqb]
    rows = np.repeat(same, bq, axis=-1)[..., :T]
    assert same.mean() >= 0.9
    assert np.abs(o - Oo)[rows].max() <= TOL[dt]


# ------------------------------------------------------------------------------------------------
# Full-size configuration (BASELINE C2 shape, sampled): the launch bench.py times
# ------------------------------------------------------------------------------------------------
@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["c2", "c4", "c5"])
def test_full_size_sampled(orc, cfg):
    """The launches bench.py times (C2 32 heads x 32k, C4 40 x 128k, C5 32 x 1M; bf16, llm inputs),
    checked on sampled query blocks — the regime boundaries q in {0, 15, 16, 31, 32, N_qb - 1} plus
    random ones — against the oracle run on the sub-problem (the block's Q rows, the K/V prefix:
    bottom-right alignment makes it exact)."""
    Hq, T, n_heads, per_head = {"c2": (32, 32768, 48, 7), "c4": (40, 131072, 8, 7), "c5": (32, 1048576, 3, 7)}[cfg]
    B, d, k, bq, bk = 1, 128, 512, 32, 2
    from test_gpu_replay import check_unit
    Q, K, V = synth.gen_qkv(B, Hq, Hq, T, T, d, "llm", seed=0, dtype=torch.bfloat16, device="cuda")
    nqb = T // bq
    rng = np.random.default_rng(0)
    units = [(int(h), q) for h in rng.integers(0, Hq, n_heads) for q in
             [0, 15, 16, 31, 32, nqb - 1, int(rng.integers(33, nqb - 1))][:per_head]]
    units = sorted(set(units))
    dump = torch.full((len(units), T // bk), float("nan"), dtype=torch.float32, device="cuda")
    with H.debug_score_dump(_slot_map([h * nqb + q for h, q in units], Hq * nqb), dump):
        idx, cnt = H.mask_estimate(Q, K, k_budget=k, b_q=bq, b_k=bk)
    o = H.sparse_attention_prefill(Q, K, V, idx, cnt, k_budget=k, b_q=bq, b_k=bk)
    torch.cuda.synchronize()
    st = dict(units=0, scores=0, replayed=0, mismatch=0, certified=0, unexplained=0)
    for u, (h, q) in enumerate(units):
        t1 = (q + 1) * bq
        Qs = Q[:, h:h + 1, q * bq:t1].cpu()
        Ks, Vs = K[:, h:h + 1, :t1].cpu(), V[:, h:h + 1, :t1].cpu()
        gi = idx[0, h, q].cpu().numpy()
        assert int(cnt[0, h, q]) == min(k // bk, t1 // bk)
        check_unit(orc, Qs, Ks, k, bq, bk, True, 0, gi, dump[u, :t1 // bk].cpu().numpy(), d, st)
        # C-3: attention on the GPU's own selection
        Oo, _ = orc.sparse_attention(Qs, Ks, Vs, k, bq, bk, True, gi[None, None, None], cnt[0, h, q].view(1, 1, 1).cpu())
        assert np.abs(o[0, h, q * bq:t1].float().cpu().numpy() - Oo[0, 0]).max() <= 2e-2
    print(f"\n[parity] {cfg} sampled: {st}")
    assert st["unexplained"] == 0
    del Q, K, V, o, idx, cnt
    torch.cuda.empty_cache()


# ------------------------------------------------------------------------------------------------
# Sink + sliding window fused into the sparse kernels (f1; oracle: the S:285-301 union)
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("Tq,Tk,bq,bk,k,causal,sink,window", [
    (1000, 1000, 32, 2, 512, True, 32, 128),   # the paper's sizes
    (333, 900, 32, 4, 256, True, 4, 16),       # T_q < T_k, small sizes, overlaps with the blocks
    (257, 257, 16, 2, 128, False, 8, 33),      # non-causal
    (300, 300, 32, 2, 2, True, 0, 64),         # one block per query block: mostly window
])
def test_attention_sinkwin_prefill_parity(orc, dt, Tq, Tk, bq, bk, k, causal, sink, window):
    B, Hq, Hkv, d = 1, 2, 1, 128
    Q, K, V = synth.gen_qkv(B, Hq, Hkv, Tq, Tk, d, "llm", seed=20, dtype=dt)
    idx, cnt = _synthetic_selection(B, Hq, Tq, Tk, k, bq, bk, causal, seed=20)
    o, lse = H.sparse_attention_prefill(Q.cuda(), K.cuda(), V.cuda(), idx.cuda(), cnt.cuda(), k_budget=k, b_q=bq,
                                        b_k=bk, causal=causal, sink=sink, window=window, return_lse=True)
    torch.cuda.synchronize()
    Oo, lo = orc.sparse_attention(Q, K, V, k, bq, bk, causal, idx, cnt, sink=sink, window=window)
    assert np.abs(o.float().cpu().numpy() - Oo).max() <= TOL[dt]
    fin = np.isfinite(lo)
    lg = lse.cpu().numpy()
    assert np.array_equal(np.isfinite(lg), fin)
    assert np.abs(lg[fin] - lo[fin]).max() <= 1e-3


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float32])
def test_attention_sinkwin_decode_parity(orc, dt):
    B, Hq, Hkv, d, k, bk, ps = 4, 8, 2, 128, 512, 2, 64
    seq = [5000, 1, 200, 4096]
    T = max(seq)
    Q = synth.gen_decode_q(B, Hq, d, seed=21, dtype=dt)
    kp, vp, bt, sl = synth.gen_paged_direct(B, Hkv, seq, d, ps, seed=21, dtype=dt)
    oi, oc = orc.mask_paged(Q, kp, bt, sl, k, 1, bk, True)
    o, lse = H.sparse_attention_decode(Q.cuda(), kp.cuda(), vp.cuda(), bt.cuda(), sl.cuda(), T,
                                       torch.from_numpy(oi).cuda(), torch.from_numpy(oc).cuda(), k_budget=k, b_q=1,
                                       b_k=bk, causal=True, sink=32, window=128, return_lse=True)
    torch.cuda.synchronize()
    Oo, lo = orc.sparse_attention_paged(Q, kp, vp, bt, sl, k, 1, bk, True, oi, oc, sink=32, window=128)
    assert np.abs(o.float().cpu().numpy() - Oo).max() <= TOL[dt]
    assert np.abs(lse.cpu().numpy() - lo).max() <= 1e-3


def test_attention_sinkwin_validation():
    Q, K, V = (x.cuda() for x in synth.gen_qkv(1, 1, 1, 64, 64, 128, "iid", seed=22))
    idx, cnt = H.mask_estimate(Q, K, k_budget=64, b_q=32, b_k=2)
    with pytest.raises(H.HipError):
        H.sparse_attention_prefill(Q, K, V, idx, cnt, k_budget=64, b_q=32, b_k=2, sink=-1)
    with pytest.raises(H.HipError):
        H.sparse_attention_prefill(Q, K, V, idx, cnt, k_budget=64, b_q=32, b_k=2, sink=200, window=100)


# ------------------------------------------------------------------------------------------------
# f2: multi-query (speculative) decode and the r_m mask-caching loop (Alg. 2)
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("dt,dist", [(torch.bfloat16, "int"), (torch.float32, "iid")])
@pytest.mark.parametrize("Tq", [4, 16])
def test_multi_query_decode_parity(orc, dt, dist, Tq):
    """T_q > 1 query rows per sequence at positions seq_len - T_q + t, b_q = T_q."""
    B, Hq, Hkv, d, k, bk, ps = 3, 4, 2, 128, 256, 2, 16
    seq = [3000, 40, 777]
    T = max(seq)
    Q = synth.gen_decode_q(B, Hq, d, seed=30, dtype=dt, dist=dist, Tq=Tq)
    kp, vp, bt, sl = synth.gen_paged_direct(B, Hkv, seq, d, ps, seed=30, dtype=dt, dist=dist)
    idx, cnt = H.mask_estimate_paged(Q.cuda(), kp.cuda(), bt.cuda(), sl.cuda(), T, k_budget=k, b_q=Tq, b_k=bk)
    torch.cuda.synchronize()
    mode = orc.F32L if dt == torch.float32 and Tq <= 4 else orc.F32C
    oi, oc = orc.mask_paged(Q, kp, bt, sl, k, Tq, bk, True, mode=mode)
    _assert_mask_equal(idx.cpu().numpy(), cnt.cpu().numpy(), oi, oc)
    o, lse = H.sparse_attention_decode(Q.cuda(), kp.cuda(), vp.cuda(), bt.cuda(), sl.cuda(), T, idx, cnt, k_budget=k,
                                       b_q=Tq, b_k=bk, sink=4, window=32, return_lse=True)
    torch.cuda.synchronize()
    Oo, lo = orc.sparse_attention_paged(Q, kp, vp, bt, sl, k, Tq, bk, True, oi, oc, sink=4, window=32)
    assert np.abs(o.float().cpu().numpy() - Oo).max() <= TOL[dt]
    assert np.abs(lse.cpu().numpy() - lo).max() <= 1e-3


@pytest.mark.parametrize("shared,chunks", [(False, 1), (True, 2)])
def test_decoder_rm_cache_schedule(orc, shared, chunks):
    """HipDecoder: the mask is re-estimated exactly when a sequence's length is divisible by r_m
    (Alg. 2 line 8) and reused in between; every step's output is the oracle's attention over the
    cached selection at the current length (the steps 'append' tokens already present in pages).
    Also with the GQA-shared + chunked mask options."""
    from paper_2406_09827_b200.decode import HipDecoder
    B, Hq, Hkv, d, k, bk, ps, r_m = 2, 4, 2, 128, 128, 2, 16, 4
    full = [700, 901]
    kp, vp, bt, _ = synth.gen_paged_direct(B, Hkv, full, d, ps, seed=31, dist="int")
    dec = HipDecoder(r_m=r_m, k_budget=k, b_k=bk, b_q=1, sink=4, window=16, gqa_shared=shared, chunks=chunks)
    lens = [690, 893]
    cached = None
    for step in range(8):
        cur = [lens[0] + step, lens[1] + step]
        q = synth.gen_decode_q(B, Hq, d, seed=100 + step, dist="int")
        sl = torch.tensor(cur, dtype=torch.int32)
        expect_refresh = [cached is None or t % r_m == 0 for t in cur]
        o = dec.step(q.cuda(), kp.cuda(), vp.cuda(), bt.cuda(), sl.cuda(), cur)
        torch.cuda.synchronize()
        # integer inputs: exact in any order
        oi, oc = orc.mask_paged(q, kp, bt, sl, k, 1, bk, True, gqa_shared=shared, chunks=chunks)
        gi, gc = dec.idx.cpu().numpy(), dec.cnt.cpu().numpy()
        for b in range(B):
            if expect_refresh[b]:
                assert np.array_equal(gi[b], oi[b]) and np.array_equal(gc[b], oc[b])
            else:
                assert np.array_equal(gi[b], cached[0][b]) and np.array_equal(gc[b], cached[1][b])
        cached = (gi.copy(), gc.copy())
        ei, ec = orc.expand_gqa(gi, gc, Hq) if shared else (gi, gc)
        Oo, _ = orc.sparse_attention_paged(q, kp, vp, bt, sl, k, 1, bk, True, ei, ec, sink=4, window=16)
        assert np.abs(o.float().cpu().numpy() - Oo).max() <= TOL[torch.bfloat16]
    assert 1 < dec.refreshes < 8


@pytest.mark.parametrize("lens", [[690, 893], [692, 896]])
def test_decoder_graphed_step_equals_eager(lens):
    """HipDecoder.graphed_step (CUDA graphs: refresh graph = mask + attention, cached graph =
    attention; mixed-refresh steps merge an eager mask) gives the eager step's indices and outputs
    bit-for-bit over an r_m = 4 schedule.  lens[0] % 4 != lens[1] % 4 exercises the mixed case, the
    second set (both divisible by 4 together) the all / none cases.  Static buffers updated in place."""
    from paper_2406_09827_b200.decode import HipDecoder
    B, Hq, Hkv, d, k, bk, ps, r_m = 2, 4, 2, 128, 128, 2, 16, 4
    kp, vp, bt, _ = (x.cuda() for x in synth.gen_paged_direct(B, Hkv, [1000, 1000], d, ps, seed=32))
    eager = HipDecoder(r_m=r_m, k_budget=k, b_k=bk, b_q=1, sink=4, window=16)
    graphed = HipDecoder(r_m=r_m, k_budget=k, b_k=bk, b_q=1, sink=4, window=16)
    q = torch.empty(B, Hq, 1, d, dtype=torch.bfloat16, device="cuda")
    sl = torch.empty(B, dtype=torch.int32, device="cuda")
    out = torch.empty_like(q)
    for step in range(9):
        cur = [lens[0] + step, lens[1] + step]
        q.copy_(synth.gen_decode_q(B, Hq, d, seed=200 + step))
        sl.copy_(torch.tensor(cur, dtype=torch.int32))
        oe = eager.step(q, kp, vp, bt, sl, cur)
        graphed.graphed_step(q, kp, vp, bt, sl, cur, out)
        torch.cuda.synchronize()
        assert torch.equal(graphed.idx, eager.idx) and torch.equal(graphed.cnt, eager.cnt), step
        assert torch.equal(out, oe), step
    assert graphed.refreshes == eager.refreshes


def test_decoder_non_refresh_step_attends_current_token(orc):
    """with a cached mask (r_m = 8, the paper's default) a step between refreshes must still
    attend the token just generated — the default sliding window (128) covers it.  Changing
    that token's V row changes the output, and the output matches the oracle's union mask."""
    from paper_2406_09827_b200.decode import HipDecoder
    B, Hq, Hkv, d, ps = 1, 2, 1, 128, 16
    L0 = 4000                              # divisible by 8: refresh step
    kp, vp, bt, _ = synth.gen_paged_direct(B, Hkv, [L0 + 16], d, ps, seed=90, dtype=torch.bfloat16)
    kp, vp, bt = kp.cuda(), vp.cuda(), bt.cuda()
    dec = HipDecoder(k_budget=256, b_k=2, b_q=1)
    q0 = synth.gen_decode_q(B, Hq, d, seed=91).cuda()
    dec.step(q0, kp, vp, bt, torch.tensor([L0], dtype=torch.int32, device="cuda"), [L0])
    assert dec.refreshes == 1
    L = L0 + 3                             # not divisible by 8: the cached mask is reused
    q = synth.gen_decode_q(B, Hq, d, seed=92).cuda()
    sl = torch.tensor([L], dtype=torch.int32, device="cuda")
    o1 = dec.step(q, kp, vp, bt, sl, [L]).float()
    assert dec.refreshes == 1
    page, slot = int(bt[0, (L - 1) // ps]), (L - 1) % ps
    vp[page, :, slot] = 512.0              # the current token's value row (weight ~1/700 -> ~0.7 change)
    o2 = dec.step(q, kp, vp, bt, sl, [L]).float()
    torch.cuda.synchronize()
    assert dec.refreshes == 1
    assert (o2 - o1).abs().min() > 0.1, "the current token is not attended"
    Oo, _ = orc.sparse_attention_paged(q.cpu(), kp.cpu(), vp.cpu(), bt.cpu(), sl.cpu(), 256, 1, 2, True,
                                       dec.idx.cpu().numpy(), dec.cnt.cpu().numpy(), sink=32, window=128)
    assert np.abs(o2.cpu().numpy() - Oo).max() <= TOL[torch.bfloat16]


# ------------------------------------------------------------------------------------------------
# f3: stridden partial top-k (S chunks per query block; reading G21)
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("S", [2, 4])
@pytest.mark.parametrize("dt,dist", [(torch.float32, "llm"), (torch.bfloat16, "int")])
def test_mask_chunked_parity(orc, S, dt, dist):
    Tq, Tk, k, bq, bk = 1500, 1700, 256, 32, 2
    Q, K, _ = synth.gen_qkv(1, 2, 1, Tq, Tk, 128, dist, seed=60, dtype=dt, make_v=False)
    idx, cnt = H.mask_estimate(Q.cuda(), K.cuda(), k_budget=k, b_q=bq, b_k=bk, chunks=S)
    torch.cuda.synchronize()
    oi, oc = orc.mask(Q, K, k, bq, bk, True, chunks=S)
    _assert_mask_equal(idx.cpu().numpy(), cnt.cpu().numpy(), oi, oc)


@pytest.mark.parametrize("dt,dist", [(torch.float32, "iid"), (torch.bfloat16, "int")])
def test_mask_chunked_decode_parity(orc, dt, dist):
    B, Hq, Hkv, d, k, bk, ps, S = 3, 4, 2, 128, 512, 2, 64, 4
    seq = [5000, 100, 3333]
    T = max(seq)
    Q = synth.gen_decode_q(B, Hq, d, seed=61, dtype=dt, dist=dist)
    kp, vp, bt, sl = synth.gen_paged_direct(B, Hkv, seq, d, ps, seed=61, dtype=dt, dist=dist)
    idx, cnt = H.mask_estimate_paged(Q.cuda(), kp.cuda(), bt.cuda(), sl.cuda(), T, k_budget=k, b_q=1, b_k=bk,
                                     chunks=S)
    torch.cuda.synchronize()
    gi, gc = idx.cpu().numpy(), cnt.cpu().numpy()
    for b in range(B):  # the oracle's chunked mask on the contiguous view of each sequence
        Kb = _paged_to_contiguous(kp, bt, sl, b)
        mode = orc.F32L if dt == torch.float32 else orc.F32C
        oi, oc = orc.mask(Q[b:b + 1], Kb, k, 1, bk, True, mode=mode, chunks=S)
        _assert_mask_equal(gi[b:b + 1], gc[b:b + 1], oi, oc)


# ------------------------------------------------------------------------------------------------
# f4: top-r approximation (G22), ensemble samples (G23) and vote
# (G24).  Bit-exact tiers as for the plain mask: fp32 kernels issue the oracle's fmaf
# order with the dropped components zeroed (exact zeros), tcgen05 on integer-valued inputs.
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("r", [16, 40])
@pytest.mark.parametrize("dt,dist", [(torch.float32, "llm"), (torch.bfloat16, "int")])
def test_mask_topr_parity(orc, r, dt, dist):
    Tq, Tk, k, bq, bk = 2500, 2600, 256, 32, 2
    Q, K, _ = synth.gen_qkv(1, 2, 1, Tq, Tk, 128, dist, seed=80, dtype=dt, make_v=False)
    idx, cnt = H.mask_estimate(Q.cuda(), K.cuda(), k_budget=k, b_q=bq, b_k=bk, top_r=r)
    torch.cuda.synchronize()
    oi, oc = orc.mask(Q, K, k, bq, bk, True, top_r=r)
    _assert_mask_equal(idx.cpu().numpy(), cnt.cpu().numpy(), oi, oc)
    pi, _ = orc.mask(Q, K, k, bq, bk, True)
    assert not np.array_equal(pi, oi)  # the approximation is active


@pytest.mark.parametrize("dt,dist", [(torch.float32, "iid"), (torch.bfloat16, "int")])
def test_mask_topr_decode_parity(orc, dt, dist):
    B, Hq, Hkv, d, k, bk, ps, r = 3, 4, 2, 128, 256, 2, 16, 24
    seq = [5000, 100, 3333]
    Q = synth.gen_decode_q(B, Hq, d, seed=81, dtype=dt, dist=dist)
    kp, vp, bt, sl = synth.gen_paged_direct(B, Hkv, seq, d, ps, seed=81, dtype=dt, dist=dist)
    idx, cnt = H.mask_estimate_paged(Q.cuda(), kp.cuda(), bt.cuda(), sl.cuda(), max(seq), k_budget=k, b_q=1, b_k=bk,
                                     top_r=r)
    torch.cuda.synchronize()
    mode = orc.F32L if dt == torch.float32 else orc.F32C
    oi, oc = orc.mask_paged(Q, kp, bt, sl, k, 1, bk, True, mode=mode, top_r=r)
    _assert_mask_equal(idx.cpu().numpy(), cnt.cpu().numpy(), oi, oc)


@pytest.mark.parametrize("R,seed,S", [(3, 1, 1), (5, 2, 1), (4, 3, 2)])
@pytest.mark.parametrize("dt,dist", [(torch.float32, "llm"), (torch.bfloat16, "int")])
def test_mask_jitter_parity(orc, R, seed, S, dt, dist):
    Tq, Tk, k, bq, bk = 3000, 3000, 128, 32, 2
    Q, K, _ = synth.gen_qkv(1, 3, 1, Tq, Tk, 128, dist, seed=82, dtype=dt, make_v=False)
    idx, cnt = H.mask_estimate(Q.cuda(), K.cuda(), k_budget=k, b_q=bq, b_k=bk, jitter=R, seed=seed, chunks=S)
    torch.cuda.synchronize()
    oi, oc = orc.mask(Q, K, k, bq, bk, True, jitter=R, seed=seed, chunks=S)
    _assert_mask_equal(idx.cpu().numpy(), cnt.cpu().numpy(), oi, oc)


@pytest.mark.parametrize("dt,dist", [(torch.float32, "iid"), (torch.bfloat16, "int")])
def test_mask_jitter_decode_parity(orc, dt, dist):
    B, Hq, Hkv, d, k, bk, ps = 3, 4, 2, 128, 128, 2, 64
    seq = [6000, 90, 3333]
    Q = synth.gen_decode_q(B, Hq, d, seed=83, dtype=dt, dist=dist)
    kp, vp, bt, sl = synth.gen_paged_direct(B, Hkv, seq, d, ps, seed=83, dtype=dt, dist=dist)
    idx, cnt = H.mask_estimate_paged(Q.cuda(), kp.cuda(), bt.cuda(), sl.cuda(), max(seq), k_budget=k, b_q=1, b_k=bk,
                                     jitter=5, seed=11, top_r=32)
    torch.cuda.synchronize()
    mode = orc.F32L if dt == torch.float32 else orc.F32C
    oi, oc = orc.mask_paged(Q, kp, bt, sl, k, 1, bk, True, mode=mode, jitter=5, seed=11, top_r=32)
    _assert_mask_equal(idx.cpu().numpy(), cnt.cpu().numpy(), oi, oc)


@pytest.mark.parametrize("n_e,theta,tau", [(1, 1, 1), (3, 1, 0), (3, 2, 1), (4, 2, 0), (4, 4, 1), (8, 3, 1)])
def test_vote_parity_synthetic(orc, n_e, theta, tau):
    """GPU vote vs oracle vote on seeded synthetic sample masks (bit-exact)."""
    B, Hq, nqb, n = 1, 3, 40, 64
    hi = torch.randint(1, 300, (B, Hq, nqb), generator=torch.Generator().manual_seed(n_e))
    samples = [synth.gen_block_indices(B, Hq, nqb, n, hi, seed=100 + e) for e in range(n_e)]
    I = torch.stack([s[0] for s in samples])
    C = torch.stack([s[1] for s in samples])
    gi, gc = H.mask_vote(I.cuda(), C.cuda(), theta=theta, tau=tau)
    torch.cuda.synchronize()
    oi, oc = orc.vote(I, C, theta, tau)
    assert np.array_equal(gc.cpu().numpy(), oc)
    assert np.array_equal(gi.cpu().numpy(), oi)


def test_ensemble_end_to_end(orc):
    """n_e jittered samples -> vote -> sparse attention, on integer bf16 inputs: the GPU samples and
    vote equal the oracle's bit-for-bit, and the attention on that selection (tau = 0: up to
    n_e * k tokens per row) matches the fp64 oracle within the bf16 bar."""
    Tq = Tk = 2048
    k, bq, bk, n_e, R = 128, 32, 2, 3, 5
    Q, K, V = synth.gen_qkv(1, 2, 1, Tq, Tk, 128, "int", seed=84, dtype=torch.bfloat16)
    Qd, Kd, Vd = Q.cuda(), K.cuda(), V.cuda()
    gs = [H.mask_estimate(Qd, Kd, k_budget=k, b_q=bq, b_k=bk, jitter=R, seed=s) for s in range(n_e)]
    os_ = [orc.mask(Q, K, k, bq, bk, True, jitter=R, seed=s) for s in range(n_e)]
    for (gi, gc), (oi, oc) in zip(gs, os_):
        torch.cuda.synchronize()
        _assert_mask_equal(gi.cpu().numpy(), gc.cpu().numpy(), oi, oc)
    for theta, tau in ((1, 0), (2, 1)):
        vi, vc = H.mask_vote(torch.stack([g[0] for g in gs]), torch.stack([g[1] for g in gs]), theta=theta, tau=tau)
        oi, oc = orc.vote(np.stack([o[0] for o in os_]), np.stack([o[1] for o in os_]), theta, tau)
        torch.cuda.synchronize()
        assert np.array_equal(vi.cpu().numpy(), oi) and np.array_equal(vc.cpu().numpy(), oc)
        kk = oi.shape[-1] * bk
        o = H.sparse_attention_prefill(Qd, Kd, Vd, vi, vc, k_budget=kk, b_q=bq, b_k=bk)
        Oo, _ = orc.sparse_attention(Q, K, V, kk, bq, bk, True, oi, oc)
        torch.cuda.synchronize()
        assert np.abs(o.float().cpu().numpy() - Oo).max() <= TOL[torch.bfloat16]


@pytest.mark.parametrize("paged", [False, True])
def test_attention_wide_selection_parity(orc, paged):
    """Selections longer than k = 512 keys (the ensemble's tau = 0 union: up to n_e * n blocks) run on
    the wide tcgen05 instantiation; seeded synthetic selections of up to 1024 blocks = 2048 keys."""
    Tq, Tk, bq, bk, n = 700, 4000, 32, 2, 1024
    Q, K, V = synth.gen_qkv(1, 2, 1, Tq, Tk, 128, "iid", seed=85, dtype=torch.bfloat16)
    idx, cnt = _synthetic_selection(1, 2, Tq, Tk, n * bk, bq, bk, True, seed=85)
    if not paged:
        o = H.sparse_attention_prefill(Q.cuda(), K.cuda(), V.cuda(), idx.cuda(), cnt.cuda(), k_budget=n * bk, b_q=bq,
                                       b_k=bk, sink=32, window=128)
        Oo, _ = orc.sparse_attention(Q, K, V, n * bk, bq, bk, True, idx, cnt, sink=32, window=128)
    else:
        kp, vp, bt, sl = synth.to_paged(K, V, [Tk], 64, seed=85)
        o = H.sparse_attention_decode(Q.cuda(), kp.cuda(), vp.cuda(), bt.cuda(), sl.cuda(), Tk, idx.cuda(), cnt.cuda(),
                                      k_budget=n * bk, b_q=bq, b_k=bk)
        Oo, _ = orc.sparse_attention_paged(Q, kp, vp, bt, sl, n * bk, bq, bk, True, idx, cnt)
    torch.cuda.synchronize()
    assert int(cnt.max()) > 256
    assert np.abs(o.float().cpu().numpy() - Oo).max() <= TOL[torch.bfloat16]


# ------------------------------------------------------------------------------------------------
# f3b: GQA-shared masks (reading G25): one mask per kv head, scored over all its query heads' rows
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("dt,dist,bq", [(torch.float32, "llm", 8), (torch.bfloat16, "int", 8), (torch.bfloat16, "int", 4)])
def test_mask_gqa_shared_prefill_parity(orc, dt, dist, bq):
    B, Hq, Hkv, Tq, Tk, k, bk = 1, 8, 2, 1200, 1300, 256, 2
    Q, K, V = synth.gen_qkv(B, Hq, Hkv, Tq, Tk, 128, dist, seed=95, dtype=dt)
    idx, cnt = H.mask_estimate(Q.cuda(), K.cuda(), k_budget=k, b_q=bq, b_k=bk, gqa_shared=True)
    o = H.sparse_attention_prefill(Q.cuda(), K.cuda(), V.cuda(), idx, cnt, k_budget=k, b_q=bq, b_k=bk, gqa_shared=True)
    torch.cuda.synchronize()
    oi, oc = orc.mask(Q, K, k, bq, bk, True, gqa_shared=True)
    assert idx.shape[1] == Hkv
    _assert_mask_equal(idx.cpu().numpy(), cnt.cpu().numpy(), oi, oc)
    ei, ec = orc.expand_gqa(oi, oc, Hq)
    Oo, _ = orc.sparse_attention(Q, K, V, k, bq, bk, True, ei, ec)
    assert np.abs(o.float().cpu().numpy() - Oo).max() <= TOL[dt]


@pytest.mark.parametrize("dt,dist", [(torch.float32, "iid"), (torch.bfloat16, "int")])
@pytest.mark.parametrize("chunks", [1, 4])
def test_mask_gqa_shared_decode_parity(orc, dt, dist, chunks):
    B, Hq, Hkv, d, k, bk, ps = 3, 8, 2, 128, 512, 2, 64
    seq = [6000, 77, 3333]
    T = max(seq)
    Q = synth.gen_decode_q(B, Hq, d, seed=96, dtype=dt, dist=dist)
    kp, vp, bt, sl = synth.gen_paged_direct(B, Hkv, seq, d, ps, seed=96, dtype=dt, dist=dist)
    idx, cnt = H.mask_estimate_paged(Q.cuda(), kp.cuda(), bt.cuda(), sl.cuda(), T, k_budget=k, b_q=1, b_k=bk,
                                     chunks=chunks, gqa_shared=True)
    o = H.sparse_attention_decode(Q.cuda(), kp.cuda(), vp.cuda(), bt.cuda(), sl.cuda(), T, idx, cnt, k_budget=k, b_q=1,
                                  b_k=bk, gqa_shared=True)
    torch.cuda.synchronize()
    mode = orc.F32L if dt == torch.float32 else orc.F32C
    oi, oc = orc.mask_paged(Q, kp, bt, sl, k, 1, bk, True, mode=mode, chunks=chunks, gqa_shared=True)
    _assert_mask_equal(idx.cpu().numpy(), cnt.cpu().numpy(), oi, oc)
    ei, ec = orc.expand_gqa(oi, oc, Hq)
    Oo, _ = orc.sparse_attention_paged(Q, kp, vp, bt, sl, k, 1, bk, True, ei, ec)
    assert np.abs(o.float().cpu().numpy() - Oo).max() <= TOL[dt]


@pytest.mark.parametrize("chunk", [1, 3])
def test_hip_attention_host_pipelined_equals_device(chunk):
    """The pinned-host pipelined layer (3 streams, double-buffered head chunks) gives bit-for-bit the
    device layer's output (results never depend on launch composition, PIN-9)."""
    B, Hq, Hkv, T = 2, 8, 4, 1500
    Q, K, V = synth.gen_qkv(B, Hq, Hkv, T, T, 128, "llm", seed=97, dtype=torch.bfloat16)
    ref = H.hip_attention(Q.cuda(), K.cuda(), V.cuda(), k_budget=256, b_q=32, b_k=2)
    Qh, Kh, Vh = Q.pin_memory(), K.pin_memory(), V.pin_memory()
    Oh = torch.empty_like(Q).pin_memory()
    done = H.hip_attention_host(Qh, Kh, Vh, Oh, k_budget=256, b_q=32, b_k=2, kv_heads_per_chunk=chunk)
    done.synchronize()
    torch.cuda.synchronize()
    assert torch.equal(Oh, ref.cpu())


def test_vote_edge_cases(orc):
    """Empty sample rows, all-identical samples, theta = n_e with disjoint samples (empty result)."""
    n, units = 8, 4
    I = torch.full((3, units, n), -1, dtype=torch.int32)
    C = torch.zeros((3, units), dtype=torch.int32)
    I[:, 1, :3] = torch.tensor([2, 5, 9], dtype=torch.int32)       # identical in every sample
    C[:, 1] = 3
    for e in range(3):                                              # disjoint
        I[e, 2, :2] = torch.tensor([10 * e, 10 * e + 1], dtype=torch.int32)
        C[e, 2] = 2
    I[0, 3, :n] = torch.arange(n, dtype=torch.int32)                # one full row, others empty
    C[0, 3] = n
    for theta, tau in ((1, 0), (1, 1), (3, 1), (2, 0)):
        gi, gc = H.mask_vote(I.cuda(), C.cuda(), theta=theta, tau=tau)
        oi, oc = orc.vote(I, C, theta, tau)
        torch.cuda.synchronize()
        assert np.array_equal(gi.cpu().numpy(), oi) and np.array_equal(gc.cpu().numpy(), oc)
    assert oc[0] == 0


def test_gqa_shared_with_sinkwin_prefill(orc):
    """GQA-shared mask + sink / window tokens in the prefill attention (the two options compose)."""
    B, Hq, Hkv, T, k, bq, bk = 1, 4, 2, 900, 128, 16, 2
    Q, K, V = synth.gen_qkv(B, Hq, Hkv, T, T, 128, "int", seed=98, dtype=torch.bfloat16)
    idx, cnt = H.mask_estimate(Q.cuda(), K.cuda(), k_budget=k, b_q=bq, b_k=bk, gqa_shared=True)
    o = H.sparse_attention_prefill(Q.cuda(), K.cuda(), V.cuda(), idx, cnt, k_budget=k, b_q=bq, b_k=bk, sink=32,
                                   window=128, gqa_shared=True)
    torch.cuda.synchronize()
    oi, oc = orc.mask(Q, K, k, bq, bk, True, gqa_shared=True)
    _assert_mask_equal(idx.cpu().numpy(), cnt.cpu().numpy(), oi, oc)
    ei, ec = orc.expand_gqa(oi, oc, Hq)
    Oo, _ = orc.sparse_attention(Q, K, V, k, bq, bk, True, ei, ec, sink=32, window=128)
    assert np.abs(o.float().cpu().numpy() - Oo).max() <= TOL[torch.bfloat16]


def test_vote_max_size(orc):
    """n_e = 16 samples of n = 256 (the largest staged list, 4096 entries) — bit-exact vs the oracle."""
    B, Hq, nqb, n, n_e = 1, 2, 24, 256, 16
    hi = torch.randint(256, 900, (B, Hq, nqb), generator=torch.Generator().manual_seed(3))
    samples = [synth.gen_block_indices(B, Hq, nqb, n, hi, seed=200 + e) for e in range(n_e)]
    I, C = torch.stack([s[0] for s in samples]), torch.stack([s[1] for s in samples])
    for theta, tau in ((1, 0), (8, 1), (16, 1)):
        gi, gc = H.mask_vote(I.cuda(), C.cuda(), theta=theta, tau=tau)
        oi, oc = orc.vote(I, C, theta, tau)
        torch.cuda.synchronize()
        assert np.array_equal(gi.cpu().numpy(), oi) and np.array_equal(gc.cpu().numpy(), oc)


# ------------------------------------------------------------------------------------------------
# Split-K single-row attention (decode) and the dynamic job queue
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("B,Hq,Hkv,sw", [
    (2, 4, 1, False),    # 8 units: S = 8, most splits empty (<= 4 chunks)
    (16, 32, 8, True),   # 512 units (the C3 shape): S = 3, sink + window extras
    (20, 32, 8, False),  # 640 units >= the GPU's 592 slots: no split, dynamic queue
])
def test_decode_split_k_parity(orc, B, Hq, Hkv, sw):
    """Split-K partials merged in the kernel (max-rescaled softmax states) == the fp64 oracle on the
    oracle's own selection, for split counts 8 / 3 / 1 (units below / near / above the CTA slots),
    ragged sequence lengths (some shorter than one chunk, so whole splits are empty), bf16 2e-2,
    lse 1e-3."""
    d, k, bk, ps = 128, 512, 2, 16
    rng = np.random.default_rng(B)
    seq = [int(x) for x in rng.integers(1, 3000, size=B)]
    seq[0] = 1
    T = max(seq)
    Q = synth.gen_decode_q(B, Hq, d, seed=31 + B, dtype=torch.bfloat16)
    kp, vp, bt, sl = synth.gen_paged_direct(B, Hkv, seq, d, ps, seed=31 + B, dtype=torch.bfloat16)
    oi, oc = orc.mask_paged(Q, kp, bt, sl, k, 1, bk, True)
    kw = dict(sink=32, window=128) if sw else {}
    o, lse = H.sparse_attention_decode(Q.cuda(), kp.cuda(), vp.cuda(), bt.cuda(), sl.cuda(), T,
                                       torch.from_numpy(oi).cuda(), torch.from_numpy(oc).cuda(), k_budget=k, b_q=1,
                                       b_k=bk, causal=True, return_lse=True, **kw)
    torch.cuda.synchronize()
    Oo, lo = orc.sparse_attention_paged(Q, kp, vp, bt, sl, k, 1, bk, True, oi, oc, **kw)
    assert np.abs(o.float().cpu().numpy() - Oo).max() <= TOL[torch.bfloat16]
    assert np.abs(lse.cpu().numpy() - lo).max() <= 1e-3


@pytest.mark.parametrize("Tq,causal,sw", [(1, True, False), (40, True, False), (40, True, True), (40, False, True)])
def test_single_row_prefill_parity(orc, Tq, causal, sw):
    """Single-row query blocks through the contiguous prefill entry (the decode kernel): T_q = 1
    (split-K), and b_q = 1 with T_q = 40 rows at increasing positions, where the token-level causal
    mask cuts selected blocks and the sink / window sets differ per row."""
    B, Hq, Hkv, Tk, d, k, bk = 3, 4, 2, 2500, 128, 256, 2
    Q, K, V = synth.gen_qkv(B, Hq, Hkv, Tq, Tk, d, "iid", seed=41, dtype=torch.bfloat16)
    hi = torch.tensor([[[_visible(t, 1, bk, Tq, Tk, causal) for t in range(Tq)] for _ in range(Hq)] for _ in range(B)])
    idx, cnt = synth.gen_block_indices(B, Hq, Tq, k // bk, hi, seed=41)
    kw = dict(sink=32, window=128) if sw else {}
    o, lse = H.sparse_attention_prefill(Q.cuda(), K.cuda(), V.cuda(), idx.cuda(), cnt.cuda(), k_budget=k, b_q=1,
                                        b_k=bk, causal=causal, return_lse=True, **kw)
    torch.cuda.synchronize()
    Oo, lo = orc.sparse_attention(Q, K, V, k, 1, bk, causal, idx.numpy(), cnt.numpy(), **kw)
    assert np.abs(o.float().cpu().numpy() - Oo).max() <= TOL[torch.bfloat16]
    fin = np.isfinite(lo)
    assert np.array_equal(fin, np.isfinite(lse.cpu().numpy()))
    assert np.abs(lse.cpu().numpy()[fin] - lo[fin]).max() <= 1e-3


def test_concurrent_streams_own_workspaces():
    """Each call gets its own workspace (job counter, split-K partials), so the same launches
    issued concurrently on two streams give the bits of the sequential run."""
    B, Hq, Hkv, d, k, bk, ps = 16, 32, 8, 128, 512, 2, 64
    seq = [4096] * B
    q = synth.gen_decode_q(B, Hq, d, seed=51).cuda()
    kp, vp, bt, sl = (x.cuda() for x in synth.gen_paged_direct(B, Hkv, seq, d, ps, seed=51))
    Q, K, V = (x.cuda() for x in synth.gen_qkv(1, 8, 8, 8192, 8192, d, "llm", seed=52))
    kw = dict(k_budget=k, b_q=1, b_k=bk, causal=True)
    ref_i, ref_c = H.mask_estimate_paged(q, kp, bt, sl, 4096, **kw)
    ref_o = H.sparse_attention_decode(q, kp, vp, bt, sl, 4096, ref_i, ref_c, **kw)
    ref_pi, ref_pc = H.mask_estimate(Q, K)
    ref_po = H.sparse_attention_prefill(Q, K, V, ref_pi, ref_pc)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        s1.wait_stream(torch.cuda.current_stream())
        s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s1):
            i1, c1 = H.mask_estimate_paged(q, kp, bt, sl, 4096, **kw)
            o1 = H.sparse_attention_decode(q, kp, vp, bt, sl, 4096, i1, c1, **kw)
        with torch.cuda.stream(s2):
            pi, pc = H.mask_estimate(Q, K)
            po = H.sparse_attention_prefill(Q, K, V, pi, pc)
        torch.cuda.synchronize()
        assert torch.equal(i1, ref_i) and torch.equal(o1, ref_o)
        assert torch.equal(pi, ref_pi) and torch.equal(po, ref_po)


def test_decode_attention_batch_composition_invariant():
    """Split-K is chosen from the unit count (S = min(8, CTA slots / units)), but the output of a unit
    does not depend on it: every path merges the same 128-key chunk states in chunk order.  One
    sequence alone (32 units: split 8) and inside a batch of 20 (640 units: no split) give the same
    bits, lse included; so do sequence subsets (the decode batch shard of dist.py)."""
    B, Hq, Hkv, d, k, bk, ps = 20, 32, 8, 128, 512, 2, 16
    seq = [3000 - 37 * b for b in range(B)]
    q = synth.gen_decode_q(B, Hq, d, seed=71).cuda()
    kp, vp, bt, sl = (x.cuda() for x in synth.gen_paged_direct(B, Hkv, seq, d, ps, seed=71))
    kw = dict(k_budget=k, b_q=1, b_k=bk, causal=True, sink=32, window=128, return_lse=True)
    idx, cnt = H.mask_estimate_paged(q, kp, bt, sl, max(seq), k_budget=k, b_q=1, b_k=bk)
    o_all, l_all = H.sparse_attention_decode(q, kp, vp, bt, sl, max(seq), idx, cnt, **kw)
    for lo, hi in ((0, 1), (5, 6), (3, 7), (10, 20)):
        o, l = H.sparse_attention_decode(q[lo:hi].contiguous(), kp, vp, bt[lo:hi].contiguous(), sl[lo:hi].contiguous(),
                                         max(seq[lo:hi]), idx[lo:hi].contiguous(), cnt[lo:hi].contiguous(), **kw)
        torch.cuda.synchronize()
        assert torch.equal(o, o_all[lo:hi]) and torch.equal(l, l_all[lo:hi]), (lo, hi)
