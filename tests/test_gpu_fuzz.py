"""Randomised GPU-vs-oracle parity over the shape space the C ABI accepts (seeded, -m gpu).

Each case draws (B, H_q, H_kv, T_q, T_k, d, k, b_q, b_k, causal, dtype, contiguous or paged) from a
fixed generator, so the run is reproducible, and crosses the combinations the hand-written cases in
test_gpu_parity.py do not enumerate: every kernel the dispatch in csrc/api.cu can pick (tcgen05 mask
and attention, the CUDA-core fp32 / exact kernels, the decode GEMV, the single-row attention, d = 64),
ragged tails, T_q < T_k, b_q > T_q, b_k > T_k, n = 1, GQA ratios, non-causal, sink + sliding window.

Bars:
  * mask: bit-exact with the oracle in the order the dispatched kernel computes in — integer-valued
    bf16 inputs (every fp32 sum exact, any order) on the tcgen05 / CUDA-core kernels; fp32 with
    HIP_FLAG_EXACT_SCORES == oracle F32C; fp32 without it == F32L where the decode GEMV runs
    (min(b_q, T_q) <= 4 rows, b_k <= 16, power of two), F32C otherwise.
  * attention on the ORACLE's mask (no GPU output ever feeds the oracle): max-abs <= 1e-4 (fp32) /
    2e-2 (bf16), lse <= 1e-3 where finite, identical -inf pattern.
"""
import numpy as np
import pytest
import torch

from paper_2406_09827_b200 import hipattn as H
from paper_2406_09827_b200 import synth

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-4, torch.bfloat16: 2e-2}
N_CASES = 96


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    H.load()


def _case(i):
    """Case i of the fixed stream: a dict of shape / option parameters, always a valid ABI call."""
    r = np.random.default_rng(20261018 + 7919 * i)
    dt = torch.bfloat16 if r.random() < 0.6 else torch.float32
    d = 128 if r.random() < 0.8 else 64
    Hkv = int(r.choice([1, 2]))
    Hq = Hkv * int(r.choice([1, 2, 4]))
    B = int(r.choice([1, 2]))
    bk = int(r.choice([1, 2, 2, 4, 8, 16]))
    bq = int(r.choice([1, 4, 16, 32, 32, 64]))
    n = int(r.choice([1, 8, 32, 64, 128, 256]))
    k = n * bk
    Tk = int(r.integers(1, 2600))
    causal = bool(r.random() < 0.75)
    Tq = int(r.integers(1, Tk + 1)) if r.random() < 0.4 else Tk
    if not causal and r.random() < 0.3:
        Tq = int(r.integers(1, 700))  # non-causal: any T_q
    paged = bool(r.random() < 0.25)
    if paged:  # decode / speculative-decode regime over a paged cache
        Tq = min(Tq, int(r.choice([1, 1, 4, 16, 64])))
    ps = int(r.choice([p for p in (16, 32, 64) if p % bk == 0] or [bk]))
    sink = window = 0
    if r.random() < 0.3:  # attention sink + sliding window, sink + window + b_q - 1 <= 256
        sink, window = int(r.choice([0, 4, 32])), int(r.choice([0, 16, 128]))
        if sink + window + bq - 1 > 256:
            sink, window = 4, 16
    return dict(dt=dt, d=d, B=B, Hq=Hq, Hkv=Hkv, Tq=Tq, Tk=Tk, bq=bq, bk=bk, k=k, causal=causal, paged=paged,
                ps=ps, sink=sink, window=window)


def _decode_gemv(c):
    """Mirror of csrc/mask_decode.cu mask_decode_supported for the plain mask (group = 1)."""
    rows = min(c["bq"], c["Tq"])
    return rows <= 4 and c["bk"] <= 16 and (c["bk"] & (c["bk"] - 1)) == 0 and c["d"] in (64, 128)


def _to_paged(K, V, ps, seed):
    """Contiguous [B, H_kv, T, d] -> ([pages, H_kv, ps, d] x 2, block table, seq lens), pages in a seeded
    permuted order (the oracle reads the same pages through the same table)."""
    B, Hkv, T, d = K.shape
    npg = -(-T // ps)
    perm = torch.randperm(B * npg, generator=torch.Generator().manual_seed(seed))
    kp = torch.zeros(B * npg, Hkv, ps, d, dtype=K.dtype)
    vp = torch.zeros_like(kp)
    bt = torch.zeros(B, npg, dtype=torch.int32)
    for b in range(B):
        for j in range(npg):
            p = int(perm[b * npg + j])
            bt[b, j] = p
            t0, t1 = j * ps, min((j + 1) * ps, T)
            kp[p, :, : t1 - t0] = K[b, :, t0:t1]
            vp[p, :, : t1 - t0] = V[b, :, t0:t1]
    return kp, vp, bt, torch.full((B,), T, dtype=torch.int32)


@pytest.mark.parametrize("i", range(N_CASES))
def test_fuzz_mask_and_attention(orc, i):
    c = _case(i)
    dt, causal, k, bq, bk = c["dt"], c["causal"], c["k"], c["bq"], c["bk"]
    dist = "int" if dt == torch.bfloat16 else ("llm" if i % 2 else "iid")
    Q, K, V = synth.gen_qkv(c["B"], c["Hq"], c["Hkv"], c["Tq"], c["Tk"], c["d"], dist, seed=100 + i, dtype=dt)
    if c["paged"]:
        kp, vp, bt, sl = _to_paged(K, V, c["ps"], seed=100 + i)
        T = c["Tk"]
        run_mask = lambda exact: H.mask_estimate_paged(  # noqa: E731
            Q.cuda(), kp.cuda(), bt.cuda(), sl.cuda(), T, k_budget=k, b_q=bq, b_k=bk, causal=causal, exact=exact)
        oracle_mask = lambda mode: orc.mask_paged(Q, kp, bt, sl, k, bq, bk, causal, mode=mode)  # noqa: E731
    else:
        run_mask = lambda exact: H.mask_estimate(Q.cuda(), K.cuda(), k_budget=k, b_q=bq, b_k=bk,  # noqa: E731
                                                 causal=causal, exact=exact)
        oracle_mask = lambda mode: orc.mask(Q, K, k, bq, bk, causal, mode=mode)  # noqa: E731

    # mask: the dispatched kernel's own order
    oi, oc = oracle_mask(orc.F32C)
    gi, gc = run_mask(False)
    torch.cuda.synchronize()
    if dt == torch.float32 and _decode_gemv(c):
        oi_l, oc_l = oracle_mask(orc.F32L)
        ref_i, ref_c = oi_l, oc_l
    else:
        ref_i, ref_c = oi, oc
    gi, gc = gi.cpu().numpy(), gc.cpu().numpy()
    assert np.array_equal(gc, ref_c), f"case {c}: cnt differs"
    bad = np.argwhere((gi != ref_i).any(-1))
    assert len(bad) == 0, f"case {c}: {len(bad)} query blocks differ, first {bad[:3].tolist()}"
    if dt == torch.float32:  # HIP_FLAG_EXACT_SCORES: the sequential chain == F32C
        ei, ec = run_mask(True)
        torch.cuda.synchronize()
        assert np.array_equal(ei.cpu().numpy(), oi) and np.array_equal(ec.cpu().numpy(), oc), f"case {c}: exact"

    # attention on the oracle's selection (with the case's sink / sliding window, if any)
    sw = (c["sink"], c["window"])
    idx, cnt = torch.from_numpy(oi).cuda(), torch.from_numpy(oc).cuda()
    if c["paged"]:
        o, lse = H.sparse_attention_decode(Q.cuda(), kp.cuda(), vp.cuda(), bt.cuda(), sl.cuda(), T, idx, cnt,
                                           k_budget=k, b_q=bq, b_k=bk, causal=causal, sink=sw[0], window=sw[1],
                                           return_lse=True)
        Oo, lo = orc.sparse_attention_paged(Q, kp, vp, bt, sl, k, bq, bk, causal, oi, oc, sink=sw[0], window=sw[1])
    else:
        o, lse = H.sparse_attention_prefill(Q.cuda(), K.cuda(), V.cuda(), idx, cnt, k_budget=k, b_q=bq, b_k=bk,
                                            causal=causal, sink=sw[0], window=sw[1], return_lse=True)
        Oo, lo = orc.sparse_attention(Q, K, V, k, bq, bk, causal, oi, oc, sink=sw[0], window=sw[1])
    torch.cuda.synchronize()
    err = float(np.abs(o.float().cpu().numpy() - Oo).max())
    assert err <= TOL[dt], f"case {c}: attention max-abs {err}"
    lg = lse.cpu().numpy()
    fin = np.isfinite(lo)
    assert np.array_equal(np.isfinite(lg), fin), f"case {c}: lse -inf pattern"
    if fin.any():
        assert float(np.abs(lg[fin] - lo[fin]).max()) <= 1e-3, f"case {c}: lse"


def _option_case(i):
    """Case i of the mask-option stream: shape plus a random combination of the SURVEY §8(f) options
    (stridden partial top-k S, top-r, ensemble jitter R / seed, GQA-shared masks)."""
    r = np.random.default_rng(9001 + 104729 * i)
    dt = torch.bfloat16 if r.random() < 0.5 else torch.float32
    Hkv = int(r.choice([1, 2]))
    Hq = Hkv * int(r.choice([1, 2, 4]))
    bk = int(r.choice([1, 2, 2, 4]))
    n = int(r.choice([16, 64, 128, 256]))
    Tk = int(r.integers(64, 3000))
    Tq = Tk if r.random() < 0.6 else int(r.integers(1, Tk + 1))
    bq = int(r.choice([1, 8, 16, 32]))
    gqa = bool(r.random() < 0.3)
    if gqa:
        bq = min(bq, 32 // (Hq // Hkv))  # the group's rows share one <= 32-row tile
    return dict(dt=dt, B=int(r.choice([1, 2])), Hq=Hq, Hkv=Hkv, Tq=Tq, Tk=Tk, bq=bq, bk=bk, k=n * bk,
                causal=bool(r.random() < 0.8), chunks=int(r.choice([1, 1, 2, 4])), top_r=int(r.choice([0, 0, 16, 40])),
                jitter=int(r.choice([0, 0, 3])), seed=int(r.integers(0, 1000)), gqa=gqa)


@pytest.mark.parametrize("i", range(48))
def test_fuzz_mask_options(orc, i):
    """Every option combination against the oracle, bit-exact in the dispatched kernel's order."""
    c = _option_case(i)
    dt = c["dt"]
    dist = "int" if dt == torch.bfloat16 else "llm"
    Q, K, _ = synth.gen_qkv(c["B"], c["Hq"], c["Hkv"], c["Tq"], c["Tk"], 128, dist, seed=300 + i, dtype=dt,
                            make_v=False)
    opt = dict(chunks=c["chunks"], top_r=c["top_r"], jitter=c["jitter"], seed=c["seed"])
    gi, gc = H.mask_estimate(Q.cuda(), K.cuda(), k_budget=c["k"], b_q=c["bq"], b_k=c["bk"], causal=c["causal"],
                             gqa_shared=c["gqa"], **opt)
    torch.cuda.synchronize()
    group = c["Hq"] // c["Hkv"] if c["gqa"] else 1
    gemv = min(c["bq"], c["Tq"]) * group <= 4 and c["bk"] <= 16
    mode = orc.F32L if (dt == torch.float32 and gemv) else orc.F32C
    oi, oc = orc.mask(Q, K, c["k"], c["bq"], c["bk"], c["causal"], mode=mode, gqa_shared=c["gqa"], **opt)
    gi, gc = gi.cpu().numpy(), gc.cpu().numpy()
    assert np.array_equal(gc, oc), f"case {c}: cnt differs"
    bad = np.argwhere((gi != oi).any(-1))
    assert len(bad) == 0, f"case {c}: {len(bad)} query blocks differ, first {bad[:3].tolist()}"


def _decode_case(i):
    """Case i of the decode stream: a batch of sequences of mixed lengths on a paged cache."""
    r = np.random.default_rng(424242 + 7727 * i)
    dt = torch.bfloat16 if r.random() < 0.6 else torch.float32
    B = int(r.integers(1, 7))
    Hkv = int(r.choice([1, 2, 4]))
    Hq = Hkv * int(r.choice([1, 2, 4]))
    bk = int(r.choice([1, 2, 2, 4]))
    ps = int(r.choice([p for p in (16, 32, 64) if p % bk == 0]))
    n = int(r.choice([8, 64, 256]))
    seq = [int(x) for x in r.integers(1, 6000, size=B)]
    Tq = int(r.choice([1, 1, 1, 4]))
    seq = [max(s, Tq) for s in seq]
    gqa = bool(r.random() < 0.25)
    sw = (32, 128) if r.random() < 0.4 else (0, 0)
    return dict(dt=dt, B=B, Hq=Hq, Hkv=Hkv, bk=bk, ps=ps, k=n * bk, seq=seq, Tq=Tq, gqa=gqa, sink=sw[0], window=sw[1],
                chunks=int(r.choice([1, 1, 2])), top_r=int(r.choice([0, 0, 32])), jitter=int(r.choice([0, 0, 2])),
                seed=int(r.integers(0, 100)))


@pytest.mark.parametrize("i", range(32))
def test_fuzz_decode_mixed_lengths(orc, i):
    """Paged decode over a batch of different lengths (and T_q = 4 speculative rows), with random
    mask options and sink / window: mask bit-exact, attention within tolerance of the oracle."""
    c = _decode_case(i)
    dt, bk, k, Tq = c["dt"], c["bk"], c["k"], c["Tq"]
    dist = "int" if dt == torch.bfloat16 else "iid"
    q = synth.gen_decode_q(c["B"], c["Hq"], 128, seed=500 + i, dtype=dt, dist=dist, Tq=Tq)
    kp, vp, bt, sl = synth.gen_paged_direct(c["B"], c["Hkv"], c["seq"], 128, c["ps"], seed=500 + i, dtype=dt,
                                            dist=dist)
    T = max(c["seq"])
    bq = 32 // (c["Hq"] // c["Hkv"]) if c["gqa"] else 32
    opt = dict(chunks=c["chunks"], top_r=c["top_r"], jitter=c["jitter"], seed=c["seed"])
    gi, gc = H.mask_estimate_paged(q.cuda(), kp.cuda(), bt.cuda(), sl.cuda(), T, k_budget=k, b_q=bq, b_k=bk,
                                   causal=True, gqa_shared=c["gqa"], **opt)
    torch.cuda.synchronize()
    group = c["Hq"] // c["Hkv"] if c["gqa"] else 1
    gemv = min(bq, Tq) * group <= 4 and bk <= 16
    mode = orc.F32L if (dt == torch.float32 and gemv) else orc.F32C
    oi, oc = orc.mask_paged(q, kp, bt, sl, k, bq, bk, True, mode=mode, gqa_shared=c["gqa"], **opt)
    gi, gc = gi.cpu().numpy(), gc.cpu().numpy()
    assert np.array_equal(gc, oc), f"case {c}: cnt differs"
    bad = np.argwhere((gi != oi).any(-1))
    assert len(bad) == 0, f"case {c}: {len(bad)} units differ, first {bad[:3].tolist()}"
    o, lse = H.sparse_attention_decode(q.cuda(), kp.cuda(), vp.cuda(), bt.cuda(), sl.cuda(), T,
                                       torch.from_numpy(oi).cuda(), torch.from_numpy(oc).cuda(), k_budget=k, b_q=bq,
                                       b_k=bk, causal=True, sink=c["sink"], window=c["window"], return_lse=True,
                                       gqa_shared=c["gqa"])
    torch.cuda.synchronize()
    ei, ec = orc.expand_gqa(oi, oc, c["Hq"]) if c["gqa"] else (oi, oc)  # the group's mask for each head
    Oo, lo = orc.sparse_attention_paged(q, kp, vp, bt, sl, k, bq, bk, True, ei, ec, sink=c["sink"],
                                        window=c["window"])
    err = float(np.abs(o.float().cpu().numpy() - Oo).max())
    assert err <= TOL[dt], f"case {c}: attention max-abs {err}"
    fin = np.isfinite(lo)
    assert np.array_equal(np.isfinite(lse.cpu().numpy()), fin), f"case {c}: lse -inf pattern"
    if fin.any():
        assert float(np.abs(lse.cpu().numpy()[fin] - lo[fin]).max()) <= 1e-3, f"case {c}: lse"


@pytest.mark.parametrize("i", range(16))
def test_fuzz_tcgen05_gaussian_replay(orc, i):
    """The tcgen05 mask on Gaussian bf16 inputs over random shapes (b_q, b_k, n, T, causal, GQA):
    sampled units checked as in test_gpu_replay — every dumped score within the fp32 error bound of
    fp64, the oracle's selection replayed on the GPU's scores equals the GPU mask, and any difference
    from the fp64 mask is certified at its first divergent iteration."""
    from test_gpu_replay import _slot_map, _stats, check_unit
    r = np.random.default_rng(77 + 31337 * i)
    Hkv = int(r.choice([1, 2]))
    Hq = Hkv * int(r.choice([1, 2]))
    bq = int(r.choice([1, 4, 16, 32]))
    bk = int(r.choice([1, 2, 4, 8, 16, 32]))
    n = int(r.choice([8, 64, 256]))
    k = n * bk
    Tk = int(r.integers(2 * n * bk // 2 + 1, 3000)) if n * bk < 3000 else 3000
    causal = bool(r.random() < 0.75)
    Tq = Tk if r.random() < 0.6 else int(r.integers(1, Tk + 1))
    d = 128
    Q, K, _ = synth.gen_qkv(1, Hq, Hkv, Tq, Tk, d, "iid" if i % 2 else "llm", seed=700 + i, dtype=torch.bfloat16,
                            make_v=False)
    nqb, nkb = -(-Tq // bq), -(-Tk // bk)
    units = sorted(set(int(u) for u in r.integers(0, Hq * nqb, size=min(48, Hq * nqb))))
    dump = torch.full((len(units), nkb), float("nan"), dtype=torch.float32, device="cuda")
    with H.debug_score_dump(_slot_map(units, Hq * nqb, "cuda"), dump):
        idx, _ = H.mask_estimate(Q.cuda(), K.cuda(), k_budget=k, b_q=bq, b_k=bk, causal=causal)
    torch.cuda.synchronize()
    gi, gs = idx.cpu().numpy(), dump.cpu().numpy()
    st = _stats()
    g = Hq // Hkv
    for s, u in enumerate(units):
        h, q = divmod(u, nqb)
        check_unit(orc, Q[:, h:h + 1], K[:, h // g:h // g + 1], k, bq, bk, causal, q, gi[0, h, q], gs[s], d, st)
    print(f"\n[fuzz replay] case {i} (bq={bq} bk={bk} n={n} Tq={Tq} Tk={Tk} causal={causal}): {st}")
    assert st["unexplained"] == 0
