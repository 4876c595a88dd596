"""Seeded synthetic inputs shared by the tests, the bench and the smoke run.

This module holds NONE of HiP's arithmetic (no scores, splits, selections or softmax): it only draws
random tensors with the shapes and structure of the paper's workloads and
moves bytes into a paged layout.  Both the CUDA path and the CPU oracle consume its output, so it is
the one module they share.

Distributions
  iid  Q, K, V ~ N(0, 1).                                    (structureless worst case)
  int  Q, K uniform integers in [-4, 4]; V ~ N(0, 1).         (every fp32 score sum is exact)
  llm  block-local, sink-heavy, partly long-range structure like LLaMA attention (P:90-95,
       P:1082-1084): segment topics u_g ~ N(0, I) for segments of 128 tokens; keys
       k~_s = z_s + u_{g(s)}; queries q~_t = z'_t + u_{src(t)}, where the source segment is drawn per
       16-token phrase of queries (neighbouring queries attend to the same places — the locality
       HiP's b_q blocks rely on): src = g(t) w.p. 0.7, else uniform over [0, g(t)];
       z, z' ~ N(0, 0.5^2 I); a sink direction w ~ N(0, I) is added as +2.5 w to the first 4 keys
       and +0.5 w to every query; RoPE (NeoX pairing (c, c + d/2), base 10 000 or 500 000).
       At d = 128 a query's own-topic logit q.k / sqrt(d) is ~11 above the rest and the 4 sink keys
       carry a share comparable to a whole topic segment: peaked, LLM-like attention rows.
Seeds: sub-seed = seed * 16 + {0: Q, 1: K, 2: V, 3: page permutation, 4: indices}.
"""
from __future__ import annotations

import torch

SEGMENT = 128
P_LOCAL = 0.7
NOISE = 0.5
SINK_KEYS = 4
SINK_K = 2.5
SINK_Q = 0.5
LLM_SCALE = 1.0
PHRASE = 16


def _gen(seed: int, sub: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) * 16 + sub)
    return g


def _rope(x: torch.Tensor, pos: torch.Tensor, base: float) -> torch.Tensor:
    """Rotary position embedding on the last dim (NeoX pairing), computed in fp32."""
    d = x.shape[-1]
    half = d // 2
    inv = base ** (-torch.arange(half, device=x.device, dtype=torch.float32) * 2.0 / d)
    ang = pos.to(torch.float32)[:, None] * inv[None, :]
    c, s = torch.cos(ang), torch.sin(ang)
    x1, x2 = x[..., :half], x[..., half:]
    return torch.cat([x1 * c - x2 * s, x1 * s + x2 * c], dim=-1)


def gen_qkv(B: int, Hq: int, Hkv: int, Tq: int, Tk: int, d: int, dist: str = "iid", seed: int = 0,
            dtype: torch.dtype = torch.bfloat16, device="cpu", rope_base: float = 10000.0,
            make_v: bool = True):
    """Q [B,Hq,Tq,d], K/V [B,Hkv,Tk,d] contiguous, rounded once to `dtype`.

    Query row t is taken to sit at key position t + Tk - Tq (bottom-right alignment)."""
    device = torch.device(device)
    gq, gk, gv = _gen(seed, 0, device), _gen(seed, 1, device), _gen(seed, 2, device)
    if dist == "iid":
        Q = torch.randn(B, Hq, Tq, d, generator=gq, device=device)
        K = torch.randn(B, Hkv, Tk, d, generator=gk, device=device)
    elif dist == "int":
        Q = torch.randint(-4, 5, (B, Hq, Tq, d), generator=gq, device=device).float()
        K = torch.randint(-4, 5, (B, Hkv, Tk, d), generator=gk, device=device).float()
    elif dist == "llm":
        nseg = (Tk + SEGMENT - 1) // SEGMENT
        topics = torch.randn(B, Hkv, nseg, d, generator=gk, device=device)
        spos = torch.arange(Tk, device=device)
        K = NOISE * torch.randn(B, Hkv, Tk, d, generator=gk, device=device) + topics[:, :, spos // SEGMENT]
        sink = torch.randn(B, Hkv, 1, d, generator=gk, device=device)
        nsink = min(SINK_KEYS, Tk)
        K[:, :, :nsink] += SINK_K * sink
        qpos = torch.arange(Tq, device=device) + (Tk - Tq)
        g = (qpos // SEGMENT).clamp(max=nseg - 1)
        # one source draw per 16-token phrase of query positions
        nph = (int(qpos[-1]) // PHRASE) + 1 if Tq > 0 else 1
        ph = qpos // PHRASE
        local = (torch.rand(B, Hq, nph, generator=gq, device=device) < P_LOCAL)[:, :, ph]
        u = torch.rand(B, Hq, nph, generator=gq, device=device)[:, :, ph]
        far = (u * (g + 1).float()).floor().long()
        src = torch.where(local, g.expand(B, Hq, Tq), far)
        grp = Hq // Hkv
        kvh = torch.arange(Hq, device=device) // grp
        tq = topics[:, kvh]  # [B,Hq,nseg,d]
        Q = NOISE * torch.randn(B, Hq, Tq, d, generator=gq, device=device)
        Q = Q + torch.gather(tq, 2, src[..., None].expand(B, Hq, Tq, d))
        Q = Q + SINK_Q * sink[:, kvh]
        Q = _rope(LLM_SCALE * Q, qpos, rope_base)
        K = _rope(LLM_SCALE * K, spos, rope_base)
    else:
        raise ValueError(f"unknown distribution {dist!r}")
    V = torch.randn(B, Hkv, Tk, d, generator=gv, device=device) if make_v else None
    cast = lambda x: None if x is None else x.to(dtype).contiguous()
    return cast(Q), cast(K), cast(V)


def gen_block_indices(B: int, Hq: int, nqb: int, n: int, hi, seed: int = 0, device="cpu",
                      edge_cases: bool = True):
    """Random selections for attention-only parity: per unit a sorted set of distinct key-block
    indices drawn from [0, hi[b,h,q]) with a random count in [0, min(n, hi)]; -1 padded.

    `hi` is an int tensor [B,Hq,nqb] supplied by the caller.  With edge_cases the first units get
    count 0, 1 and min(n, hi) so that empty, single-block and full rows are always present."""
    device = torch.device(device)
    g = _gen(seed, 4, device)
    hi = torch.as_tensor(hi, device=device).long().reshape(B * Hq * nqb)
    U = hi.numel()
    cap = torch.minimum(hi, torch.full_like(hi, n))
    cnt = (torch.rand(U, generator=g, device=device) * (cap + 1).float()).floor().long().clamp(max=cap)
    if edge_cases and U >= 3:
        cnt[0] = 0
        cnt[1] = torch.clamp(cap[1], max=1)
        cnt[2] = cap[2]
    idx = torch.full((U, n), -1, dtype=torch.int32, device=device)
    for u in range(U):
        c = int(cnt[u])
        if c == 0:
            continue
        perm = torch.randperm(int(hi[u]), generator=g, device=device)[:c]
        idx[u, :c] = torch.sort(perm).values.to(torch.int32)
    return idx.reshape(B, Hq, nqb, n), cnt.to(torch.int32).reshape(B, Hq, nqb)


def to_paged(K: torch.Tensor, V: torch.Tensor, seq_lens, page_size: int, seed: int = 0, extra_pages: int = 3):
    """Copy contiguous K/V [B,Hkv,Tmax,d] into a paged cache [num_pages,Hkv,page_size,d] whose
    physical pages are a seeded random permutation (plus a few unused pages).

    Returns (k_pages, v_pages, block_table int32 [B, max_pages], seq_lens int32 [B])."""
    B, Hkv, Tmax, d = K.shape
    device = K.device
    seq_lens = torch.as_tensor(seq_lens, dtype=torch.int32).reshape(B)
    npg = [(int(s) + page_size - 1) // page_size for s in seq_lens.tolist()]
    max_pages = max(max(npg), 1)
    total = sum(npg) + extra_pages
    perm = torch.randperm(total, generator=_gen(seed, 3, torch.device("cpu")))
    kp = torch.zeros(total, Hkv, page_size, d, dtype=K.dtype, device=device)
    vp = torch.zeros(total, Hkv, page_size, d, dtype=V.dtype, device=device)
    bt = torch.full((B, max_pages), -1, dtype=torch.int32)
    nxt = 0
    for b in range(B):
        for p in range(npg[b]):
            phys = int(perm[nxt]); nxt += 1
            bt[b, p] = phys
            s0, s1 = p * page_size, min((p + 1) * page_size, int(seq_lens[b]))
            kp[phys, :, : s1 - s0] = K[b, :, s0:s1]
            vp[phys, :, : s1 - s0] = V[b, :, s0:s1]
    # unused block-table slots point at page 0 (never dereferenced: beyond seq_len)
    bt[bt < 0] = 0
    return kp, vp, bt.to(device), seq_lens.to(device)


def gen_paged_direct(B: int, Hkv: int, seq_lens, d: int, page_size: int, seed: int = 0,
                     dtype: torch.dtype = torch.bfloat16, device="cpu", dist: str = "iid"):
    """Large decode caches straight in paged form (no contiguous copy): pages drawn iid (or int),
    physical order a seeded permutation.  Returns (k_pages, v_pages, block_table, seq_lens)."""
    device = torch.device(device)
    seq_lens = torch.as_tensor(seq_lens, dtype=torch.int32).reshape(B)
    npg = [(int(s) + page_size - 1) // page_size for s in seq_lens.tolist()]
    max_pages = max(max(npg), 1)
    total = sum(npg)
    gk, gv = _gen(seed, 1, device), _gen(seed, 2, device)
    if dist == "int":
        kp = torch.randint(-4, 5, (total, Hkv, page_size, d), generator=gk, device=device).to(dtype)
    else:
        kp = torch.randn(total, Hkv, page_size, d, generator=gk, device=device, dtype=torch.float32).to(dtype)
    vp = torch.randn(total, Hkv, page_size, d, generator=gv, device=device, dtype=torch.float32).to(dtype)
    perm = torch.randperm(total, generator=_gen(seed, 3, torch.device("cpu")))
    bt = torch.zeros((B, max_pages), dtype=torch.int32)
    nxt = 0
    for b in range(B):
        bt[b, : npg[b]] = perm[nxt: nxt + npg[b]].to(torch.int32)
        nxt += npg[b]
    return kp, vp, bt.to(device), seq_lens.to(device)


def gen_decode_q(B: int, Hq: int, d: int, seed: int = 0, dtype=torch.bfloat16, device="cpu", dist="iid",
                 Tq: int = 1):
    g = _gen(seed, 0, torch.device(device))
    if dist == "int":
        q = torch.randint(-4, 5, (B, Hq, Tq, d), generator=g, device=device).float()
    else:
        q = torch.randn(B, Hq, Tq, d, generator=g, device=device)
    return q.to(dtype).contiguous()

