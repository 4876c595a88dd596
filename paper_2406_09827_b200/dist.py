"""Multi-GPU sharding of the HiP hot path (one process per GPU, torch.distributed over NCCL).

Every (batch, head, query block) unit of HiP is independent given its head's K/V (Alg. 1 runs "for
each query block"; decoding "for each head"), so the path partitions with no exchange
inside the hot loop.  The only collective is the final gather of the output (BASELINE.json
north_star: "NCCL over NVLink used only for the final gather").

  heads     rank r owns heads [r H/G, (r+1) H/G) of every sequence (default; C2/C4/C5)
  sequence  rank r owns a contiguous range of query blocks of every head whose boundaries balance
            the per-block cost model ((n_it(q) + 3) n gathered blocks, logarithmic in position),
            for B*H < G or very long T.  A query range [t0, t1) is run as its own problem on
            (Q[t0:t1], K[:t1], V[:t1]): with bottom-right alignment (reading G7) its rows sit at the
            same key positions, so the result is bit-identical to the unsharded run.

Sharding changes no arithmetic: sharded outputs equal single-GPU outputs bit-for-bit (PIN-9).
"""
from __future__ import annotations

import math
from typing import Callable, List, Sequence, Tuple

import torch
import torch.distributed as dist


def head_range(H: int, world: int, rank: int) -> range:
    if H % world:
        raise ValueError(f"{H} heads do not divide over {world} ranks")
    per = H // world
    return range(rank * per, (rank + 1) * per)


def block_cost(q: int, bq: int, bk: int, k: int, T: int) -> float:
    """Gathered key blocks of query block q (causal, T_q = T_k = T): tree search
    2n + (n_it - 1) n when B_q > n (PIN-7), plus n blocks of K and V for the attention."""
    n = k // bk
    Bq = min(((q + 1) * bq - 1) // bk + 1, (T + bk - 1) // bk)
    if Bq <= n:
        return float(Bq * 2)
    it = math.ceil(math.log2(math.ceil(Bq / n)))
    return float(2 * n + (it - 1) * n + 2 * n)


def balanced_block_ranges(T: int, bq: int, bk: int, k: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous query-block ranges [q0, q1) per rank with near-equal modelled cost."""
    nqb = (T + bq - 1) // bq
    costs = [block_cost(q, bq, bk, k, T) for q in range(nqb)]
    total = sum(costs)
    bounds, acc, r = [0], 0.0, 1
    for q, c in enumerate(costs):
        acc += c
        while r < world and acc >= total * r / world:
            bounds.append(q + 1)
            r += 1
    while len(bounds) < world:
        bounds.append(nqb)
    bounds.append(nqb)
    return [(bounds[i], bounds[i + 1]) for i in range(world)]


def gather_heads(o_shard: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather head shards [B, H/G, T, d] -> [B, H, T, d] (ncclAllGather on NVLink)."""
    world = dist.get_world_size(group)
    B, h, T, d = o_shard.shape
    out = torch.empty((world * B, h, T, d), dtype=o_shard.dtype, device=o_shard.device)
    dist.all_gather_into_tensor(out, o_shard.contiguous(), group=group)
    return out.view(world, B, h, T, d).permute(1, 0, 2, 3, 4).reshape(B, world * h, T, d)


def gather_rows(o_shard: torch.Tensor, ranges: Sequence[Tuple[int, int]], bq: int, T: int, group=None) -> torch.Tensor:
    """All-gather query-range shards (rank r holds rows [q0 bq, min(q1 bq, T))) -> [B, H, T, d]."""
    world = dist.get_world_size(group)
    rows = [min(q1 * bq, T) - q0 * bq for q0, q1 in ranges]
    mx = max(rows)
    B, H, r, d = o_shard.shape
    pad = torch.zeros(B, H, mx, d, dtype=o_shard.dtype, device=o_shard.device)
    pad[:, :, :r] = o_shard
    out = torch.empty((world * B, H, mx, d), dtype=o_shard.dtype, device=o_shard.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    out = out.view(world, B, H, mx, d)
    return torch.cat([out[i, :, :, : rows[i]] for i in range(world)], dim=2)


def sharded_layer(layer: Callable, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, mode: str = "heads",
                  bq: int = 32, bk: int = 2, k_budget: int = 512, group=None) -> torch.Tensor:
    """Run `layer(q, k, v) -> o` (e.g. hipattn.hip_attention with fixed params) on this rank's shard
    of the FULL inputs and return the gathered [B, H, T, d] output on every rank."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if mode == "heads":
        Hq, Hkv = q.shape[1], k.shape[1]
        hr = head_range(Hq, world, rank)
        g = Hq // Hkv
        if hr.start % g or len(hr) % g:
            raise ValueError("head shards must hold whole GQA groups")
        kr = range(hr.start // g, hr.stop // g)
        o = layer(q[:, hr.start:hr.stop], k[:, kr.start:kr.stop], v[:, kr.start:kr.stop])
        return gather_heads(o, group)
    if mode == "sequence":
        T = q.shape[2]
        if k.shape[2] != T:
            raise ValueError("sequence sharding expects T_q == T_k (prefill)")
        ranges = balanced_block_ranges(T, bq, bk, k_budget, world)
        q0, q1 = ranges[rank]
        t0, t1 = q0 * bq, min(q1 * bq, T)
        o = layer(q[:, :, t0:t1], k[:, :, :t1], v[:, :, :t1])
        return gather_rows(o, ranges, bq, T, group)
    raise ValueError(mode)
