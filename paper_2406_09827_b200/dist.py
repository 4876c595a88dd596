"""Multi-GPU sharding of the HiP hot path (one process per GPU, torch.distributed over NCCL).

Every (batch, head, query block) unit of HiP is independent given its head's K/V (Alg. 1 runs "for
each query block"; decoding "for each head"; jobs are laid out over (N*H, Q)),
so the path partitions with no exchange inside the hot loop.  The only collective is the final
gather of the output (BASELINE.json north_star: "heads, batch and long sequences are partitioned
... NCCL over NVLink used only for the final gather").

Prefill (T_q = T_k):
  heads     rank r owns H/G query heads (whole GQA groups).  With `chunks` = C > 1 the heads are
            assigned interleaved — chunk c of rank r is heads [(cG + r) h_c, (cG + r + 1) h_c),
            h_c = H / (G C) — so chunk c of all ranks is ONE contiguous head range of the output and
            its all-gather lands in place (B = 1) while the ranks compute chunk c + 1 (the gather runs
            on a second stream: the transfer overlaps the kernels).
  sequence  rank r owns a contiguous range of query blocks of every head, the boundaries balancing
            the per-block cost model ((n_it(q) + 4) n gathered blocks, logarithmic in position); a
            range [t0, t1) runs as its own problem on (Q[t0:t1], K[:t1], V[:t1]): with bottom-right
            alignment (reading G7) its rows sit at the same key positions, so the result is
            bit-identical to the unsharded run.
Decode (paged KV, T_q query rows per sequence):
  batch     rank r owns B / G sequences (their block-table rows and lengths); O gathers along batch.
  kvgroup   rank r owns H_kv / G kv heads with their H_q / H_kv query heads each (the page tensors are
            sliced along their head axis, a strided view the C ABI takes as is); O gathers along heads.

Sharding changes no arithmetic: sharded outputs equal single-GPU outputs bit-for-bit (PIN-9).
"""
from __future__ import annotations

import math
from typing import Callable, List, Sequence, Tuple

import torch
import torch.distributed as dist


# ------------------------------------------------------------------------------------------------
# shard maps (pure host logic)
# ------------------------------------------------------------------------------------------------
def head_range(H: int, world: int, rank: int) -> range:
    if H % world:
        raise ValueError(f"{H} heads do not divide over {world} ranks")
    per = H // world
    return range(rank * per, (rank + 1) * per)


def head_chunks(H: int, world: int, rank: int, chunks: int = 1, group: int = 1) -> List[range]:
    """Query heads of rank r as `chunks` contiguous ranges, interleaved over the ranks (see the
    module docstring); chunks = 1 is the plain contiguous split head_range.  Every range holds whole
    GQA groups of `group` query heads."""
    if chunks < 1 or H % (world * chunks):
        raise ValueError(f"{H} heads do not divide into {world} ranks x {chunks} chunks")
    hc = H // (world * chunks)
    if hc % group:
        raise ValueError(f"a chunk of {hc} query heads does not hold whole GQA groups of {group}")
    return [range((c * world + rank) * hc, (c * world + rank + 1) * hc) for c in range(chunks)]


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
    """Contiguous query-block ranges [q0, q1) per rank with near-equal modelled cost.  Boundary r is
    the first block where the cumulative cost reaches r/world of the total, clamped to
    [r, nqb - world + r] so that every rank keeps at least one query block."""
    nqb = (T + bq - 1) // bq
    if world > nqb:
        raise ValueError(f"{world} ranks for {nqb} query blocks: every rank needs at least one")
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
    for r in range(1, world):  # at least one block per rank, boundaries strictly increasing
        bounds[r] = min(max(bounds[r], bounds[r - 1] + 1), nqb - world + r)
    return [(bounds[i], bounds[i + 1]) for i in range(world)]


def batch_range(B: int, world: int, rank: int) -> range:
    if B % world:
        raise ValueError(f"batch {B} does not divide over {world} ranks")
    per = B // world
    return range(rank * per, (rank + 1) * per)


# ------------------------------------------------------------------------------------------------
# gathers (the one collective)
# ------------------------------------------------------------------------------------------------
def _gather_dim1(dst: torch.Tensor, shard: torch.Tensor, group=None):
    """dst[:, w*h:(w+1)*h] <- shard of rank w (shard [B, h, ...]).  B = 1 with a contiguous dst: the
    all-gather writes in place; otherwise through a world-major buffer and one permuting copy."""
    world = dist.get_world_size(group)
    shard = shard.contiguous()
    B, h = shard.shape[:2]
    if B == 1 and dst.is_contiguous():
        dist.all_gather_into_tensor(dst.view(world * B, h, *shard.shape[2:]), shard, group=group)
        return
    buf = torch.empty((world * B, h) + tuple(shard.shape[2:]), dtype=shard.dtype, device=shard.device)
    dist.all_gather_into_tensor(buf, shard, group=group)
    dst.copy_(buf.view(world, B, h, *shard.shape[2:]).transpose(0, 1).reshape(dst.shape))


def gather_heads(o_shard: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather contiguous head shards [B, H/G, T, d] -> [B, H, T, d] (ncclAllGather on NVLink)."""
    world = dist.get_world_size(group)
    B, h, T, d = o_shard.shape
    out = torch.empty((B, world * h, T, d), dtype=o_shard.dtype, device=o_shard.device)
    _gather_dim1(out, o_shard, group)
    return out


def gather_batch(o_shard: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather batch shards [B/G, ...] -> [B, ...] (world-major = batch order: in place)."""
    world = dist.get_world_size(group)
    out = torch.empty((world * o_shard.shape[0],) + tuple(o_shard.shape[1:]), dtype=o_shard.dtype,
                      device=o_shard.device)
    dist.all_gather_into_tensor(out, o_shard.contiguous(), group=group)
    return out


def gather_rows(o_shard: torch.Tensor, ranges: Sequence[Tuple[int, int]], bq: int, T: int, group=None) -> torch.Tensor:
    """All-gather query-range shards (rank r holds rows [q0 bq, min(q1 bq, T))) -> [B, H, T, d]."""
    world = dist.get_world_size(group)
    rows = [max(0, min(q1 * bq, T) - q0 * bq) for q0, q1 in ranges]
    mx = max(rows)
    B, H, r, d = o_shard.shape
    pad = torch.zeros(B, H, mx, d, dtype=o_shard.dtype, device=o_shard.device)
    pad[:, :, :r] = o_shard
    out = torch.empty((world * B, H, mx, d), dtype=o_shard.dtype, device=o_shard.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    out = out.view(world, B, H, mx, d)
    return torch.cat([out[i, :, :, : rows[i]] for i in range(world)], dim=2)


class ChunkGather:
    """All-gathers of per-chunk head shards on a side stream (CUDA) so that chunk c's transfer
    overlaps the kernels of chunk c + 1; synchronous on CPU (gloo).  The output [B, H, T, d] (dtype
    and device of the shards, allocated at the first push unless `out` is given) receives chunk c of
    every rank at heads [c G h_c, (c + 1) G h_c) (head_chunks' interleaved map)."""

    def __init__(self, H: int, out: torch.Tensor = None, group=None):
        self.H, self.out, self.group = H, out, group
        self.world = dist.get_world_size(group)
        self.stream = None

    def push(self, c: int, shard: torch.Tensor):
        if self.out is None:
            B, _, T, d = shard.shape
            self.out = torch.empty((B, self.H, T, d), dtype=shard.dtype, device=shard.device)
        if self.stream is None and shard.is_cuda:
            self.stream = torch.cuda.Stream(shard.device)
        hc = shard.shape[1]
        dst = self.out[:, c * self.world * hc:(c + 1) * self.world * hc]
        if not shard.is_cuda:
            _gather_dim1(dst, shard, self.group)
            return
        cur = torch.cuda.current_stream(shard.device)
        self.stream.wait_stream(cur)          # the chunk's kernels are done before it is sent
        shard.record_stream(self.stream)      # and its memory is not reused while in flight
        with torch.cuda.stream(self.stream):
            _gather_dim1(dst, shard, self.group)

    def finish(self) -> torch.Tensor:
        if self.stream is not None:
            torch.cuda.current_stream(self.out.device).wait_stream(self.stream)
        return self.out


# ------------------------------------------------------------------------------------------------
# sharded layers on FULL inputs (every rank passes the same tensors, keeps only its shard's work)
# ------------------------------------------------------------------------------------------------
def sharded_layer(layer: Callable, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, mode: str = "heads",
                  chunks: int = 1, bq: int = 32, bk: int = 2, k_budget: int = 512, group=None) -> torch.Tensor:
    """Prefill: run `layer(q, k, v) -> o` (e.g. hipattn.hip_attention with fixed params) on this
    rank's shard of the FULL inputs and return the gathered [B, H, T, d] output on every rank."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if mode == "heads":
        Hq, Hkv = q.shape[1], k.shape[1]
        g = Hq // Hkv
        ranges = head_chunks(Hq, world, rank, chunks, g)
        if chunks == 1:
            hr = ranges[0]
            return gather_heads(layer(q[:, hr.start:hr.stop], k[:, hr.start // g:hr.stop // g],
                                      v[:, hr.start // g:hr.stop // g]), group)
        gat = ChunkGather(Hq, group=group)
        for c, hr in enumerate(ranges):
            gat.push(c, layer(q[:, hr.start:hr.stop], k[:, hr.start // g:hr.stop // g],
                              v[:, hr.start // g:hr.stop // g]))
        return gat.finish()
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


def sharded_decode(step: Callable, q: torch.Tensor, k_pages: torch.Tensor, v_pages: torch.Tensor,
                   block_table: torch.Tensor, seq_lens: torch.Tensor, *, mode: str = "batch",
                   group=None) -> torch.Tensor:
    """Decode: run `step(q, k_pages, v_pages, block_table, seq_lens) -> o` (mask estimation over the
    paged cache + paged sparse attention, e.g. a HipDecoder step) on this rank's shard and return the
    gathered O [B, H_q, T_q, d] on every rank.  batch: sequences [r B/G, (r+1) B/G); kvgroup: kv heads
    [r H_kv/G, (r+1) H_kv/G) with their query heads."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if mode == "batch":
        br = batch_range(q.shape[0], world, rank)
        o = step(q[br.start:br.stop], k_pages, v_pages, block_table[br.start:br.stop].contiguous(),
                 seq_lens[br.start:br.stop].contiguous())
        return gather_batch(o, group)
    if mode == "kvgroup":
        Hq, Hkv = q.shape[1], k_pages.shape[1]
        g = Hq // Hkv
        kr = head_range(Hkv, world, rank)
        o = step(q[:, kr.start * g:kr.stop * g], k_pages[:, kr.start:kr.stop], v_pages[:, kr.start:kr.stop],
                 block_table, seq_lens)
        return gather_heads(o, group)
    raise ValueError(mode)
