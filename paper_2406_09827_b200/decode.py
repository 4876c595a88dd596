"""decode.py — the HiP decoding loop policy (Alg. 2).

Per HiP layer and decode step: if the current sequence length is divisible by the mask estimation
period r_m, estimate the attention mask (Alg. 1, O(T log T)) and cache it (O(T) space);
then run the fused sparse attention with the cached mask.  The paper's default is r_m = 8
(P:815); r_m = 1 re-estimates every step (its latency benchmarks).  Multi-query
(speculative) steps pass T_q > 1 query rows per sequence, at positions seq_len - T_q + t
(P:1154-1159); b_q <= 32 rows form one query block.

A batch holds sequences of different lengths, so the refresh decision is taken per sequence: the
new mask is estimated for the batch and kept only for the sequences whose length is divisible by
r_m (the others keep their cached rows).  Policy only: every step runs in the C-ABI kernels
(hipattn); nothing here computes on the CPU.
"""
from __future__ import annotations

import torch

from . import hipattn as H


class HipDecoder:
    """Cached-mask HiP attention for one layer of a decoder (Alg. 2 lines 8-12)."""

    def __init__(self, r_m: int = 8, k_budget: int = 512, b_k: int = 2, b_q: int = 32, causal: bool = True,
                 sink: int = 32, window: int = 128, sm_scale=None, gqa_shared: bool = False, chunks: int = 1):
        """sink / window: StreamingLLM sink and sliding-window tokens added to every row; the paper
        fixes (window, sink) = (128, 32) for every experiment (SPEC's defaults too).  With
        a cached mask (r_m > 1) the window is what covers the up to r_m - 1 tokens generated since
        the last refresh and the current token itself, so it must span at least r_m tokens.
        gqa_shared / chunks: the mask options of SURVEY §8 f3 — one mask per GQA group (reading
        G25) and the stridden partial top-k with S chunks (G21) — the low-latency decode
        configuration when the batch gives fewer units than the GPU has CTA slots."""
        if r_m < 1:
            raise ValueError("r_m must be >= 1")
        if r_m > 1 and window < r_m:
            raise ValueError(f"window={window} < r_m={r_m}: tokens generated since the last mask refresh "
                             "(including the current one) would never be attended")
        self.r_m, self.k_budget, self.b_k, self.b_q = int(r_m), int(k_budget), int(b_k), int(b_q)
        self.causal, self.sink, self.window, self.sm_scale = bool(causal), int(sink), int(window), sm_scale
        self.gqa_shared, self.chunks = bool(gqa_shared), int(chunks)
        self.idx = None
        self.cnt = None
        self.refreshes = 0  # number of steps that ran the mask estimation (for tests / stats)
        self._graphs = None  # graphed_step state: (buffers key, refresh graph, cached graph)

    def refresh_rows(self, seq_lens_host) -> list:
        """Per-sequence refresh decision for this step (Alg. 2 line 8)."""
        return [self.idx is None or int(t) % self.r_m == 0 for t in seq_lens_host]

    def step(self, q, k_pages, v_pages, block_table, seq_lens, seq_lens_host, *, return_lse: bool = False,
             stream=None):
        """One decode step: q [B, H_q, T_q, d] against the paged cache whose sequence b holds
        seq_lens[b] tokens (seq_lens_host: the same lengths on the host, which decide refreshes)."""
        max_len = int(max(int(t) for t in seq_lens_host))
        rows = self.refresh_rows(seq_lens_host)
        if any(rows):
            idx, cnt = H.mask_estimate_paged(q, k_pages, block_table, seq_lens, max_len, k_budget=self.k_budget,
                                             b_q=self.b_q, b_k=self.b_k, causal=self.causal,
                                             gqa_shared=self.gqa_shared, chunks=self.chunks, stream=stream)
            if self.idx is None or self.idx.shape != idx.shape or all(rows):
                self.idx, self.cnt = idx, cnt
            else:
                sel = torch.tensor(rows, device=idx.device)
                self.idx = torch.where(sel.view(-1, 1, 1, 1), idx, self.idx)
                self.cnt = torch.where(sel.view(-1, 1, 1), cnt, self.cnt)
            self.refreshes += 1
        return H.sparse_attention_decode(q, k_pages, v_pages, block_table, seq_lens, max_len, self.idx, self.cnt,
                                         k_budget=self.k_budget, b_q=self.b_q, b_k=self.b_k, causal=self.causal,
                                         sm_scale=self.sm_scale, sink=self.sink, window=self.window,
                                         return_lse=return_lse, gqa_shared=self.gqa_shared, stream=stream)

    def graphed_step(self, q, k_pages, v_pages, block_table, seq_lens, seq_lens_host, out):
        """The same Alg. 2 step replayed from CUDA graphs (how a serving loop launches it: one graph
        launch per step instead of a chain of host calls).  q, seq_lens, out (and the cache) are
        STATIC buffers the caller updates in place between steps.  Two graphs are captured on the
        first call for a set of buffers: refresh (mask estimation into the cached idx / cnt, then the
        sparse attention) and cached (the attention only).  The kernels take each sequence's length
        from seq_lens, so the graphs are captured once with max_seq_len = the cache capacity
        (block_table columns x page size).  Per step (Alg. 2 line 8, from seq_lens_host): every
        sequence refreshes -> the refresh graph; none -> the cached graph; a mix -> the mask is
        estimated eagerly for the batch, the refreshing rows are merged into the cached buffers,
        then the cached graph runs.  Returns out."""
        cap = int(block_table.shape[1]) * int(k_pages.shape[2])
        key = tuple(int(t.data_ptr()) for t in (q, k_pages, v_pages, block_table, seq_lens, out)) + (
            tuple(q.shape), tuple(k_pages.shape), tuple(block_table.shape))
        if self._graphs is None or self._graphs[0] != key:
            mkw = dict(k_budget=self.k_budget, b_q=self.b_q, b_k=self.b_k, causal=self.causal,
                       gqa_shared=self.gqa_shared, chunks=self.chunks)
            akw = dict(k_budget=self.k_budget, b_q=self.b_q, b_k=self.b_k, causal=self.causal, sm_scale=self.sm_scale,
                       sink=self.sink, window=self.window, gqa_shared=self.gqa_shared)
            idx, cnt = H.mask_estimate_paged(q, k_pages, block_table, seq_lens, cap, **mkw)  # buffers + warm-up
            if self.idx is not None and self.idx.shape == idx.shape:
                idx.copy_(self.idx)
                cnt.copy_(self.cnt)
            H.sparse_attention_decode(q, k_pages, v_pages, block_table, seq_lens, cap, idx, cnt, out=out, **akw)
            torch.cuda.synchronize(q.device)
            g_ref, g_att = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_ref):
                H.mask_estimate_paged(q, k_pages, block_table, seq_lens, cap, out=(idx, cnt), **mkw)
                H.sparse_attention_decode(q, k_pages, v_pages, block_table, seq_lens, cap, idx, cnt, out=out, **akw)
            with torch.cuda.graph(g_att):
                H.sparse_attention_decode(q, k_pages, v_pages, block_table, seq_lens, cap, idx, cnt, out=out, **akw)
            self._graphs = (key, g_ref, g_att, idx, cnt, cap, mkw)
            had_mask = self.idx is not None
            self.idx, self.cnt = idx, cnt
            if not had_mask:
                self.idx = None  # nothing cached yet: the first step refreshes
        _, g_ref, g_att, idx, cnt, cap, mkw = self._graphs
        rows = self.refresh_rows(seq_lens_host)
        if all(rows):
            g_ref.replay()
            self.refreshes += 1
        elif not any(rows):
            g_att.replay()
        else:
            ni, nc = H.mask_estimate_paged(q, k_pages, block_table, seq_lens, cap, **mkw)
            sel = torch.tensor(rows, device=idx.device)
            idx.copy_(torch.where(sel.view(-1, 1, 1, 1), ni, idx))
            cnt.copy_(torch.where(sel.view(-1, 1, 1), nc, cnt))
            self.refreshes += 1
            g_att.replay()
        self.idx, self.cnt = idx, cnt
        return out

