"""ctypes front-end of the CPU oracle (oracle/hip_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module; the product package never does.

Every function takes numpy arrays (or anything numpy can view) and widens them to float32 exactly
(bf16 -> fp32 is exact); the arithmetic happens in C (see the header of hip_oracle.c for the
citations of each step).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hip_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

F32C = 0  # canonical fp32: acc = fmaf(q[c], k[c], acc), c = 0..d-1 (reading G9)
F64 = 1   # fp64 dot products
F32L = 2  # reading G9b: 16 sequential fmaf segments of d/16 terms + pairwise tree (o = 8, 4, 2, 1)

_ERR = {1: "invalid value", 2: "out of memory", 3: "index out of range", 4: "replay: a block score was not supplied"}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C99 + OpenMP, no fast-math, no FP contraction).

    HIP_ORACLE_LIB overrides the library path (used by tests/mutants.py to check that the pins
    kill deliberately broken oracles)."""
    if os.environ.get("HIP_ORACLE_LIB"):
        return os.environ["HIP_ORACLE_LIB"]
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c99", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-fPIC", "-shared", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        i32, i64, f64 = ctypes.c_int, ctypes.c_int64, ctypes.c_double
        P = ctypes.c_void_p
        _lib.oracle_mask.argtypes = [P, P] + [i32] * 11 + [P] * 6
        _lib.oracle_mask_chunked.argtypes = [P, P] + [i32] * 12 + [P] * 4
        _lib.oracle_mask_trace.argtypes = [P, P] + [i32] * 11 + [i32] * 3 + [P, P, P, P, i32, P, P]
        _lib.oracle_exact_block_topn.argtypes = [P, P] + [i32] * 11 + [P, P]
        _lib.oracle_block_scores.argtypes = [P, P] + [i32] * 10 + [P, i64, P, P]
        _lib.oracle_sparse_attention.argtypes = [P, P, P] + [i32] * 10 + [f64, P, P, P, P]
        _lib.oracle_dense_attention.argtypes = [P, P, P] + [i32] * 7 + [f64, P, P]
        _lib.oracle_mask_paged.argtypes = [P, P, i32, i32, P, i32, P] + [i32] * 10 + [P] * 6
        _lib.oracle_sparse_attention_paged.argtypes = ([P, P, P, i32, i32, P, i32, P] + [i32] * 9
                                                       + [f64, P, P, P, P])
        _lib.oracle_sparse_attention_sw.argtypes = [P, P, P] + [i32] * 10 + [f64, P, P, i32, i32, P, P]
        _lib.oracle_sparse_attention_paged_sw.argtypes = ([P, P, P, i32, i32, P, i32, P] + [i32] * 9
                                                          + [f64, P, P, i32, i32, P, P])
        u64 = ctypes.c_uint64
        _lib.oracle_mask_ext.argtypes = [P, P] + [i32] * 14 + [u64, i32] + [P] * 4
        _lib.oracle_mask_trace_ext.argtypes = ([P, P] + [i32] * 11 + [i32] * 3 + [P, P, P, P, i32, P, P]
                                               + [i32, i32, u64])
        _lib.oracle_mask_paged_ext.argtypes = ([P, P, i32, i32, P, i32, P] + [i32] * 10 + [P] * 6
                                               + [i32, i32, i32, u64, i32])
        _lib.oracle_top_r_components.argtypes = [P, i32, i32, i32, P]
        _lib.oracle_splitmix64.argtypes = [u64]
        _lib.oracle_splitmix64.restype = u64
        _lib.oracle_jitter.argtypes = [u64, i64, i32, i64, i32]
        _lib.oracle_jitter.restype = i64
        _lib.oracle_vote.argtypes = [i32, i64, i32, P, P, i32, i32, i32, P, P]
        _lib.oracle_mask_replay.argtypes = [i32] * 6 + [i64, P, P, i64, P, P, P, i32]
        _lib.oracle_mask_replay.restype = i32
        for name in ("oracle_mask_ext", "oracle_mask_trace_ext", "oracle_mask_paged_ext", "oracle_top_r_components",
                     "oracle_vote"):
            getattr(_lib, name).restype = i32
        _lib.oracle_num_threads.restype = i32
        _lib.oracle_set_num_threads.argtypes = [i32]
        for name in ("oracle_mask", "oracle_mask_trace", "oracle_exact_block_topn", "oracle_block_scores",
                     "oracle_sparse_attention", "oracle_dense_attention", "oracle_mask_paged",
                     "oracle_sparse_attention_paged", "oracle_sparse_attention_sw", "oracle_mask_chunked",
                     "oracle_sparse_attention_paged_sw"):
            getattr(_lib, name).restype = i32
    return _lib


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_num_threads(t: int) -> None:
    lib().oracle_set_num_threads(int(t))


def _f32(a) -> np.ndarray:
    if hasattr(a, "detach"):  # torch tensor: widen exactly on the host
        a = a.detach().cpu().float().numpy()
    return np.ascontiguousarray(a, dtype=np.float32)


def _i32(a) -> np.ndarray:
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    return np.ascontiguousarray(a, dtype=np.int32)


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise ValueError(f"{what}: {_ERR.get(rc, rc)}")


def n_blocks(k: int, bk: int) -> int:
    return k // bk


def mask(Q, K, k: int, bq: int, bk: int, causal: bool, mode: int = F32C, diag: bool = False, chunks: int = 1,
         top_r: int = 0, jitter: int = 0, seed: int = 0, gqa_shared: bool = False):
    """Alg. 1 mask. Q [B,Hq,Tq,d], K [B,Hkv,Tk,d] -> idx [B,Hq,Nqb,n] (asc, -1 pad), cnt [B,Hq,Nqb].

    diag=True also returns dict(margin_min, emax, n_scored, n_iter) per unit.  chunks = S > 1: the
    stridden partial top-k (reading G21; diag then carries margin_min and emax only).
    top_r = r in (0, d): top-r approximation (G22).  jitter = R > 0: an ensemble sample
    with split offsets in [-R, R] from generator seed `seed` (G23).  gqa_shared: one mask
    per GQA group over all its query heads' rows (G25) -> idx [B, Hkv, Nqb, n]."""
    Q, K = _f32(Q), _f32(K)
    B, Hq, Tq, d = Q.shape
    _, Hkv, Tk, _ = K.shape
    n = k // bk if bk > 0 else 0
    nqb = -(-Tq // bq) if bq > 0 else 0
    Hm = Hkv if gqa_shared else Hq
    idx = np.empty((B, Hm, nqb, max(n, 1)), np.int32)
    cnt = np.empty((B, Hm, nqb), np.int32)
    mg = np.empty((B, Hm, nqb), np.float64)
    em = np.empty((B, Hm, nqb), np.float64)
    ns = np.empty((B, Hm, nqb), np.int64)
    ni = np.empty((B, Hm, nqb), np.int32)
    if chunks != 1 or top_r or jitter or gqa_shared:
        rc = lib().oracle_mask_ext(_p(Q), _p(K), B, Hq, Hkv, Tq, Tk, d, k, bq, bk, int(causal), mode, int(chunks),
                                   int(top_r), int(jitter), int(seed) & (2**64 - 1), int(bool(gqa_shared)), _p(idx),
                                   _p(cnt), _p(mg), _p(em))
        _check(rc, "oracle_mask_ext")
        if diag:
            return idx, cnt, dict(margin_min=mg, emax=em)
        return idx, cnt
    rc = lib().oracle_mask(_p(Q), _p(K), B, Hq, Hkv, Tq, Tk, d, k, bq, bk, int(causal), mode, _p(idx), _p(cnt),
                           _p(mg), _p(em), _p(ns), _p(ni))
    _check(rc, "oracle_mask")
    if diag:
        return idx, cnt, dict(margin_min=mg, emax=em, n_scored=ns, n_iter=ni)
    return idx, cnt


def mask_trace(Q, K, k: int, bq: int, bk: int, causal: bool, b: int, h: int, q: int, mode: int = F32C,
               max_trace: int = 64, top_r: int = 0, jitter: int = 0, seed: int = 0):
    """Node ranges after every iteration of one unit: list of [n,2] arrays (entry 0 = initial)."""
    Q, K = _f32(Q), _f32(K)
    B, Hq, Tq, d = Q.shape
    _, Hkv, Tk, _ = K.shape
    n = k // bk
    idx = np.empty(n, np.int32)
    cnt = np.empty(1, np.int32)
    tn = np.full(((max_trace + 1), n, 2), -7, np.int32)
    ts = np.full((max_trace, n), np.nan, np.float64)
    nit = np.zeros(1, np.int32)
    nsc = np.zeros(1, np.int64)
    rc = lib().oracle_mask_trace_ext(_p(Q), _p(K), B, Hq, Hkv, Tq, Tk, d, k, bq, bk, int(causal), mode, b, h, q,
                                     _p(idx), _p(cnt), _p(tn), _p(ts), max_trace, _p(nit), _p(nsc), int(top_r),
                                     int(jitter), int(seed) & (2**64 - 1))
    _check(rc, "oracle_mask_trace")
    it = int(nit[0])
    return dict(idx=idx, cnt=int(cnt[0]), nodes=[tn[i] for i in range(it + 1)] if it else [],
                scores=[ts[i] for i in range(it)], n_iter=it, n_scored=int(nsc[0]))


def exact_block_topn(Q, K, k: int, bq: int, bk: int, causal: bool, mode: int = F32C):
    Q, K = _f32(Q), _f32(K)
    B, Hq, Tq, d = Q.shape
    _, Hkv, Tk, _ = K.shape
    n = k // bk
    nqb = -(-Tq // bq)
    idx = np.empty((B, Hq, nqb, n), np.int32)
    cnt = np.empty((B, Hq, nqb), np.int32)
    rc = lib().oracle_exact_block_topn(_p(Q), _p(K), B, Hq, Hkv, Tq, Tk, d, k, bq, bk, int(causal), mode,
                                       _p(idx), _p(cnt))
    _check(rc, "oracle_exact_block_topn")
    return idx, cnt


def block_scores(Q, K, bq: int, bk: int, causal: bool, tuples, mode: int = F64):
    """Tile-max scores for (b, h, q, j) tuples -> (scores, emax)."""
    Q, K = _f32(Q), _f32(K)
    B, Hq, Tq, d = Q.shape
    _, Hkv, Tk, _ = K.shape
    t = np.ascontiguousarray(np.asarray(tuples, np.int32).reshape(-1, 4))
    sc = np.empty(len(t), np.float64)
    em = np.empty(len(t), np.float64)
    rc = lib().oracle_block_scores(_p(Q), _p(K), B, Hq, Hkv, Tq, Tk, d, bq, bk, int(causal), mode, _p(t),
                                   len(t), _p(sc), _p(em))
    _check(rc, "oracle_block_scores")
    return sc, em


def sparse_attention(Q, K, V, k: int, bq: int, bk: int, causal: bool, idx, cnt, sm_scale: float = 0.0,
                     sink: int = 0, window: int = 0):
    """Eq. 2-3 in fp64 over the selection idx/cnt -> (O [B,Hq,Tq,d] f64, lse [B,Hq,Tq] f64).  With
    sink/window > 0 the selection is united with the sink and sliding-window tokens."""
    Q, K, V = _f32(Q), _f32(K), _f32(V)
    idx, cnt = _i32(idx), _i32(cnt)
    B, Hq, Tq, d = Q.shape
    _, Hkv, Tk, _ = K.shape
    O = np.empty((B, Hq, Tq, d), np.float64)
    lse = np.empty((B, Hq, Tq), np.float64)
    if sink or window:
        rc = lib().oracle_sparse_attention_sw(_p(Q), _p(K), _p(V), B, Hq, Hkv, Tq, Tk, d, k, bq, bk, int(causal),
                                              float(sm_scale), _p(idx), _p(cnt), int(sink), int(window), _p(O),
                                              _p(lse))
    else:
        rc = lib().oracle_sparse_attention(_p(Q), _p(K), _p(V), B, Hq, Hkv, Tq, Tk, d, k, bq, bk, int(causal),
                                           float(sm_scale), _p(idx), _p(cnt), _p(O), _p(lse))
    _check(rc, "oracle_sparse_attention")
    return O, lse


def dense_attention(Q, K, V, causal: bool, sm_scale: float = 0.0):
    Q, K, V = _f32(Q), _f32(K), _f32(V)
    B, Hq, Tq, d = Q.shape
    _, Hkv, Tk, _ = K.shape
    O = np.empty((B, Hq, Tq, d), np.float64)
    lse = np.empty((B, Hq, Tq), np.float64)
    rc = lib().oracle_dense_attention(_p(Q), _p(K), _p(V), B, Hq, Hkv, Tq, Tk, d, int(causal),
                                      float(sm_scale), _p(O), _p(lse))
    _check(rc, "oracle_dense_attention")
    return O, lse


def mask_replay(Tq: int, Tk: int, k: int, bq: int, bk: int, causal: bool, q_of_unit, scores, trace: bool = False,
                max_trace: int = 40):
    """Alg. 1's split / rank / keep on SUPPLIED scores (C-2 replay parity): scores [u, nkb] fp32 holds
    the score of every key block the u-th listed query block q_of_unit[u] needs (NaN elsewhere).
    Returns (idx [u, n], cnt [u]) (+ per unit the list of [n, 2] node ranges after every iteration,
    entry 0 = initial, if trace); raises if the search needs a score that was not supplied."""
    qs = np.ascontiguousarray(np.asarray(q_of_unit, np.int64))
    sc = np.ascontiguousarray(np.asarray(scores, np.float32))
    n = k // bk
    idx = np.empty((len(qs), n), np.int32)
    cnt = np.empty(len(qs), np.int32)
    tn = np.full((len(qs), max_trace + 1, n, 2), -7, np.int32) if trace else None
    rc = lib().oracle_mask_replay(Tq, Tk, k, bq, bk, int(causal), len(qs), _p(qs), _p(sc), sc.shape[1], _p(idx),
                                  _p(cnt), _p(tn), max_trace)
    _check(rc, "oracle_mask_replay")
    if not trace:
        return idx, cnt
    nodes = [[tn[u, i] for i in range(max_trace + 1) if tn[u, i, 0, 0] != -7] for u in range(len(qs))]
    return idx, cnt, nodes


def mask_paged(Q, Kpages, block_table, seq_lens, k: int, bq: int, bk: int, causal: bool, mode: int = F32C,
               diag: bool = False, chunks: int = 1, top_r: int = 0, jitter: int = 0, seed: int = 0,
               gqa_shared: bool = False):
    """Mask on a paged cache. Kpages [num_pages, Hkv, page_size, d]; block_table [B, max_pages]."""
    Q, Kp = _f32(Q), _f32(Kpages)
    bt, sl = _i32(block_table), _i32(seq_lens)
    B, Hq, Tq, d = Q.shape
    num_pages, Hkv, ps, _ = Kp.shape
    n = k // bk
    nqb = -(-Tq // bq)
    Hm = Hkv if gqa_shared else Hq
    idx = np.empty((B, Hm, nqb, n), np.int32)
    cnt = np.empty((B, Hm, nqb), np.int32)
    mg = np.empty((B, Hm, nqb), np.float64)
    em = np.empty((B, Hm, nqb), np.float64)
    ns = np.empty((B, Hm, nqb), np.int64)
    ni = np.empty((B, Hm, nqb), np.int32)
    rc = lib().oracle_mask_paged_ext(_p(Q), _p(Kp), num_pages, ps, _p(bt), bt.shape[1], _p(sl), B, Hq, Hkv, Tq,
                                     d, k, bq, bk, int(causal), mode, _p(idx), _p(cnt), _p(mg), _p(em), _p(ns),
                                     _p(ni), int(chunks), int(top_r), int(jitter), int(seed) & (2**64 - 1),
                                     int(bool(gqa_shared)))
    _check(rc, "oracle_mask_paged")
    if diag:
        return idx, cnt, dict(margin_min=mg, emax=em, n_scored=ns, n_iter=ni)
    return idx, cnt


def sparse_attention_paged(Q, Kpages, Vpages, block_table, seq_lens, k: int, bq: int, bk: int, causal: bool,
                           idx, cnt, sm_scale: float = 0.0, sink: int = 0, window: int = 0):
    Q, Kp, Vp = _f32(Q), _f32(Kpages), _f32(Vpages)
    bt, sl = _i32(block_table), _i32(seq_lens)
    idx, cnt = _i32(idx), _i32(cnt)
    B, Hq, Tq, d = Q.shape
    num_pages, Hkv, ps, _ = Kp.shape
    O = np.empty((B, Hq, Tq, d), np.float64)
    lse = np.empty((B, Hq, Tq), np.float64)
    rc = lib().oracle_sparse_attention_paged_sw(_p(Q), _p(Kp), _p(Vp), num_pages, ps, _p(bt), bt.shape[1],
                                                _p(sl), B, Hq, Hkv, Tq, d, k, bq, bk, int(causal),
                                                float(sm_scale), _p(idx), _p(cnt), int(sink), int(window), _p(O),
                                                _p(lse))
    _check(rc, "oracle_sparse_attention_paged")
    return O, lse


def top_r_components(Qb, r: int) -> np.ndarray:
    """argtop_r(|q|) of one query block Qb [rows, d] (reading G22) -> r components, ascending."""
    Qb = _f32(Qb)
    rows, d = Qb.shape
    out = np.empty(r, np.int32)
    _check(lib().oracle_top_r_components(_p(Qb), rows, d, int(r), _p(out)), "oracle_top_r_components")
    return out


def splitmix64(state: int) -> int:
    """First output of splitmix64 seeded with `state` (the ensemble's counter-based generator)."""
    return int(lib().oracle_splitmix64(int(state) & (2**64 - 1)))


def jitter_offset(seed: int, lin: int, it: int, f: int, R: int) -> int:
    """Split offset u in [-R, R] of node (first block f) at iteration it of unit lin (reading G23)."""
    return int(lib().oracle_jitter(int(seed) & (2**64 - 1), int(lin), int(it), int(f), int(R)))


def vote(idx_samples, cnt_samples, theta: int, tau: int, n_out: int | None = None):
    """Ensemble vote (reading G24).  idx_samples [n_e, ..., n], cnt_samples [n_e, ...]
    -> (idx [..., n_out] ascending, -1 pad, cnt [...]).  n_out defaults to n (tau = 1) or n_e * n."""
    I, C = _i32(idx_samples), _i32(cnt_samples)
    n_e, n = I.shape[0], I.shape[-1]
    lead = I.shape[1:-1]
    units = int(np.prod(lead)) if lead else 1
    if n_out is None:
        n_out = n if tau else n_e * n
    out = np.empty(lead + (n_out,), np.int32)
    oc = np.empty(lead, np.int32)
    _check(lib().oracle_vote(n_e, units, n, _p(I), _p(C), int(theta), int(tau), int(n_out), _p(out), _p(oc)),
           "oracle_vote")
    return out, oc


def expand_gqa(idx, cnt, Hq: int):
    """A GQA-shared mask [B, Hkv, ...] as per-query-head masks [B, Hq, ...]: head h uses group h // G."""
    idx, cnt = np.asarray(idx), np.asarray(cnt)
    G = Hq // idx.shape[1]
    return np.repeat(idx, G, axis=1), np.repeat(cnt, G, axis=1)
