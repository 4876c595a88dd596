"""Thin Python binding of the C ABI in include/hip_attn.h (libhipattn.so, sm_100a).

Argument marshalling only: every step of the hot path runs in the CUDA kernels behind the ABI.
PyTorch supplies device memory and the current stream.  There is no CPU fallback: if the library
is missing or the device is not an sm_100 B200, calls raise.

Names follow the paper (arXiv 2406.09827): k = token budget per query block, b_q / b_k = query /
key block sizes, n = k / b_k selected key blocks per query block (reading G1).
"""
from __future__ import annotations

import contextlib
import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libhipattn.so")

HIP_SUCCESS, HIP_ERROR_INVALID_VALUE, HIP_ERROR_NOT_SUPPORTED, HIP_ERROR_WORKSPACE, HIP_ERROR_CUDA = range(5)
HIP_DTYPE_F32, HIP_DTYPE_BF16 = 0, 1
HIP_FLAG_EXACT_SCORES = 1
HIP_FLAG_GQA_SHARED_MASK = 2
HIP_OP_MASK, HIP_OP_PREFILL, HIP_OP_DECODE = 0, 1, 2

EXPORTS = ("hip_version", "hip_last_error", "hip_num_blocks", "hip_workspace_bytes", "hip_mask_estimate",
           "hip_sparse_attention_prefill", "hip_sparse_attention_decode", "hip_mask_vote")


class HipError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[hip status {status}] {msg}")
        self.status = status


class Params(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("b_q", ctypes.c_int32), ("b_k", ctypes.c_int32), ("causal", ctypes.c_int32),
                ("sm_scale", ctypes.c_float), ("flags", ctypes.c_uint32), ("sink_tokens", ctypes.c_int32),
                ("window_tokens", ctypes.c_int32), ("chunks", ctypes.c_int32), ("top_r", ctypes.c_int32),
                ("split_jitter", ctypes.c_int32), ("sample_seed", ctypes.c_uint64)]


class TensorDesc(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("stride_b", ctypes.c_int64), ("stride_h", ctypes.c_int64),
                ("stride_t", ctypes.c_int64)]


class PagedKV(ctypes.Structure):
    _fields_ = [("k_pages", ctypes.c_void_p), ("v_pages", ctypes.c_void_p), ("stride_page", ctypes.c_int64),
                ("stride_h", ctypes.c_int64), ("stride_t", ctypes.c_int64), ("block_table", ctypes.c_void_p),
                ("seq_lens", ctypes.c_void_p), ("page_size", ctypes.c_int32), ("max_pages_per_seq", ctypes.c_int32),
                ("num_pages", ctypes.c_int32), ("max_seq_len", ctypes.c_int32)]


_lib = None
_libs: dict = {}


def load(path: str = LIB_PATH):
    """Load libhipattn.so (ctypes).  Raises if it has not been built: there is no fallback."""
    global _lib
    if _lib is not None and path == LIB_PATH:
        return _lib
    lib = _open(path)
    if path == LIB_PATH:
        _lib = lib
    return lib


def _open(path: str):
    if path in _libs:
        return _libs[path]
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P, i32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
    lib.hip_version.restype = i32
    lib.hip_last_error.restype = ctypes.c_char_p
    lib.hip_num_blocks.restype = i32
    lib.hip_num_blocks.argtypes = [ctypes.POINTER(Params)]
    lib.hip_workspace_bytes.restype = sz
    lib.hip_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_int] + [i32] * 6 + [ctypes.POINTER(Params)]
    lib.hip_mask_estimate.restype = ctypes.c_int
    lib.hip_mask_estimate.argtypes = ([ctypes.c_int] + [i32] * 6 + [TensorDesc, TensorDesc, ctypes.POINTER(PagedKV),
                                      ctypes.POINTER(Params), P, P, P, sz, P])
    lib.hip_sparse_attention_prefill.restype = ctypes.c_int
    lib.hip_sparse_attention_prefill.argtypes = ([ctypes.c_int] + [i32] * 6 + [TensorDesc] * 3 +
                                                 [ctypes.POINTER(Params), P, P, TensorDesc, P, P, sz, P])
    lib.hip_mask_vote.restype = ctypes.c_int
    lib.hip_mask_vote.argtypes = [i32, ctypes.c_int64, i32, P, P, i32, i32, i32, P, P, P]
    lib.hip_sparse_attention_decode.restype = ctypes.c_int
    lib.hip_sparse_attention_decode.argtypes = ([ctypes.c_int] + [i32] * 5 + [TensorDesc, ctypes.POINTER(PagedKV),
                                                ctypes.POINTER(Params), P, P, TensorDesc, P, P, sz, P])
    _libs[path] = lib
    return lib


DEBUG_LIB_PATH = os.path.join(_PKG, "libhipattn_debug.so")


@contextlib.contextmanager
def debug_score_dump(slot_of_unit: torch.Tensor, dump: torch.Tensor):
    """TEST INFRASTRUCTURE (SURVEY 8(c) C-2 replay parity): inside the block, the mask calls of this
    module go through libhipattn_debug.so, whose tcgen05 mask kernel writes the score of every
    representative block of unit row `lin` (b * H_m + h) * N_qb + q with slot_of_unit[lin] = s >= 0 to
    dump[s, block].  slot_of_unit: int32 [units] on the device; dump: fp32 [slots, N_kb] on the device."""
    global _lib
    if slot_of_unit.dtype != torch.int32 or dump.dtype != torch.float32 or dump.dim() != 2:
        raise TypeError("slot_of_unit int32 [units], dump float32 [slots, N_kb]")
    if not (slot_of_unit.is_contiguous() and dump.is_contiguous()):
        raise ValueError("contiguous buffers")
    dbg = _open(DEBUG_LIB_PATH)
    dbg.hip_debug_score_dump.restype = ctypes.c_int
    dbg.hip_debug_score_dump.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
    with torch.cuda.device(dump.device):
        if dbg.hip_debug_score_dump(slot_of_unit.data_ptr(), dump.data_ptr(), dump.shape[1]) != 0:
            raise RuntimeError("hip_debug_score_dump failed")
        saved = load()
        _lib = dbg
        try:
            yield
        finally:
            torch.cuda.synchronize(dump.device)
            dbg.hip_debug_score_dump(None, None, 0)
            _lib = saved


def _check(status: int):
    if status != HIP_SUCCESS:
        raise HipError(status, load().hip_last_error().decode())


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return HIP_DTYPE_BF16
    if t.dtype == torch.float32:
        return HIP_DTYPE_F32
    raise TypeError(f"unsupported dtype {t.dtype} (bf16 or fp32)")


def _desc(t: torch.Tensor) -> TensorDesc:
    if t.dim() != 4:
        raise ValueError("expected a [B, H, T, d] tensor")
    if t.stride(3) != 1:
        raise ValueError("the head dimension must be contiguous (stride 1)")
    return TensorDesc(t.data_ptr(), t.stride(0), t.stride(1), t.stride(2))


def _stream(t: torch.Tensor, stream=None) -> int:
    if stream is not None:
        return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    return torch.cuda.current_stream(t.device).cuda_stream


def _workspace(op: int, dtype: int, B, Hq, Hkv, Tq, Tk, d, p: Params, device, stream=None):
    """Device scratch of hip_workspace_bytes(...) bytes (the launch's job counter; split-K partials
    for single-row attention), allocated per call from torch's caching allocator.  If the call runs
    on a stream other than the current one, the block is recorded on it so the allocator does not
    hand it out again before the kernel is done."""
    n = int(load().hip_workspace_bytes(op, dtype, B, Hq, Hkv, Tq, Tk, d, ctypes.byref(p)))
    if n == 0:
        return None
    ws = torch.empty(n, dtype=torch.uint8, device=device)
    if stream is not None:
        st = stream if isinstance(stream, torch.cuda.Stream) else torch.cuda.ExternalStream(int(
            stream.cuda_stream if hasattr(stream, "cuda_stream") else stream), device=device)
        if st.cuda_stream != torch.cuda.current_stream(device).cuda_stream:
            ws.record_stream(st)
    return ws


def _ws_args(ws):
    return (ws.data_ptr(), ws.numel()) if ws is not None else (None, 0)


def _params(k: int, b_q: int, b_k: int, causal: bool, sm_scale=None, exact: bool = False, sink: int = 0,
            window: int = 0, chunks: int = 1, top_r: int = 0, jitter: int = 0, seed: int = 0,
            gqa_shared: bool = False) -> Params:
    flags = (HIP_FLAG_EXACT_SCORES if exact else 0) | (HIP_FLAG_GQA_SHARED_MASK if gqa_shared else 0)
    return Params(int(k), int(b_q), int(b_k), int(bool(causal)), float(sm_scale or 0.0), flags, int(sink),
                  int(window), int(chunks), int(top_r), int(jitter), int(seed) & (2**64 - 1))


def _require_cuda(*ts):
    for t in ts:
        if not t.is_cuda:
            raise ValueError("all tensors must be CUDA tensors (no CPU path)")


def _same_as_q(q, **ts):
    """The C ABI takes ONE dtype for q, k, v, o and the pages: every one must match q's dtype and
    device (a mismatch would be read as the wrong element type)."""
    for name, t in ts.items():
        if t is None:
            continue
        if t.dtype != q.dtype:
            raise TypeError(f"{name} is {t.dtype}, q is {q.dtype}: q, k, v, o (and pages) share one dtype")
        if t.device != q.device:
            raise ValueError(f"{name} is on {t.device}, q on {q.device}")


def _int32_buffer(name, t, shape, device):
    """idx / cnt buffers are read and written as contiguous int32 of exactly `shape`."""
    if t.dtype != torch.int32:
        raise TypeError(f"{name} must be int32, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")


def _mask_shape(B, Hm, Tq, b_q, n):
    bq = max(1, min(int(b_q), Tq))
    nqb = (Tq + bq - 1) // bq
    return (B, Hm, nqb, max(n, 1)), (B, Hm, nqb)


def num_blocks(k: int, b_k: int) -> int:
    p = _params(k, 1, b_k, False)
    return int(load().hip_num_blocks(ctypes.byref(p)))


def mask_estimate(q: torch.Tensor, k: torch.Tensor, *, k_budget: int = 512, b_q: int = 32, b_k: int = 2,
                  causal: bool = True, exact: bool = False, chunks: int = 1, top_r: int = 0, jitter: int = 0,
                  seed: int = 0, gqa_shared: bool = False, out=None, stream=None):
    """hip_mask_estimate on contiguous keys.  q [B,Hq,Tq,d], k [B,Hkv,Tk,d] -> (idx, cnt).  chunks = S:
    stridden partial top-k; top_r: top-r approximation; jitter / seed: one
    ensemble sample (combine with mask_vote); gqa_shared: one mask per kv head over the
    group's query heads (reading G25) -> idx [B, Hkv, Nqb, n]."""
    _require_cuda(q, k)
    _same_as_q(q, k=k)
    lib = load()
    B, Hq, Tq, d = q.shape
    _, Hkv, Tk, _ = k.shape
    p = _params(k_budget, b_q, b_k, causal, exact=exact, chunks=chunks, top_r=top_r, jitter=jitter, seed=seed,
                gqa_shared=gqa_shared)
    n = int(lib.hip_num_blocks(ctypes.byref(p)))
    ishape, cshape = _mask_shape(B, Hkv if gqa_shared else Hq, Tq, b_q, n)
    if out is None:
        idx = torch.empty(ishape, dtype=torch.int32, device=q.device)
        cnt = torch.empty(cshape, dtype=torch.int32, device=q.device)
    else:
        idx, cnt = out
        _int32_buffer("out idx", idx, ishape, q.device)
        _int32_buffer("out cnt", cnt, cshape, q.device)
    with torch.cuda.device(q.device):
        ws = _workspace(HIP_OP_MASK, _dtype_code(q), B, Hq, Hkv, Tq, Tk, d, p, q.device, stream)
        _check(lib.hip_mask_estimate(_dtype_code(q), B, Hq, Hkv, Tq, Tk, d, _desc(q), _desc(k), None,
                                     ctypes.byref(p), idx.data_ptr(), cnt.data_ptr(), *_ws_args(ws), _stream(q, stream)))
    return idx, cnt


def mask_vote(idx_samples: torch.Tensor, cnt_samples: torch.Tensor, *, theta: int, tau: int, n_out=None,
              stream=None):
    """hip_mask_vote: idx_samples [n_e, ..., n] int32, cnt_samples [n_e, ...] -> (idx [..., n_out], cnt [...]).
    n_out defaults to n (tau = 1) or n_e * n (tau = 0).  Feed the result to the attention with
    k_budget = n_out * b_k."""
    _require_cuda(idx_samples, cnt_samples)
    if idx_samples.dtype != torch.int32 or cnt_samples.dtype != torch.int32:
        raise TypeError("int32 indices / counts")
    if not (idx_samples.is_contiguous() and cnt_samples.is_contiguous()):
        raise ValueError("idx_samples / cnt_samples must be contiguous")  # no temporaries freed under a kernel
    if tuple(cnt_samples.shape) != tuple(idx_samples.shape[:-1]):
        raise ValueError("cnt_samples must have idx_samples' shape without the last axis")
    lib = load()
    I, C = idx_samples, cnt_samples
    n_e, n = I.shape[0], I.shape[-1]
    lead = tuple(I.shape[1:-1])
    units = 1
    for x in lead:
        units *= int(x)
    if n_out is None:
        n_out = n if tau else n_e * n
    idx = torch.empty(lead + (int(n_out),), dtype=torch.int32, device=I.device)
    cnt = torch.empty(lead, dtype=torch.int32, device=I.device)
    with torch.cuda.device(I.device):
        _check(lib.hip_mask_vote(n_e, units, n, I.data_ptr(), C.data_ptr(), int(theta), int(tau), int(n_out),
                                 idx.data_ptr(), cnt.data_ptr(), _stream(I, stream)))
    return idx, cnt


def _paged(k_pages, v_pages, block_table, seq_lens, max_seq_len: int) -> PagedKV:
    if k_pages.dim() != 4 or k_pages.stride(3) != 1:
        raise ValueError("pages must be [num_pages, Hkv, page_size, d] with d contiguous")
    if v_pages is not None and v_pages.stride() != k_pages.stride():
        raise ValueError("k_pages and v_pages must share strides")
    if block_table.dtype != torch.int32 or seq_lens.dtype != torch.int32:
        raise TypeError("block_table and seq_lens must be int32")
    # no contiguous() temporaries: a copy freed right after the enqueue could be reused by the
    # allocator while the kernel (possibly on another stream) still reads it
    if block_table.dim() != 2 or not block_table.is_contiguous():
        raise ValueError("block_table must be a contiguous [B, max_pages_per_seq] int32 tensor")
    if seq_lens.dim() != 1 or not seq_lens.is_contiguous():
        raise ValueError("seq_lens must be a contiguous [B] int32 tensor")
    if v_pages is not None and (v_pages.dtype != k_pages.dtype or v_pages.device != k_pages.device):
        raise TypeError("k_pages and v_pages must share dtype and device")
    for t in (block_table, seq_lens):
        if t.device != k_pages.device:
            raise ValueError("block_table / seq_lens must be on the pages' device")
    return PagedKV(k_pages.data_ptr(), v_pages.data_ptr() if v_pages is not None else None, k_pages.stride(0),
                   k_pages.stride(1), k_pages.stride(2), block_table.data_ptr(), seq_lens.data_ptr(),
                   k_pages.shape[2], block_table.shape[1], k_pages.shape[0], int(max_seq_len))


def mask_estimate_paged(q, k_pages, block_table, seq_lens, max_seq_len: int, *, k_budget: int = 512, b_q: int = 32,
                        b_k: int = 2, causal: bool = True, exact: bool = False, chunks: int = 1, top_r: int = 0,
                        jitter: int = 0, seed: int = 0, gqa_shared: bool = False, out=None, stream=None):
    """hip_mask_estimate on a paged cache (decode: q [B,Hq,Tq,d], Tq rows at positions seq_len-Tq+t)."""
    _require_cuda(q, k_pages, block_table, seq_lens)
    _same_as_q(q, k_pages=k_pages)
    lib = load()
    B, Hq, Tq, d = q.shape
    Hkv = k_pages.shape[1]
    p = _params(k_budget, b_q, b_k, causal, exact=exact, chunks=chunks, top_r=top_r, jitter=jitter, seed=seed,
                gqa_shared=gqa_shared)
    n = int(lib.hip_num_blocks(ctypes.byref(p)))
    pg = _paged(k_pages, None, block_table, seq_lens, max_seq_len)
    ishape, cshape = _mask_shape(B, Hkv if gqa_shared else Hq, Tq, b_q, n)
    if out is None:
        idx = torch.empty(ishape, dtype=torch.int32, device=q.device)
        cnt = torch.empty(cshape, dtype=torch.int32, device=q.device)
    else:
        idx, cnt = out
        _int32_buffer("out idx", idx, ishape, q.device)
        _int32_buffer("out cnt", cnt, cshape, q.device)
    with torch.cuda.device(q.device):
        ws = _workspace(HIP_OP_MASK, _dtype_code(q), B, Hq, Hkv, Tq, int(max_seq_len), d, p, q.device, stream)
        _check(lib.hip_mask_estimate(_dtype_code(q), B, Hq, Hkv, Tq, int(max_seq_len), d, _desc(q),
                                     TensorDesc(None, 0, 0, 0), ctypes.byref(pg), ctypes.byref(p), idx.data_ptr(),
                                     cnt.data_ptr(), *_ws_args(ws), _stream(q, stream)))
    return idx, cnt


def sparse_attention_prefill(q, k, v, idx, cnt, *, k_budget: int = 512, b_q: int = 32, b_k: int = 2,
                             causal: bool = True, sm_scale=None, sink: int = 0, window: int = 0, out=None,
                             return_lse: bool = False, gqa_shared: bool = False, stream=None):
    """hip_sparse_attention_prefill.  Returns o (and lse fp32 [B,Hq,Tq] if return_lse).  sink/window
    add StreamingLLM sink and sliding-window tokens to every row (the paper: 32 / 128)."""
    _require_cuda(q, k, v, idx, cnt)
    _same_as_q(q, k=k, v=v, out=out)
    lib = load()
    B, Hq, Tq, d = q.shape
    _, Hkv, Tk, _ = k.shape
    p = _params(k_budget, b_q, b_k, causal, sm_scale, sink=sink, window=window, gqa_shared=gqa_shared)
    ishape, cshape = _mask_shape(B, Hkv if gqa_shared else Hq, Tq, b_q, int(lib.hip_num_blocks(ctypes.byref(p))))
    _int32_buffer("idx", idx, ishape, q.device)
    _int32_buffer("cnt", cnt, cshape, q.device)
    o = torch.empty_like(q) if out is None else out
    lse = torch.empty((B, Hq, Tq), dtype=torch.float32, device=q.device) if return_lse else None
    with torch.cuda.device(q.device):
        ws = _workspace(HIP_OP_PREFILL, _dtype_code(q), B, Hq, Hkv, Tq, Tk, d, p, q.device, stream)
        _check(lib.hip_sparse_attention_prefill(_dtype_code(q), B, Hq, Hkv, Tq, Tk, d, _desc(q), _desc(k), _desc(v),
                                                ctypes.byref(p), idx.data_ptr(), cnt.data_ptr(), _desc(o),
                                                lse.data_ptr() if lse is not None else None, *_ws_args(ws),
                                                _stream(q, stream)))
    return (o, lse) if return_lse else o


def sparse_attention_decode(q, k_pages, v_pages, block_table, seq_lens, max_seq_len: int, idx, cnt, *,
                            k_budget: int = 512, b_q: int = 32, b_k: int = 2, causal: bool = True, sm_scale=None,
                            sink: int = 0, window: int = 0, out=None, return_lse: bool = False,
                            gqa_shared: bool = False, stream=None):
    """hip_sparse_attention_decode on a paged cache.  q [B,Hq,Tq,d] -> o (and lse).  gqa_shared: idx/cnt
    hold one mask per kv head (mask_estimate_paged(..., gqa_shared=True))."""
    _require_cuda(q, k_pages, v_pages, block_table, seq_lens, idx, cnt)
    _same_as_q(q, k_pages=k_pages, v_pages=v_pages, out=out)
    lib = load()
    B, Hq, Tq, d = q.shape
    Hkv = k_pages.shape[1]
    p = _params(k_budget, b_q, b_k, causal, sm_scale, sink=sink, window=window, gqa_shared=gqa_shared)
    ishape, cshape = _mask_shape(B, Hkv if gqa_shared else Hq, Tq, b_q, int(lib.hip_num_blocks(ctypes.byref(p))))
    _int32_buffer("idx", idx, ishape, q.device)
    _int32_buffer("cnt", cnt, cshape, q.device)
    pg = _paged(k_pages, v_pages, block_table, seq_lens, max_seq_len)
    o = torch.empty_like(q) if out is None else out
    lse = torch.empty((B, Hq, Tq), dtype=torch.float32, device=q.device) if return_lse else None
    with torch.cuda.device(q.device):
        ws = _workspace(HIP_OP_DECODE, _dtype_code(q), B, Hq, Hkv, Tq, int(max_seq_len), d, p, q.device, stream)
        _check(lib.hip_sparse_attention_decode(_dtype_code(q), B, Hq, Hkv, Tq, d, _desc(q), ctypes.byref(pg),
                                               ctypes.byref(p), idx.data_ptr(), cnt.data_ptr(), _desc(o),
                                               lse.data_ptr() if lse is not None else None, *_ws_args(ws),
                                               _stream(q, stream)))
    return (o, lse) if return_lse else o


def hip_attention(q, k, v, *, k_budget: int = 512, b_q: int = 32, b_k: int = 2, causal: bool = True,
                  sm_scale=None, sink: int = 0, window: int = 0, gqa_shared: bool = False, out=None, stream=None):
    """One HiP attention layer (prefill): mask estimation then block-sparse attention (with the
    optional sink / sliding-window tokens and GQA-shared masks)."""
    idx, cnt = mask_estimate(q, k, k_budget=k_budget, b_q=b_q, b_k=b_k, causal=causal, gqa_shared=gqa_shared,
                             stream=stream)
    return sparse_attention_prefill(q, k, v, idx, cnt, k_budget=k_budget, b_q=b_q, b_k=b_k, causal=causal,
                                    sm_scale=sm_scale, sink=sink, window=window, gqa_shared=gqa_shared, out=out,
                                    stream=stream)


_HOST_CTX: dict = {}


def hip_attention_host(q, k, v, out, *, k_budget: int = 512, b_q: int = 32, b_k: int = 2, causal: bool = True,
                       sm_scale=None, sink: int = 0, window: int = 0, device=None, kv_heads_per_chunk: int = 2):
    """One HiP prefill layer on PINNED HOST tensors q [B,Hq,T,d], k/v [B,Hkv,T,d] -> out (pinned host,
    like q).  The kv heads (with their query heads) stream through the device in chunks on three CUDA
    streams — host->device copy, mask + attention kernels, device->host copy — double-buffered, so the
    PCIe transfers of one chunk overlap the kernels of its neighbours.  Returns an event recorded on
    the copy-out stream when `out` is complete (the caller synchronises on it).  Marshalling and
    scheduling only: all arithmetic runs in the library's kernels."""
    if q.is_cuda or k.is_cuda or v.is_cuda or out.is_cuda:
        raise ValueError("hip_attention_host takes host tensors (pinned for asynchronous copies)")
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    B, Hq, Tq, d = q.shape
    _, Hkv, Tk, _ = k.shape
    G = Hq // Hkv
    ck = max(1, min(int(kv_heads_per_chunk), Hkv))
    chunks = [(h, min(h + ck, Hkv)) for h in range(0, Hkv, ck)]
    bq = max(1, min(int(b_q), Tq))
    nqb = (Tq + bq - 1) // bq
    n = k_budget // b_k
    key = (device, B, Hq, Hkv, Tq, Tk, d, q.dtype, k.dtype, ck, nqb, n)
    ctx = _HOST_CTX.get(key)
    if ctx is None:  # device buffers (double-buffered) and the three streams, reused across calls
        mk = lambda shape, dt: [torch.empty(shape, dtype=dt, device=device) for _ in range(2)]  # noqa: E731
        ctx = dict(Q=mk((B, G * ck, Tq, d), q.dtype), O=mk((B, G * ck, Tq, d), q.dtype),
                   K=mk((B, ck, Tk, d), k.dtype), V=mk((B, ck, Tk, d), v.dtype),
                   I=mk((B, G * ck, nqb, n), torch.int32), C=mk((B, G * ck, nqb), torch.int32),
                   streams=tuple(torch.cuda.Stream(device) for _ in range(3)))
        for old in _HOST_CTX.values():  # keep one configuration's buffers alive at a time: the old
            for st_ in old["streams"]:    # buffers are freed only once their side streams are done
                st_.synchronize()
        _HOST_CTX.clear()
        _HOST_CTX[key] = ctx
    Qd, Od, Kd, Vd, Id, Cd = ctx["Q"], ctx["O"], ctx["K"], ctx["V"], ctx["I"], ctx["C"]
    s_in, s_run, s_out = ctx["streams"]
    # the previous call's work on these buffers must be finished before they are rewritten
    cur = torch.cuda.current_stream(device)
    for st_ in (s_in, s_run, s_out):
        st_.wait_stream(cur)
    s_in.wait_stream(s_out)
    s_in.wait_stream(s_run)
    ev = lambda: torch.cuda.Event()  # noqa: E731
    run_done, out_done = [None, None], [None, None]
    with torch.cuda.device(device):
        for c, (g0, g1) in enumerate(chunks):
            i, hq0, hq1, w = c % 2, g0 * G, g1 * G, g1 - g0
            with torch.cuda.stream(s_in):
                if run_done[i] is not None:
                    s_in.wait_event(run_done[i])  # the kernels of chunk c - 2 have read buffer i
                for b in range(B):
                    Qd[i][b, :G * w].copy_(q[b, hq0:hq1], non_blocking=True)
                    Kd[i][b, :w].copy_(k[b, g0:g1], non_blocking=True)
                    Vd[i][b, :w].copy_(v[b, g0:g1], non_blocking=True)
                in_done = ev()
                in_done.record(s_in)
            with torch.cuda.stream(s_run):
                s_run.wait_event(in_done)
                if out_done[i] is not None:
                    s_run.wait_event(out_done[i])  # chunk c - 2's output has left buffer i
                qq, kk, vv, oo = Qd[i][:, :G * w], Kd[i][:, :w], Vd[i][:, :w], Od[i][:, :G * w]
                # mask outputs: contiguous [B, G*w, N_qb, n] views at the start of the buffers
                ii = Id[i].view(-1)[:B * G * w * nqb * n].view(B, G * w, nqb, n)
                cc = Cd[i].view(-1)[:B * G * w * nqb].view(B, G * w, nqb)
                mask_estimate(qq, kk, k_budget=k_budget, b_q=b_q, b_k=b_k, causal=causal, out=(ii, cc), stream=s_run)
                sparse_attention_prefill(qq, kk, vv, ii, cc, k_budget=k_budget,
                                         b_q=b_q, b_k=b_k, causal=causal, sm_scale=sm_scale, sink=sink,
                                         window=window, out=oo, stream=s_run)
                run_done[i] = ev()
                run_done[i].record(s_run)
            with torch.cuda.stream(s_out):
                s_out.wait_event(run_done[i])
                for b in range(B):
                    out[b, hq0:hq1].copy_(Od[i][b, :G * w], non_blocking=True)
                out_done[i] = ev()
                out_done[i].record(s_out)
    done = ev()
    done.record(s_out)
    return done
