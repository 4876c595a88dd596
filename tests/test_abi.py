"""The C-ABI library loads and exports every symbol include/hip_attn.h declares; host-side
validation rejects bad arguments before touching the device (CPU only, no compute)."""
import ctypes
import os
import re

import pytest
import torch

from paper_2406_09827_b200 import hipattn as H

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hip_attn.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hip_[a-z_]+)\s*\(", src)))


def test_header_declares_north_star_calls():
    names = _declared()
    for fn in ("hip_mask_estimate", "hip_sparse_attention_prefill", "hip_sparse_attention_decode"):
        assert fn in names
    assert set(names) == set(H.EXPORTS)


def test_library_exports_every_symbol():
    lib = H.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.hip_version() == 201


def test_nm_dynamic_symbols():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", H.LIB_PATH], capture_output=True, text=True).stdout
    syms = {l.split()[-1] for l in out.splitlines() if l.strip()}
    for name in _declared():
        assert name in syms, name


def test_sm100a_cubin_and_tcgen05_in_sass():
    """The library carries sm_100a SASS, with tcgen05 MMAs (UTC*MMA) and TMEM loads (LDTM)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", H.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert re.search(r"UTC\w*MMA", out) and "LDTM" in out


def test_num_blocks_and_workspace():
    lib = H.load()
    assert H.num_blocks(512, 2) == 256
    assert H.num_blocks(512, 3) == 0  # k % b_k != 0 (G12)
    p = H._params(512, 32, 2, True)
    ws = lambda op, B, Hq, Tq, pp=p, d=128: lib.hip_workspace_bytes(op, H.HIP_DTYPE_BF16, B, Hq, 8, Tq, 131072, d,  # noqa: E731
                                                                ctypes.byref(pp))
    # every op: the launch's 256-byte job counter
    assert ws(H.HIP_OP_MASK, 1, 32, 32768) == 256
    assert ws(H.HIP_OP_PREFILL, 1, 32, 32768) == 256
    # single-row attention units split over a thread-block cluster merge in shared memory: nothing more
    assert ws(H.HIP_OP_DECODE, 16, 32, 1) == 256
    p1 = H._params(512, 1, 2, True)
    assert ws(H.HIP_OP_PREFILL, 2, 4, 3, pp=p1) == 256
    assert ws(H.HIP_OP_DECODE, 16, 32, 1, d=64) == 256
    assert lib.hip_workspace_bytes(H.HIP_OP_DECODE, H.HIP_DTYPE_BF16, 0, 32, 8, 1, 10, 128, ctypes.byref(p)) == 0


def _call_mask(dtype=H.HIP_DTYPE_BF16, B=1, Hq=2, Hkv=1, Tq=64, Tk=64, d=128, params=None, qptr=0x1000, kptr=0x2000,
               st=(8192, 8192, 128), idx=0x3000, cnt=0x4000, ws=0x8000, ws_bytes=256):
    lib = H.load()
    p = params if params is not None else H._params(512, 32, 2, True)
    q = H.TensorDesc(qptr, *st)
    k = H.TensorDesc(kptr, *st)
    return lib.hip_mask_estimate(dtype, B, Hq, Hkv, Tq, Tk, d, q, k, None, ctypes.byref(p) if p else None, idx, cnt,
                                 ws, ws_bytes, None)


@pytest.mark.parametrize("kw,status", [
    (dict(params=False), H.HIP_ERROR_INVALID_VALUE),
    (dict(Tk=0), H.HIP_ERROR_INVALID_VALUE),                      # empty K
    (dict(B=0), H.HIP_ERROR_INVALID_VALUE),
    (dict(Hq=3, Hkv=2), H.HIP_ERROR_INVALID_VALUE),               # GQA divisibility
    (dict(d=96), H.HIP_ERROR_NOT_SUPPORTED),
    (dict(dtype=7), H.HIP_ERROR_NOT_SUPPORTED),
    (dict(params=H._params(511, 32, 2, True)), H.HIP_ERROR_INVALID_VALUE),   # k % b_k (G12)
    (dict(params=H._params(1, 32, 2, True)), H.HIP_ERROR_INVALID_VALUE),     # k < b_k
    (dict(params=H._params(512, 0, 2, True)), H.HIP_ERROR_INVALID_VALUE),
    (dict(params=H._params(4096, 32, 2, True)), H.HIP_ERROR_INVALID_VALUE),  # n > 1024
    (dict(Tq=65, Tk=64), H.HIP_ERROR_INVALID_VALUE),              # causal with T_q > T_k
    (dict(qptr=0), H.HIP_ERROR_INVALID_VALUE),
    (dict(qptr=0x1008), H.HIP_ERROR_INVALID_VALUE),               # misaligned
    (dict(st=(8192, 8192, 100)), H.HIP_ERROR_INVALID_VALUE),      # row stride not 16-byte multiple
    (dict(idx=0), H.HIP_ERROR_INVALID_VALUE),
    (dict(ws=None, ws_bytes=0), H.HIP_ERROR_WORKSPACE),           # workspace required (job counter)
    (dict(ws_bytes=255), H.HIP_ERROR_WORKSPACE),                  # shorter than hip_workspace_bytes
    (dict(ws=0x8008), H.HIP_ERROR_WORKSPACE),                     # misaligned
])
def test_validation_before_launch(kw, status):
    if kw.get("params") is False:
        kw["params"] = None
        lib = H.load()
        q = H.TensorDesc(0x1000, 8192, 8192, 128)
        rc = lib.hip_mask_estimate(1, 1, 2, 1, 64, 64, 128, q, q, None, None, 0x3000, 0x4000, None, 0, None)
    else:
        rc = _call_mask(**kw)
    assert rc == status, H.load().hip_last_error()
    assert H.load().hip_last_error()


def test_non_causal_tq_gt_tk_is_valid_and_ragged_blocks_are_not_errors():
    """b_q > T_q and b_k > T_k give one ragged block, not an error: validation passes and
    the call only fails at the device query when no GPU is present."""
    p = H._params(512, 64, 8, False)
    rc = _call_mask(Tq=20, Tk=5, params=p)
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    assert rc == H.HIP_ERROR_CUDA


def test_paged_validation():
    lib = H.load()
    p = H._params(512, 32, 2, True)
    q = H.TensorDesc(0x1000, 128, 128, 128)
    pg = H.PagedKV(0x2000, 0x3000, 8 * 64 * 128, 64 * 128, 128, 0x4000, 0x5000, 63, 10, 100, 600)
    rc = lib.hip_mask_estimate(1, 2, 8, 8, 1, 600, 128, q, H.TensorDesc(0, 0, 0, 0), ctypes.byref(pg),
                               ctypes.byref(p), 0x6000, 0x7000, None, 0, None)
    assert rc == H.HIP_ERROR_INVALID_VALUE  # page_size % b_k
    pg.page_size = 64
    pg.max_pages_per_seq = 5  # 5 * 64 < 600
    rc = lib.hip_mask_estimate(1, 2, 8, 8, 1, 600, 128, q, H.TensorDesc(0, 0, 0, 0), ctypes.byref(pg),
                               ctypes.byref(p), 0x6000, 0x7000, None, 0, None)
    assert rc == H.HIP_ERROR_INVALID_VALUE
    pg.max_pages_per_seq = 10
    rc = lib.hip_mask_estimate(1, 2, 8, 8, 1, 599, 128, q, H.TensorDesc(0, 0, 0, 0), ctypes.byref(pg),
                               ctypes.byref(p), 0x6000, 0x7000, None, 0, None)
    assert rc == H.HIP_ERROR_INVALID_VALUE  # T_k must equal max_seq_len
    rc = lib.hip_sparse_attention_decode(1, 2, 8, 8, 1, 128, q, None, ctypes.byref(p), 0x6000, 0x7000, q, None,
                                         None, 0, None)
    assert rc == H.HIP_ERROR_INVALID_VALUE


def test_no_cpu_path():
    """The product path refuses CPU tensors (no silent fallback)."""
    x = torch.zeros(1, 1, 64, 128, dtype=torch.bfloat16)
    with pytest.raises(ValueError):
        H.mask_estimate(x, x)
    with pytest.raises(ValueError):
        H.sparse_attention_prefill(x, x, x, torch.zeros(1, 1, 2, 256, dtype=torch.int32),
                                   torch.zeros(1, 1, 2, dtype=torch.int32))


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2406_09827_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dp, f)).read()
                for pat in (r"import\s+oracle", r"from\s+oracle", "liboracle", "hip_oracle", r'#include\s+".*oracle'):
                    assert not re.search(pat, src), (f, pat)


def test_decoder_refresh_rule_host():
    """Alg. 2 line 8: refresh when the sequence length is divisible by r_m; always on the
    first step (nothing cached).  Host logic only."""
    from paper_2406_09827_b200.decode import HipDecoder
    d = HipDecoder(r_m=8)
    assert d.refresh_rows([5, 13]) == [True, True]
    d.idx = object()  # pretend a mask is cached
    assert d.refresh_rows([8, 13, 16, 1]) == [True, False, True, False]
    assert HipDecoder(r_m=1).refresh_rows([3]) == [True]
    import pytest
    with pytest.raises(ValueError):
        HipDecoder(r_m=0)
    # the paper's (window, sink) = (128, 32) by default; a cached mask needs a window
    # covering the tokens generated since the refresh
    d = HipDecoder()
    assert (d.r_m, d.window, d.sink) == (8, 128, 32)
    with pytest.raises(ValueError):
        HipDecoder(r_m=8, window=0, sink=0)
    with pytest.raises(ValueError):
        HipDecoder(r_m=8, window=7)
    HipDecoder(r_m=8, window=8)
    HipDecoder(r_m=1, window=0, sink=0)


def test_params_struct_layout_matches_header(tmp_path):
    """The ctypes mirrors of hip_params_t / hip_paged_kv_t have the C compiler's size and offsets."""
    import subprocess
    src = tmp_path / "off.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "hip_attn.h"\nint main(void){'
                   'printf("%zu %zu %zu %zu %zu\\n", sizeof(hip_params_t), offsetof(hip_params_t, chunks),'
                   'offsetof(hip_params_t, top_r), offsetof(hip_params_t, sample_seed), sizeof(hip_paged_kv_t));}')
    exe = tmp_path / "off"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert got == [ctypes.sizeof(H.Params), H.Params.chunks.offset, H.Params.top_r.offset,
                   H.Params.sample_seed.offset, ctypes.sizeof(H.PagedKV)]


def test_appendix_params_validation():
    lib = H.load()
    q = H.TensorDesc(0x1000, 64 * 128, 64 * 128, 128)
    for bad in (dict(top_r=-1), dict(jitter=-2), dict(jitter=70000)):
        p = H._params(512, 32, 2, True, **bad)
        rc = lib.hip_mask_estimate(1, 1, 1, 1, 64, 64, 128, q, q, None, ctypes.byref(p), 0x3000, 0x4000, None, 0, None)
        assert rc == H.HIP_ERROR_INVALID_VALUE, bad


def test_vote_validation():
    lib = H.load()
    P = 0x1000
    cases = [(0, 4, 8, 1, 1, 8), (17, 4, 8, 1, 1, 8), (2, 4, 8, 0, 1, 8), (2, 4, 8, 3, 1, 8), (2, 4, 8, 1, 2, 8),
             (2, 4, 8, 1, 0, 8), (2, 4, 8, 1, 1, 7), (8, 4, 1024, 1, 1, 1024)]
    for n_e, units, n_in, theta, tau, n_out in cases:
        rc = lib.hip_mask_vote(n_e, units, n_in, P, P, theta, tau, n_out, P, P, None)
        assert rc == H.HIP_ERROR_INVALID_VALUE, (n_e, n_in, theta, tau, n_out)
    assert lib.hip_mask_vote(2, 4, 8, None, P, 1, 1, 8, P, P, None) == H.HIP_ERROR_INVALID_VALUE
