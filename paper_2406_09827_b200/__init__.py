"""B200-native (sm_100a) hot path of HiP — Hierarchically Pruned Attention (arXiv 2406.09827).

The compute lives in libhipattn.so (C ABI, include/hip_attn.h); `hipattn` is its ctypes binding.
"""
from . import hipattn  # noqa: F401
from .hipattn import (hip_attention, mask_estimate, mask_estimate_paged, sparse_attention_decode,  # noqa: F401
                      sparse_attention_prefill)
