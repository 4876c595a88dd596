"""fp32 paged decode (C3 shape: 16 x 128k, 32 q-heads / 8 kv-heads, page 64, k = 512, b_k = 2):
the CUDA-core mask_decode (F32L order) + attention timing.  Profiling aid."""
import statistics
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_09827_b200 import hipattn as H, synth  # noqa: E402

dev = torch.device("cuda:0")
B, Hq, Hkv, T, d = 16, 32, 8, 131072, 128
q = synth.gen_decode_q(B, Hq, d, seed=0, dtype=torch.float32, device=dev)
kp, vp, bt, sl = synth.gen_paged_direct(B, Hkv, [T] * B, d, 64, seed=0, dtype=torch.float32, device=dev)
kw = dict(k_budget=512, b_q=1, b_k=2)


def t(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return 1e3 * statistics.median(out)


idx, cnt = H.mask_estimate_paged(q, kp, bt, sl, T, **kw)
print("fp32 decode mask_us", round(t(lambda: H.mask_estimate_paged(q, kp, bt, sl, T, **kw)), 1),
      "attn_us", round(t(lambda: H.sparse_attention_decode(q, kp, vp, bt, sl, T, idx, cnt, **kw)), 1))
