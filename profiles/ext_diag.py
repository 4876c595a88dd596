"""Timing of the mask kernel instantiations: plain Alg. 1 vs the option kernels (top-r, ensemble
jitter, GQA-shared rows) on the C2 inputs.  Profiling aid."""
import sys, statistics, torch
sys.path.insert(0, '/root/repo')
from paper_2406_09827_b200 import hipattn as H, synth
dev = torch.device('cuda:0')
Hh, T = 32, 32768
Q = torch.empty(1, Hh, T, 128, dtype=torch.bfloat16, device=dev); K = torch.empty_like(Q)
for h in range(Hh):
    q, k, _ = synth.gen_qkv(1, 1, 1, T, T, 128, "llm", seed=h, dtype=torch.bfloat16, device=dev, make_v=False)
    Q[:, h:h+1].copy_(q); K[:, h:h+1].copy_(k)
def t(fn):
    for _ in range(3): fn()
    torch.cuda.synchronize(); out = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); out.append(a.elapsed_time(b))
    return statistics.median(out)
import os
tag = os.environ.get("TAG", "")
print(tag, "plain", t(lambda: H.mask_estimate(Q, K)))
print(tag, "top_r64", t(lambda: H.mask_estimate(Q, K, top_r=64)))
print(tag, "jitter5", t(lambda: H.mask_estimate(Q, K, jitter=5, seed=1)))
print(tag, "plain b_q=8", t(lambda: H.mask_estimate(Q, K, b_q=8)))
print(tag, "gqa G=4 b_q=8", t(lambda: H.mask_estimate(Q, K[:, :8], b_q=8, gqa_shared=True)))
