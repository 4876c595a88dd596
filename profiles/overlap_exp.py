"""Experiment: does running the mask estimation of head group g+1 concurrently with the sparse
attention of head group g (two streams) beat the sequential layer?  Profiling aid only.

usage: HIPATTN_CTAS_PER_SM=<c> python profiles/overlap_exp.py [groups]
(needs a -DHIPATTN_TUNING build of the library: the product build reads no environment)"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2406_09827_b200 import hipattn as H, synth  # noqa: E402


def main():
    G = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    Hh, T, d = 32, 32768, 128
    Q = torch.empty(1, Hh, T, d, dtype=torch.bfloat16, device="cuda")
    K, V = torch.empty_like(Q), torch.empty_like(Q)
    for h in range(Hh):
        q, k, v = synth.gen_qkv(1, 1, 1, T, T, d, "llm", seed=h, device="cuda")
        Q[:, h:h + 1].copy_(q); K[:, h:h + 1].copy_(k); V[:, h:h + 1].copy_(v)
    idx = torch.empty(1, Hh, T // 32, 256, dtype=torch.int32, device="cuda")
    cnt = torch.empty(1, Hh, T // 32, dtype=torch.int32, device="cuda")
    O = torch.empty_like(Q)
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()

    def seq():
        H.mask_estimate(Q, K, out=(idx, cnt))
        H.sparse_attention_prefill(Q, K, V, idx, cnt, out=O)

    def overlap():
        hg = Hh // G
        evs = []
        for g in range(G):
            sl = slice(g * hg, (g + 1) * hg)
            with torch.cuda.stream(s0):
                H.mask_estimate(Q[:, sl], K[:, sl], out=(idx[:, sl], cnt[:, sl]), stream=s0)
                e = torch.cuda.Event()
                e.record(s0)
            evs.append(e)
        for g in range(G):
            sl = slice(g * hg, (g + 1) * hg)
            s1.wait_event(evs[g])
            with torch.cuda.stream(s1):
                H.sparse_attention_prefill(Q[:, sl], K[:, sl], V[:, sl], idx[:, sl], cnt[:, sl], out=O[:, sl],
                                           stream=s1)
        torch.cuda.current_stream().wait_stream(s1)

    for name, fn in (("sequential", seq), ("overlap", overlap)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            fn()
        b.record()
        torch.cuda.synchronize()
        print(name, G, os.environ.get("HIPATTN_CTAS_PER_SM", "-"), round(a.elapsed_time(b) / 10, 3), "ms")


if __name__ == "__main__":
    main()
