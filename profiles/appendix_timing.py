"""Timing of the appendix extensions on the C2 workload (32 heads x 32k, bf16, llm inputs):
top-r approximation at r in {128 (off), 64, 32, 16} and one HiP-ensemble layer
(P:1162-1184): n_e jittered samples + vote + sparse attention.  CUDA events on the launching
stream, 3 warm-ups, median of 5.  Prints one JSON object."""
import json
import statistics
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_09827_b200 import hipattn as H  # noqa: E402
from paper_2406_09827_b200 import synth  # noqa: E402


def t(fn, reps=5, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


def main():
    dev = torch.device("cuda:0")
    Hh, T, d = 32, 32768, 128
    Q = torch.empty(1, Hh, T, d, dtype=torch.bfloat16, device=dev)
    K, V = torch.empty_like(Q), torch.empty_like(Q)
    for h in range(Hh):
        q, k, v = synth.gen_qkv(1, 1, 1, T, T, d, "llm", seed=h, dtype=torch.bfloat16, device=dev)
        Q[:, h:h + 1].copy_(q), K[:, h:h + 1].copy_(k), V[:, h:h + 1].copy_(v)
    kw = dict(k_budget=512, b_q=32, b_k=2)
    res = {"workload": "C2 32 heads x 32k bf16 llm", "top_r_mask_ms": {}, "top_r_recall_vs_exact_mask": {}}
    base_idx, _ = H.mask_estimate(Q, K, **kw)
    for r in (0, 64, 32, 16):
        res["top_r_mask_ms"][str(r or 128)] = round(t(lambda: H.mask_estimate(Q, K, top_r=r, **kw)), 4)
        idx, cnt = H.mask_estimate(Q, K, top_r=r, **kw)
        # fraction of the exact-score mask's blocks the approximate mask keeps (sampled heads)
        a, b = base_idx[:, :4], idx[:, :4]
        same = (a.unsqueeze(-1) == b.unsqueeze(-2)).any(-1) & (a >= 0)
        res["top_r_recall_vs_exact_mask"][str(r or 128)] = round(float(same.sum() / (a >= 0).sum()), 4)
    for n_e, theta, tau in ((4, 2, 1), (4, 1, 0)):
        def layer():
            S = [H.mask_estimate(Q, K, jitter=5, seed=s, **kw) for s in range(n_e)]
            vi, vc = H.mask_vote(torch.stack([x[0] for x in S]), torch.stack([x[1] for x in S]), theta=theta, tau=tau)
            return H.sparse_attention_prefill(Q, K, V, vi, vc, k_budget=vi.shape[-1] * 2, b_q=32, b_k=2)
        S = [H.mask_estimate(Q, K, jitter=5, seed=s, **kw) for s in range(n_e)]
        I, C = torch.stack([x[0] for x in S]), torch.stack([x[1] for x in S])
        vote_ms = t(lambda: H.mask_vote(I, C, theta=theta, tau=tau))
        vi, vc = H.mask_vote(I, C, theta=theta, tau=tau)
        res[f"ensemble_ne{n_e}_theta{theta}_tau{tau}"] = {
            "layer_ms": round(t(layer, reps=3), 3), "vote_ms": round(vote_ms, 4),
            "mean_blocks_per_row": round(float(vc.float().mean()), 2)}
    res["plain_layer_ms"] = round(t(lambda: H.hip_attention(Q, K, V, **kw)), 3)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
