"""Runs every kernel instantiation of the library once on small inputs (profiling aid, for
compute-sanitizer; no checking here — the parity tests do that):

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python profiles/sanitize.py

Cases (kernel, instantiation): mask_tc prefill b_k = 2 / b_k = 4, paged decode b_k = 2 / 4, ensemble
jitter, top-r, GQA-shared; mask_cc (fp32, exact bf16); mask_decode (fp32 GEMV); attn_tc prefill
plain / sink + window / wide (union masks), paged decode split-K and unsplit; the small-batch decode
mask rings (8 and 4 slots); attn_cc (fp32);
attn_decode (fp32 GEMV); the ensemble vote.  Sizes span several tiles and ragged tails and stay
small enough for racecheck.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2406_09827_b200 import hipattn as H
    from paper_2406_09827_b200 import synth
    dev = torch.device("cuda:0")
    bf, f32 = torch.bfloat16, torch.float32
    small = "--small" in sys.argv
    T = 1536 if small else 2600

    def run(name, fn):
        fn()
        torch.cuda.synchronize()
        print(f"[sanitize] {name}: done", flush=True)

    Q, K, V = (x.to(dev) for x in synth.gen_qkv(1, 4, 2, T, T, 128, "llm", seed=1, dtype=bf))
    Qf, Kf, Vf = (x.float() for x in (Q, K, V))
    kw = dict(k_budget=256, b_q=32, b_k=2)
    run("mask_tc prefill b_k=2", lambda: H.mask_estimate(Q, K, **kw))
    run("mask_tc prefill b_k=4", lambda: H.mask_estimate(Q, K, k_budget=256, b_q=32, b_k=4))
    run("mask_tc jitter", lambda: H.mask_estimate(Q, K, jitter=3, seed=5, **kw))
    run("mask_tc top-r", lambda: H.mask_estimate(Q, K, top_r=32, **kw))
    run("mask_tc chunks", lambda: H.mask_estimate(Q, K, chunks=2, **kw))
    run("mask_tc gqa-shared", lambda: H.mask_estimate(Q, K, k_budget=256, b_q=8, b_k=2, gqa_shared=True))
    run("mask_cc fp32", lambda: H.mask_estimate(Qf, Kf, **kw))
    run("mask_cc bf16 exact", lambda: H.mask_estimate(Q, K, exact=True, **kw))
    idx, cnt = H.mask_estimate(Q, K, **kw)
    run("attn_tc prefill", lambda: H.sparse_attention_prefill(Q, K, V, idx, cnt, return_lse=True, **kw))
    run("attn_tc prefill sink+window", lambda: H.sparse_attention_prefill(Q, K, V, idx, cnt, sink=32, window=128, **kw))
    idf, cnf = H.mask_estimate(Qf, Kf, **kw)
    run("attn_cc fp32", lambda: H.sparse_attention_prefill(Qf, Kf, Vf, idf, cnf, return_lse=True, **kw))
    # ensemble: samples -> vote -> wide attention (tau = 0 union)
    samples = [H.mask_estimate(Q, K, jitter=3, seed=s, **kw) for s in range(3)]
    I = torch.stack([s[0] for s in samples])
    C = torch.stack([s[1] for s in samples])
    vi, vc = H.mask_vote(I, C, theta=1, tau=0)
    run("vote", lambda: H.mask_vote(I, C, theta=2, tau=1))
    run("attn_tc wide", lambda: H.sparse_attention_prefill(Q, K, V, vi, vc, k_budget=vi.shape[-1] * 2, b_q=32, b_k=2))
    # paged decode: split-K (few units) and unsplit (>= the CTA slots)
    for B, Hq, Hkv, Tmax, tag in ((3, 8, 2, T, "split-K"), (20, 32, 8, 400, "unsplit"), (1, 32, 8, T, "batch-1")):
        seq = [max(1, Tmax - 97 * b) for b in range(B)]
        q = synth.gen_decode_q(B, Hq, 128, seed=2, dtype=bf, device=dev)
        kp, vp, bt, sl = (x.to(dev) for x in synth.gen_paged_direct(B, Hkv, seq, 128, 16, seed=2, dtype=bf))
        dk = dict(k_budget=256, b_q=1, b_k=2)
        di, dc = H.mask_estimate_paged(q, kp, bt, sl, Tmax, **dk)
        run(f"mask_tc decode b_k=2 ({tag})", lambda: H.mask_estimate_paged(q, kp, bt, sl, Tmax, **dk))
        run(f"attn_tc decode {tag}", lambda: H.sparse_attention_decode(q, kp, vp, bt, sl, Tmax, di, dc, return_lse=True,
                                                                      **dk))
        run(f"attn_tc decode {tag} sink+window",
            lambda: H.sparse_attention_decode(q, kp, vp, bt, sl, Tmax, di, dc, sink=32, window=128, **dk))
        if tag == "split-K":
            run("mask_tc decode b_k=4", lambda: H.mask_estimate_paged(q, kp, bt, sl, Tmax, k_budget=256, b_q=1, b_k=4))
            qf, kpf, vpf = q.float(), kp.float(), vp.float()
            run("mask_decode fp32", lambda: H.mask_estimate_paged(qf, kpf, bt, sl, Tmax, **dk))
            run("attn_decode fp32", lambda: H.sparse_attention_decode(qf, kpf, vpf, bt, sl, Tmax, di, dc, **dk))
            run("mask_tc decode gqa-shared", lambda: H.mask_estimate_paged(q, kp, bt, sl, Tmax, gqa_shared=True, **dk))
    # decode mask, 2 units per SM or fewer: the 4-slot ring instantiation
    q4 = synth.gen_decode_q(8, 32, 128, seed=3, dtype=bf, device=dev)
    kp4, vp4, bt4, sl4 = (x.to(dev) for x in synth.gen_paged_direct(8, 8, [T] * 8, 128, 16, seed=3, dtype=bf))
    run("mask_tc decode 4-slot ring", lambda: H.mask_estimate_paged(q4, kp4, bt4, sl4, T, k_budget=256, b_q=1, b_k=2))
    print("[sanitize] all cases ran", flush=True)


if __name__ == "__main__":
    main()
