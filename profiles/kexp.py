"""Kernel-variant experiments (profiling aid, never used by the product path).

    python profiles/kexp.py build NAME [-DFLAG ...]      -> build/variants/libhipattn_NAME.so
    python profiles/kexp.py time NAME[,NAME...] [--cfg c2,c4,c3,c3_32k,c3b1] [--reps 7] [--rounds R]

`build` compiles every csrc/*.cu with the extra defines into its own library; `time` runs each
library in a fresh process on the same seeded inputs (the bench's: per-head `llm` recipe, paged C3
cache) and prints one JSON line per (variant, config): median CUDA-event ms of the mask and the
attention launch, one L2 flush (256 MB read, leaving clean lines) before every timed launch.  "base" = the product
library paper_2406_09827_b200/libhipattn.so.
"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "build", "variants")


def lib_path(name):
    if name == "base":
        return os.path.join(ROOT, "paper_2406_09827_b200", "libhipattn.so")
    return os.path.join(VDIR, f"libhipattn_{name}.so")


def build(name, defines):
    from concurrent.futures import ThreadPoolExecutor
    from paper_2406_09827_b200 import build as b
    objdir = os.path.join(VDIR, name)
    os.makedirs(objdir, exist_ok=True)
    flags = [b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler",
             "-fPIC", "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), *defines]

    def one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        subprocess.check_call(flags + ["-c", src, "-o", obj])
        return obj

    with ThreadPoolExecutor(max_workers=8) as ex:
        objs = list(ex.map(one, b.sources()))
    subprocess.check_call([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o",
                           lib_path(name), *objs])
    print(lib_path(name))


def checksum(idx, o):
    """Order-sensitive digest of the mask and the output (variants must agree with base)."""
    w = (idx.long().flatten() * 2654435761 + idx.long().flatten().roll(1)) % 1000000007
    return [int(w.sum().item()), round(float(o.float().abs().sum().item()), 2)]


def _time_one(path, cfgs, reps):
    import torch
    import bench
    from paper_2406_09827_b200 import hipattn as H
    from paper_2406_09827_b200 import synth
    H._lib = H._open(path)
    dev = torch.device("cuda:0")
    flush = torch.ones(bench.L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream(dev)
    out = []

    def timed(fns):
        ts = [[] for _ in fns]
        for f in fns:  # warm-up
            f()
        for _ in range(reps):
            for i, f in enumerate(fns):
                flush.sum()  # read-flush: L2 left holding clean lines (a write flush leaves ~126 MB of dirty
                #              lines whose write-back lands inside the next short kernel)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                f()
                e1.record(st)
                torch.cuda.synchronize(dev)
                ts[i].append(e0.elapsed_time(e1))
        return [statistics.median(t) for t in ts]

    for cn in cfgs:
        if cn.startswith("c3"):  # c3, c3_32k, c3b1 / c3b4 (batch 1 / 4)
            c = dict(bench.DECODE)
            if cn.startswith("c3_32k"):
                c["T"] = 32768
            sw = {}
            if cn.endswith("sw"):  # attention with the paper's sink 32 + window 128 (Alg. 2 cached steps)
                sw = dict(sink=32, window=128)
                cn0 = cn[:-2]
            else:
                cn0 = cn
            if cn0.startswith("c3b"):
                c["B"] = int(cn0[3:])
            seq = [c["T"]] * c["B"]
            q = synth.gen_decode_q(c["B"], c["Hq"], c["d"], seed=0, device=dev)
            kp, vp, bt, sl = synth.gen_paged_direct(c["B"], c["Hkv"], seq, c["d"], c["page"], seed=0, device=dev)
            kw = dict(k_budget=c["k"], b_q=1, b_k=c["bk"], causal=True)
            n = c["k"] // c["bk"]
            idx = torch.empty(c["B"], c["Hq"], 1, n, dtype=torch.int32, device=dev)
            cnt = torch.empty(c["B"], c["Hq"], 1, dtype=torch.int32, device=dev)
            o = torch.empty_like(q)
            m, a = timed([lambda: H.mask_estimate_paged(q, kp, bt, sl, c["T"], out=(idx, cnt), **kw),
                          lambda: H.sparse_attention_decode(q, kp, vp, bt, sl, c["T"], idx, cnt, out=o, **kw, **sw)])
            out.append({"cfg": cn, "mask_us": round(m * 1e3, 2), "attn_us": round(a * 1e3, 2),
                        "step_us": round((m + a) * 1e3, 2), "chk": checksum(idx, o)})
            del kp, vp
        else:
            cfg = bench.CONFIGS[cn]
            Q, K, V = bench.make_prefill_inputs(cfg, list(range(cfg["H"])), 0, dev)
            kw = dict(k_budget=cfg["k"], b_q=cfg["bq"], b_k=cfg["bk"], causal=True)
            idx, cnt = H.mask_estimate(Q, K, **kw)
            o = torch.empty_like(Q)
            m, a = timed([lambda: H.mask_estimate(Q, K, out=(idx, cnt), **kw),
                          lambda: H.sparse_attention_prefill(Q, K, V, idx, cnt, out=o, **kw)])
            out.append({"cfg": cn, "mask_ms": round(m, 4), "attn_ms": round(a, 4), "layer_ms": round(m + a, 4),
                        "chk": checksum(idx, o)})
            del Q, K, V, o
        torch.cuda.empty_cache()
    return out


def main():
    if sys.argv[1] == "build":
        build(sys.argv[2], sys.argv[3:])
    elif sys.argv[1] == "time":
        names = sys.argv[2].split(",")
        cfgs = "c2,c4,c3"
        reps = 7
        a = sys.argv[3:]
        if "--cfg" in a:
            cfgs = a[a.index("--cfg") + 1]
        if "--reps" in a:
            reps = int(a[a.index("--reps") + 1])
        rounds = int(a[a.index("--rounds") + 1]) if "--rounds" in a else 1
        for nm in [x for _ in range(rounds) for x in names]:  # A B A B ...: box drift hits all alike
            r = subprocess.run([sys.executable, __file__, "_time", lib_path(nm), cfgs, str(reps)], capture_output=True,
                               text=True)
            if r.returncode:
                print(json.dumps({"variant": nm, "error": r.stderr[-2000:]}), flush=True)
                continue
            for ln in r.stdout.splitlines():
                if ln.startswith("{"):
                    d = json.loads(ln)
                    print(json.dumps({"variant": nm, **d}), flush=True)
    elif sys.argv[1] == "_time":
        for d in _time_one(sys.argv[2], sys.argv[3].split(","), int(sys.argv[4])):
            print(json.dumps(d), flush=True)


if __name__ == "__main__":
    main()
