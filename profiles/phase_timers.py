"""Per-phase cycle breakdown of the tcgen05 mask kernel (profiling aid).

Builds a separate library with -DHIPATTN_PHASES (libhipattn_phases.so, never used by the product
path), runs one C2-sized mask estimation and prints the share of CTA time per phase."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PHASES = ["split+scan", "gather+MMA issue", "MMA drain", "epilogue", "radix select", "compaction",
          "output", "unit setup", "keys"]


def build():
    from paper_2406_09827_b200 import build as b
    out = os.path.join(ROOT, "paper_2406_09827_b200", "libhipattn_phases.so")
    cmd = [b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler",
           "-fPIC", "-shared", "-cudart", "static", "-DHIPATTN_PHASES", "-I", os.path.join(ROOT, "include"), "-o", out,
           *b.sources()]
    subprocess.check_call(cmd)
    return out


def main():
    import torch
    from paper_2406_09827_b200 import hipattn as H, synth
    lib_path = build() if "--build" in sys.argv else os.path.join(ROOT, "paper_2406_09827_b200", "libhipattn_phases.so")
    H._lib = None
    lib = H.load(lib_path)
    H._lib = lib  # route the binding through the phase-timer build
    fn = lib.hip_debug_phase_cycles
    fn.argtypes = [ctypes.c_void_p]
    T, Hh = int(os.environ.get("PT_T", 32768)), int(os.environ.get("PT_H", 32))
    if os.environ.get("PT_DECODE"):  # paged decode mask, batch PT_DECODE, 32 q / 8 kv heads (C3 shape)
        B = int(os.environ["PT_DECODE"])
        q = synth.gen_decode_q(B, 32, 128, seed=0, device="cuda")
        kp, vp, bt, sl = synth.gen_paged_direct(B, 8, [T] * B, 128, 64, seed=0, device="cuda")
        run = lambda: H.mask_estimate_paged(q, kp, bt, sl, T, k_budget=512, b_q=1, b_k=2)  # noqa: E731
    else:
        Q, K, _ = synth.gen_qkv(1, Hh, Hh, T, T, 128, "llm", seed=0, device="cuda", make_v=False)
        run = lambda: H.mask_estimate(Q, K)  # noqa: E731
    run()
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 16)()
    fn(buf)
    run()
    fn(buf)
    tot = sum(buf[i] for i in range(9)) + sum(buf[i] for i in range(11, 15))
    for i, nm in enumerate(PHASES):
        print(f"{nm:22s} {100 * buf[i] / tot:5.1f}%   {buf[i] / 1e9:8.3f} Gcyc")
    # per-item split of the gather loop (mask_tc.cu marks 11-14).  The clock read after BAR.SYNC sees the
    # barrier's ISSUE, not its release (the block is deferred to the next dependent instruction), so
    # the barrier wait lands in the "MMA issue" slice: read 11 + 12 together as landing + barrier + issue.
    sub = {11: "  landing wait+barrier", 12: "  MMA issue", 13: "  MMA completion wait", 14: "  refill issue"}
    for i, nm in sub.items():
        print(f"{nm:22s} {100 * buf[i] / tot:5.1f}%   {buf[i] / 1e9:8.3f} Gcyc")
    if buf[10]:
        print(f"radix passes per select: {buf[9] / buf[10]:.2f} over {buf[10]} selections")


if __name__ == "__main__":
    main()
