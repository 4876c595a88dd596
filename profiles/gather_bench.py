"""Random 512-byte block gather bandwidth (the pattern of HiP's mask / attention gathers) on B200:
L2-resident (8 MB, 32 MB) vs HBM-resident (4 GB) source, for several CTAs/SM and ring depths.
Writes profiles/r01/gather_ceiling.json.  Profiling tool only (own .so, not the product)."""
import ctypes
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libgather_bench.so")


def build():
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                           "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-o", SO,
                           os.path.join(HERE, "gather_bench.cu")])


def main():
    if "--build" in sys.argv:
        build()
        return
    import torch
    lib = ctypes.CDLL(SO)
    lib.gather_bench.argtypes = [ctypes.c_void_p, ctypes.c_ulonglong, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.POINTER(ctypes.c_float)]
    big = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
    big.random_()
    out = []
    for size_mb in (8, 32, 4096):
        nbytes = size_mb << 20
        for nbuf, cps in ((1, 4), (2, 2), (2, 3), (3, 2), (4, 1), (2, 1), (1, 6)):
            iters = 400
            ms = ctypes.c_float(0)
            rc = lib.gather_bench(big.data_ptr(), nbytes, nbuf, cps, iters, ctypes.byref(ms))
            sms = torch.cuda.get_device_properties(0).multi_processor_count
            moved = sms * cps * iters * 32768
            gbs = moved / (ms.value * 1e-3) / 1e9
            r = dict(source_mb=size_mb, ring_tiles=nbuf, ctas_per_sm=cps, gbs=round(gbs, 1), rc=rc)
            out.append(r)
            print(r, flush=True)
    os.makedirs(os.path.join(HERE, "r01"), exist_ok=True)
    json.dump(out, open(os.path.join(HERE, "r01", "gather_ceiling.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
