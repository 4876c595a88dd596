"""Multi-process sharding with the CUDA kernels on the GPU (PIN-9 on hardware): world_size 2 processes
share the one GPU of the test box, each runs its shard of the layer through the C ABI, and the shards
are gathered with gloo (the outputs move to the host for the collective; on an 8-GPU box the same
dist.py code gathers with NCCL over NVLink).  Sharded == unsharded, bit for bit, for the prefill
head / interleaved-head-chunk / balanced-query-range splits and the decode batch / kv-group splits."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_09827_b200 import dist as hd
from paper_2406_09827_b200 import synth

pytestmark = pytest.mark.gpu

KW = dict(k_budget=256, b_q=32, b_k=2, causal=True)
DKW = dict(k_budget=256, b_q=1, b_k=2, causal=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gpu_layer(q, k, v):
    from paper_2406_09827_b200 import hipattn as H
    o = H.hip_attention(q.cuda(), k.cuda(), v.cuda(), **KW)
    return o.cpu()


def _gpu_decode_step(q, kp, vp, bt, sl):
    from paper_2406_09827_b200 import hipattn as H
    T = int(sl.max())
    q, kp, vp, bt, sl = (x.cuda() for x in (q, kp, vp, bt, sl))
    idx, cnt = H.mask_estimate_paged(q, kp, bt, sl, T, **DKW)
    o = H.sparse_attention_decode(q, kp, vp, bt, sl, T, idx, cnt, sink=32, window=128, **DKW)
    return o.cpu()


def _worker(rank, world, port, kind, mode, chunks, tensors, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if kind == "prefill":
            o = hd.sharded_layer(_gpu_layer, *tensors, mode=mode, chunks=chunks, bq=KW["b_q"], bk=KW["b_k"],
                                 k_budget=KW["k_budget"])
        else:
            o = hd.sharded_decode(_gpu_decode_step, *tensors, mode=mode)
        ret[rank] = o
    finally:
        dist.destroy_process_group()


def _run(kind, mode, tensors, world=2, chunks=1):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    ret = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), kind, mode, chunks, tensors, ret), nprocs=world, join=True,
                       start_method="spawn")
    return [ret[r] for r in range(world)]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("mode,chunks", [("heads", 1), ("heads", 2), ("sequence", 1)])
def test_gpu_sharded_prefill_equals_unsharded(mode, chunks):
    q, k, v = synth.gen_qkv(1, 8, 4, 3000, 3000, 128, "llm", seed=61, dtype=torch.bfloat16)
    ref = _gpu_layer(q, k, v)
    for o in _run("prefill", mode, (q, k, v), chunks=chunks):
        assert torch.equal(o, ref)


@pytest.mark.parametrize("mode", ["batch", "kvgroup"])
def test_gpu_sharded_decode_equals_unsharded(mode):
    B, Hq, Hkv, d = 4, 8, 4, 128
    seq = [2100, 700, 3000, 1]
    q = synth.gen_decode_q(B, Hq, d, seed=62)
    kp, vp, bt, sl = synth.gen_paged_direct(B, Hkv, seq, d, 16, seed=62)
    ref = _gpu_decode_step(q, kp, vp, bt, sl)
    for o in _run("decode", mode, (q, kp, vp, bt, sl)):
        assert torch.equal(o, ref)
