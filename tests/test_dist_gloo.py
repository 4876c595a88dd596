"""Multi-process (gloo, CPU, world_size 2 and 4) tests of the sharding layer paper_2406_09827_b200/dist.py.

The layer run on each shard here is the CPU oracle (mask + attention), so the tests check the host
logic of the N > 1 path — shard maps, bottom-right alignment of query ranges, the interleaved
head-chunk gathers, batch / kv-group decode shards and the reassembly — against the unsharded
oracle result, bit-for-bit (PIN-9)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_09827_b200 import dist as hd
from paper_2406_09827_b200 import synth

K_BUDGET, BQ, BK = 64, 16, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_layer(q, k, v, bq=BQ):
    from oracle import oracle as orc
    idx, cnt = orc.mask(q, k, K_BUDGET, bq, BK, True)
    O, _ = orc.sparse_attention(q, k, v, K_BUDGET, bq, BK, True, idx, cnt)
    return torch.from_numpy(O)


def _oracle_decode_step(q, kp, vp, bt, sl):
    """One decode step on a paged cache, with the paper's sink / window."""
    from oracle import oracle as orc
    Tq = q.shape[2]
    idx, cnt = orc.mask_paged(q, kp, bt, sl, K_BUDGET, Tq, BK, True)
    O, _ = orc.sparse_attention_paged(q, kp, vp, bt, sl, K_BUDGET, Tq, BK, True, idx, cnt, sink=8, window=16)
    return torch.from_numpy(O)


def _worker(rank, world, port, kind, mode, chunks, bq, tensors, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if kind == "prefill":
            q, k, v = tensors
            layer = lambda a, b, c: _oracle_layer(a, b, c, bq)  # noqa: E731
            o = hd.sharded_layer(layer, q, k, v, mode=mode, chunks=chunks, bq=bq, bk=BK, k_budget=K_BUDGET)
        else:
            o = hd.sharded_decode(_oracle_decode_step, *tensors, mode=mode)
        ret[rank] = o.numpy()
    finally:
        dist.destroy_process_group()


def _run(kind, mode, tensors, world, chunks=1, bq=BQ):
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), kind, mode, chunks, bq, tensors, ret), nprocs=world, join=True)
    return [ret[r] for r in range(world)]


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("mode,chunks", [("heads", 1), ("heads", 2), ("sequence", 1)])
def test_sharded_prefill_equals_unsharded(mode, chunks, world):
    # 8 query heads over 4 kv heads (GQA group of 2); T = 700 is not a multiple of b_q (ragged tail)
    Q, K, V = synth.gen_qkv(2, 8, 4, 700, 700, 32, "llm", seed=3, dtype=torch.float32)
    if mode == "heads" and 8 % (world * chunks * 2):
        pytest.skip("a chunk must hold whole GQA groups")
    full = _oracle_layer(Q, K, V).numpy()
    for o in _run("prefill", mode, (Q, K, V), world, chunks):
        assert o.shape == full.shape
        assert np.array_equal(o, full)


def test_sharded_sequence_uneven_world4():
    """T = 300, b_q = 64 gives 5 query blocks; 4 ranks must each get >= 1 of them."""
    Q, K, V = synth.gen_qkv(1, 2, 2, 300, 300, 32, "iid", seed=4, dtype=torch.float32)
    r = hd.balanced_block_ranges(300, 64, BK, K_BUDGET, 4)
    assert all(q1 > q0 for q0, q1 in r) and r[0][0] == 0 and r[-1][1] == 5
    full = _oracle_layer(Q, K, V, 64).numpy()
    for o in _run("prefill", "sequence", (Q, K, V), 4, bq=64):
        assert np.array_equal(o, full)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("mode", ["batch", "kvgroup"])
def test_sharded_decode_equals_unsharded(mode, world):
    # 4 sequences of different lengths, 8 query heads over 4 kv heads, 2 query rows per step
    B, Hq, Hkv, d, ps = 4, 8, 4, 32, 16
    seq = [300, 71, 512, 199]
    q = synth.gen_decode_q(B, Hq, d, seed=5, dtype=torch.float32, Tq=2)
    kp, vp, bt, sl = synth.gen_paged_direct(B, Hkv, seq, d, ps, seed=5, dtype=torch.float32)
    full = _oracle_decode_step(q, kp, vp, bt, sl).numpy()
    for o in _run("decode", mode, (q, kp, vp, bt, sl), world):
        assert o.shape == full.shape
        assert np.array_equal(o, full)


def test_balanced_ranges_cover_and_balance():
    T, bq, bk, k = 1 << 20, 32, 2, 512
    for world in (2, 4, 8):
        r = hd.balanced_block_ranges(T, bq, bk, k, world)
        assert r[0][0] == 0 and r[-1][1] == T // bq
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
        cost = [sum(hd.block_cost(q, bq, bk, k, T) for q in range(q0, q1)) for q0, q1 in r]
        assert max(cost) / min(cost) < 1.01


@pytest.mark.parametrize("T,bq,world", [(300, 64, 4), (100, 32, 4), (64, 32, 2), (1000, 16, 8), (33, 32, 2)])
def test_balanced_ranges_never_empty(T, bq, world):
    r = hd.balanced_block_ranges(T, bq, BK, K_BUDGET, world)
    nqb = -(-T // bq)
    assert len(r) == world and r[0][0] == 0 and r[-1][1] == nqb
    assert all(q1 > q0 for q0, q1 in r)
    assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
    with pytest.raises(ValueError):
        hd.balanced_block_ranges(T, bq, BK, K_BUDGET, nqb + 1)


def test_head_maps():
    with pytest.raises(ValueError):
        hd.head_range(40, 3, 0)
    assert list(hd.head_range(40, 8, 7)) == [35, 36, 37, 38, 39]
    # interleaved chunks: chunk c of all ranks is one contiguous range, every head exactly once
    H, world, chunks = 32, 4, 2
    maps = [hd.head_chunks(H, world, r, chunks) for r in range(world)]
    for c in range(chunks):
        assert sorted(h for r in range(world) for h in maps[r][c]) == list(range(c * H // chunks, (c + 1) * H // chunks))
    assert sorted(h for m in maps for rg in m for h in rg) == list(range(H))
    assert hd.head_chunks(H, world, 1, 1) == [hd.head_range(H, world, 1)]
    with pytest.raises(ValueError):
        hd.head_chunks(32, 4, 0, 4, group=4)  # 2 heads per chunk cannot hold a group of 4
    assert list(hd.batch_range(16, 4, 3)) == [12, 13, 14, 15]
