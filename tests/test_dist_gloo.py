"""Multi-process (world_size 2, gloo, CPU) tests of the sharding layer paper_2406_09827_b200/dist.py.

The layer run on each shard here is the CPU oracle (mask + attention), so the tests check the host
logic of the N > 1 path — shard boundaries, bottom-right alignment of query ranges, the gather and
reassembly — against the unsharded oracle result, bit-for-bit (PIN-9)."""
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


def _oracle_layer(q, k, v):
    from oracle import oracle as orc
    idx, cnt = orc.mask(q, k, K_BUDGET, BQ, BK, True)
    O, _ = orc.sparse_attention(q, k, v, K_BUDGET, BQ, BK, True, idx, cnt)
    return torch.from_numpy(O)


def _worker(rank, world, port, mode, q, k, v, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = hd.sharded_layer(_oracle_layer, q, k, v, mode=mode, bq=BQ, bk=BK, k_budget=K_BUDGET)
        ret[rank] = o.numpy()
    finally:
        dist.destroy_process_group()


def _run(mode, q, k, v, world=2):
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), mode, q, k, v, ret), nprocs=world, join=True)
    return [ret[r] for r in range(world)]


@pytest.mark.parametrize("mode", ["heads", "sequence"])
def test_sharded_equals_unsharded(mode):
    Q, K, V = synth.gen_qkv(2, 4, 2, 700, 700, 32, "llm", seed=3, dtype=torch.float32)
    full = _oracle_layer(Q, K, V).numpy()
    outs = _run(mode, Q, K, V)
    for o in outs:
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


def test_head_range_rejects_uneven():
    with pytest.raises(ValueError):
        hd.head_range(40, 3, 0)
    assert list(hd.head_range(40, 8, 7)) == [35, 36, 37, 38, 39]
