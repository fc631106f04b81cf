"""Multi-GPU path on CPU: world_size-2 gloo processes exchange their local
best (peak, id) exactly as the NCCL path does; the result must equal the
reference's first strict minimum over the global candidate order
(tests/oracles.py:46-56).  Shard ranges are contiguous and disjoint."""

from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import memplan_oracle as O
from paper_2310_19295_b200.sharding import NONE_PEAK, allgather_best, lex_min, shard_range


def test_shard_ranges_partition():
    for total in (0, 1, 7, 16384, 1_048_576 + 3):
        for world in (1, 2, 3, 4, 8):
            rs = [shard_range(total, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, peaks, valids, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_range(len(peaks), world, rank)
        local = lex_min((peaks[i], i) for i in range(lo, hi) if valids[i])
        got = allgather_best(torch.tensor(local, dtype=torch.int64))
        q.put((rank, tuple(int(x) for x in got.tolist())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["ties_across_ranks", "none_valid_on_one_rank", "none_valid", "random"])
def test_gloo_world2_argmin_equals_first_strict_min(case):
    import random
    rng = random.Random(4)
    if case == "ties_across_ranks":
        peaks, valids = [9, 5, 7, 5, 5, 6], [True] * 6      # tie spans both shards -> id 1
    elif case == "none_valid_on_one_rank":
        peaks, valids = [3, 3, 3, 8, 2, 9], [False, False, False, True, True, True]
    elif case == "none_valid":
        peaks, valids = [1, 2, 3], [False] * 3
    else:
        peaks = [rng.randint(0, 5) for _ in range(101)]
        valids = [rng.random() < 0.8 for _ in range(101)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, peaks, valids, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    want = O.first_strict_min(peaks, valids)
    want = (NONE_PEAK, -1) if want[0] is None else want
    assert res[0] == res[1] == want


def _key_worker(rank, world, port, keys, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2310_19295_b200.sharding import allreduce_key
        k = torch.tensor([keys[rank]], dtype=torch.int64)
        q.put((rank, int(allreduce_key(k).item())))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_packed_key_allreduce():
    from paper_2310_19295_b200.sharding import decode_key, key_bits
    bits = key_bits(1_048_576)
    peaks, valids = [9, 5, 7, 5, 5, 6, 5, 8], [True, False, True, True, True, True, True, True]
    keys = []
    for r in range(2):
        lo, hi = shard_range(len(peaks), 2, r)
        p, i = lex_min((peaks[j], j) for j in range(lo, hi) if valids[j])
        keys.append(NONE_PEAK if i < 0 else (p << bits) | i)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_key_worker, args=(r, 2, port, keys, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[0] == res[1]
    assert decode_key(res[0], bits) == O.first_strict_min(peaks, valids) == (5, 3)
