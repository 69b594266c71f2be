"""Multi-rank host logic on CPU: token-balanced shards, max-over-ranks job time and
the optional logits gather, over a real gloo process group (world_size 2)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2209_09130_b200.sharding import partition_by_tokens


def test_partition_properties():
    rng = np.random.default_rng(0)
    for world in (1, 2, 4, 8):
        lens = rng.integers(16, 513, 64)
        parts = partition_by_tokens(lens, world)
        assert parts[0][0] == 0 and parts[-1][1] == 64
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
        assert all(s1 > s0 for s0, s1 in parts)
        loads = [lens[s0:s1].sum() for s0, s1 in parts]
        assert max(loads) - min(loads) <= 2 * lens.max()
    assert partition_by_tokens([128] * 32, 4) == [(0, 8), (8, 16), (16, 24), (24, 32)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2209_09130_b200.sharding import gather_rows, max_over_ranks, partition_by_tokens
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lens = [64] * 10 + [32] * 6
    s0, s1 = partition_by_tokens(lens, world)[rank]
    local = np.arange(s0, s1, dtype=np.float32)[:, None].repeat(2, axis=1)   # stand-in logits
    t = max_over_ranks(1.5 if rank == 0 else 2.5)
    g = gather_rows(local)
    q.put((rank, t, None if g is None else g[:, 0].tolist()))
    dist.destroy_process_group()


def test_two_rank_gloo_group():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [r[1] for r in res] == [2.5, 2.5]
    assert res[0][2] == list(range(16)) and res[1][2] is None
