"""N > 1 host path on CPU: world_size-2 gloo, cell sharding, metric reduction."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_23397_b200.dist import cell_seed, reduce_metrics, shard_cells


def test_shard_cells_partition():
    for n in (1, 7, 64, 1024):
        for w in (1, 2, 3, 8):
            got = [list(shard_cells(n, r, w)) for r in range(w)]
            flat = [c for g in got for c in g]
            assert flat == list(range(n))
            assert max(map(len, got)) - min(map(len, got)) <= 1
    assert cell_seed(1000, 3) == 1003


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cells = shard_cells(64, rank, world)
    # each rank "processes" its cells for a rank-dependent time
    t, n = reduce_metrics(10.0 * (rank + 1), len(cells) * 256)
    q.put((rank, t, n, list(cells)[:2]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [o[1] for o in out] == [20.0, 20.0]           # max over ranks
    assert [o[2] for o in out] == [64 * 256, 64 * 256]   # all units counted once
    assert out[0][3] == [0, 1] and out[1][3] == [32, 33]
