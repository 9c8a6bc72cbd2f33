"""The N>1 path of bench.py on CPU: world_size-2 gloo.  Streams shard by rank
with no data-path collective; only the barrier and the max-over-ranks timing
reduction cross processes."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import bench
    dist, r, w, local = bench.dist_setup(world)
    bench.dist_barrier(dist)
    # each rank times its own shard; the job time is the slowest rank
    mx = bench.dist_max(dist, 1.0 + rank * 0.5)
    q.put((r, w, local, mx))
    bench.dist_barrier(dist)
    dist.destroy_process_group()


def test_two_rank_barrier_and_max_over_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[0] for r in res] == [0, 1]
    assert all(r[1] == 2 for r in res)
    assert [r[2] for r in res] == [0, 1]          # one GPU per rank (LOCAL_RANK)
    assert all(r[3] == pytest.approx(1.5) for r in res)


def test_single_process_default_has_no_group():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.dist_setup(1) == (None, 0, 1, 0)
    assert bench.dist_max(None, 3.0) == 3.0
