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


class _FakeC5Lib:
    """Stands in for libgpuos_bench.so's config-5 entry points on CPU: records
    which streams each rank opens and reports a per-rank device time."""

    def __init__(self, rank, log):
        self.rank, self.log = rank, log

        def gb_c5_open(local, ids, n, tasks_per_stream, workers, out_cap):
            self.log.append(("open", rank, [ids[i] for i in range(n)], workers))
            return 1000 + rank

        def gb_c5_run(h, warm, verify, res):
            n = len(self.log[-1][2])
            res[0] = 1000.0 * n                 # tasks
            res[1] = 10.0 + 5.0 * self.rank      # this rank's union ms
            res[2] = 1e6 * n                     # algorithmic bytes
            res[3] = 0.0                         # failed
            res[4], res[5], res[6], res[7], res[8] = 0.0, float(n), 100.0 * n, 1.0, 0.0
            res[9] = 90.0
            return 0

        def gb_c5_survivors(h):
            return 10.0

        def gb_c5_close(h):
            self.log.append(("close", rank))

        for f in (gb_c5_open, gb_c5_run, gb_c5_survivors, gb_c5_close):
            setattr(self, f.__name__, f)


def _c5_worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import bench
    dist, r, w, local = bench.dist_setup(world)
    log = []
    res = bench.run_config5(_FakeC5Lib(r, log), dist, r, w, local, tasks_per_stream=1000, streams=8)
    q.put((r, res, [e for e in log if e[0] == "open"]))
    bench.dist_barrier(dist)
    dist.destroy_process_group()


def test_two_rank_config5_shards_streams_and_aggregates():
    """bench.py's config-5 rank path at G=2 over gloo: stream s runs on rank
    s mod 2, tasks and bytes add across ranks, the device time is the max over
    ranks, and the G=1 reference run happens on rank 0 only."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_c5_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=180) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, res0, opens0), (r1, res1, opens1) = res
    assert opens0[0][2] == [0, 2, 4, 6] and opens1[0][2] == [1, 3, 5, 7]
    assert len(opens0) == 2 and opens0[1][2] == list(range(8))   # G=1 rerun on rank 0
    assert len(opens1) == 1
    assert res0["G"] == 2
    assert res0["union_ms"] == pytest.approx(15.0)                # max over ranks (rank 1: 15 ms)
    assert res0["per_gpu_ms"] == [10.0, 15.0]
    assert res0["tasks_per_s"] == pytest.approx(8000 / 15e-3)     # all ranks' tasks / max time
    assert res0["rate_G1_tasks_per_s"] == pytest.approx(8000 / 10e-3)
    assert res0["scaling_efficiency"] == pytest.approx((8000 / 15e-3) / (2 * 8000 / 10e-3))
    assert res0["parity"]["checked"] == 8
