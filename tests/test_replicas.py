"""Multi-process host logic of the N>1 path on CPU (gloo, world_size 2).

The path does not shard (lexicographic Gauss-Seidel is one global dependency
chain), so N GPUs run N independent replicas: the only
cross-rank traffic is the timing/work aggregation of bench.py, and the
reference arm runs on rank 0 alone.
"""

from __future__ import annotations

import os
import socket
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, REPO)
    import bench

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank r took (r + 1) ms for 10 + r iterations
        t, u = bench.aggregate_over_ranks(1.0 + rank, 10 + rank, world, "cpu")
        # the reference arm: ranks other than 0 return without work or output
        class A:
            steps, warmup = 1, 0

        if rank != 0:
            bench.run_reference(A())
        out.put((rank, t, u))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_replica_aggregation_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    for rank, t, u in res:
        assert t == 2.0  # max over ranks
        assert u == 21.0  # work summed over ranks


def test_single_rank_aggregation_is_identity():
    sys.path.insert(0, REPO)
    import bench

    assert bench.aggregate_over_ranks(3.5, 7, 1, "cpu") == (3.5, 7.0)
