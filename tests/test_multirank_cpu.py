"""Multi-rank host logic on CPU (gloo, world_size 2): the NCCL unique-id
broadcast, slab partition and the max-over-ranks timing reduction the bench
and the slab contexts rely on.  No GPU needed."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2403_10706_b200 import hysco as H


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2403_10706_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nid = D.share_nccl_id()
        tmax = D.max_over_ranks(1.5 + rank)
        tsum = D.sum_over_ranks(1.0)
        q.put((rank, nid, tmax, tsum, D.slab_bounds(512, world, rank)))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_share_id_and_reduce():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    (r0, id0, m0, s0, b0), (r1, id1, m1, s1, b1) = out
    assert id0 == id1 and len(id0) == 128 and any(id0)
    assert m0 == m1 == 2.5 and s0 == s1 == 2.0
    assert b0 == (0, 256) and b1 == (256, 512)


@pytest.mark.parametrize("n1,world", [(512, 8), (168, 3), (7, 3), (16, 16), (5, 4)])
def test_slab_bounds_partition(n1, world):
    spans = [H.slab_bounds(n1, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n1
    assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
    sizes = [b - a for a, b in spans]
    assert min(sizes) >= 1 and max(sizes) - min(sizes) <= 1
