"""The multi-GPU exchange layer on CPU with gloo, world size 2: the three collectives of
a distributed round (slabs.DistWorld) on fixed-capacity buffers whose counts travel
inside them -- all-gather of merge buffers, all-reduce MIN of the int64 stats, equal-split
all-to-all of delta blocks -- deliver exactly what the slab kernels expect, through the
host-staged wrapper the multi-process GPU test uses (slabs.HostStagedDist)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_03519_b200 import slabs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        hd = slabs.HostStagedDist(dist)
        # merge buffers: [count links, count clusters, 0, 0, records ...] per rank
        cap = 4
        mb = torch.zeros(4 + 6 * cap, dtype=torch.int32)
        mb[0] = rank + 1
        mb[4:4 + 2 * (rank + 1)] = torch.arange(2 * (rank + 1), dtype=torch.int32) + 100 * rank
        mall = torch.empty((world, 4 + 6 * cap), dtype=torch.int32)
        hd.all_gather_into_tensor(mall.view(-1), mb)
        ok1 = all(int(mall[r, 0]) == r + 1 and
                  torch.equal(mall[r, 4:4 + 2 * (r + 1)], torch.arange(2 * (r + 1), dtype=torch.int32) + 100 * r)
                  for r in range(world))
        # stats: int64 MIN (next event, W, -S, inactive)
        st = torch.tensor([1000 + rank, 5 + rank, -(10 + rank), 1 - rank], dtype=torch.int64)
        hd.all_reduce(st, op=dist.ReduceOp.MIN)
        ok2 = st.tolist() == [1000, 5, -(10 + world - 1), 0]
        # delta blocks: block j of rank r goes to rank j; header = record count
        capp = 3
        ds = torch.zeros((world, 6 + 12 * capp), dtype=torch.int32)
        for j in range(world):
            if j != rank:
                ds[j, 0] = rank + 1
                ds[j, 6] = 1000 * rank + j
        dr = torch.empty_like(ds)
        hd.all_to_all_single(dr, ds)
        ok3 = all((int(dr[r, 0]) == (r + 1 if r != rank else 0)) and
                  (r == rank or int(dr[r, 6]) == 1000 * r + rank) for r in range(world))
        q.put((rank, ok1, ok2, ok3))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, ok1, ok2, ok3 in res:
        assert ok1 and ok2 and ok3, (rank, ok1, ok2, ok3)


def test_partition_rows_and_halo():
    rows = slabs.slab_of_rows(100, 3)
    assert rows == [(0, 33), (33, 66), (66, 100)]
    y = torch.tensor([0, 32, 33, 65, 66, 99])
    assert slabs.partition(y, 100, 3).tolist() == [0, 0, 1, 1, 2, 2]
    # R_b(spread + 1) + (K + 1) v  (P:406 plus K rounds of growth at one step per round)
    assert slabs.halo_needed(0, 4, 1, 16) == (0 + 2) * 1 + 4 + 17
    assert slabs.halo_needed(80, 4, 1, 16) == 82 + 4 + 17
