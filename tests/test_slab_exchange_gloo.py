"""The multi-GPU exchange layer (slabs.round_distributed's collectives) on CPU with
gloo, world size 2: the variable-size all-gather and the counts-then-payload
all-to-all deliver exactly the records the slab kernels would send."""
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
        dev = torch.device("cpu")
        # variable all-gather of link records: rank k contributes k+1 pairs
        t = torch.arange(2 * (rank + 1), dtype=torch.int32).reshape(-1, 2) + 100 * rank
        g = slabs._all_gather_var(dist, t, world, dev)
        exp = torch.cat([torch.arange(2 * (k + 1), dtype=torch.int32).reshape(-1, 2) + 100 * k
                         for k in range(world)])
        ok1 = torch.equal(g, exp)
        # counts then payload (halo records): rank k sends k+2 records to every other rank
        out = [torch.full((0 if j == rank else rank + 2, 4), rank, dtype=torch.int32) for j in range(world)]
        sc = torch.tensor([int(o.shape[0]) for o in out], dtype=torch.int64)
        rc = torch.empty_like(sc)
        dist.all_to_all_single(rc, sc)
        recv = torch.empty((int(rc.sum()), 4), dtype=torch.int32)
        dist.all_to_all_single(recv, torch.cat(out), output_split_sizes=rc.tolist(),
                               input_split_sizes=sc.tolist())
        exp2 = torch.cat([torch.full((0 if j == rank else j + 2, 4), j, dtype=torch.int32) for j in range(world)])
        ok2 = torch.equal(recv, exp2)
        ws = torch.tensor([5 + rank, -(10 + rank)], dtype=torch.int32)
        dist.all_reduce(ws, op=dist.ReduceOp.MIN)
        ok3 = ws.tolist() == [5, -(10 + world - 1)]
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


def test_partition_rows():
    rows = slabs.slab_of_rows(100, 3)
    assert rows == [(0, 33), (33, 66), (66, 100)]
    y = torch.tensor([0, 32, 33, 65, 66, 99])
    assert slabs.partition(y, 100, 3).tolist() == [0, 0, 1, 1, 2, 2]
