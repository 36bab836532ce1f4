"""slabs.DistWorld itself -- the distributed round as bench.py --gpus N runs it -- with
two processes (two ranks, two slabs) on ONE GPU: torch.distributed over gloo with the
CUDA buffers staged through the host (NCCL refuses two ranks per device).  The replay of
C2 (500 agents, 25 steps) equals the oracle's round by round (the ranks' orders merged)
and in its final state -- synchronous, and with stale-halo rounds (a sync round every
P = 4 rounds, orc_replay_stale)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, P):
    import torch
    import torch.distributed as dist

    import amgen
    from paper_2411_03519_b200 import slabs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        w = amgen.config("C2", steps=25)
        lm = amgen.latency_model(w.profile)
        sy = slabs.Synth(lm, wall=w.wall)
        wd = slabs.DistWorld(slabs.HostStagedDist(dist), w.map_w, w.map_h, w.r_p, w.v, w.x, w.y, w.steps, sy, w.Q,
                             check_rounds=4, stale_rounds=P)
        logs = []
        k = 0
        while True:
            log = []
            wd.round(log)
            o = log[0]
            logs.append({key: v.cpu().numpy() for key, v in o.items()})
            k += 1
            if k % wd.K == 0 and wd.check():
                break
        res = wd.results()
        q.put((rank, logs, {kk: (vv if not isinstance(vv, np.ndarray) else vv) for kk, vv in res.items()}, None))
        wd.close()
    except Exception as e:   # report instead of hanging the parent
        import traceback
        q.put((rank, None, None, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P", [1, 4])
def test_dist_world_two_ranks_one_gpu_vs_oracle(P):
    import torch.multiprocessing as mp

    import amgen
    import oracle as O
    from paper_2411_03519_b200 import slabs
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q, P)) for r in range(2)]
    for p in ps:
        p.start()
    got = {}
    for _ in ps:
        rank, logs, res, err = q.get(timeout=900)
        assert err is None, err
        got[rank] = (logs, res)
    for p in ps:
        p.join(timeout=120)
    w = amgen.config("C2", steps=25)
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, wall=w.wall)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps)
    if P == 1:
        r = O.replay(p, sy, w.x, w.y, Q=w.Q, log_rounds=10**6, log_entries=len(w.x) * w.steps + 10)
    else:
        r = O.replay_stale(p, sy, w.x, w.y, G=2, P=P, Q=w.Q, log_rounds=10**6, log_entries=len(w.x) * w.steps + 10)
    ologs, k = [], 0
    for nr in r["log_nready"]:
        if nr:
            ologs.append((r["log_id"][k:k + nr], r["log_label"][k:k + nr]))
        k += nr
    import torch
    glogs = []
    for a, b in zip(got[0][0], got[1][0]):
        outs = [{kk: torch.as_tensor(vv) for kk, vv in o.items()} for o in (a, b)]
        ids, lab = slabs.merged_order(outs)
        if len(ids):
            glogs.append((ids, lab))
    assert len(glogs) == len(ologs)
    for (gi, gl), (oi, ol) in zip(glogs, ologs):
        np.testing.assert_array_equal(gi, oi)
        np.testing.assert_array_equal(gl, ol)
    res = got[0][1]
    np.testing.assert_array_equal(res["traj"], r["traj"])
    np.testing.assert_array_equal(res["x"], r["x"])
    assert res["T_ooo"] == int(r["T_ooo"][0]) and res["rounds"] == int(r["rounds"][0])
    assert res["dispatched"] == len(w.x) * w.steps
