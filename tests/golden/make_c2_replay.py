"""Writes tests/golden/c2_replay_T1000.txt: the CPU oracle's out-of-order replay of
BASELINE config 2 (500 agents on 20 replicated Smallville maps, busy-hour latencies,
exact events, T = 1000; Alg. 3 with infinite capacity, replay mode P:228) -- the
oracle takes ~10 min for it, too long to rerun inside every GPU test session.

Calls only oracle/ and amgen (seeded inputs).  Run:  python tests/golden/make_c2_replay.py

Contents: the round count, T_ooo, a blake2b-128 chain over the per-round logs (for
every round that dispatched agents: the count, the dispatched ids in priority order,
their cluster labels; int32 little-endian) with a checkpoint every 1000 logged rounds,
and a blake2b-128 of the final positions and trajectory hashes.  The same oracle run's
lock-step result (Alg. 1) must give the same trajectory hashes."""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import amgen  # noqa: E402
import oracle as O  # noqa: E402

CHECK_EVERY = 1000


def log_chain(rounds):
    """rounds: iterable of (ids int32[], labels int32[]) of the non-empty rounds."""
    h = hashlib.blake2b(digest_size=16)
    marks = []
    k = 0
    for ids, lab in rounds:
        h.update(np.int32(len(ids)).tobytes())
        h.update(np.ascontiguousarray(ids, np.int32).tobytes())
        h.update(np.ascontiguousarray(lab, np.int32).tobytes())
        k += 1
        if k % CHECK_EVERY == 0:
            marks.append(h.hexdigest())
    return k, marks, h.hexdigest()


def state_hash(x, y, traj):
    h = hashlib.blake2b(digest_size=16)
    for a in (np.asarray(x, np.int32), np.asarray(y, np.int32), np.asarray(traj, np.uint64)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    w = amgen.config("C2")
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, wall=w.wall)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps)
    r = O.replay(p, sy, w.x, w.y, Q=w.Q, log_rounds=2_000_000, log_entries=len(w.x) * w.steps + 10)
    assert r["log_complete"]
    ls = O.lockstep(p, sy, w.x, w.y, w.steps)
    assert np.array_equal(r["traj"], ls["traj"]), "OoO != lock-step (P:27)"

    def rounds():
        k = 0
        for nr in r["log_nready"]:
            if nr:
                yield r["log_id"][k:k + nr], r["log_label"][k:k + nr]
            k += nr

    nlog, marks, final = log_chain(rounds())
    with open(os.path.join(HERE, "c2_replay_T1000.txt"), "w") as f:
        f.write("# C2 (500 agents, 700x400 replicated town, busy hour, exact events, T=1000):\n")
        f.write("# oracle.replay + oracle.lockstep, written by tests/golden/make_c2_replay.py\n")
        f.write(f"rounds {int(r['rounds'][0])}\n")
        f.write(f"T_ooo {int(r['T_ooo'][0])}\n")
        f.write(f"T_sync {int(ls['T_sync'][0])}\n")
        f.write(f"logged_rounds {nlog}\n")
        f.write(f"state {state_hash(r['x'], r['y'], r['traj'])}\n")
        f.write(f"log_final {final}\n")
        for i, m in enumerate(marks):
            f.write(f"log_mark {(i + 1) * CHECK_EVERY} {m}\n")


if __name__ == "__main__":
    main()
