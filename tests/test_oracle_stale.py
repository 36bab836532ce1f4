"""Pins of the oracle's stale-halo slab replay (orc_replay_stale).

Stale rounds are this repo's construction, derived from App. A: the
blocking radius R_b(s_A - s_B) = (s_A - s_B + 1) v + r_p shrinks by exactly v per step
the blocker advances, and a blocker moves at most v per step, so a blocker seen at an
older (step, position) blocks whenever the real one does; an agent coupled with a
foreign agent (same step) is either blocked by that agent's stale copy or in a
cluster with it (RUNNING: deferred).  The pins below do not re-derive that argument
from the oracle's code:

* P = 1 equals the plain replay round for round (no stale round exists);
* hand-worked schedules (a blocker seen one sync period late; a coupled pair across a
  slab edge that only sync rounds can dispatch, with idle stale rounds);
* for random workloads and every (G, P): zero I1 / I2 violations (nobody dispatched
  within a blocker's radius, no committed state invalid) and the lock-step final
  state (outcome preservation)."""
import numpy as np
import pytest

import amgen
import oracle as O


def _stay_synth(dur):
    lm = amgen.latency_model()
    return O.SynthTables.from_model(lm, dur_table=np.asarray(dur, np.int64), policy=1)


def _rounds(r):
    """Per round: (time, dispatched ids in order, their labels)."""
    out, k = [], 0
    for t, nr in zip(r["log_t"], r["log_nready"]):
        out.append((int(t), list(r["log_id"][k:k + nr]), list(r["log_label"][k:k + nr])))
        k += nr
    return out


def test_stale_blocker_seen_late_hand_schedule():
    """A (id 0, slab 0 at row 9) takes 1 us per step, B (id 1, slab 1 at row 13) 10 us;
    r_p = 1, v = 1: |AB| = 4, never coupled (R_c = 2), B blocks A iff s_A - s_B >= 2.

    Synchronous (P = 1), worked by hand:
      t=0 both; t=1 A; t=2 - (A at 2, B at 0); t=10 B, A; t=11 -; t=20 B, A; t=21 -;
      t=30 B (A done); t=40 end.
    P = 3 (sync rounds 0, 3, 6): round 5 (t=20) is stale -- slab 0 still sees B at the
    round-3 snapshot (step 1) while B is at step 2, so A (step 3) stays blocked; slab 1
    dispatches B.  Round 6 (sync, t=30) dispatches both at step 3; round 7 (t=31) idle."""
    p = O.params(10, 20, 1, 1, target=4)
    sy = _stay_synth([[1] * 4, [10] * 4])
    sync = O.replay(p, sy, [5, 5], [9, 13], log_rounds=50, log_entries=50, check=True)
    assert _rounds(sync) == [(0, [0, 1], [0, 1]), (1, [0], [0]), (2, [], []), (10, [1, 0], [1, 0]),
                             (11, [], []), (20, [1, 0], [1, 0]), (21, [], []), (30, [1], [1])]
    st = O.replay_stale(p, sy, [5, 5], [9, 13], G=2, P=3, log_rounds=50, log_entries=50, check=True)
    assert _rounds(st) == [(0, [0, 1], [0, 1]), (1, [0], [0]), (2, [], []), (10, [1, 0], [1, 0]),
                           (11, [], []), (20, [1], [1]), (30, [0, 1], [0, 1]), (31, [], [])]
    for r in (sync, st):
        assert int(r["T_ooo"][0]) == 40 and int(r["rounds"][0]) == 8 and r["violations"] == 0
    np.testing.assert_array_equal(st["traj"], sync["traj"])
    # one slab: no foreign agent, the stale rounds see everything current
    one = O.replay_stale(p, sy, [5, 5], [9, 13], G=1, P=3, log_rounds=50, log_entries=50)
    assert _rounds(one) == _rounds(sync)


def test_coupled_pair_across_the_slab_edge_waits_for_sync_rounds():
    """A (row 9, slab 0) and B (row 10, slab 1) are always coupled (|AB| = 1 <= R_c = 2,
    equal steps): a cluster spanning two slabs.  In a stale round each slab sees the
    other member at its snapshot step (one behind), which blocks (|AB| = 1 <= R_b(1)):
    nothing is dispatched, nothing is pending, the clock stays, and the pair advances
    only at sync rounds (0, 3, 6): rounds 1-2 and 4-5 are idle."""
    p = O.params(10, 20, 1, 1, target=3)
    sy = _stay_synth([[4, 4, 4], [7, 7, 7]])
    st = O.replay_stale(p, sy, [5, 5], [9, 10], G=2, P=3, log_rounds=50, log_entries=50, check=True)
    assert _rounds(st) == [(0, [0, 1], [0, 0]), (7, [], []), (7, [], []), (7, [0, 1], [0, 0]),
                           (14, [], []), (14, [], []), (14, [0, 1], [0, 0])]
    assert int(st["T_ooo"][0]) == 21 and int(st["rounds"][0]) == 7 and st["violations"] == 0
    sync = O.replay(p, sy, [5, 5], [9, 10], log_rounds=50, log_entries=50)
    assert _rounds(sync) == [(0, [0, 1], [0, 0]), (7, [0, 1], [0, 0]), (14, [0, 1], [0, 0])]
    np.testing.assert_array_equal(st["traj"], sync["traj"])


def test_arguments():
    p = O.params(10, 20, 1, 1, target=2)
    sy = _stay_synth([[1, 1]])
    for G, P in ((0, 1), (1, 0)):
        with pytest.raises(RuntimeError):
            O.replay_stale(p, sy, [1], [1], G=G, P=P)


@pytest.mark.parametrize("G", [1, 2, 4])
def test_period_one_is_the_synchronous_replay(G):
    w = amgen.config("C1", steps=120)
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, wall=w.wall)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps)
    a = O.replay(p, sy, w.x, w.y, Q=w.Q, log_rounds=10**5, log_entries=10**5)
    b = O.replay_stale(p, sy, w.x, w.y, G=G, P=1, Q=w.Q, log_rounds=10**5, log_entries=10**5)
    for k in ("x", "y", "traj", "T_ooo", "rounds", "log_t", "log_nready", "log_id", "log_label"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


@pytest.mark.parametrize("G,P", [(2, 2), (3, 3), (4, 5), (8, 4)])
def test_stale_replay_is_safe_and_outcome_preserving(G, P):
    """Random state on a 120 x 160 map (one row band per slab holds ~50 agents): zero
    violations at every dispatch and commit, and the final state of lock-step."""
    rng = np.random.default_rng(100 * G + P)
    n, W, H, T = 200, 120, 160, 30
    x = rng.integers(0, W, n).astype(np.int32)
    y = rng.integers(0, H, n).astype(np.int32)
    lm = amgen.latency_model()
    sy = O.SynthTables.from_model(lm)
    p = O.params(W, H, 4, 1, target=T)
    st = O.replay_stale(p, sy, x, y, G=G, P=P, Q=50_000, log_rounds=10**5, log_entries=10**6, check=True)
    assert st["violations"] == 0 and st["log_complete"]
    ls = O.lockstep(p, sy, x, y, T)
    np.testing.assert_array_equal(st["x"], ls["x"])
    np.testing.assert_array_equal(st["y"], ls["y"])
    np.testing.assert_array_equal(st["traj"], ls["traj"])
    # every agent-step dispatched exactly once
    assert int(st["log_nready"].sum()) == n * T
    sync = O.replay(p, sy, x, y, Q=50_000, log_rounds=10**5, log_entries=10**6)
    assert not np.array_equal(sync["log_nready"], st["log_nready"]) or G == 1   # the stale rounds changed the schedule
