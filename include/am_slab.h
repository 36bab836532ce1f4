/*
 * am_slab.h -- the tracker and the trace-replay driver split across GPUs by spatial
 * slabs (the paper runs one controller process, and
 * scales its workers "beyond a single machine", P:194 -- the slab exchange is this
 * repo's design).  Implemented by libametro.so (am_slab.cu); driven round by round by
 * paper_2411_03519_b200/slabs.py, which only marshals pointers and runs the three
 * collectives through torch.distributed (NCCL over NVLink) or an in-process loopback.
 *
 * PARTITION.  The map's rows are split into G horizontal slabs; slab k owns the rows
 * [k*H/G, (k+1)*H/G) and every agent whose y lies there (ownership follows the agent).
 * Rank k keeps a WINDOW: every agent whose y lies within `halo` rows of its slab, in
 * stable slots (a global-id -> slot map; departures free a slot, arrivals take one).
 * Owned agents carry their real status; the other window agents ("ghosts") are
 * tracked as RUNNING (their blocking verdicts are their owner's business; DONE ones as
 * DONE).  With halo >= R_b(S - W) + v (P:406 at the global step spread, plus one move)
 * every agent that can block or couple with an owned agent (R_c = R_b(0)) is in
 * the window, and an agent entering the window cannot affect an owned verdict, so the
 * window's tracker runs the INCREMENTAL round (am_update_replica: only changed agents
 * are re-examined).
 *
 * ONE DISTRIBUTED ROUND (Alg. 3 controller + workers, replay mode P:228):
 *   am_slab_round_local   replica update + tracker round (PEEK) on the window; per local
 *                         cluster: min global id, OR of (owned member RUNNING or
 *                         blocked), max duration of the owned IDLE members; records for
 *                         every cluster that touches the boundary (a ghost, or an owned
 *                         agent inside another rank's window): links {gid, cluster min
 *                         gid} and cluster records {min gid, bad, max duration};
 *     -> all-gather of the records (fixed capacity per rank, device counts)
 *   am_slab_merge         identical on every rank: union-find over the link records in a
 *                         global-id forest (roots = min id, Q10), bad OR-ed and durations
 *                         max-ed per root; for the owned agents the global cluster label,
 *                         the ready bit (IDLE and cluster not bad, P:162 / P:184), dispatch
 *                         of the ready ones (completion time t + the cluster's max
 *                         duration, the move from the perception digest -- all perceived
 *                         agents are in the window), the priority order of the rank's
 *                         ready agents by (step, label, id) (Q9; the global order is
 *                         the merge of the ranks' orders), and this rank's next event and
 *                         activity;
 *     -> all-reduce MIN of {next event, W, -S, no agent active}
 *   am_slab_commit        the common clock advances to the global next event (rounded up
 *                         to the quantum); owned agents whose cluster completed commit their
 *                         move (step + 1, trajectory hash); every commit inside another
 *                         rank's window (old or new position) becomes a delta record for it;
 *     -> all-to-all of the delta records (fixed capacity per peer, device counts)
 *   am_slab_apply         the received deltas update the window: moved agents, arrivals
 *                         (new slots), departures (freed slots); ownership changes with y.
 * The merged result equals the single-GPU round bit for bit (tests/test_gpu_slabs.py),
 * and the replay equals the single-GPU replay and the oracle's.
 *
 * STALE-HALO ROUNDS (stale_rounds = P > 1).  Only every P-th round
 * is a sync round as above; the exchange (all-to-all + apply) happens only after the
 * commits of the round before a sync round, and ownership changes only there.  In the
 * P - 1 rounds in between each rank runs am_slab_round_stale: its window's tracker round
 * with the ghosts at their state of the last exchange (RUNNING), the local clusters, and
 * the dispatch of the owned agents whose cluster holds no ghost and no owned RUNNING or
 * blocked member -- no merge records, no all-gather; the all-reduce of the stats stays
 * (the common clock).  Exact by App. A: the blocking radius shrinks by v per
 * step the blocker advances and the blocker moves at most v per step, so a stale ghost
 * blocks whenever the real agent does, and a real same-step neighbour is either
 * blocked-on through its stale copy or that copy sits in the cluster (deferred).  The
 * schedule equals oracle/orc_replay_stale round for round (tests/test_gpu_slabs.py); the
 * outcome equals lock-step.  A stale round may leave nothing pending: the clock
 * then stays and the rounds up to the next sync round are idle.
 *
 * All arrays are DEVICE pointers; every call is stream-ordered on the slab's stream and
 * none synchronises the host.  Capacity overflows and a halo narrower than the step
 * spread needs are reported through am_slab_flags (checked by the caller every few
 * rounds; the spread grows by at most one step per round, so a check every K rounds
 * with K v of margin keeps every round exact).  Errors: AM_E_ARG, AM_E_WORKSPACE,
 * AM_E_CUDA.
 */
#ifndef AM_SLAB_H_
#define AM_SLAB_H_

#include <stddef.h>
#include <stdint.h>
#include "am.h"
#include "am_driver.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t map_w, map_h;     /* map (tiles): map_w <= 32768, map_h <= 2^30 -- the map may be
                                 taller than one tracker's 32768 rows as long as every window
                                 (slab rows + 2 halo) fits in 32768 rows (its own frame,
                                 y - y0); am_slab_create returns AM_E_ARG otherwise          */
    int32_t r_p, v_max;       /* radius_p, max_vel                                   */
    int32_t metric;           /* AM_METRIC_L2 / AM_METRIC_LINF                               */
    int32_t n_slabs;          /* G >= 1                                                      */
    int32_t my_slab;          /* this rank's slab                                            */
    int32_t n_total;          /* agents over all slabs (global ids 0..n_total-1, < 2^28)     */
    int32_t target_step;      /* agents reaching it become DONE (> 0)                        */
    int32_t halo;             /* window rows beyond the slab on each side (>= r_p + 2 v)     */
    int32_t cap_window;       /* window slots                                                */
    int32_t cap_peer;         /* delta records per peer per round                            */
    int32_t cap_merge;        /* link records and cluster records (each) per rank per round, even */
    int32_t check_rounds;     /* K: the caller checks am_slab_flags at least every K rounds  */
    int32_t stale_rounds;     /* P: a sync round (and exchange) every P rounds; 0 or 1 = every
                                 round.  halo >= r_p + (P + 1) v                              */
} am_slab_geom;

typedef struct am_slab am_slab;

/* flags (am_slab_flags) */
#define AM_SLAB_OVF_WINDOW  0x1   /* no free window slot for an arrival                     */
#define AM_SLAB_OVF_PEER    0x2   /* more delta records for a peer than cap_peer            */
#define AM_SLAB_OVF_MERGE   0x4   /* more link / cluster records than cap_merge             */
#define AM_SLAB_HALO        0x8   /* R_b(S - W) + (K + 1) v > halo: re-window before K rounds */
#define AM_SLAB_LIVENESS    0x10  /* agents not DONE but nothing running after a sync round  */
#define AM_SLAB_LAG         0x20  /* the step spread exceeds the priority key's lag field    */

/* Exchange buffers (int32 words; fixed capacity, counts inside, so a collective moves
 * them without any host synchronisation):
 *   merge buffer of one rank, AM_SLAB_MERGE_WORDS(cap_merge) words (cap_merge even):
 *     [0] link count, [1] cluster count, [2..3] 0, then cap_merge links {gid, cluster min
 *     gid}, then cap_merge cluster records {min gid, bad, max duration lo, hi};
 *   delta block for one peer, AM_SLAB_DELTA_WORDS(cap_peer) words:
 *     [0] record count, [1..5] 0, then cap_peer records {gid, x, y, step, traj lo, traj hi,
 *     status, completion time lo, hi, move x, move y, 0} (the owner's state: a RUNNING
 *     agent that changes owner carries its completion time and move);
 *   stats: int64 [4] {next event, W, -S, no agent active} (all-reduce MIN). */
#define AM_SLAB_MERGE_WORDS(cap) (4 + 6 * (int64_t)(cap))
#define AM_SLAB_DELTA_WORDS(cap) (6 + 12 * (int64_t)(cap))

/* Device workspace bytes of a slab (window arrays, its tracker's workspace, the global-id
 * map and merge forest, exchange buffers). */
size_t am_slab_workspace_size(const am_slab_geom* g);

/* Create rank g->my_slab's slab.  synth: the synthetic policy / latency model
 * (am_driver.h), quantum_us: the event quantum.  workspace: >= am_slab_workspace_size
 * bytes, 256-byte aligned, caller-owned (NULL: the slab allocates its own).  stream:
 * cudaStream_t of every call. */
int am_slab_create(am_slab** out, const am_slab_geom* g, const am_synth* synth, int64_t quantum_us,
                   void* workspace, size_t workspace_bytes, void* stream);

/* (Re)load the window: m agents (global ids, positions int32 [m][2] in GLOBAL map
 * coordinates, steps, statuses -- real ones for owned agents --, trajectory hashes,
 * completion times and moves of owned RUNNING agents), clock t.  Device arrays.  The
 * next round recomputes the window from scratch. */
int am_slab_load(am_slab* s, int32_t m, const int32_t* gid, const int32_t* pos, const int32_t* steps,
                 const uint8_t* status, const uint64_t* traj, const int64_t* tcommit, const int32_t* newpos,
                 int64_t t);

/* Step 1: the window's tracker round; this rank's merge buffer (mbuf). */
int am_slab_round_local(am_slab* s, int32_t* mbuf);

/* Step 2: merge the G ranks' all-gathered merge buffers (mbufs, G consecutive buffers),
 * dispatch this rank's ready agents, write their global ids in priority order to
 * order_out (int32, capacity cap_window) and their count to n_order (device int32), and
 * this rank's stats (int64 [4]). */
int am_slab_merge(am_slab* s, const int32_t* mbufs, int32_t* order_out, int32_t* n_order, int64_t* stats);

/* The round of a stale-halo round (instead of round_local + all-gather + merge):
 * dispatch of the owned agents whose local cluster holds no ghost and no owned RUNNING
 * or blocked member; outputs as am_slab_merge. */
int am_slab_round_stale(am_slab* s, int32_t* order_out, int32_t* n_order, int64_t* stats);

/* order_out of am_slab_merge / am_slab_round_stale is written by the rank's priority sort
 * on a library side stream, beside commit, exchange and apply (none of them reads it),
 * after the merge forest's restore (which reads mbufs: the caller leaves mbufs untouched
 * until the join); n_order and everything else are ordered on the slab's stream as
 * usual.  The slab's stream waits for the side work (an event wait, no host
 * synchronisation) at the start of the next am_slab_round_local / am_slab_round_stale /
 * am_slab_load, or at am_slab_wait_order -- call it before reading order_out on the
 * slab's stream. */
int am_slab_wait_order(am_slab* s);

/* Device time of the last side-stream work (forest restore + priority sort) in ms
 * (timing events around it; blocks the host until it is done).  AM_E_STATE before the
 * first round. */
int am_slab_order_ms(am_slab* s, float* ms);

/* Step 3: commit at the global next event (stats_global: the all-reduced MIN of the
 * ranks' stats).  dsend non-NULL (an exchange follows): pack the delta records of every
 * owned agent committed since the last exchange -- dsend = G delta blocks (block j for
 * rank j; this rank's own block stays empty) -- and hand the agents that left the slab
 * over (ghosts here from now on).  dsend NULL: the commits stay local until the next
 * exchange (stale-halo rounds). */
int am_slab_commit(am_slab* s, const int64_t* stats_global, int32_t* dsend);

/* Step 4: apply the received delta blocks (drecv: block r from rank r). */
int am_slab_apply(am_slab* s, const int32_t* drecv);

/* Per window slot, after the last merge (device pointers owned by the slab): the global
 * id (-1 free), the global cluster label (-1 for DONE agents and ghosts), the ready bit
 * (owned agents). */
int am_slab_outputs(am_slab* s, const int32_t** slot_gid, const int32_t** slot_label, const uint8_t** slot_ready);

/* The window state (device pointers owned by the slab): positions int32 [L][2] (global
 * coordinates), steps, statuses (owned: real; ghosts: RUNNING / DONE), owned flags,
 * trajectory hashes; and device counters int64 [4]: {clock t, time of the last commit
 * that finished an agent, agent-steps dispatched by this rank, rounds}. */
int am_slab_state(am_slab* s, const int32_t** pos, const int32_t** steps, const uint8_t** status,
                  const uint64_t** traj, const int64_t** tcommit, const int32_t** newpos, const int64_t** counters);

/* Per window slot: 1 if this rank owns the agent (device pointer owned by the slab). */
int am_slab_owned(am_slab* s, const uint8_t** own);

/* Sticky flags (AM_SLAB_*) and the window occupancy; synchronises the slab's stream and
 * clears the flags. */
int am_slab_flags(am_slab* s, int32_t* flags, int32_t* window_used);

/* The slab's tracker context (statistics, profiling) and its stream. */
am_ctx* am_slab_tracker(am_slab* s);
void* am_slab_stream(am_slab* s);

int am_slab_destroy(am_slab* s);

#ifdef __cplusplus
}
#endif
#endif /* AM_SLAB_H_ */
