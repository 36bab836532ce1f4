/*
 * am.h -- C ABI of the B200-native spatio-temporal dependency tracker of
 * AI Metropolis (arXiv 2411.03519), the per-round hot path of its out-of-order
 * scheduler.  Implemented by libametro.so (paper_2411_03519_b200/csrc, sm_100a).
 *
 * Citations "P:<line>" refer to /root/reference/PAPER.md.
 *
 * The method, per scheduling round (one controller iteration of Alg. 3):
 *   - coupling (App. A): A,B coupled iff Step_A == Step_B and
 *     dist(A,B) <= radius_p + max_vel;
 *   - blocking (App. A): A blocked by B iff Step_B < Step_A and
 *     dist(A,B) <= (Step_A - Step_B + 1) * max_vel + radius_p;
 *   - clusters = connected components of the coupling graph over the agents that are
 *     not DONE ("group of coupled agents at the same step"; geo_clustering P:109);
 *   - a cluster is ready iff none of its members is blocked and none is
 *     still RUNNING (in flight);
 *   - ready agents are reported in priority order: by step first (priority queues
 *     "sort tasks based on their associated steps", section 3.5), then
 *     by cluster label, then agent id (our tie-break, Q9).
 * dist is Euclidean on integer tile coordinates unless AM_METRIC_LINF.
 *
 * Agent states: IDLE (waiting at its step), RUNNING (dispatched by am_ready, its
 * step not committed yet), DONE (reached target_step; never blocks, never ready).
 *
 * MEMORY / OWNERSHIP.  All array arguments are DEVICE pointers (e.g. torch CUDA
 * tensors' data_ptr()) owned by the caller, unless marked "host".  Work is enqueued
 * on the context's stream (am_config.stream, a cudaStream_t; NULL = legacy default
 * stream) and is asynchronous: the caller keeps every input/output array alive and
 * untouched until that stream work completes (am_ready / am_sync synchronise).
 * DEVICE WORKSPACE (two-phase idiom): am_workspace_size() gives the bytes a context
 * with these arguments needs; the caller allocates them (e.g. a torch uint8 CUDA
 * tensor, so PyTorch's allocator serves all device memory), passes the pointer in
 * am_config.workspace and keeps it alive until am_destroy.  With workspace == NULL the
 * context allocates its own (cudaMalloc in am_init, cudaFree in am_destroy).  The
 * context otherwise owns only small host state, a pinned control-block mirror, and
 * its side streams / events.  Nothing is allocated after am_init.  A context is not
 * thread-safe: one host thread at a time.
 *
 * ERRORS.  Every call returns AM_OK (0) or a negative AM_E_* code; no exception
 * crosses the ABI.  Commit validation happens on the device inside am_update; its
 * verdict is reported by the next synchronising call (am_ready or am_sync).  A
 * rejected update is not applied: the context stays at the last good state.
 * am_last_error() gives a human-readable message for the last failing call.
 */
#ifndef AM_H_
#define AM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes */
#define AM_OK            0
#define AM_E_ARG        -1   /* bad argument (NULL pointer, negative size, map too large) */
#define AM_E_BOUNDS     -2   /* a position outside [0,map_w) x [0,map_h)                  */
#define AM_E_PROTOCOL   -3   /* step change not in {0,+1}; +1 for a non-RUNNING agent;    */
                             /* moved without stepping; step outside [0,target]          */
#define AM_E_VELOCITY   -4   /* a commit moved farther than max_vel              */
#define AM_E_CUDA       -5   /* CUDA runtime error (message in am_last_error)             */
#define AM_E_NCCL       -6   /* reserved for the multi-GPU exchange                       */
#define AM_E_STATE      -11  /* call out of order (e.g. am_ready before any am_update)    */
#define AM_E_WORKSPACE  -13  /* caller workspace too small or not 256-byte aligned         */
#define AM_E_LIVENESS   -12  /* replay driver: nothing running but agents not DONE        */

/* agent status values (am_set_state / am_status) */
#define AM_IDLE     0
#define AM_RUNNING  1
#define AM_DONE     2

/* distance metric */
#define AM_METRIC_L2    0    /* Euclidean, compared as squared integers (default)        */
#define AM_METRIC_LINF  1    /* Chebyshev variant                                         */
#define AM_METRIC_GRAPH 2    /* hop count on a graph (am_set_graph; "non-Euclidean spaces   */
                             /* such as social networks"): positions are nodes        */
                             /* (x = node in [0, map_w), map_h = 1); fused path only         */

/* flags (am_config.flags, am_set_flags) */
#define AM_VALIDATE     0x1u /* validate commits in am_update (protocol + velocity)       */
#define AM_PEEK         0x2u /* am_ready does not dispatch (IDLE -> RUNNING)              */
#define AM_DIGEST       0x4u /* compute perception digests for the replay driver          */
#define AM_ASYNC        0x8u /* am_ready does not synchronise; n_ready may be NULL        */
#define AM_FORCE_BINNED 0x10u/* always use the cell-binned pipeline (tests)                */
#define AM_FORCE_SMALL  0x20u/* always use the fused per-simulation kernel (<=1024/sim)    */
#define AM_STATS        0x40u/* count scan work (cells, candidate pairs) for am_scan_stats  */
#define AM_SCAN_THREAD  0x80u/* one thread per agent neighbour scan (ablation baseline)    */
#define AM_NO_ORDER     0x100u/* am_ready leaves `order` unwritten (the mask, labels and the  */
                              /* ready count are computed; the spatial-slab window tracker   */
                              /* orders its ranks' ready agents itself)                      */
#define AM_LABELS_ONLY  0x200u/* binned path: am_ready stops after the labels and blocking   */
                              /* verdicts (am_clusters, am_blocked): no mask, order, ready   */
                              /* count or dispatch (mask / order may be NULL) -- the slab    */
                              /* window tracker decides readiness in its merge               */
#define AM_DBG_SKIP_NEAR 0x1000u /* PROFILING ONLY: skip the scan's near phase (wrong results) */
#define AM_DBG_SKIP_FAR  0x2000u /* PROFILING ONLY: skip the scan's far phase (wrong results)  */

typedef struct am_ctx am_ctx;                 /* opaque */

typedef struct {
    int32_t  target_step;  /* agents reaching it become DONE (Alg. 3); 0 = none    */
    int32_t  n_sims;       /* >= 1 independent simulations; sim b owns agents             */
                           /* [b*n/n_sims, (b+1)*n/n_sims); no interaction across sims    */
    int32_t  cell;         /* cell edge in tiles for binning, power of two; 0 = auto      */
    int32_t  metric;       /* AM_METRIC_L2 or AM_METRIC_LINF                              */
    uint32_t flags;        /* AM_* flags                                                  */
    void*    stream;       /* cudaStream_t                                                */
    void*    workspace;    /* caller-owned device memory of >= am_workspace_size() bytes, */
                           /* 256-byte aligned; NULL = the context allocates its own       */
    size_t   workspace_bytes;
} am_config;

/* Round statistics of the most recent am_ready (host copy, filled at its sync). */
typedef struct {
    int32_t n_ready;       /* agents reported ready (and dispatched unless AM_PEEK)       */
    int32_t n_active;      /* agents not DONE                                             */
    int32_t n_running;     /* agents RUNNING when the round started                       */
    int32_t watermark;     /* W = min step over non-DONE agents (base_step)        */
    int32_t max_step;      /* S = max step over non-DONE agents                           */
    int32_t n_clusters;    /* ready clusters                                              */
    int32_t path;          /* 0 = fused per-simulation kernel, 1 = cell-binned pipeline   */
    int32_t cell;          /* cell edge used by the binned pipeline                       */
    int32_t n_work;        /* binned: agents re-scanned this round (incremental work queue) */
    int32_t n_far;         /* binned: queued IDLE agents ahead of W (far blocking test due)  */
    int32_t n_items;       /* binned: 4x4-cell blocks the far test walked in the pyramid   */
    int32_t n_edges;       /* binned: coupling edges of this round (carried + new)        */
    int32_t n_passes;      /* binned: radix passes the priority order needed              */
    int32_t rebuilt;       /* binned: 1 if the round rebuilt the cell binning, 0 if it kept  */
                           /* the loose cells of the last rebuild (records updated in place) */
    int32_t drift;         /* binned: tiles any agent lies outside its record's cell (D)     */
    int32_t n_rebuilds;    /* binned: cell-binning rebuilds since am_init                    */
} am_round_stats;

/* Device workspace bytes am_init needs for these arguments (the same validation as
 * am_init; 0 if they are invalid).  No CUDA call: usable before any device work. */
size_t am_workspace_size(int32_t map_w, int32_t map_h, int32_t radius_p, int32_t v_max, int32_t n_agents,
                         const am_config* cfg);

/* Create a tracker for n_agents agents on a map_w x map_h tile map (1..32768 each),
 * perception radius radius_p >= 0 and max speed v_max >= 0 tiles per step.
 * cfg may be NULL (defaults: no target, 1 sim, auto cell, L2, AM_VALIDATE, own workspace).
 * *out receives the context.  Radii >= 46340 tiles are clamped (they already cover
 * every distance on a <= 32768^2 map; no result changes).  Errors: AM_E_ARG, AM_E_WORKSPACE,
 * AM_E_CUDA. */
int am_init(am_ctx** out, int32_t map_w, int32_t map_h, int32_t radius_p, int32_t v_max,
            int32_t n_agents, const am_config* cfg);

/* Agents' positions and simulation steps (update_agents, Alg. 3 l.11 P:112).
 * positions: int32 [n_agents][2] (x, y); sim_steps: int32 [n_agents].
 * The first call after am_init (or am_reset) sets the initial state: every agent IDLE,
 * or DONE if its step equals target_step.  Later calls are commits: an agent may
 * change only if RUNNING, by exactly +1 step and a move of at most v_max (P:153,
 * App. A); it then becomes IDLE (DONE at target_step).  Unchanged agents keep
 * their status.  Validation (AM_VALIDATE) is reported by the next am_ready/am_sync. */
int am_update(am_ctx* ctx, const int32_t* positions, const int32_t* sim_steps);

/* The graph of AM_METRIC_GRAPH: dist = uint16 [n_nodes][n_nodes] hop distances (device,
 * caller-owned, 0xFFFF = unreachable; a shortest-path metric, so App. A's derivation --
 * triangle inequality and at most v hops per step -- holds), n_nodes == map_w.  Call
 * before the first am_update.  Errors: AM_E_ARG (wrong metric / size / path). */
int am_set_graph(am_ctx* ctx, const uint16_t* dist, int32_t n_nodes);

/* Set the full state, including statuses (uint8 [n_agents], AM_IDLE/RUNNING/DONE),
 * without commit validation (snapshots).  Bounds and status values are checked; the call
 * synchronises and reports them, unless AM_ASYNC is set (then it is stream-ordered and a
 * rejected state is reported by the next synchronising call). */
int am_set_state(am_ctx* ctx, const int32_t* positions, const int32_t* sim_steps,
                 const uint8_t* status);

/* Replica update (the spatial-slab window of am_slab.h): the full state including
 * statuses (uint8 [n_agents]; AM_DONE also marks an absent slot), diffed against the
 * current one without commit validation.  An agent whose position or step changed, that
 * arrived (absent -> present) or departed (present -> absent) is re-examined by the next
 * round; every other verdict, coupling edge and cluster is reused (the incremental
 * round).  Status changes IDLE <-> RUNNING alone are not changes.
 * Stream-ordered (no synchronisation); errors (bounds, status values) surface at the
 * next synchronising call.  The first call after am_init / am_reset acts as am_set_state. */
int am_update_replica(am_ctx* ctx, const int32_t* positions, const int32_t* sim_steps,
                      const uint8_t* status);

/* One scheduling round (geo_clustering + ready filter + priority order, Alg. 3 l.8-9).
 * mask:  uint8 [n_agents]   1 iff the agent is ready (IDLE and its cluster unblocked).
 * order: int32 [n_agents]   capacity; the first *n_ready entries are the ready agents
 *                           sorted by (sim, step, cluster label, id).
 * n_ready: host int32*, receives the count (may be NULL with AM_ASYNC).
 * Unless AM_PEEK, ready agents become RUNNING (dispatched to the ready queue).
 * Synchronises the stream unless AM_ASYNC.  Returns a pending validation error. */
int am_ready(am_ctx* ctx, uint8_t* mask, int32_t* order, int32_t* n_ready);

/* Cluster labels of the most recent round: int32 [n_agents]; label = smallest agent
 * id of the agent's cluster, -1 for DONE agents.  Stream-ordered copy. */
int am_clusters(am_ctx* ctx, int32_t* labels);

/* Blocking verdicts of the most recent round: uint8 [n_agents] (device), 1 iff the
 * agent is IDLE and blocked by some agent behind it in time; 0 for
 * RUNNING and DONE agents (their clusters are never ready anyway).  Used by the
 * spatial-slab merge (am_slab.h).  Stream-ordered copy. */
int am_blocked(am_ctx* ctx, uint8_t* blocked);

/* Current statuses (uint8 [n_agents], device), stream-ordered copy. */
int am_status(am_ctx* ctx, uint8_t* status);

/* Statistics of the most recent synchronised am_ready (host struct). */
int am_stats(const am_ctx* ctx, am_round_stats* out);

/* Synchronise the stream; returns (and clears) a pending validation/CUDA error. */
int am_sync(am_ctx* ctx);

/* Replace the flags / the stream. */
int am_set_flags(am_ctx* ctx, uint32_t flags);
int am_set_stream(am_ctx* ctx, void* stream);

/* The stream the context's work is ordered on now (a replay driver moves its context
 * onto the replay's own stream, am_driver.h): a caller reading an output of a
 * stream-ordered getter (am_status, am_clusters, am_blocked) from another stream makes
 * that stream wait on this one first. */
void* am_get_stream(const am_ctx* ctx);

/* Forget the state: the next am_update is an initial state again. */
int am_reset(am_ctx* ctx);

/* Device workspace bytes of the context (caller-provided or its own). */
size_t am_workspace_bytes(const am_ctx* ctx);

/* Device pointer of the round's device-side ready count (int32), for graph capture. */
const int32_t* am_ready_count_device(const am_ctx* ctx);

int am_destroy(am_ctx* ctx);

/* Message of the last failing call on ctx ("" if none); ctx may be NULL (init errors). */
const char* am_last_error(const am_ctx* ctx);

/* Per-kernel device timing (tracing).  mask selects kernel ids (bit k = kernel k,
 * names from am_profile_name; 0 disables).  Every selected kernel launch of the
 * context (tracker and replay driver) is bracketed by CUDA events recorded on the
 * context's stream (external event records, so they work inside CUDA graphs); each
 * synchronising call adds the elapsed times to per-kernel totals.  Enabling resets
 * the totals.  am_profile_read fills ms[k] / counts[k] for k < max (host arrays) and
 * returns the number of kernel ids; am_profile_name gives kernel k's name. */
int am_profile_enable(am_ctx* ctx, uint32_t mask);
int am_profile_read(am_ctx* ctx, double* ms, int64_t* counts, int32_t max);
const char* am_profile_name(int32_t id);

/* Work counters of the neighbour scan accumulated while AM_STATS is set (host
 * array out[6]: cells visited, candidate pairs tested, agents entering the far
 * (time-dilated) phase, 16x16-cell blocks tested, 4x4-cell blocks tested, blocked
 * agents); resets them.  Synchronises. */
int am_scan_stats(am_ctx* ctx, uint64_t* out);

/* Kernel launches of one am_update + am_ready on this context (host-side count; a
 * replay round on the binned path fuses two of them, see am_driver.h). */
int32_t am_launches_per_round(const am_ctx* ctx);

/* Library version string. */
const char* am_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AM_H_ */
