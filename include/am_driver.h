/*
 * am_driver.h -- C ABI of the GPU-resident trace-replay driver (libametro.so).
 *
 * The paper evaluates AI Metropolis by replaying recorded GenAgent traces (replay
 * mode) through its controller/worker loop (Alg. 3).  Those traces
 * and the LLM are out of scope here: agent actions come from a deterministic
 * random-walk policy and LLM latencies are sampled from integer tables
 * (SURVEY 8(c.4)).  LLM capacity is infinite: every ready
 * cluster starts at once.
 *
 * Event rules (integer microseconds), per simulation b with clock t_b (start 0):
 *   1. commit every RUNNING agent whose cluster completion time <= t_b: apply the
 *      move computed at dispatch, step += 1 (worker l.20-21, controller l.11-12);
 *   2. one tracker round (am_update + am_ready, Alg. 3 l.8-9);
 *   3. each ready cluster C gets completion time t_b + max_{i in C} dur(i, s_i);
 *      every member's move is computed now from its perception (all perceived agents
 *      are cluster-mates, so the inputs equal the lock-step run's);
 *   4. t_b = min pending completion time (quantum 0), else rounded up to a multiple
 *      of the quantum.
 * A simulation ends when all its agents are DONE (step == target); T_ooo[b] is the
 * time of that last commit.  All simulations advance one round per am_replay_round.
 *
 * Synthetic model (identical definition implemented independently by the oracle):
 *   mix64 = splitmix64 finaliser; key3(s,a,b) = mix64(mix64(mix64(s+a)+b))
 *   digest_i = sum_{j perceived} mix64((j<<32) ^ ((u16)dx<<16) ^ (u16)dy),
 *              perceived = same-step non-DONE j != i with dist <= radius_p
 *   h = mix64(key3(policy_seed, i, s) + digest_i); move = {0,+x,-x,+y,-y}[h % 5]
 *       (policy 2, the 8-connected walk for the L-infinity metric: those five then
 *       (+1,+1), (-1,+1), (+1,-1), (-1,-1), [h % 9]; policy 3, the graph walk:
 *       {stay, neighbour 0, ..., neighbour deg-1}[h % (deg + 1)]),
 *       cancelled if the target tile is a wall or off the map
 *   K = vals[min{m : (key3(lat_seed,i,s) >> 32) < cdf32[m]}]
 *   dur(i,s) = base_us + sum_{k<K} lat[key3(lat_seed ^ 0xC0FFEE, (i<<20) ^ s, k) >> 54]
 *
 * Ownership: every pointer in am_synth and every array argument is a caller-owned
 * DEVICE pointer that must stay alive while the replay exists; outputs marked
 * "host" are host memory.  Errors as in am.h.
 */
#ifndef AM_DRIVER_H_
#define AM_DRIVER_H_

#include <stdint.h>
#include "am.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    const uint32_t* lat;        /* [1024] per-call latency quantiles, microseconds        */
    const uint64_t* cdf32;      /* [n_vals] cumulative call-count probability * 2^32      */
    const int32_t*  vals;       /* [n_vals] call counts                                    */
    int32_t  n_vals;            /* 1..16                                                   */
    int32_t  base_us;           /* fixed per-step cost                                     */
    uint64_t lat_seed;
    uint64_t policy_seed;
    const uint8_t* wall;        /* [map_h*map_w] row-major, 1 = wall; NULL = open map      */
    const int64_t* dur_table;   /* optional explicit durations [n_agents][dur_T]; NULL     */
    int32_t  dur_T;
    int32_t  policy;            /* 0 = random walk, 1 = always stay, 2 = 8-connected walk   */
    int32_t  conflict;          /* 0 = co-occupancy allowed; 1 = exclusive tiles: a move is
                                   cancelled if its target is occupied by a cluster-mate or
                                   a lower-id cluster-mate proposes it (Alg. 3 l.20;
                                   needs r_p >= 2 v; fused per-simulation path only,
                                   through am_replay_run / am_replay_launch)              */
    const int32_t* graph_off;   /* policy 3 (graph walk, AM_METRIC_GRAPH): CSR adjacency,  */
    const int32_t* graph_adj;   /* [n_nodes + 1] offsets and the neighbour lists; a move is
                                   {stay, neighbour 0..deg-1}[h % (deg + 1)]              */
} am_synth;

typedef struct am_replay am_replay;

/* Device workspace bytes of a replay on ctx (event clock, dispatch times, moves,
 * trajectory hashes, round outputs, the host-loop shadow): the two-phase idiom of am.h. */
size_t am_replay_workspace_size(const am_ctx* ctx);

/* Create a replay on ctx (which must have been created with target_step > 0; the
 * replay sets AM_DIGEST and clears AM_PEEK/AM_ASYNC on it as needed).
 * positions int32 [n][2] and steps int32 [n] are the world state, updated in place
 * by commits; the replay starts from the current contents (steps normally all 0).
 * workspace: caller-owned device memory of >= am_replay_workspace_size(ctx) bytes,
 * 256-byte aligned, alive until am_replay_destroy (NULL: the replay allocates its own).
 * Nothing is allocated after creation (am_replay_io included).  Errors: AM_E_ARG,
 * AM_E_WORKSPACE, AM_E_CUDA. */
int am_replay_create(am_replay** out, am_ctx* ctx, const am_synth* synth,
                     int64_t quantum_us, int32_t* positions, int32_t* steps, void* workspace,
                     size_t workspace_bytes);

/* Run up to max_rounds rounds without host synchronisation, then synchronise.  On the
 * cell-binned path the rounds are a CUDA graph of one round replayed; when every
 * simulation has <= 1024 agents (the fused per-simulation path) and tracing is off, one
 * persistent kernel runs all the rounds with one CTA per simulation (identical rounds;
 * am_replay_launch likewise).  *active (host) receives the number of agents not yet
 * DONE (0 = every simulation finished).  Rounds after a simulation finished are no-ops. */
int am_replay_run(am_replay* r, int64_t max_rounds, int64_t* active);

/* Exactly one round with its outputs kept for inspection (tests): mask uint8 [n],
 * order int32 [n], labels int32 [n] device arrays (may be NULL); *n_ready host. */
int am_replay_step(am_replay* r, uint8_t* mask, int32_t* order, int32_t* labels,
                   int32_t* n_ready);

/* Results: T_ooo int64 [n_sims] (host), rounds int64 [n_sims] (host; rounds in which
 * the simulation had at least one active agent), traj uint64 [n] (device, may be NULL:
 * per-agent trajectory hash chained at every commit). */
int am_replay_results(am_replay* r, int64_t* T_ooo, int64_t* rounds, uint64_t* traj);

/* Finite LLM capacity (call before the first round): at most
 * `capacity` agent-steps in service at once (0 = infinite, the default).  Ready clusters
 * are queued (members RUNNING, moves computed at queueing) and started -- completion =
 * start + max member duration -- in the order of the key (step << 32 | label) when
 * priority != 0 (the paper's step-priority ready_queue, section 3.5),
 * else (round << 32 | label) (FIFO); strict order, a cluster larger than the capacity
 * starts only when nothing is in service.  The fused per-simulation path runs it in the
 * persistent kernel (am_replay_run / am_replay_launch; am_replay_step / am_replay_io
 * return AM_E_ARG there); the cell-binned path (one simulation) keeps a device queue of
 * ready clusters, sorted each round by the one-kernel cluster sort and started in key
 * order while they fit (every call).  Errors: AM_E_ARG, AM_E_STATE (rounds already ran). */
int am_replay_set_capacity(am_replay* r, int64_t capacity, int32_t priority);

/* LLM busy time dispatched so far per simulation (host int64 [n_sims], microseconds):
 * the sum over dispatched agent-steps of dur(i, s) - base_us (the time spent in LLM
 * calls; calls of one agent-step are sequential, one outstanding request at a time).
 * Divided by T_ooo it is the achieved parallelism of the paper's evaluation (average
 * outstanding LLM requests over the execution time).  Synchronises. */
int am_replay_llm_time(am_replay* r, int64_t* llm_us);

/* The parallel-sync baseline (Algorithm 1's barrier per step): T_sync[b]
 * = sum_{s < T} max_{i in simulation b} dur(i, s) for n agents in n_sims simulations
 * under the synthetic latency model, computed on the device (host int64 [n_sims] out;
 * temporary device memory from the stream-ordered allocator).  Synchronises. */
int am_lockstep_time(const am_synth* synth, int32_t n, int32_t n_sims, int32_t T, int64_t* T_sync, void* stream);

/* Total agent-steps dispatched so far (host). */
int am_replay_dispatched(am_replay* r, int64_t* agent_steps);

/* One round with the world state in HOST memory (pinned for asynchronous copies):
 * copies h_pos_in int32[n][2] / h_steps_in int32[n] to the replay's world arrays, runs
 * the round, copies back the committed state (h_pos_out, h_steps_out; may alias the
 * inputs), the ready mask uint8[n] and the order int32[n] (capacity n; only the first
 * n_ready entries are written when h_order is page-locked, the whole capacity
 * otherwise).  When the state outputs alias the inputs and are page-locked, only the
 * agents committed by the round are written back (the arrays already hold the rest).
 * Output pointers may be NULL.  If n_ready is non-NULL the call synchronises and stores the round's ready
 * count (first *n_ready order entries valid); otherwise call am_replay_sync.  This
 * is the end-to-end user loop measured by bench.py. */
int am_replay_io(am_replay* r, const int32_t* h_pos_in, const int32_t* h_steps_in,
                 int32_t* h_pos_out, int32_t* h_steps_out, uint8_t* h_mask, int32_t* h_order,
                 int32_t* n_ready);

/* Enqueue `rounds` rounds (CUDA graphs) without synchronising. */
int am_replay_launch(am_replay* r, int64_t rounds);

/* Synchronise; *active = agents not DONE, *n_ready = last round's ready count
 * (either may be NULL).  Reports validation / liveness errors. */
int am_replay_sync(am_replay* r, int64_t* active, int32_t* n_ready);

/* The cudaStream_t the replay launches on (for timing events). */
void* am_replay_stream(am_replay* r);

int am_replay_destroy(am_replay* r);

#ifdef __cplusplus
}
#endif
#endif /* AM_DRIVER_H_ */
