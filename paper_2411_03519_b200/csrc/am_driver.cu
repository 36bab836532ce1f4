// am_driver.cu -- GPU-resident trace-replay driver (include/am_driver.h).
//
// One replay round for every simulation at once (Alg. 3 with infinite LLM capacity,
// replay mode P:228): am_update -> am_ready -> k_disp_a -> k_disp_b -> k_commit.
// The synthetic policy/latency model is the same definition the oracle implements
// independently (am_driver.h); nothing here is shared with oracle/.
#include <climits>
#include <cstdlib>
#include <cstdio>
#include <new>

#include "am_driver.h"
#include "am_internal.cuh"
#include "am_synth.cuh"

int am_internal_csort(am_ctx* c, const am::Dev& sd, int32_t* order, cudaStream_t s);

namespace am {

struct RepDev {
    Dev d;                      // tracker context (labels, digests, status)
    am_synth sy;
    long long Q;
    int2* pos;                  // world state (caller-owned)
    int32_t* steps;
    long long* tcommit;         // [n] completion time of the agent's dispatched step
    int2* newpos;               // [n] move computed at dispatch
    unsigned long long* traj;   // [n]
    long long* tcl;             // [n] cluster completion time, indexed by root label
    long long* t_sim;           // [S] current event time
    long long* tnext;           // [S] accumulator: min pending completion (LLONG_MAX)
    long long* tdone;           // [S] time of the last commit that finished an agent
    long long* rounds;          // [S]
    int32_t* active_flag;       // [S]
    const int32_t* order;       // this round's ready agents (any order: the ready list of the
                                // binned path, the priority order of the fused path)
    long long* dispatched;      // [1]
    int32_t* liveness;          // [1]
    Chain* chain;               // last-block counter of k_disp_b
    unsigned long long* qkey;   // [n] queue key of a queued (RUNNING, not started) agent (finite capacity)
    long long K;                // agent-steps in service at once; 0 = infinite capacity
    int32_t* part;              // [2 x 4 x commit blocks] post-commit partials (in-place commits)
    long long* llm;             // [S] LLM busy time dispatched so far: sum of (duration - base_us), us
    int32_t* clist;             // [n] this round's committing agents (AM_COMMIT_SPLIT)
    // finite capacity on the cell-binned path (one simulation): the queue of ready clusters
    // waiting to start, one entry each {key, label, size, max duration}
    int32_t* qsz;               // [n] members of this round's ready cluster, by label
    unsigned long long* qe_key[2];   // [n] entry keys (ping-pong)
    int32_t* qe_lab[2];
    int32_t* qe_size[2];
    long long* qe_dur[2];
    int32_t* qn;                // [2] entries in each buffer
    int32_t* qcur;              // [1] the current buffer
    long long* qstart_t;        // [n] by label: completion time of a cluster started this round
    uint32_t* qstart_ep;        // [n] by label: the epoch it started in
    long long* busy;            // [1] agent-steps in service
    int32_t* qorder;            // [n] entry indices in key order (the queue's sort)
    Ctl* qctl;                  // the queue sort's control block (n_ready = entries, sort_or)
    unsigned long long* qrk[2]; // the queue sort's ping-pong keys / values
    uint32_t* qrv[2];
    int32_t qidb;               // bits of an agent id in the compact entry key
    int32_t prio;               // 1: queue by (step, label); 0: by (round, label)
};

__device__ __forceinline__ int sim_of(const Dev& d, int i)
{
    return d.n_sims == 1 ? 0 : (int)(((long long)i * d.n_sims + d.n_sims - 1) / d.n);
}

__device__ __forceinline__ int2 policy_move(const RepDev& r, int i, int s, int2 p, unsigned long long dig)
{
    return policy_move_g(r.sy, r.d.map_w, r.d.map_h, i, s, p, dig);
}

// The commit of one agent i (old step s0) at time t of its simulation b: world state,
// trajectory hash, the tracker's state in place (inplace), the loose-cell drift.
// Returns the new step; done = reached the target.
__device__ __forceinline__ int commit_agent(const RepDev& r, int i, int s0, int b, long long t, bool inplace,
                                            uint32_t c, uint32_t tag, bool& done, int& dmax, int& err)
{
    const Dev& d = r.d;
    const int2 np = r.newpos[i];
    const int2 op = r.pos[i];
    const int s = (inplace ? s0 : r.steps[i]) + 1;
    r.pos[i] = np;
    r.steps[i] = s;
    r.traj[i] = traj_step(r.traj[i], s, np.x, np.y);
    done = d.target > 0 && s == d.target;
    if (done) atomicMax((unsigned long long*)(r.tdone + b), (unsigned long long)t);
    if (inplace) {
        // the speed limit the soundness of the rules rests on
        if (!within_pts(d, op.x, op.y, np.x, np.y, (uint32_t)d.v)) err |= ERR_VELOCITY;
        const uint8_t nst = done ? ST_DONE : ST_IDLE;
        d.pos[c][i] = np;
        d.step[c][i] = s;
        d.status[c][i] = nst;
        d.chg8[i] = 1;
        const int lab = d.labels[i];
        if (lab >= 0) d.dirty[lab] = d.ctl->epoch + 1u;
        const uint32_t rr = d.slot[i];
        AM_CHECK(rr == kSentinel || rr < (uint32_t)d.n);
        if (rr != kSentinel) {
            d.rec[rr] = make_int4(np.x | (np.y << 16), s, i, (int)nst | (int)(tag << kTagShift));
            int cx, cy;
            mkey_decode(d, d.key[i], cx, cy);
            const int x0 = cx << d.clog, y0 = cy << d.clog;
            const int x1 = x0 + (1 << d.clog) - 1, y1 = y0 + (1 << d.clog) - 1;
            dmax = max(dmax, max(max(x0 - np.x, np.x - x1), max(y0 - np.y, np.y - y1)));
        }
    }
    return s;
}

// commit every RUNNING agent whose cluster completed (tcommit <= t_sim, the clock
// k_disp_b just advanced): the move computed at dispatch is applied and the step
// advances (worker l.20-21).  Agents that stay RUNNING bound the next
// event; any agent left active marks its simulation active for the next round.
// inplace (cell-binned path, the driver's own rounds): the commit is also applied to
// the tracker's state in place -- exactly what the next am_update would find by diffing
// the world arrays (update_agents, Alg. 3 l.11): IDLE (DONE at the target), the changed
// mark, the last-round cluster made dirty, the agent's loose-cell record and its drift
// -- and every block adds its {min step, max step, active, running} of the post-commit
// state to one of 64 reduction stripes for k_replay_begin, so the next round needs no
// O(N) ingest.
// Each thread reads kCommitItems agents' status / completion time / step (all loads in
// flight together); the ~4% that commit are compacted per warp (ballot) into a shared
// list and committed by consecutive lanes, so a warp runs the scattered commit path
// once per 32 commits instead of once per 32 agents with any commit among them.
__global__ void __launch_bounds__(256) k_commit(RepDev r, int inplace)
{
#if !(AM_PDL_EARLY & 2)
    pdl_begin();
#endif
    constexpr int KC = kCommitItems;
    __shared__ int2 s_cl[8][32 * KC];   // per warp: {agent, old step} of the committing agents
    const Dev& d = r.d;
    const bool one = d.n_sims == 1;
    const uint32_t c = d.ctl->cur;
    const uint32_t tag = (d.ctl->epoch + 1u) & kTagMask;   // the round this commit feeds
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long tmin = ~0ull;  // pending completions (single-simulation case)
    int any_active = 0;
    int wmin = INT_MAX, smax = INT_MIN, nact = 0, nrun = 0, dmax = 0, err = 0;
    // loads of all items first (independent chains in flight), then the commits
    uint8_t st[KC];
    long long tc[KC];
    int sw[KC];
#pragma unroll
    for (int k = 0; k < KC; k++) {
        const int i = blockIdx.x * (256 * KC) + k * 256 + threadIdx.x;
        st[k] = ST_DONE;
        tc[k] = 0;
        sw[k] = 0;
        if (i < d.n) {
            st[k] = d.status[c][i];  // after this round's dispatch
            if (inplace) sw[k] = r.steps[i];   // (post-commit W / S: issued with the others)
#if !(AM_PDL_EARLY & 2)
            tc[k] = r.tcommit[i];
#endif
        }
    }
#if AM_PDL_EARLY & 2
    // statuses (k_ready) and steps (the last commit) were final before this kernel's
    // predecessor began: loaded above while k_disp_b still runs (PDL); the completion
    // times k_disp_b writes and the clock its last block sets, after the wait
    pdl_begin();
#pragma unroll
    for (int k = 0; k < KC; k++) {
        const int i = blockIdx.x * (256 * KC) + k * 256 + threadIdx.x;
        if (i < d.n) tc[k] = r.tcommit[i];
    }
#endif
    const long long t1 = one ? r.t_sim[0] : 0;
    int nlist = 0;   // warp uniform
#pragma unroll
    for (int k = 0; k < KC; k++) {
        const int i = blockIdx.x * (256 * KC) + k * 256 + threadIdx.x;
        bool commit = false;
        if (st[k] != ST_DONE) {
            if (r.K > 0 && st[k] == ST_RUNNING && tc[k] == LLONG_MAX) {
                // queued: did its cluster start this round (k_qstart)?
                const int lab = (int)(r.qkey[i] & ((1ull << r.qidb) - 1ull));
                if (r.qstart_ep[lab] == d.ctl->epoch) {
                    tc[k] = r.qstart_t[lab];
                    r.tcommit[i] = tc[k];
                }
            }
            const int b = sim_of(d, i);
            const long long t = one ? t1 : r.t_sim[b];
            commit = st[k] == ST_RUNNING && tc[k] <= t;
            if (!commit) {
                if (st[k] == ST_RUNNING) {
                    // stays RUNNING through this round: bounds the next event
                    if (one) tmin = min(tmin, (unsigned long long)tc[k]);
                    else atomicMin((unsigned long long*)(r.tnext + b), (unsigned long long)tc[k]);
                }
                if (one) any_active = 1;
                else r.active_flag[b] = 1;
                if (inplace) {
                    wmin = min(wmin, sw[k]);
                    smax = max(smax, sw[k]);
                    nact++;
                    nrun += st[k] == ST_RUNNING;
                }
            }
        }
        const unsigned bal = __ballot_sync(0xFFFFFFFFu, commit);
        AM_CHECK(!commit || (i < d.n && nlist + __popc(bal & ((1u << lane) - 1u)) < 32 * KC));
        if (commit) s_cl[w][nlist + __popc(bal & ((1u << lane) - 1u))] = make_int2(i, sw[k]);
        nlist += __popc(bal);
    }
    __syncwarp();
    // the warp's committing agents, one per lane
    for (int j = lane; j < nlist; j += 32) {
        const int2 e = s_cl[w][j];
        const int b = sim_of(d, e.x);
        const long long t = one ? t1 : r.t_sim[b];
        bool done;
        const int s = commit_agent(r, e.x, e.y, b, t, inplace != 0, c, tag, done, dmax, err);
        if (!done) {
            if (one) any_active = 1;
            else r.active_flag[b] = 1;
            if (inplace) {
                wmin = min(wmin, s);
                smax = max(smax, s);
                nact++;
            }
        }
    }
    if (r.K > 0 && one) {   // agent-steps leaving service (finite capacity)
        if (lane == 0 && nlist) atomicAdd((unsigned long long*)r.busy, (unsigned long long)(-(long long)nlist));
    }
    if (one) {  // block reduction, one atomic per block
        __shared__ unsigned long long s_min[8];
        __shared__ int s_act[8];
        for (int o = 16; o > 0; o >>= 1) tmin = min(tmin, __shfl_xor_sync(0xFFFFFFFFu, tmin, o));
        any_active = __reduce_or_sync(0xFFFFFFFFu, (unsigned)any_active);
        if (lane == 0) { s_min[w] = tmin; s_act[w] = any_active; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int q = 1; q < 8; q++) { tmin = min(tmin, s_min[q]); any_active |= s_act[q]; }
            if (tmin != ~0ull) atomicMin((unsigned long long*)r.tnext, tmin);
            if (any_active) r.active_flag[0] = 1;
        }
    }
    if (inplace) {   // the post-commit state's reduction: one atomic per quantity per block, 64 stripes
        __shared__ int p_w[8], p_s[8], p_a[8], p_r[8], p_d[8], p_e[8];
        wmin = __reduce_min_sync(0xFFFFFFFFu, wmin);
        smax = __reduce_max_sync(0xFFFFFFFFu, smax);
        nact = (int)__reduce_add_sync(0xFFFFFFFFu, (unsigned)nact);
        nrun = (int)__reduce_add_sync(0xFFFFFFFFu, (unsigned)nrun);
        dmax = __reduce_max_sync(0xFFFFFFFFu, dmax);
        err = (int)__reduce_or_sync(0xFFFFFFFFu, (unsigned)err);
        if (lane == 0) { p_w[w] = wmin; p_s[w] = smax; p_a[w] = nact; p_r[w] = nrun; p_d[w] = dmax; p_e[w] = err; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int q = 1; q < 8; q++) {
                wmin = min(wmin, p_w[q]); smax = max(smax, p_s[q]); nact += p_a[q]; nrun += p_r[q];
                dmax = max(dmax, p_d[q]); err |= p_e[q];
            }
            int32_t* st = d.cstripe + 32 * (blockIdx.x & (kCommitStripes - 1));   // its own 128-byte line
            if (wmin != INT_MAX) atomicMin(st, wmin);
            if (smax != INT_MIN) atomicMax(st + 1, smax);
            if (nact) atomicAdd(st + 2, nact);
            if (nrun) atomicAdd(st + 3, nrun);
            if (blockIdx.x == 0) d.ctl->part_valid = 1;
            // the drift and a velocity violation go to the accumulators both round starts
            // merge (k_replay_begin, or k_ingest_done after a host-buffer ingest)
            if (dmax > 0) atomicMax(&d.ctl->acc_D, dmax);
            if (err) atomicOr(&d.ctl->err_new, err);
        }
    }
}

// ---- the commit as two passes (AM_COMMIT_SPLIT, one simulation, binned path) ----
// k_commit_scan: the O(N) part only -- statuses, completion times and steps, read
// coalesced with no dependent chain: which agents commit (appended to a list), the next
// event from the agents that stay RUNNING, activity, and the post-commit {min step, max
// step, active, running} into the reduction stripes.  k_commit_apply then commits the
// listed agents densely, one thread each (world state, trajectory hash, the tracker's
// state in place, loose-cell record and drift) -- the scattered work leaves the O(N) pass.
__global__ void __launch_bounds__(256) k_commit_scan(RepDev r)
{
    pdl_begin();
    const Dev& d = r.d;
    const uint32_t c = d.ctl->cur;
    const long long t = r.t_sim[0];
    unsigned long long tmin = ~0ull;
    int wmin = INT_MAX, smax = INT_MIN, nact = 0, nrun = 0, any_active = 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int base = blockIdx.x * blockDim.x; base < d.n; base += gridDim.x * blockDim.x) {   // block uniform
        const int i = base + threadIdx.x;
        bool com = false;
        if (i < d.n) {
            const uint8_t st = d.status[c][i];
            if (st != ST_DONE) {
                const int s0 = r.steps[i];
                int s = s0;
                bool run = st == ST_RUNNING;
                if (run) {
                    const long long tc = r.tcommit[i];
                    if (tc <= t) {
                        com = true;
                        run = false;
                        s = s0 + 1;
                    } else {
                        tmin = min(tmin, (unsigned long long)tc);
                    }
                }
                const bool done = com && d.target > 0 && s == d.target;
                if (!done) {
                    any_active = 1;
                    wmin = min(wmin, s);
                    smax = max(smax, s);
                    nact++;
                    nrun += run;
                } else {
                    atomicMax((unsigned long long*)r.tdone, (unsigned long long)t);
                }
            }
        }
        // warp-aggregated append of the committing agents
        const unsigned m = __ballot_sync(0xFFFFFFFFu, com);
        int b0 = 0;
        if (lane == 0 && m) b0 = atomicAdd(&d.ctl->n_commit, __popc(m));
        b0 = __shfl_sync(0xFFFFFFFFu, b0, 0);
        if (com) r.clist[b0 + __popc(m & ((1u << lane) - 1u))] = i;
    }
    __shared__ unsigned long long s_min[8];
    __shared__ int p_w[8], p_s[8], p_a[8], p_r[8], p_y[8];
    for (int o = 16; o > 0; o >>= 1) tmin = min(tmin, __shfl_xor_sync(0xFFFFFFFFu, tmin, o));
    wmin = __reduce_min_sync(0xFFFFFFFFu, wmin);
    smax = __reduce_max_sync(0xFFFFFFFFu, smax);
    nact = (int)__reduce_add_sync(0xFFFFFFFFu, (unsigned)nact);
    nrun = (int)__reduce_add_sync(0xFFFFFFFFu, (unsigned)nrun);
    any_active = (int)__reduce_or_sync(0xFFFFFFFFu, (unsigned)any_active);
    if (lane == 0) { s_min[w] = tmin; p_w[w] = wmin; p_s[w] = smax; p_a[w] = nact; p_r[w] = nrun; p_y[w] = any_active; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < 8; q++) {
            tmin = min(tmin, s_min[q]); wmin = min(wmin, p_w[q]); smax = max(smax, p_s[q]);
            nact += p_a[q]; nrun += p_r[q]; any_active |= p_y[q];
        }
        if (tmin != ~0ull) atomicMin((unsigned long long*)r.tnext, tmin);
        if (any_active) r.active_flag[0] = 1;
        int32_t* sp = d.cstripe + 32 * (blockIdx.x & (kCommitStripes - 1));
        if (wmin != INT_MAX) atomicMin(sp, wmin);
        if (smax != INT_MIN) atomicMax(sp + 1, smax);
        if (nact) atomicAdd(sp + 2, nact);
        if (nrun) atomicAdd(sp + 3, nrun);
        if (blockIdx.x == 0) d.ctl->part_valid = 1;
    }
}

__global__ void __launch_bounds__(256) k_commit_apply(RepDev r)
{
    pdl_begin();
    const Dev& d = r.d;
    const uint32_t c = d.ctl->cur;
    const uint32_t tag = (d.ctl->epoch + 1u) & kTagMask;
    const int nc = d.ctl->n_commit;
    int dmax = 0, err = 0;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nc; k += gridDim.x * blockDim.x) {
        const int i = r.clist[k];
        // every load first (independent), then the stores
        const int2 np = r.newpos[i];
        const int2 op = r.pos[i];
        const int s = r.steps[i] + 1;
        const unsigned long long th = r.traj[i];
        const int lab = d.labels[i];
        const uint32_t rr = d.slot[i];
        const uint32_t key = d.key[i];
        const bool done = d.target > 0 && s == d.target;
        const uint8_t nst = done ? ST_DONE : ST_IDLE;
        r.pos[i] = np;
        r.steps[i] = s;
        r.traj[i] = traj_step(th, s, np.x, np.y);
        if (!within_pts(d, op.x, op.y, np.x, np.y, (uint32_t)d.v)) err |= ERR_VELOCITY;
        d.pos[c][i] = np;
        d.step[c][i] = s;
        d.status[c][i] = nst;
        d.chg8[i] = 1;
        if (lab >= 0) d.dirty[lab] = d.ctl->epoch + 1u;
        if (rr != kSentinel) {
            d.rec[rr] = make_int4(np.x | (np.y << 16), s, i, (int)nst | (int)(tag << kTagShift));
            int cx, cy;
            mkey_decode(d, key, cx, cy);
            const int x0 = cx << d.clog, y0 = cy << d.clog;
            const int x1 = x0 + (1 << d.clog) - 1, y1 = y0 + (1 << d.clog) - 1;
            dmax = max(dmax, max(max(x0 - np.x, np.x - x1), max(y0 - np.y, np.y - y1)));
        }
    }
    dmax = __reduce_max_sync(0xFFFFFFFFu, dmax);
    err = (int)__reduce_or_sync(0xFFFFFFFFu, (unsigned)err);
    if ((threadIdx.x & 31) == 0) {
        if (dmax > 0) atomicMax(&d.ctl->acc_D, dmax);
        if (err) atomicOr(&d.ctl->err_new, err);
    }
}

// The driver's own round begins (cell-binned path, after an in-place k_commit): the
// 64 reduction stripes of the post-commit state give W, S and the counts k_ingest_done
// would publish (nothing else changed since the commit), the drift is merged, a velocity
// violation is reported and forces a full recompute; then the round's counters reset.
__global__ void __launch_bounds__(32) k_replay_begin(RepDev r, int nparts)
{
    pdl_begin();
    (void)nparts;
    Ctl* ctl = r.d.ctl;
    const Dev& d = r.d;
    // one warp reduces the 64 stripes (two per lane) and resets them
    const int lane = threadIdx.x;
    int w = INT_MAX, s = INT_MIN, a = 0, run = 0;
    const bool valid = ctl->part_valid != 0;
    for (int k = lane; k < kCommitStripes; k += 32) {
        int32_t* c = d.cstripe + 32 * k;
        w = min(w, c[0]); s = max(s, c[1]); a += c[2]; run += c[3];
        c[0] = INT_MAX; c[1] = INT_MIN; c[2] = 0; c[3] = 0;
    }
    w = __reduce_min_sync(0xFFFFFFFFu, w);
    s = __reduce_max_sync(0xFFFFFFFFu, s);
    a = (int)__reduce_add_sync(0xFFFFFFFFu, (unsigned)a);
    run = (int)__reduce_add_sync(0xFFFFFFFFu, (unsigned)run);
    if (lane == 0) {
        if (valid) {
            ctl->W = w;
            ctl->S = s;
            ctl->n_active = a;
            ctl->n_running = run;
            ctl->part_valid = 0;
        }
        ctl->D = max(ctl->D, ctl->acc_D);
        ctl->acc_D = 0;
        if (ctl->err_new) {   // a commit broke the speed limit: reported, full recompute next
            ctl->err_sticky |= ctl->err_new;
            ctl->full_next = 1;
            ctl->err_new = 0;
        }
        round_begin(r.d);
    }
}

// ---- finite capacity on the cell-binned path (one simulation) ---------------------
// k_qprep: the queue's entries become the sort's input (compact keys, entry indices)
__global__ void __launch_bounds__(256) k_qprep(RepDev r)
{
    pdl_begin();
    const int q = *r.qcur, n = r.qn[q];
    unsigned long long kor = 0;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const unsigned long long key = r.qe_key[q][k];
        r.qrk[0][k] = key;
        r.qrv[0][k] = (uint32_t)k;
        kor |= key;
    }
    for (int o = 16; o > 0; o >>= 1) kor |= __shfl_xor_sync(0xFFFFFFFFu, kor, o);
    if ((threadIdx.x & 31) == 0 && kor) atomicOr(&r.qctl->sort_or, kor);
    if (blockIdx.x == 0 && threadIdx.x == 0) r.qctl->n_ready = n;
}

// k_qstart (one block): start the queued clusters in key order while they fit -- strict
// order, no bypass; a cluster larger than the capacity starts only when nothing is in
// service (the oracle's orc_replay_cap) -- then the event clock (k_disp_b's last block
// without capacity): the next event is the earliest completion of what is in service.
__global__ void __launch_bounds__(1024) k_qstart(RepDev r)
{
    pdl_begin();
    __shared__ int s_wsum[32];
    __shared__ long long s_base;
    __shared__ int s_cut, s_keep;
    __shared__ unsigned long long s_tmin;
    const int q = *r.qcur, n = r.qn[q];
    const long long t = r.t_sim[0];
    const uint32_t ep = r.d.ctl->epoch;
    const long long busy0 = *r.busy;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) { s_base = 0; s_cut = n; s_keep = 0; s_tmin = ~0ull; }
    __syncthreads();
    // pass 1: the cutoff in key order (sizes' prefix sums, chunk by chunk)
    for (int c0 = 0; c0 < n; c0 += blockDim.x) {
        if (s_cut < c0) break;   // block uniform (written before the last barrier)
        const int k = c0 + threadIdx.x;
        const int e = k < n ? (int)r.qorder[k] : 0;
        const int sz = k < n ? r.qe_size[q][e] : 0;
        int incl = sz;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_wsum[w] = incl;
        __syncthreads();
        if (w == 0) {
            const int v = lane < (int)(blockDim.x >> 5) ? s_wsum[lane] : 0;
            int sc = v;
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xFFFFFFFFu, sc, o);
                if (lane >= o) sc += y;
            }
            s_wsum[lane] = sc - v;
        }
        __syncthreads();
        const long long P = s_base + s_wsum[w] + incl;   // sizes of entries [0, k]
        const bool fits = (busy0 + P <= r.K) || (k == 0 && busy0 == 0);
        if (k < n && !fits) atomicMin(&s_cut, k);
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_base = P;
        __syncthreads();
    }
    const int cut = s_cut;
    // pass 2: start the prefix, keep the rest (any order: the queue is re-sorted next round)
    long long started = 0;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const int e = (int)r.qorder[k];
        if (k < cut) {
            const int lab = r.qe_lab[q][e];
            const long long tc = t + r.qe_dur[q][e];
            r.qstart_t[lab] = tc;
            r.qstart_ep[lab] = ep;
            started += r.qe_size[q][e];
            atomicMin(&s_tmin, (unsigned long long)tc);
        } else {
            const int j = atomicAdd(&s_keep, 1);
            r.qe_key[q ^ 1][j] = r.qe_key[q][e];
            r.qe_lab[q ^ 1][j] = r.qe_lab[q][e];
            r.qe_size[q ^ 1][j] = r.qe_size[q][e];
            r.qe_dur[q ^ 1][j] = r.qe_dur[q][e];
        }
    }
    started = __reduce_add_sync(0xFFFFFFFFu, (unsigned)started);
    if (lane == 0 && started) atomicAdd((unsigned long long*)r.busy, (unsigned long long)started);
    __syncthreads();
    if (threadIdx.x == 0) {
        r.qn[q ^ 1] = s_keep;
        r.qn[q] = 0;
        *r.qcur = q ^ 1;
        r.qctl->sort_or = 0;
        // the clock (k_disp_b's last block without capacity)
        unsigned long long tn = *(volatile unsigned long long*)r.tnext;
        tn = min(tn, s_tmin);
        const int act = *(volatile int32_t*)r.active_flag;
        if (act) {
            r.rounds[0] += 1;
            if (tn == (unsigned long long)LLONG_MAX || tn == ~0ull) *r.liveness = 1;
            else r.t_sim[0] = r.Q > 0 ? (((long long)tn + r.Q - 1) / r.Q) * r.Q : (long long)tn;
        }
        r.tnext[0] = LLONG_MAX;
        r.active_flag[0] = 0;
    }
}

// dispatch, part a: cluster completion time = t + max member duration (atomicMax at
// the cluster's root label; a stale value is <= t).
__global__ void __launch_bounds__(256) k_disp_a(RepDev r)
{
    pdl_begin();
    const Dev& d = r.d;
    const int nr = d.ctl->n_ready;
    if (blockIdx.x == 0 && threadIdx.x == 0) *r.dispatched += nr;
    unsigned long long busy = 0;   // LLM time of the dispatched agent-steps (one simulation)
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nr; k += gridDim.x * blockDim.x) {
        const int i = r.order[k];
        const int b = sim_of(d, i);
        const long long du = duration(r.sy, i, r.steps[i]);
        const long long tc = r.t_sim[b] + du;
        atomicMax((unsigned long long*)(r.tcl + d.labels[i]), (unsigned long long)tc);
        if (r.K > 0) atomicAdd(r.qsz + d.labels[i], 1);   // the cluster's size (finite capacity)
        if (d.n_sims > 1) atomicAdd((unsigned long long*)(r.llm + b), (unsigned long long)(du - r.sy.base_us));
        else busy += (unsigned long long)(du - r.sy.base_us);
    }
    if (d.n_sims == 1) {   // block reduction, one atomic per block on one of 64 stripes
        __shared__ unsigned long long s_b[8];
        for (int o = 16; o > 0; o >>= 1) busy += __shfl_xor_sync(0xFFFFFFFFu, busy, o);
        if ((threadIdx.x & 31) == 0) s_b[threadIdx.x >> 5] = busy;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int q = 1; q < 8; q++) busy += s_b[q];
            if (busy) atomicAdd((unsigned long long*)(r.llm + 16 * (blockIdx.x & 63)), busy);
        }
    }
}

// dispatch, part b: member completion times and moves (random-walk policy on the
// perception digest), next event per simulation (last block).
__global__ void __launch_bounds__(256) k_disp_b(RepDev r)
{
    pdl_begin();
    const Dev& d = r.d;
    const int nr = d.ctl->n_ready;
    unsigned long long tmin = ~0ull;
    const bool cap = r.K > 0;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nr; k += gridDim.x * blockDim.x) {
        const int i = r.order[k];
        const int b = sim_of(d, i);
        const int lab = d.labels[i];
        const long long tc = r.tcl[lab];
        r.newpos[i] = policy_move(r, i, r.steps[i], r.pos[i], d.digest[i]);
        if (cap) {
            // queued (members RUNNING, moves computed now): key (step, label) in step-priority
            // order (section 3.5) or (round, label) in FIFO order
            const unsigned long long hi = r.prio ? (unsigned long long)(uint32_t)r.steps[i]
                                                 : (unsigned long long)r.rounds[0];
            const unsigned long long key = (hi << r.qidb) | (unsigned long long)(uint32_t)lab;
            r.tcommit[i] = LLONG_MAX;
            r.qkey[i] = key;
            if (i == lab) {   // the cluster's entry, from its min-id member
                const int q = *r.qcur;
                const int e = atomicAdd(r.qn + q, 1);
                r.qe_key[q][e] = key;
                r.qe_lab[q][e] = lab;
                r.qe_size[q][e] = r.qsz[lab];
                r.qe_dur[q][e] = tc - r.t_sim[0];
                r.qsz[lab] = 0;
            }
            continue;
        }
        r.tcommit[i] = tc;
        if (d.n_sims > 1) atomicMin((unsigned long long*)(r.tnext + b), (unsigned long long)tc);
        else tmin = min(tmin, (unsigned long long)tc);
    }
    if (cap) return;   // the queue's starts and the clock: k_qprep / k_csort / k_qstart
    if (d.n_sims == 1) {  // block reduction, one atomic per block
        __shared__ unsigned long long s_min[8];
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        for (int o = 16; o > 0; o >>= 1) tmin = min(tmin, __shfl_xor_sync(0xFFFFFFFFu, tmin, o));
        if (lane == 0) s_min[w] = tmin;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int q = 1; q < 8; q++) tmin = min(tmin, s_min[q]);
            if (tmin != ~0ull) atomicMin((unsigned long long*)r.tnext, tmin);
        }
    }
    // (agents still RUNNING from earlier rounds were folded into tnext by k_commit)
    if (finish_block(r.chain, gridDim.x)) {
        for (int b = threadIdx.x; b < d.n_sims; b += blockDim.x) {
            const long long tn = *(volatile long long*)(r.tnext + b);
            const int act = *(volatile int32_t*)(r.active_flag + b);
            if (act) {
                r.rounds[b] += 1;
                if (tn == LLONG_MAX) {
                    *r.liveness = 1;
                } else {
                    r.t_sim[b] = r.Q > 0 ? ((tn + r.Q - 1) / r.Q) * r.Q : tn;
                }
            }
            r.tnext[b] = LLONG_MAX;
            r.active_flag[b] = 0;
        }
    }
}

// ============================================================== persistent small replay
// The whole replay of one simulation (<= 1024 agents) in one CTA, up to max_rounds
// rounds without leaving the kernel: the fused round of k_small (pairwise blocking and
// coupling tests, shared-memory union-find, ready filter, perception digests), the
// dispatch of k_disp_a / k_disp_b (cluster completion time = t + max member duration,
// moves computed at dispatch), the event clock of k_disp_b's last block and the commits
// of k_commit -- each step in the same order and with the same arithmetic as the
// multi-kernel round, so every round's outcome is identical.  Entry and exit state is
// the multi-kernel round's (world arrays, context state, tcommit / newpos / traj,
// per-simulation clock and counters), so the two paths can alternate.  Grid = one CTA
// per simulation of M x G threads: G lanes (a power of two <= 32, one warp) share an
// agent's pair tests (lane q takes partners j = q, q + G, ...; verdicts and digests are
// combined by shuffles), lane 0 of the group does the agent's serial work.  Dynamic
// shared memory is sized by the largest simulation (M agents).
template <int kMetric>
__global__ void __launch_bounds__(1024) k_small_replay(RepDev r, long long max_rounds, int M, int G)
{
    const Dev& d = r.d;
    extern __shared__ __align__(16) unsigned char sm_raw[];
    long long* stc = reinterpret_cast<long long*>(sm_raw);                       // [M] tcommit
    unsigned long long* stcl = reinterpret_cast<unsigned long long*>(stc + M);   // [M] cluster time by label
    int2* snp = reinterpret_cast<int2*>(stcl + M);                               // [M] move computed at dispatch
    int4* sa = reinterpret_cast<int4*>(snp + M);                                 // [M] {x, y, step, status}
    unsigned long long* sq = reinterpret_cast<unsigned long long*>(sa + M);   // [M] queue keys (finite capacity)
    int* slab = reinterpret_cast<int*>(sq + M);                                  // [M] this round's labels
    uint32_t* par = reinterpret_cast<uint32_t*>(slab + M);
    uint8_t* sbad = reinterpret_cast<uint8_t*>(par + M);
    __shared__ unsigned long long s_tmin, s_best;
    __shared__ long long s_busy, s_size, s_dmax;
    __shared__ int s_any, s_fin, s_nr;
    const int b = blockIdx.x;
    const int t = threadIdx.x / G, q = threadIdx.x % G;   // agent slot, lane within its group
    const bool lead = q == 0;
    const int lo = (int)((long long)b * d.n / d.n_sims);
    const int m = (int)((long long)(b + 1) * d.n / d.n_sims) - lo;
    const uint32_t c = d.ctl->cur;
    const int i = lo + t;
    const bool mine = t < m;
    unsigned long long traj = 0;
    // entry: the world arrays (after the last commits) and the context's statuses; an
    // agent the last commit advanced is IDLE (or DONE) again, as the next ingest makes it
    if (mine && lead) {
        const int2 p = r.pos[i];
        const int s = r.steps[i];
        uint8_t st = d.status[c][i];
        if (st == ST_RUNNING && s == d.step[c][i] + 1) st = (d.target > 0 && s == d.target) ? ST_DONE : ST_IDLE;
        sa[t] = make_int4(p.x, p.y, s, st);
        stc[t] = r.tcommit[i];
        snp[t] = r.newpos[i];
        sq[t] = r.qkey[i];
        traj = r.traj[i];
    }
    long long tsim = r.t_sim[b], tdone = r.tdone[b], nrounds = r.rounds[b], disp = 0, busy = 0;
    int act = r.active_flag[b], live_err = 0, lab = -1;
    const uint32_t Rc = (uint32_t)min((long long)d.r_p + d.v, (long long)kRClamp);
    const uint32_t Rc2 = Rc * Rc, Rp = (uint32_t)d.r_p, Rp2 = Rp * Rp;
    // R_b(lag) = (lag + 1) v + r_p in 32 bits: lags beyond lagcap give >= kRClamp anyway
    const int lagcap = (int)(kRClamp / (uint32_t)max(1, d.v)) + 1;
    const uint32_t vv = (uint32_t)d.v, vr = (uint32_t)(d.v + d.r_p);
    __syncthreads();
    for (long long k = 0; k < max_rounds && act; k++) {
        // ---- the tracker round (k_small)
        if (mine && lead) { par[t] = (uint32_t)t; sbad[t] = 0; stcl[t] = 0; }
        if (threadIdx.x == 0) { s_tmin = ~0ull; s_any = 0; s_fin = 0; s_nr = 0; }
        __syncthreads();
        bool blocked = false;
        unsigned long long dig = 0;
        const int4 A = mine ? sa[t] : make_int4(0, 0, 0, ST_DONE);
        const int st = A.w;
        if (st != ST_DONE) {
            for (int j = q; j < m; j += G) {
                const int4 B = sa[j];
                if (j == t || B.w == ST_DONE) continue;
                const int dx = B.x - A.x, dy = B.y - A.y;
                // the metric (template): coordinates, or the graph's hop table
                const uint32_t hop = kMetric == AM_METRIC_GRAPH ? (uint32_t)d.gdist[(size_t)A.x * d.gV + B.x] : 0u;
                auto in = [&](uint32_t R2, uint32_t R) {
                    return kMetric == AM_METRIC_GRAPH ? (hop != 0xFFFFu && hop <= R) : within2(dx, dy, R2, R, kMetric);
                };
                if (B.z == A.z) {
                    if (in(Rc2, Rc)) {
                        if (t < j) suf_unite(par, (uint32_t)t, (uint32_t)j);
                        if (in(Rp2, Rp)) dig += digest_term((uint32_t)(lo + j), dx, dy);
                    }
                } else if (!blocked && B.z < A.z) {
                    const uint32_t R = min((uint32_t)min(A.z - B.z, lagcap) * vv + vr, kRClamp);
                    blocked = in(R * R, R);
                }
            }
        }
        for (int o = 1; o < G; o <<= 1) {   // combine the group's lanes (one warp)
            blocked |= __shfl_xor_sync(0xFFFFFFFFu, blocked, o) != 0;
            dig += __shfl_xor_sync(0xFFFFFFFFu, dig, o);
        }
        __syncthreads();
        lab = -1;
        if (st != ST_DONE) {
            lab = (int)suf_find(par, (uint32_t)t);
            if (lead && (blocked || st == ST_RUNNING)) sbad[lab] = 1;
        }
        __syncthreads();
        const bool rdy = lead && st == ST_IDLE && !sbad[lab];
        if (mine && lead) slab[t] = rdy ? lab : -1;   // ready clusters' members (exclusive tiles)
        // ---- dispatch part a (k_disp_a): cluster completion time
        if (rdy) {
            const long long du = duration(r.sy, i, A.z);
            atomicMax(stcl + lab, (unsigned long long)(tsim + du));
            busy += du - r.sy.base_us;
        }
        __syncthreads();
        // ---- dispatch part b (k_disp_b): member completion times and moves
        if (rdy) snp[t] = policy_move(r, i, A.z, make_int2(A.x, A.y), dig);
        if (r.sy.conflict) {
            // exclusive tiles, per ready cluster (resolve_exclusive in the oracle): a
            // move is cancelled if its target is a cluster-mate's current tile or a
            // lower-id cluster-mate proposes the same tile
            __syncthreads();
            bool keep = true;
            if (rdy) {
                const int2 q = snp[t];
                if (q.x != A.x || q.y != A.y) {
                    for (int j = 0; j < m && keep; j++) {
                        if (j == t || slab[j] != lab) continue;
                        const int4 B = sa[j];
                        const int2 qj = snp[j];
                        if ((B.x == q.x && B.y == q.y) || (j < t && qj.x == q.x && qj.y == q.y)) keep = false;
                    }
                }
            }
            __syncthreads();
            if (rdy && !keep) snp[t] = make_int2(A.x, A.y);
        }
        if (rdy) {
            sa[t].w = ST_RUNNING;
            stc[t] = (long long)stcl[lab];
            atomicAdd(&s_nr, 1);
            if (r.K > 0) {   // finite capacity: queued now, started below in key order
                stc[t] = LLONG_MAX;
                sq[t] = ((unsigned long long)(r.prio ? (uint32_t)A.z : (uint32_t)nrounds) << 32) | (uint32_t)(lo + lab);
            }
        }
        if (r.K > 0) {
            // start queued clusters in key order while they fit (strict order; a cluster
            // larger than K starts only when nothing is in service) -- orc_replay_cap
            if (threadIdx.x == 0) s_busy = 0;
            __syncthreads();
            if (mine && lead && sa[t].w == ST_RUNNING && stc[t] != LLONG_MAX) atomicAdd((unsigned long long*)&s_busy, 1ull);
            for (;;) {
                if (threadIdx.x == 0) { s_best = ~0ull; s_size = 0; s_dmax = 0; }
                __syncthreads();
                const bool queued = mine && lead && sa[t].w == ST_RUNNING && stc[t] == LLONG_MAX;
                if (queued) atomicMin(&s_best, sq[t]);
                __syncthreads();
                const unsigned long long best = s_best;
                if (best == ~0ull) break;
                const bool head = queued && sq[t] == best;
                if (head) {
                    atomicAdd((unsigned long long*)&s_size, 1ull);
                    atomicMax((unsigned long long*)&s_dmax, (unsigned long long)duration(r.sy, i, sa[t].z));
                }
                __syncthreads();
                if (s_busy > 0 && s_busy + s_size > r.K) break;
                if (head) stc[t] = tsim + s_dmax;
                __syncthreads();
                if (threadIdx.x == 0) s_busy += s_size;
            }
            __syncthreads();
        }
        if (mine && lead && (rdy || st == ST_RUNNING)) atomicMin(&s_tmin, (unsigned long long)stc[t]);
        __syncthreads();
        // ---- next event (k_disp_b's last block); this round counts (an agent was active)
        const unsigned long long tn = s_tmin;
        disp += s_nr;
        nrounds += 1;
        if (tn >= (unsigned long long)LLONG_MAX) {   // agents left, nothing in service: liveness violation
            live_err = 1;
            break;
        }
        tsim = r.Q > 0 ? (((long long)tn + r.Q - 1) / r.Q) * r.Q : (long long)tn;
        // ---- commits at the new event time (k_commit)
        if (mine && lead) {
            int4 S = sa[t];
            if (S.w == ST_RUNNING && stc[t] <= tsim) {
                const int2 np = snp[t];
                S.x = np.x; S.y = np.y; S.z += 1;
                traj = traj_step(traj, S.z, np.x, np.y);
                const bool done = d.target > 0 && S.z == d.target;
                S.w = done ? ST_DONE : ST_IDLE;
                sa[t] = S;
                if (done) s_fin = 1;
            }
            if (S.w != ST_DONE) s_any = 1;
        }
        __syncthreads();
        if (s_fin) tdone = max(tdone, tsim);
        act = s_any;
        __syncthreads();   // s_* are reset at the top of the next round
    }
    // ---- exit: the multi-kernel round's state
    const int4 S = mine ? sa[t] : make_int4(0, 0, 0, ST_DONE);
    if (mine && lead) {
        const int2 p = make_int2(S.x, S.y);
        r.pos[i] = p;
        r.steps[i] = S.z;
        d.pos[c][i] = p;
        d.step[c][i] = S.z;
        d.status[c][i] = (uint8_t)S.w;
        r.tcommit[i] = stc[t];
        r.newpos[i] = snp[t];
        r.qkey[i] = sq[t];
        r.traj[i] = traj;
        if (lab >= 0 || S.w == ST_DONE) d.labels[i] = S.w == ST_DONE ? -1 : lo + lab;
    }
    if (threadIdx.x == 0) { s_tmin = ~0ull; s_any = 0; }
    __syncthreads();
    if (mine && lead && S.w == ST_RUNNING && stc[t] != LLONG_MAX) atomicMin(&s_tmin, (unsigned long long)stc[t]);
    if (mine && lead && S.w != ST_DONE) atomicAdd(&s_any, 1);
    if (busy) atomicAdd((unsigned long long*)(r.llm + b), (unsigned long long)busy);   // LLM time dispatched
    __syncthreads();
    if (threadIdx.x == 0) {
        r.t_sim[b] = tsim;
        r.tdone[b] = tdone;
        r.rounds[b] = nrounds;
        r.active_flag[b] = act && !live_err;
        r.tnext[b] = s_tmin == ~0ull ? LLONG_MAX : (long long)s_tmin;
        if (disp) atomicAdd((unsigned long long*)r.dispatched, (unsigned long long)disp);
        if (live_err) *r.liveness = 1;
        if (s_any) atomicAdd(&d.ctl->n_active, s_any);
    }
}

// the round's priority order straight into page-locked host memory (mapped, UVA):
// only the n_ready valid entries cross the link, not the n-entry capacity
__global__ void __launch_bounds__(256) k_order_out(const int32_t* __restrict__ order, const Ctl* ctl,
                                                   int32_t* __restrict__ h_order)
{
    const int nr = ctl->n_ready;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nr; k += gridDim.x * blockDim.x)
        h_order[k] = order[k];
}

// delta write-back of the committed world state into page-locked host arrays that
// already hold the round's input (am_replay_io with aliased in/out arrays): an agent's
// position changes only with its step (commit validation), so only agents whose step
// differs from the copied-in value need writing.  They are sparse and scattered, and
// single 4-8 byte writes over PCIe cost a transaction each, so every aligned group of 8
// agents with a change is written whole (64 B of positions + 32 B of steps, coalesced;
// the unchanged members rewrite the value the host already holds).
__global__ void __launch_bounds__(256) k_delta_out(int n, const int32_t* __restrict__ shadow,
                                                   const int2* __restrict__ pos, const int32_t* __restrict__ steps,
                                                   int2* __restrict__ h_pos, int32_t* __restrict__ h_steps)
{
    const int lane = threadIdx.x & 31;
    for (int base = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; base < n; base += gridDim.x * blockDim.x) {
        const int i = base + lane;   // warp-uniform loop: every lane takes part in the ballot
        int s = 0;
        bool ch = false;
        if (i < n) {
            s = steps[i];
            ch = s != shadow[i];
        }
        const unsigned m = __ballot_sync(0xFFFFFFFFu, ch);
        if (i < n && ((m >> (lane & 24)) & 0xFFu)) {
            h_steps[i] = s;
            h_pos[i] = pos[i];
        }
    }
}

}  // namespace am

using namespace am;

struct am_replay {
    am_ctx* ctx = nullptr;
    RepDev r{};
    void* mem = nullptr;
    bool mem_owned = false;             // allocated here (no caller workspace)
    uint8_t* mask = nullptr;
    int32_t* order = nullptr;
    cudaStream_t stream = nullptr;      // own stream (graph capture)
    cudaStream_t user_stream = nullptr;
    cudaGraphExec_t g1 = nullptr, g8 = nullptr, g1x = nullptr;   // g1x: one host-buffer (external) round
    Dev qsd{};                          // finite capacity, binned path: the queue sort's view
    unsigned graph_prof = 0;            // profiling mask the graphs were captured with
    uint32_t graph_flags = 0;           // context flags the graphs were captured with
    long long* h_buf = nullptr;         // pinned: dispatched, liveness
    int32_t* shadow = nullptr;          // am_replay_io: the steps as copied in (delta write-back)
    cudaStream_t copy = nullptr;        // am_replay_io: the mask's device->host copy beside the round
    cudaEvent_t ev_copy = nullptr;
    cudaGraphExec_t g_io = nullptr;     // one round + that copy, captured for the host mask g_io_mask
    const void* g_io_mask = nullptr;
};

static int rp_err(am_replay* rp, cudaError_t e, const char* where)
{
    char buf[256];
    snprintf(buf, sizeof buf, "%s: %s", where, cudaGetErrorString(e));
    if (rp && rp->ctx) rp->ctx->err = buf;
    return AM_E_CUDA;
}
#define RK(call)                                             \
    do {                                                     \
        cudaError_t e_ = (call);                             \
        if (e_ != cudaSuccess) return rp_err(rp, e_, #call); \
    } while (0)

// One round: update (ingest the world state) -> ready -> dispatch -> next event ->
// commit at the next event time.  Committing at the end of the round (instead of the
// start of the next) leaves the state a host-side user would hold between rounds in
// the world arrays; the sequence of rounds is unchanged.
static int enqueue_round(am_replay* rp, bool external = false)
{
    am_ctx* c = rp->ctx;
    const int n = c->d.n;
    const unsigned nb = (unsigned)((n + 255) / 256);
    const unsigned ncb = (unsigned)((n + 256 * kCommitItems - 1) / (256 * kCommitItems));
    const bool inplace = c->path == 1;   // the cell-binned tracker takes the commits in place
    int rc;
    if (inplace && !external && !c->first) {
        // the driver's own round: its last k_commit applied the commits to the tracker
        // already, so no O(N) ingest of the world arrays -- k_replay_begin publishes the
        // post-commit W / S / counts from the commit's block partials (am_ready then
        // skips k_round_begin)
        if (c->bin_pending) return AM_E_STATE;
        am_join_side(c);
        am_prof_begin(c, K_INGEST);
        RK(launch_k(c->pdl, rp->stream, k_replay_begin, 1, 32, 0, rp->r, (int)ncb));
        am_prof_end(c, K_INGEST);
        c->bin_pending = true;
    } else {
        // the world arrays as a user hands them in (am_replay_io): diffed and validated
        rc = am_update_binned(c, (const int32_t*)rp->r.pos, rp->r.steps);
        if (rc) return rc;
    }
    c->defer_join = true;   // the sort overlaps dispatch + commit; joined below
    rc = am_ready(c, rp->mask, rp->order, nullptr);
    c->defer_join = false;
    if (rc) return rc;
    rp->r.d = c->d;
    am_prof_begin(c, K_DISP_A);
    const unsigned nbd = std::min(nb, (unsigned)c->num_sms * 4);   // grid-stride over the ready list
    RK(launch_k(c->pdl, rp->stream, k_disp_a, nbd, 256, 0, rp->r));
    am_prof_end(c, K_DISP_A);
    // PROFILING ONLY (AM_DBG_LATE_DIGEST=1, wrong moves): the join after the commit
    // instead -- measures how much of the round the digests hold up beyond part a
    static const bool late_dig = [] { const char* e = getenv("AM_DBG_LATE_DIGEST"); return e && atoi(e); }();
    if (!late_dig) am_join_digest(c);   // part b reads the digests (computed beside part a)
    am_prof_begin(c, K_DISP_B);
    RK(launch_k(c->pdl, rp->stream, k_disp_b, nbd, 256, 0, rp->r));
    if (rp->r.K > 0 && c->path == 1) {
        // finite capacity: the queued clusters sorted by key, started while they fit
        RK(launch_k(c->pdl, rp->stream, k_qprep, nbd, 256, 0, rp->r));
        const int qrc = am_internal_csort(c, rp->qsd, rp->r.qorder, rp->stream);
        if (qrc) return qrc;
        RK(launch_k(false, rp->stream, k_qstart, 1, 1024, 0, rp->r));
    }
    am_prof_end(c, K_DISP_B);
    am_prof_begin(c, K_COMMIT);
    if (inplace && c->d.n_sims == 1 && AM_COMMIT_SPLIT) {
        // the O(N) scan and the dense commit of the listed agents (two passes)
        const unsigned g = std::min(ncb, (unsigned)c->num_sms * 8);
        RK(launch_k(c->pdl, rp->stream, k_commit_scan, g, 256, 0, rp->r));
        RK(launch_k(c->pdl, rp->stream, k_commit_apply, std::min(nb, (unsigned)c->num_sms * 4), 256, 0, rp->r));
    } else {
        RK(launch_k(c->pdl, rp->stream, k_commit, ncb, 256, 0, rp->r, inplace ? 1 : 0));
    }
    am_join_side(c);   // the priority sort ran beside dispatch and commit
    if (late_dig) am_join_digest(c);
    am_prof_end(c, K_COMMIT);
    RK(cudaGetLastError());
    return AM_OK;
}

// device workspace layout of a replay (caller-owned, am_replay_workspace_size)
struct RepLayout {
    size_t total, tc, np, tr, tcl, ts, tn, td, rd, af, disp, live, chain, qk, mask, order, shadow, part, llm, clist;
    size_t qsz = 0, qek[2] = {}, qel[2] = {}, qes[2] = {}, qed[2] = {}, qrk[2] = {}, qrv[2] = {}, qn = 0, qcur = 0,
           qst = 0, qsep = 0, busy = 0, qorder = 0, qctl = 0;
};
static RepLayout rep_layout(const am_ctx* ctx)
{
    RepLayout L{};
    const long long n = std::max(1, ctx->d.n), S = ctx->d.n_sims;
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += (b + 255) & ~size_t(255); return o; };
    L.tc = take(8 * n); L.np = take(8 * n); L.tr = take(8 * n); L.tcl = take(8 * n);
    L.ts = take(8 * S); L.tn = take(8 * S); L.td = take(8 * S); L.rd = take(8 * S); L.af = take(4 * S);
    L.disp = take(8); L.live = take(4); L.chain = take(sizeof(Chain)); L.qk = take(8 * n);
    L.mask = take(n); L.order = take(4 * n);
    L.shadow = take(4 * n);   // am_replay_io: the steps as copied in (delta write-back)
    L.part = take(32 * ((n + 256 * kCommitItems - 1) / (256 * kCommitItems)));   // k_commit partials
    L.llm = take(8 * std::max(S, 16LL * 64));   // one simulation: 64 stripes of 128 bytes
    L.clist = take(4 * n);
    if (ctx->path == 1) {   // finite capacity on the cell-binned path: the cluster queue
        L.qsz = take(4 * n);
        for (int b = 0; b < 2; b++) {
            L.qek[b] = take(8 * n); L.qel[b] = take(4 * n); L.qes[b] = take(4 * n); L.qed[b] = take(8 * n);
            L.qrk[b] = take(8 * n); L.qrv[b] = take(4 * n);
        }
        L.qn = take(8); L.qcur = take(4); L.qst = take(8 * n); L.qsep = take(4 * n); L.busy = take(8);
        L.qorder = take(4 * n); L.qctl = take(sizeof(Ctl));
    }
    L.total = off;
    return L;
}

extern "C" size_t am_replay_workspace_size(const am_ctx* ctx) { return ctx ? rep_layout(ctx).total : 0; }

extern "C" int am_replay_create(am_replay** out, am_ctx* ctx, const am_synth* synth, int64_t quantum_us,
                                int32_t* positions, int32_t* steps, void* workspace, size_t workspace_bytes)
{
    if (!out || !ctx || !synth || !positions || !steps) return AM_E_ARG;
    if (ctx->d.target <= 0) {
        ctx->err = "am_replay_create: the context needs target_step > 0";
        return AM_E_ARG;
    }
    if (synth->n_vals < 1 || synth->n_vals > 16 || !synth->lat || !synth->cdf32 || !synth->vals) {
        if (!synth->dur_table) {
            ctx->err = "am_replay_create: bad latency tables";
            return AM_E_ARG;
        }
    }
    if ((synth->policy == 3) != (ctx->d.metric == AM_METRIC_GRAPH) ||
        (synth->policy == 3 && (!synth->graph_off || !synth->graph_adj || !ctx->d.gdist))) {
        ctx->err = "am_replay_create: the graph walk (policy 3) goes with AM_METRIC_GRAPH and am_set_graph";
        return AM_E_ARG;
    }
    if (synth->conflict && (ctx->path != 0 || ctx->d.r_p < 2 * ctx->d.v)) {
        ctx->err = "am_replay_create: exclusive tiles need the fused per-simulation path and r_p >= 2 v";
        return AM_E_ARG;
    }
    const RepLayout L = rep_layout(ctx);
    if (workspace && (workspace_bytes < L.total || ((uintptr_t)workspace & 255))) {
        ctx->err = "am_replay_create: workspace smaller than am_replay_workspace_size() or not 256-byte aligned";
        return AM_E_WORKSPACE;
    }
    am_replay* rp = new (std::nothrow) am_replay();
    if (!rp) return AM_E_ARG;
    rp->ctx = ctx;
    rp->user_stream = ctx->stream;
    const long long S = ctx->d.n_sims;
    const size_t off = L.total;
    if (workspace) {
        rp->mem = workspace;
        rp->mem_owned = false;
    } else {   // no caller workspace: the replay allocates (and frees) its own
        cudaError_t e = cudaMalloc(&rp->mem, off);
        if (e != cudaSuccess) { delete rp; return rp_err(nullptr, e, "cudaMalloc"); }
        rp->mem_owned = true;
    }
    char* b = (char*)rp->mem;
    RepDev& r = rp->r;
    r.sy = *synth;
    r.Q = quantum_us;
    r.pos = (int2*)positions;
    r.steps = steps;
    r.tcommit = (long long*)(b + L.tc);
    r.newpos = (int2*)(b + L.np);
    r.traj = (unsigned long long*)(b + L.tr);
    r.tcl = (long long*)(b + L.tcl);
    r.t_sim = (long long*)(b + L.ts);
    r.tnext = (long long*)(b + L.tn);
    r.tdone = (long long*)(b + L.td);
    r.rounds = (long long*)(b + L.rd);
    r.active_flag = (int32_t*)(b + L.af);
    r.dispatched = (long long*)(b + L.disp);
    r.liveness = (int32_t*)(b + L.live);
    r.chain = (Chain*)(b + L.chain);
    r.qkey = (unsigned long long*)(b + L.qk);
    r.K = 0;
    r.prio = 1;
    rp->mask = (uint8_t*)(b + L.mask);
    rp->order = (int32_t*)(b + L.order);
    rp->shadow = (int32_t*)(b + L.shadow);
    r.part = (int32_t*)(b + L.part);
    r.llm = (long long*)(b + L.llm);
    r.clist = (int32_t*)(b + L.clist);
    if (ctx->path == 1) {
        r.qsz = (int32_t*)(b + L.qsz);
        for (int q = 0; q < 2; q++) {
            r.qe_key[q] = (unsigned long long*)(b + L.qek[q]); r.qe_lab[q] = (int32_t*)(b + L.qel[q]);
            r.qe_size[q] = (int32_t*)(b + L.qes[q]); r.qe_dur[q] = (long long*)(b + L.qed[q]);
            r.qrk[q] = (unsigned long long*)(b + L.qrk[q]); r.qrv[q] = (uint32_t*)(b + L.qrv[q]);
        }
        r.qn = (int32_t*)(b + L.qn); r.qcur = (int32_t*)(b + L.qcur);
        r.qstart_t = (long long*)(b + L.qst); r.qstart_ep = (uint32_t*)(b + L.qsep);
        r.busy = (long long*)(b + L.busy); r.qorder = (int32_t*)(b + L.qorder); r.qctl = (Ctl*)(b + L.qctl);
        r.qidb = ctx->d.idbits;
        rp->qsd = ctx->d;   // the queue sort's view: its keys / ids and control block
        rp->qsd.ctl = r.qctl;
        rp->qsd.rkey[0] = r.qrk[0]; rp->qsd.rkey[1] = r.qrk[1];
        rp->qsd.rval[0] = r.qrv[0]; rp->qsd.rval[1] = r.qrv[1];
    }
    r.order = ctx->path == 1 ? ctx->d.rid : rp->order;
    RK(cudaStreamCreateWithFlags(&rp->stream, cudaStreamNonBlocking));
    RK(cudaMallocHost((void**)&rp->h_buf, 64));
    RK(cudaStreamSynchronize(rp->user_stream));
    RK(cudaMemsetAsync(rp->mem, 0, off, rp->stream));
    RK(cudaMemsetAsync(r.tnext, 0x7F, 8 * S, rp->stream));  // "no pending" marker
    if (ctx->path == 1) RK(cudaMemsetAsync(r.qstart_ep, 0xFF, 4 * (size_t)std::max(1, ctx->d.n), rp->stream));
    RK(cudaStreamSynchronize(rp->stream));
    // tnext must be exactly LLONG_MAX: fill with a tiny copy
    {
        long long* h = (long long*)malloc(8 * S);
        for (long long k = 0; k < S; k++) h[k] = LLONG_MAX;
        RK(cudaMemcpy(r.tnext, h, 8 * S, cudaMemcpyHostToDevice));
        int32_t* a = (int32_t*)h;
        for (long long k = 0; k < S; k++) a[k] = 1;
        RK(cudaMemcpy(r.active_flag, a, 4 * S, cudaMemcpyHostToDevice));
        free(h);
    }
    am_set_stream(ctx, rp->stream);
    ctx->d.flags = (ctx->d.flags | AM_DIGEST | AM_ASYNC) & ~AM_PEEK;
    am_reset(ctx);
    int rc = am_update(ctx, positions, steps);  // initial state (synchronous)
    if (rc) {
        am_replay_destroy(rp);
        return rc;
    }
    r.d = ctx->d;
    *out = rp;
    return AM_OK;
}

// One round whose ready mask is copied to the page-locked host array h_mask on a
// forked stream as soon as k_ready has written it (beside dispatch, commit and the
// priority sort), captured as a graph for that host array.
static int build_io_graph(am_replay* rp, uint8_t* h_mask)
{
    am_ctx* c = rp->ctx;
    if (!rp->copy) {
        RK(cudaStreamCreateWithFlags(&rp->copy, cudaStreamNonBlocking));
        RK(cudaEventCreateWithFlags(&rp->ev_copy, cudaEventDisableTiming));
    }
    if (rp->g_io) cudaGraphExecDestroy(rp->g_io);
    rp->g_io = nullptr;
    cudaGraph_t g;
    RK(cudaStreamBeginCapture(rp->stream, cudaStreamCaptureModeThreadLocal));
    c->mask_event = true;
    int rc = enqueue_round(rp, true);   // the host-buffer round: the world state is diffed and validated
    c->mask_event = false;
    cudaError_t e = cudaSuccess;
    if (rc == AM_OK) {
        e = cudaStreamWaitEvent(rp->copy, c->ev_mask, 0);
        if (e == cudaSuccess) e = cudaMemcpyAsync(h_mask, rp->mask, (size_t)c->d.n, cudaMemcpyDeviceToHost, rp->copy);
        if (e == cudaSuccess) e = cudaEventRecord(rp->ev_copy, rp->copy);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(rp->stream, rp->ev_copy, 0);
    }
    cudaError_t e2 = cudaStreamEndCapture(rp->stream, &g);
    if (rc) return rc;
    if (e != cudaSuccess) return rp_err(rp, e, "io graph capture");
    if (e2 != cudaSuccess) return rp_err(rp, e2, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&rp->g_io, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return rp_err(rp, e, "cudaGraphInstantiate");
    rp->g_io_mask = h_mask;
    return AM_OK;
}

static int build_graph(am_replay* rp, int rounds, cudaGraphExec_t* exec, bool external = false)
{
    cudaGraph_t g;
    RK(cudaStreamBeginCapture(rp->stream, cudaStreamCaptureModeThreadLocal));
    int rc = AM_OK;
    for (int k = 0; k < rounds && rc == AM_OK; k++) rc = enqueue_round(rp, external);
    cudaError_t e = cudaStreamEndCapture(rp->stream, &g);
    if (rc) return rc;
    if (e != cudaSuccess) return rp_err(rp, e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return rp_err(rp, e, "cudaGraphInstantiate");
    return AM_OK;
}

static int finish_check(am_replay* rp, int64_t* active)
{
    am_ctx* c = rp->ctx;
    RK(cudaMemcpyAsync(rp->h_buf, rp->r.liveness, 4, cudaMemcpyDeviceToHost, rp->stream));
    int rc = am_sync(c);  // reads the control block (n_active) + validation errors
    if (rc) return rc;
    if (*(int32_t*)rp->h_buf) {
        c->err = "replay: agents not DONE but nothing running (liveness)";
        return AM_E_LIVENESS;
    }
    if (active) *active = c->h_ctl->n_active;
    return AM_OK;
}

static int ensure_graphs(am_replay* rp)
{
    if ((rp->r.K > 0 && rp->ctx->path == 0) || rp->r.sy.conflict) {   // only the persistent per-simulation kernel has these
        rp->ctx->err = "finite LLM capacity and exclusive tiles run through am_replay_run / am_replay_launch "
                       "on the fused per-simulation path (<= 1024 agents per simulation, tracing off)";
        return AM_E_ARG;
    }
    const unsigned pm = rp->ctx->prof.on ? rp->ctx->prof.mask : 0u;
    if (pm != rp->graph_prof || rp->ctx->d.flags != rp->graph_flags) {  // baked in at capture
        if (rp->g1) cudaGraphExecDestroy(rp->g1);
        if (rp->g8) cudaGraphExecDestroy(rp->g8);
        if (rp->g_io) cudaGraphExecDestroy(rp->g_io);
        if (rp->g1x) cudaGraphExecDestroy(rp->g1x);
        rp->g1 = rp->g8 = rp->g_io = rp->g1x = nullptr;
        rp->g_io_mask = nullptr;
        rp->graph_prof = pm;
        rp->graph_flags = rp->ctx->d.flags;
    }
    int rc;
    if (!rp->g8 && (rc = build_graph(rp, 8, &rp->g8))) return rc;
    if (!rp->g1 && (rc = build_graph(rp, 1, &rp->g1))) return rc;
    return AM_OK;
}

// Fused per-simulation path (every simulation <= 1024 agents), no profiling: rounds
// run inside one persistent kernel (k_small_replay), one CTA per simulation.
static bool small_persistent(am_replay* rp)
{
    am_ctx* c = rp->ctx;
    if ((rp->r.K > 0 && c->path == 0) || rp->r.sy.conflict) return c->path == 0;   // only the persistent kernel has them
    if (c->path != 0 || c->prof.on) return false;
    static const int off = [] { const char* e = getenv("AM_SMALL_PERSIST"); return e && atoi(e) == 0; }();
    return !off;   // AM_SMALL_PERSIST=0: the multi-kernel rounds (ablation)
}
static int launch_small_replay(am_replay* rp, int64_t rounds)
{
    am_ctx* c = rp->ctx;
    const int M = c->small_threads;   // >= agents of the largest simulation, multiple of 32
    const size_t smem = (size_t)M * (8 + 8 + 8 + 16 + 8 + 4 + 4 + 1);
    // lanes per agent: as many as one CTA of <= 1024 threads holds while all the
    // simulations' CTAs fit in half the GPU's thread slots (measured: C1 G = 32 3.0x
    // over G = 1; C3's 4096 simulations are best at G = 1)
    int G = 1;
    while (G < 32 && M * G * 2 <= 1024 && (long long)c->d.n_sims * M * G * 2 <= 1024LL * c->num_sms) G *= 2;
    if (const char* e = getenv("AM_SMALL_LANES")) {   // tuning knob (rounded down to a power of two)
        const int want = std::max(1, std::min(32, atoi(e)));
        G = 1;
        while (G * 2 <= want) G *= 2;
    }
    while (M * G > 1024) G /= 2;
    static bool attr = [] {   // > 48 KB of dynamic shared memory for 1024-agent simulations
        cudaFuncSetAttribute(k_small_replay<AM_METRIC_L2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        cudaFuncSetAttribute(k_small_replay<AM_METRIC_LINF>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        cudaFuncSetAttribute(k_small_replay<AM_METRIC_GRAPH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        cudaGetLastError();
        return true;
    }();
    (void)attr;
    RK(cudaMemsetAsync(&c->d.ctl->n_active, 0, sizeof(int32_t), rp->stream));
    rp->r.d = c->d;
    if (c->d.metric == AM_METRIC_GRAPH)
        RK(launch_k(false, rp->stream, k_small_replay<AM_METRIC_GRAPH>, (unsigned)c->d.n_sims, (unsigned)(M * G), smem,
                    rp->r, (long long)rounds, M, G));
    else if (c->d.metric == AM_METRIC_LINF)
        RK(launch_k(false, rp->stream, k_small_replay<AM_METRIC_LINF>, (unsigned)c->d.n_sims, (unsigned)(M * G), smem,
                    rp->r, (long long)rounds, M, G));
    else
        RK(launch_k(false, rp->stream, k_small_replay<AM_METRIC_L2>, (unsigned)c->d.n_sims, (unsigned)(M * G), smem,
                    rp->r, (long long)rounds, M, G));
    return AM_OK;
}

extern "C" int am_replay_run(am_replay* rp, int64_t max_rounds, int64_t* active)
{
    if (!rp) return AM_E_ARG;
    int rc;
    if (small_persistent(rp)) {
        if (max_rounds > 0 && (rc = launch_small_replay(rp, max_rounds))) return rc;
        return finish_check(rp, active);
    }
    if ((rc = ensure_graphs(rp))) return rc;
    int64_t k = 0;
    for (; k + 8 <= max_rounds; k += 8) RK(cudaGraphLaunch(rp->g8, rp->stream));
    for (; k < max_rounds; k++) RK(cudaGraphLaunch(rp->g1, rp->stream));
    if (max_rounds > 0) am_prof_mark(rp->ctx, rp->graph_prof);
    return finish_check(rp, active);
}

extern "C" int am_replay_set_capacity(am_replay* rp, int64_t capacity, int32_t priority)
{
    if (!rp || capacity < 0) return AM_E_ARG;
    long long rounds = 0;
    RK(cudaMemcpy(&rounds, rp->r.rounds, sizeof rounds, cudaMemcpyDeviceToHost));   // sim 0's round count
    if (rounds != 0) {
        rp->ctx->err = "am_replay_set_capacity: only before the first round";
        return AM_E_STATE;
    }
    if (capacity > 0 && rp->ctx->path == 1 && rp->ctx->d.n_sims != 1) {
        rp->ctx->err = "am_replay_set_capacity: the cell-binned path takes one simulation";
        return AM_E_ARG;
    }
    rp->r.K = capacity;
    rp->r.prio = priority ? 1 : 0;
    return AM_OK;
}

extern "C" int am_replay_step(am_replay* rp, uint8_t* mask, int32_t* order, int32_t* labels, int32_t* n_ready)
{
    if (!rp) return AM_E_ARG;
    if ((rp->r.K > 0 && rp->ctx->path == 0) || rp->r.sy.conflict) {
        rp->ctx->err = "am_replay_step: not available with a finite capacity on the fused path or exclusive tiles "
                       "(use am_replay_run)";
        return AM_E_ARG;
    }
    int rc = enqueue_round(rp);
    if (rc) return rc;
    am_ctx* c = rp->ctx;
    const size_t n = (size_t)c->d.n;
    if (mask) RK(cudaMemcpyAsync(mask, rp->mask, n, cudaMemcpyDeviceToDevice, rp->stream));
    if (order) RK(cudaMemcpyAsync(order, rp->order, 4 * n, cudaMemcpyDeviceToDevice, rp->stream));
    if (labels) RK(cudaMemcpyAsync(labels, c->d.labels, 4 * n, cudaMemcpyDeviceToDevice, rp->stream));
    int64_t act = 0;
    rc = finish_check(rp, &act);
    if (rc) return rc;
    if (n_ready) *n_ready = c->h_ctl->n_ready;
    return AM_OK;
}

extern "C" void* am_replay_stream(am_replay* rp) { return rp ? (void*)rp->stream : nullptr; }

// One round with the world state held in HOST memory (the end-to-end user loop):
// H2D of positions/steps, the round (CUDA graph), D2H of the committed state, the
// ready mask, the priority order (n entries) and the ready count, then synchronise.
extern "C" int am_replay_io(am_replay* rp, const int32_t* h_pos_in, const int32_t* h_steps_in,
                            int32_t* h_pos_out, int32_t* h_steps_out, uint8_t* h_mask, int32_t* h_order,
                            int32_t* n_ready)
{
    if (!rp || !h_pos_in || !h_steps_in) return AM_E_ARG;
    int rc;
    if ((rc = ensure_graphs(rp))) return rc;
    am_ctx* c = rp->ctx;
    const size_t n = (size_t)c->d.n;
    // delta write-back when the outputs alias the inputs and are page-locked: the host
    // arrays already hold the copied-in state, only committed agents change
    auto mapped = [](const void* p, void** dp) {
        cudaPointerAttributes pa{};
        const bool ok = p && cudaPointerGetAttributes(&pa, p) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
                        pa.devicePointer != nullptr;
        cudaGetLastError();
        if (ok) *dp = pa.devicePointer;
        return ok;
    };
    void *dpos = nullptr, *dsteps = nullptr;
    const bool delta = h_pos_out == h_pos_in && h_steps_out == h_steps_in && mapped(h_pos_out, &dpos) &&
                       mapped(h_steps_out, &dsteps);
    RK(cudaMemcpyAsync(rp->r.pos, h_pos_in, 8 * n, cudaMemcpyHostToDevice, rp->stream));
    RK(cudaMemcpyAsync(rp->r.steps, h_steps_in, 4 * n, cudaMemcpyHostToDevice, rp->stream));
    if (delta) RK(cudaMemcpyAsync(rp->shadow, rp->r.steps, 4 * n, cudaMemcpyDeviceToDevice, rp->stream));
    // page-locked host mask on the binned path: a graph whose mask copy starts right after
    // k_ready, beside dispatch, commit and the priority sort (captured per host array)
    void* dmask = nullptr;
    const bool split = c->path == 1 && h_mask && !c->prof.on && mapped(h_mask, &dmask);
    if (split) {
        if (rp->g_io_mask != (const void*)h_mask && (rc = build_io_graph(rp, h_mask))) return rc;
        RK(cudaGraphLaunch(rp->g_io, rp->stream));
    } else {
        // one round that diffs and validates the copied-in world state (captured once)
        if (!rp->g1x && (rc = build_graph(rp, 1, &rp->g1x, true))) return rc;
        RK(cudaGraphLaunch(rp->g1x, rp->stream));
        am_prof_mark(c, rp->graph_prof);
    }
    if (delta) {
        RK(launch_k(false, rp->stream, k_delta_out, (unsigned)c->num_sms * 4, 256, 0, (int)n, (const int32_t*)rp->shadow,
                    (const int2*)rp->r.pos, (const int32_t*)rp->r.steps, (int2*)dpos, (int32_t*)dsteps));
    } else {
        if (h_pos_out) RK(cudaMemcpyAsync(h_pos_out, rp->r.pos, 8 * n, cudaMemcpyDeviceToHost, rp->stream));
        if (h_steps_out) RK(cudaMemcpyAsync(h_steps_out, rp->r.steps, 4 * n, cudaMemcpyDeviceToHost, rp->stream));
    }
    if (!split && h_mask) RK(cudaMemcpyAsync(h_mask, rp->mask, n, cudaMemcpyDeviceToHost, rp->stream));
    if (h_order) {
        // page-locked (device-accessible) host order array: a kernel writes the n_ready
        // valid entries; pageable memory: a copy of the whole capacity
        void* dorder = nullptr;
        if (mapped(h_order, &dorder))
            RK(launch_k(false, rp->stream, k_order_out, (unsigned)c->num_sms, 256, 0, (const int32_t*)rp->order,
                        (const Ctl*)c->d.ctl, (int32_t*)dorder));
        else
            RK(cudaMemcpyAsync(h_order, rp->order, 4 * n, cudaMemcpyDeviceToHost, rp->stream));
    }
    if (n_ready) {
        rc = finish_check(rp, nullptr);
        if (rc) return rc;
        *n_ready = c->h_ctl->n_ready;
    }
    return AM_OK;
}

extern "C" int am_replay_launch(am_replay* rp, int64_t rounds)
{
    if (!rp || rounds < 0) return AM_E_ARG;
    int rc;
    if (small_persistent(rp)) return rounds > 0 ? launch_small_replay(rp, rounds) : AM_OK;
    if ((rc = ensure_graphs(rp))) return rc;
    int64_t k = 0;
    for (; k + 8 <= rounds; k += 8) RK(cudaGraphLaunch(rp->g8, rp->stream));
    for (; k < rounds; k++) RK(cudaGraphLaunch(rp->g1, rp->stream));
    if (rounds > 0) am_prof_mark(rp->ctx, rp->graph_prof);
    return AM_OK;
}

extern "C" int am_replay_sync(am_replay* rp, int64_t* active, int32_t* n_ready)
{
    if (!rp) return AM_E_ARG;
    int rc = finish_check(rp, active);
    if (rc) return rc;
    if (n_ready) *n_ready = rp->ctx->h_ctl->n_ready;
    return AM_OK;
}

extern "C" int am_replay_results(am_replay* rp, int64_t* T_ooo, int64_t* rounds, uint64_t* traj)
{
    if (!rp) return AM_E_ARG;
    const size_t S = (size_t)rp->ctx->d.n_sims;
    RK(cudaStreamSynchronize(rp->stream));
    if (T_ooo) RK(cudaMemcpy(T_ooo, rp->r.tdone, 8 * S, cudaMemcpyDeviceToHost));
    if (rounds) RK(cudaMemcpy(rounds, rp->r.rounds, 8 * S, cudaMemcpyDeviceToHost));
    if (traj) RK(cudaMemcpy(traj, rp->r.traj, 8 * (size_t)rp->ctx->d.n, cudaMemcpyDeviceToDevice));
    return AM_OK;
}

extern "C" int am_replay_llm_time(am_replay* rp, int64_t* llm_us)
{
    if (!rp || !llm_us) return AM_E_ARG;
    RK(cudaStreamSynchronize(rp->stream));
    if (rp->ctx->d.n_sims == 1) {   // one simulation: 64 stripes (k_disp_a); the persistent kernel adds to stripe 0
        long long h[16 * 64];
        RK(cudaMemcpy(h, rp->r.llm, sizeof h, cudaMemcpyDeviceToHost));
        long long acc = 0;
        for (int k = 0; k < 64; k++) acc += h[16 * k];
        llm_us[0] = acc;
        return AM_OK;
    }
    RK(cudaMemcpy(llm_us, rp->r.llm, 8 * (size_t)rp->ctx->d.n_sims, cudaMemcpyDeviceToHost));
    return AM_OK;
}

// T_sync[b] = sum over steps s < T of max over the agents i of simulation b of dur(i, s):
// Algorithm 1's global barrier per step, the parallel-sync baseline.
// Index k = s * n + i: a warp's lanes share the step (and mostly the simulation), so the
// max is warp-reduced before one atomic.
__global__ void k_lockstep_time(am_synth sy, int n, int n_sims, int T, unsigned long long* mx)
{
    const long long total = (long long)n * T;
    for (long long k0 = (long long)blockIdx.x * blockDim.x; k0 < total; k0 += (long long)gridDim.x * blockDim.x) {
        const long long k = k0 + threadIdx.x;
        int b = -1, s = 0;
        unsigned long long du = 0;
        if (k < total) {
            s = (int)(k / n);
            const int i = (int)(k % n);
            b = n_sims == 1 ? 0 : (int)(((long long)i * n_sims + n_sims - 1) / n);
            du = (unsigned long long)duration(sy, i, s);
        }
        const long long key = b < 0 ? -1 : (long long)b * T + s;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, key);
        unsigned long long m = du;
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long y = __shfl_xor_sync(0xFFFFFFFFu, m, o);
            const int src = (threadIdx.x & 31) ^ o;
            if ((peers >> src) & 1u) m = max(m, y);
        }
        // lanes of one key may not be a contiguous power-of-two group: finish with atomics
        if (b >= 0 && (__ffs(peers) - 1) == (int)(threadIdx.x & 31)) atomicMax(mx + key, m);
        else if (b >= 0) atomicMax(mx + key, du);
    }
}

__global__ void k_lockstep_sum(const unsigned long long* mx, int n_sims, int T, long long* out)
{
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < n_sims; b += gridDim.x * blockDim.x) {
        long long acc = 0;
        for (int s = 0; s < T; s++) acc += (long long)mx[(long long)b * T + s];
        out[b] = acc;
    }
}

extern "C" int am_lockstep_time(const am_synth* synth, int32_t n, int32_t n_sims, int32_t T, int64_t* T_sync,
                                void* stream)
{
    if (!synth || n < 1 || n_sims < 1 || n_sims > n || T < 0 || !T_sync) return AM_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long* mx = nullptr;
    long long* d_out = nullptr;
    const size_t cells = (size_t)n_sims * (size_t)std::max(1, T);
    if (cudaMallocAsync((void**)&mx, 8 * cells, st) != cudaSuccess) return AM_E_CUDA;
    if (cudaMallocAsync((void**)&d_out, 8 * (size_t)n_sims, st) != cudaSuccess) { cudaFreeAsync(mx, st); return AM_E_CUDA; }
    cudaMemsetAsync(mx, 0, 8 * cells, st);
    if (T > 0) k_lockstep_time<<<1184, 256, 0, st>>>(*synth, n, n_sims, T, mx);
    k_lockstep_sum<<<(n_sims + 255) / 256, 256, 0, st>>>(mx, n_sims, T, d_out);
    cudaError_t e = cudaMemcpyAsync(T_sync, d_out, 8 * (size_t)n_sims, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFreeAsync(mx, st);
    cudaFreeAsync(d_out, st);
    cudaStreamSynchronize(st);
    return e == cudaSuccess ? AM_OK : AM_E_CUDA;
}

extern "C" int am_replay_dispatched(am_replay* rp, int64_t* agent_steps)
{
    if (!rp || !agent_steps) return AM_E_ARG;
    RK(cudaMemcpyAsync(rp->h_buf + 1, rp->r.dispatched, 8, cudaMemcpyDeviceToHost, rp->stream));
    RK(cudaStreamSynchronize(rp->stream));
    *agent_steps = rp->h_buf[1];
    return AM_OK;
}

extern "C" int am_replay_destroy(am_replay* rp)
{
    if (!rp) return AM_OK;
    if (rp->stream) cudaStreamSynchronize(rp->stream);
    if (rp->g1) cudaGraphExecDestroy(rp->g1);
    if (rp->g8) cudaGraphExecDestroy(rp->g8);
    if (rp->g_io) cudaGraphExecDestroy(rp->g_io);
    if (rp->g1x) cudaGraphExecDestroy(rp->g1x);
    if (rp->ctx) {
        am_set_stream(rp->ctx, rp->user_stream);
        rp->ctx->d.flags &= ~AM_ASYNC;
    }
    if (rp->stream) cudaStreamDestroy(rp->stream);
    if (rp->h_buf) cudaFreeHost(rp->h_buf);
    if (rp->copy) {
        cudaStreamSynchronize(rp->copy);
        cudaStreamDestroy(rp->copy);
        cudaEventDestroy(rp->ev_copy);
    }
    if (rp->mem_owned) cudaFree(rp->mem);
    delete rp;
    return AM_OK;
}
