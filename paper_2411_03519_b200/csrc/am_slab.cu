// am_slab.cu -- the tracker and the replay driver split across GPUs by spatial slabs
// (include/am_slab.h).  One rank = one am_slab: the WINDOW of
// its slab (every agent within `halo` rows, stable slots), an incremental tracker over
// the window, and the per-round steps between the three collectives the caller runs.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstring>
#include <new>

#include "am_internal.cuh"
#include "am_slab.h"
#include "am_synth.cuh"

int am_internal_digest(am_ctx* c, const int32_t* ids, const int32_t* count, const int32_t* gidmap,
                       unsigned long long* out, int max_ids, cudaStream_t s);
int am_internal_csort(am_ctx* c, const am::Dev& sd, int32_t* order, cudaStream_t s);

namespace am {

constexpr long long kNever = LLONG_MAX;
constexpr int kDeltaRec = 12;   // words of a delta record (am_slab.h)

// everything a slab kernel needs, by value
struct SlabDev {
    am_slab_geom g;
    am_synth sy;
    long long Q;
    int lo, hi;            // the slab's rows [lo, hi)
    int y0, y1;            // the window's rows [y0, y1)
    int idb;               // bits of a global id (priority keys)
    int L;                 // window slots
    int P;                 // a sync round every P rounds (stale_rounds; 1 = every round)
    // window (slot-indexed)
    int32_t* gid;          // -1 = free slot
    int2* pos;             // GLOBAL coordinates
    int2* tpos;            // the tracker's input: window coordinates (y - y0)
    int32_t* step;
    uint8_t* stat;         // the tracker's input status: owned real, ghost RUNNING, absent/finished DONE
    uint8_t* own;          // owned by this rank: the slab of its row at the last exchange (fixed in between)
    uint8_t* dirty;        // owned and committed since the last exchange
    int32_t* ly;           // row at the last exchange
    unsigned long long* traj;
    long long* tc;         // completion time of the dispatched step (owned RUNNING)
    int2* np;              // move computed at dispatch (global coordinates)
    unsigned long long* dig;   // perception digests of the dispatched agents
    int32_t* map;          // [n_total] global id -> slot, -1
    int32_t* fstack;       // free slots
    int32_t* ftop;         // [1] number of free slots
    // per local cluster (indexed by the tracker's label = its min slot)
    int32_t* mingid;
    int32_t* csize;
    uint8_t* badl;
    uint8_t* bndl;
    long long* maxd;
    // merge forest over global ids
    uint32_t* forest;
    uint8_t* badm;
    uint8_t* touched;
    long long* maxdm;
    // outputs
    int32_t* glabel;
    uint8_t* ready;
    int32_t* rlist;        // ready slots (dispatch list)
    Ctl* sctl;             // n_ready (= ready count) and sort_or of the order sort
    unsigned long long* rkey[2];
    uint32_t* rval[2];
    // driver
    long long* counters;   // [4] clock t, last finishing commit, dispatched, rounds
    int32_t* flags;        // [1] AM_SLAB_* (sticky)
    // the tracker's arrays of the last round
    const int32_t* labels;
    const uint8_t* blocked;
    const Ctl* tctl;
};

__device__ __forceinline__ int slab_lo_(int k, int G, int H) { return (int)((long long)k * H / G); }

__device__ __forceinline__ bool in_window(const SlabDev& s, int y) { return y >= s.y0 && y < s.y1; }
__device__ __forceinline__ bool in_slab(const SlabDev& s, int y) { return y >= s.lo && y < s.hi; }
// inside some other rank's window (a neighbour's, or farther when the halo exceeds a slab)
__device__ __forceinline__ bool in_other_window(const SlabDev& s, int y)
{
    return (s.g.my_slab > 0 && y < s.lo + s.g.halo) || (s.g.my_slab < s.g.n_slabs - 1 && y >= s.hi - s.g.halo);
}
__device__ __forceinline__ bool in_window_of(const SlabDev& s, int j, int y)
{
    const int lo = slab_lo_(j, s.g.n_slabs, s.g.map_h), hi = slab_lo_(j + 1, s.g.n_slabs, s.g.map_h);
    return y >= max(0, lo - s.g.halo) && y < min(s.g.map_h, hi + s.g.halo);
}

// ------------------------------------------------------------------ load
__global__ void k_sl_load(SlabDev s, int m, const int32_t* __restrict__ gid, const int2* __restrict__ pos,
                          const int32_t* __restrict__ steps, const uint8_t* __restrict__ status,
                          const unsigned long long* __restrict__ traj, const long long* __restrict__ tcommit,
                          const int2* __restrict__ newpos, long long t)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < s.L; i += gridDim.x * blockDim.x) {
        if (i < m) {
            const int g = gid[i];
            const int2 p = pos[i];
            uint8_t st = status[i];
            const bool own = in_slab(s, p.y);
            if (!own && st != ST_DONE) st = ST_RUNNING;   // ghost
            s.own[i] = own;
            s.dirty[i] = 0;
            s.ly[i] = p.y;
            s.gid[i] = g;
            s.pos[i] = p;
            s.step[i] = steps[i];
            s.stat[i] = st;
            s.traj[i] = traj ? traj[i] : 0ull;
            s.tc[i] = tcommit ? tcommit[i] : kNever;
            s.np[i] = newpos ? newpos[i] : p;
            s.map[g] = i;
        } else {
            s.gid[i] = -1;
            s.pos[i] = make_int2(0, s.y0);
            s.step[i] = 0;
            s.stat[i] = ST_DONE;
            s.own[i] = 0;
            s.dirty[i] = 0;
            s.ly[i] = s.y0;
            s.traj[i] = 0ull;
            s.tc[i] = kNever;
            s.np[i] = make_int2(0, s.y0);
            s.fstack[i - m] = i;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *s.ftop = s.L - m;
        s.counters[0] = t;
    }
}

// ------------------------------------------------------------------ round_local
// the tracker's input positions (window coordinates) and the per-cluster scratch reset
__global__ void k_sl_prep(SlabDev s, int32_t* mbuf)
{
    pdl_begin();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < s.L; i += gridDim.x * blockDim.x) {
        const int2 p = s.pos[i];
        s.tpos[i] = s.gid[i] >= 0 ? make_int2(p.x, p.y - s.y0) : make_int2(0, 0);
        s.mingid[i] = INT_MAX;
        s.csize[i] = 0;
        s.badl[i] = 0;
        s.bndl[i] = 0;
        s.maxd[i] = 0;
    }
    if (mbuf && blockIdx.x == 0 && threadIdx.x < 4) mbuf[threadIdx.x] = 0;   // link / cluster counts
}

// per local cluster: min global id, size, bad (an OWNED member RUNNING or blocked; in a
// stale round also any ghost member: its owner's verdict is not exchanged), max duration
// of the owned IDLE members, boundary flag
__global__ void k_sl_clusters(SlabDev s, int stale)
{
    pdl_begin();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < s.L; i += gridDim.x * blockDim.x) {
        const uint8_t st = s.stat[i];
        if (st == ST_DONE) continue;
        const int l = s.labels[i];
        const int g = s.gid[i];
        const int y = s.pos[i].y;
        const bool own = s.own[i] != 0;
        atomicMin(s.mingid + l, g);
        atomicAdd(s.csize + l, 1);
        if (own) {
            if (st == ST_RUNNING || s.blocked[i]) s.badl[l] = 1;
            if (st == ST_IDLE)
                atomicMax((unsigned long long*)(s.maxd + l), (unsigned long long)duration(s.sy, g, s.step[i]));
        } else if (stale) {
            s.badl[l] = 1;
        }
        if (!own || in_other_window(s, y)) s.bndl[l] = 1;
    }
}

// link records of boundary agents in clusters of >= 2 window agents; one cluster record
// per boundary cluster (from its root slot)
__global__ void k_sl_records(SlabDev s, int32_t* __restrict__ mbuf)
{
    pdl_begin();
    int32_t* counts = mbuf;
    int2* links = reinterpret_cast<int2*>(mbuf + 4);
    int4* clusters = reinterpret_cast<int4*>(mbuf + 4 + 2 * (size_t)s.g.cap_merge);
    const int lane = threadIdx.x & 31;
    for (int base = blockIdx.x * blockDim.x; base < s.L; base += gridDim.x * blockDim.x) {   // warp uniform
        const int i = base + threadIdx.x;
        bool lk = false, cr = false;
        int2 lv = make_int2(0, 0);
        int4 cv = make_int4(0, 0, 0, 0);
        if (i < s.L && s.stat[i] != ST_DONE) {
            const int l = s.labels[i];
            if (s.bndl[l]) {
                const int y = s.pos[i].y;
                const bool bnd = !s.own[i] || in_other_window(s, y);
                if (bnd && s.csize[l] > 1) {
                    lk = true;
                    lv = make_int2(s.gid[i], s.mingid[l]);
                }
                if (i == l) {
                    cr = true;
                    const unsigned long long md = (unsigned long long)s.maxd[l];
                    cv = make_int4(s.mingid[l], s.badl[l], (int)(uint32_t)md, (int)(uint32_t)(md >> 32));
                }
            }
        }
        // warp-aggregated appends
        const unsigned ml = __ballot_sync(0xFFFFFFFFu, lk), mc = __ballot_sync(0xFFFFFFFFu, cr);
        int bl = 0, bc = 0;
        if (lane == 0) {
            if (ml) bl = atomicAdd(counts, __popc(ml));
            if (mc) bc = atomicAdd(counts + 1, __popc(mc));
        }
        bl = __shfl_sync(0xFFFFFFFFu, bl, 0);
        bc = __shfl_sync(0xFFFFFFFFu, bc, 0);
        const unsigned lt = (1u << lane) - 1u;
        if (lk) {
            const int k = bl + __popc(ml & lt);
            if (k < s.g.cap_merge) links[k] = lv; else atomicOr(s.flags, AM_SLAB_OVF_MERGE);
        }
        if (cr) {
            const int k = bc + __popc(mc & lt);
            if (k < s.g.cap_merge) clusters[k] = cv; else atomicOr(s.flags, AM_SLAB_OVF_MERGE);
        }
    }
}

// ------------------------------------------------------------------ merge
// rank r's merge buffer in the all-gathered array
__device__ __forceinline__ const int32_t* mbuf_of(const SlabDev& s, const int32_t* mbufs, int r)
{
    return mbufs + (size_t)r * (size_t)AM_SLAB_MERGE_WORDS(s.g.cap_merge);
}
__device__ __forceinline__ int2 mlink(const SlabDev& s, const int32_t* mb, int j)
{
    return reinterpret_cast<const int2*>(mb + 4)[j];
}
__device__ __forceinline__ int4 mcluster(const SlabDev& s, const int32_t* mb, int j)
{
    return reinterpret_cast<const int4*>(mb + 4 + 2 * (size_t)s.g.cap_merge)[j];
}

// neutral values of this round's stats and of the order sort's counters (one thread)
__device__ __forceinline__ void stats_reset(const SlabDev& s, long long* stats)
{
    stats[0] = kNever;   // next event
    stats[1] = kNever;   // W
    stats[2] = kNever;   // -S
    stats[3] = 1;        // no agent active
    s.sctl->n_ready = 0;
    s.sctl->sort_or = 0;
}

// merge kernels: blockIdx.y = the rank whose records a block walks, up to their count
__global__ void k_sl_unite(SlabDev s, const int32_t* __restrict__ mbufs)
{
    pdl_begin();
    const int r = blockIdx.y;
    const int32_t* mb = mbuf_of(s, mbufs, r);
    const int nl = min(mb[0], s.g.cap_merge);
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nl; j += gridDim.x * blockDim.x) {
        const int2 e = mlink(s, mb, j);
        AM_CHECK(e.x >= 0 && e.x < s.g.n_total && e.y >= 0 && e.y < s.g.n_total);
        s.touched[e.x] = 1;
        s.touched[e.y] = 1;
        if (e.x != e.y) uf_unite(s.forest, (uint32_t)e.x, (uint32_t)e.y);
    }
}

__global__ void k_sl_cbad(SlabDev s, const int32_t* __restrict__ mbufs, long long* stats)
{
    pdl_begin();
    if (stats && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) stats_reset(s, stats);   // for k_sl_final
    const int r = blockIdx.y;
    const int32_t* mb = mbuf_of(s, mbufs, r);
    const int nc = min(mb[1], s.g.cap_merge);
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nc; j += gridDim.x * blockDim.x) {
        const int4 c = mcluster(s, mb, j);
        const uint32_t f = uf_find(s.forest, (uint32_t)c.x);
        if (c.y) s.badm[f] = 1;
        const unsigned long long md = (unsigned long long)(uint32_t)c.z | ((unsigned long long)(uint32_t)c.w << 32);
        if (md) atomicMax((unsigned long long*)(s.maxdm + f), md);
    }
}

__global__ void k_sl_stats_init(SlabDev s, long long* stats)
{
    pdl_begin();
    if (threadIdx.x == 0) stats_reset(s, stats);
}

// final outputs of the owned agents: global label, ready bit, dispatch (status, completion
// time, priority key), then this rank's next event, W, S and activity
__global__ void __launch_bounds__(256) k_sl_final(SlabDev s, long long* stats)
{
    pdl_begin();
    const long long t = s.counters[0];
    const int W = s.tctl->W;
    const int idb = s.idb;
    const int lagbits = 64 - 2 * idb;
    long long tmin = kNever, wmin = kNever, nsmin = kNever;
    int act = 0;
    unsigned long long kor = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < s.L; i += gridDim.x * blockDim.x) {
        uint8_t st = s.stat[i];
        const bool own = st != ST_DONE && s.own[i];
        int lab = -1;
        bool rdy = false;
        if (own) {
            const int l = s.labels[i];
            const int L = s.mingid[l];
            long long md;
            bool bad;
            int F;
            if (s.touched[L]) {
                F = (int)uf_find(s.forest, (uint32_t)L);
                bad = s.badm[F] != 0;
                md = s.maxdm[F];
            } else {
                F = L;
                bad = s.badl[l] != 0;
                md = s.maxd[l];
            }
            lab = F;
            rdy = st == ST_IDLE && !bad;
            const int stp = s.step[i];
            if (rdy) {
                // dispatch (Alg. 3 l.9-10): completion = t + the cluster's max duration
                st = ST_RUNNING;
                s.stat[i] = ST_RUNNING;
                s.tc[i] = t + md;
                const int k = atomicAdd(&s.sctl->n_ready, 1);
                s.rlist[k] = i;
                const unsigned long long lag = (unsigned long long)(uint32_t)(stp - W);
                if (lagbits < 64 && (lag >> lagbits)) atomicOr(s.flags, AM_SLAB_LAG);
                const unsigned long long key = (lag << (2 * idb)) | ((unsigned long long)F << idb) |
                                               (unsigned long long)s.gid[i];
                s.rkey[0][k] = key;
                s.rval[0][k] = (uint32_t)s.gid[i];
                kor |= key;
            }
            act = 1;
            wmin = min(wmin, (long long)stp);
            nsmin = min(nsmin, -(long long)stp);
            if (st == ST_RUNNING) tmin = min(tmin, s.tc[i]);
        }
        s.glabel[i] = lab;
        s.ready[i] = rdy;
    }
    // block reduction, one atomic per quantity per block
    __shared__ long long r_t[8], r_w[8], r_s[8];
    __shared__ int r_a[8];
    __shared__ unsigned long long r_o[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) {
        tmin = min(tmin, __shfl_xor_sync(0xFFFFFFFFu, tmin, o));
        wmin = min(wmin, __shfl_xor_sync(0xFFFFFFFFu, wmin, o));
        nsmin = min(nsmin, __shfl_xor_sync(0xFFFFFFFFu, nsmin, o));
        kor |= __shfl_xor_sync(0xFFFFFFFFu, kor, o);
    }
    act = __reduce_or_sync(0xFFFFFFFFu, (unsigned)act);
    if (lane == 0) { r_t[w] = tmin; r_w[w] = wmin; r_s[w] = nsmin; r_a[w] = act; r_o[w] = kor; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < 8; q++) {
            tmin = min(tmin, r_t[q]); wmin = min(wmin, r_w[q]); nsmin = min(nsmin, r_s[q]);
            act |= r_a[q]; kor |= r_o[q];
        }
        if (tmin != kNever) atomicMin((long long*)stats, tmin);
        if (wmin != kNever) atomicMin((long long*)stats + 1, wmin);
        if (nsmin != kNever) atomicMin((long long*)stats + 2, nsmin);
        if (act) atomicMin((long long*)stats + 3, 0ll);
        if (kor) atomicOr(&s.sctl->sort_or, kor);
    }
}

// the forest, bad, duration and touched marks back to their neutral values
__global__ void k_sl_restore(SlabDev s, const int32_t* __restrict__ mbufs)
{
    pdl_begin();
    const int r = blockIdx.y, cap = s.g.cap_merge;
    const int32_t* mb = mbuf_of(s, mbufs, r);
    const int nmax = max(min(mb[0], cap), min(mb[1], cap));
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nmax; j += gridDim.x * blockDim.x) {
        if (j < min(mb[0], cap)) {
            const int2 e = mlink(s, mb, j);
            s.forest[e.x] = (uint32_t)e.x; s.forest[e.y] = (uint32_t)e.y;
            s.touched[e.x] = 0; s.touched[e.y] = 0;
            s.badm[e.x] = 0; s.badm[e.y] = 0;
            s.maxdm[e.x] = 0; s.maxdm[e.y] = 0;
        }
        if (j < min(mb[1], cap)) {
            const int c = mcluster(s, mb, j).x;
            s.forest[c] = (uint32_t)c;
            s.touched[c] = 0;
            s.badm[c] = 0;
            s.maxdm[c] = 0;
        }
    }
}

// moves of the dispatched agents from their perception digests (Alg. 2 "perceive"; all
// perceived agents are in the window)
__global__ void k_sl_moves(SlabDev s, int32_t* n_order)
{
    pdl_begin();
    const int nr = s.sctl->n_ready;
    if (blockIdx.x == 0 && threadIdx.x == 0) *n_order = nr;   // the order's length
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nr; k += gridDim.x * blockDim.x) {
        const int i = s.rlist[k];
        s.np[i] = policy_move_g(s.sy, s.g.map_w, s.g.map_h, s.gid[i], s.step[i], s.pos[i], s.dig[i]);
        if (k == 0) atomicAdd((unsigned long long*)(s.counters + 2), (unsigned long long)nr);
    }
}

// ------------------------------------------------------------------ commit
// the common clock: the global next event rounded up to the quantum; round count,
// liveness, the halo check (the spread grows by at most one step per round)
__device__ __forceinline__ int32_t* dblock(const SlabDev& s, int32_t* d, int r)
{
    return d + (size_t)r * (size_t)AM_SLAB_DELTA_WORDS(s.g.cap_peer);
}
__device__ __forceinline__ const int32_t* dblock(const SlabDev& s, const int32_t* d, int r)
{
    return d + (size_t)r * (size_t)AM_SLAB_DELTA_WORDS(s.g.cap_peer);
}

// (after a stale round nothing may be pending: the clock stays, the rounds up to the next
// sync round may be idle; only a sync round with nothing pending is a liveness failure)
// owned RUNNING agents whose cluster completed commit their move (worker l.20-21,
// controller l.11-12); they stay owned (IDLE, or DONE at the target) until the next
// exchange, which sends them to every rank whose window they were or are in
// The common clock first (every block computes it from the all-reduced stats; block 0
// records it with the round count, liveness and the halo check): the global next event
// rounded up to the quantum.
__global__ void k_sl_commit(SlabDev s, const long long* __restrict__ gstats, int32_t* dsend, int stale)
{
    pdl_begin();
    const long long tn = gstats[0];
    const bool active = gstats[3] == 0;
    long long t = s.counters[0];
    if (active && tn != kNever) t = s.Q > 0 ? ((tn + s.Q - 1) / s.Q) * s.Q : tn;
    if (blockIdx.x == 0) {
        if (dsend)
            for (int r = threadIdx.x; r < s.g.n_slabs; r += blockDim.x)
                for (int q = 0; q < 6; q++) dblock(s, dsend, r)[q] = 0;   // counts (headers)
        if (threadIdx.x == 0 && active) {
            s.counters[3] += 1;
            if (tn == kNever) {
                if (!stale) atomicOr(s.flags, AM_SLAB_LIVENESS);
            } else {
                s.counters[0] = t;
            }
            // the owned agents drift up to P v outside the slab between exchanges, and the
            // ghosts' snapshot is up to P rounds old: 2 P v more rows
            const long long spread = -gstats[2] - gstats[1] + 1;
            const long long need = (spread + 1) * s.g.v_max + s.g.r_p +
                                   (long long)(s.g.check_rounds + 1) * s.g.v_max +
                                   (s.P > 1 ? 2LL * s.P * s.g.v_max : 0LL);
            if (need > s.g.halo) atomicOr(s.flags, AM_SLAB_HALO);
        }
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < s.L; i += gridDim.x * blockDim.x) {
        if (s.stat[i] != ST_RUNNING || !s.own[i] || s.tc[i] > t) continue;   // ghosts are committed by their owner
        const int2 np = s.np[i];
        const int stp = s.step[i] + 1;
        s.pos[i] = np;
        s.step[i] = stp;
        s.traj[i] = traj_step(s.traj[i], stp, np.x, np.y);
        s.tc[i] = kNever;
        const bool done = s.g.target_step > 0 && stp == s.g.target_step;
        if (done) atomicMax((unsigned long long*)(s.counters + 1), (unsigned long long)t);
        s.stat[i] = done ? ST_DONE : ST_IDLE;
        s.dirty[i] = 1;
    }
}

// the exchange's send side: every owned agent that committed since the last exchange, to
// every other rank whose window holds its row then or now -- its whole state (a RUNNING
// agent changing owner carries its completion time and move) -- and ownership follows
// the row: an agent that left the slab becomes a ghost here
__global__ void k_sl_flush(SlabDev s, int32_t* __restrict__ dsend)
{
    pdl_begin();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < s.L; i += gridDim.x * blockDim.x) {
        if (!s.dirty[i]) continue;
        s.dirty[i] = 0;
        const int2 p = s.pos[i];
        const int y_old = s.ly[i];
        const uint8_t st = s.stat[i];
        const unsigned long long th = s.traj[i];
        const long long tc = s.tc[i];
        const int2 np = s.np[i];
        for (int j = 0; j < s.g.n_slabs; j++) {
            if (j == s.g.my_slab) continue;
            if (!in_window_of(s, j, y_old) && !in_window_of(s, j, p.y)) continue;
            int32_t* blk = dblock(s, dsend, j);
            const int k = atomicAdd(blk, 1);
            if (k < s.g.cap_peer) {
                int32_t* r = blk + 6 + (size_t)k * kDeltaRec;
                r[0] = s.gid[i]; r[1] = p.x; r[2] = p.y; r[3] = s.step[i];
                r[4] = (int32_t)(uint32_t)th; r[5] = (int32_t)(uint32_t)(th >> 32);
                r[6] = st; r[7] = (int32_t)(uint32_t)tc; r[8] = (int32_t)(uint32_t)((unsigned long long)tc >> 32);
                r[9] = np.x; r[10] = np.y; r[11] = 0;
            } else {
                atomicOr(s.flags, AM_SLAB_OVF_PEER);
            }
        }
        s.ly[i] = p.y;
        if (!in_slab(s, p.y)) {
            s.own[i] = 0;
            s.stat[i] = st == ST_DONE ? ST_DONE : ST_RUNNING;
            s.tc[i] = kNever;
        }
    }
}

// ------------------------------------------------------------------ apply
// departures first (their slots return to the free stack) ...
__global__ void k_sl_depart(SlabDev s, const int32_t* __restrict__ drecv)
{
    pdl_begin();
    const int r = blockIdx.y;   // the sender
    if (r == s.g.my_slab) return;
    const int32_t* blk = dblock(s, drecv, r);
    const int nd = min(blk[0], s.g.cap_peer);
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nd; j += gridDim.x * blockDim.x) {
        const int32_t* d = blk + 6 + (size_t)j * kDeltaRec;
        const int g = d[0], y = d[2];
        AM_CHECK(g >= 0 && g < s.g.n_total);
        const int i = s.map[g];
        AM_CHECK(i < s.L);
        if (i < 0 || in_window(s, y)) continue;
        s.map[g] = -1;
        s.gid[i] = -1;
        s.stat[i] = ST_DONE;
        s.own[i] = 0;
        s.pos[i] = make_int2(0, s.y0);
        const int f = atomicAdd(s.ftop, 1);
        AM_CHECK(f >= 0 && f < s.L);
        s.fstack[f] = i;
    }
}

// ... then moved agents and arrivals (a free slot each)
__global__ void k_sl_arrive(SlabDev s, const int32_t* __restrict__ drecv)
{
    pdl_begin();
    const int r = blockIdx.y;   // the sender
    if (r == s.g.my_slab) return;
    const int32_t* blk = dblock(s, drecv, r);
    const int nd = min(blk[0], s.g.cap_peer);
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nd; j += gridDim.x * blockDim.x) {
        const int32_t* d = blk + 6 + (size_t)j * kDeltaRec;
        const int g = d[0], x = d[1], y = d[2], stp = d[3];
        AM_CHECK(g >= 0 && g < s.g.n_total);
        if (!in_window(s, y)) continue;
        int i = s.map[g];
        AM_CHECK(i < s.L);
        if (i < 0) {   // arrival
            const int f = atomicSub(s.ftop, 1) - 1;
            if (f < 0) {
                atomicAdd(s.ftop, 1);
                atomicOr(s.flags, AM_SLAB_OVF_WINDOW);
                continue;
            }
            i = s.fstack[f];
            AM_CHECK(i >= 0 && i < s.L);
            s.map[g] = i;
            s.gid[i] = g;
            s.tc[i] = kNever;
        }
        s.pos[i] = make_int2(x, y);
        s.step[i] = stp;
        s.traj[i] = (unsigned long long)(uint32_t)d[4] | ((unsigned long long)(uint32_t)d[5] << 32);
        s.ly[i] = y;
        s.dirty[i] = 0;
        // mine if it is in my slab now: the owner's status (IDLE, DONE, or RUNNING with its
        // completion time and move); else a ghost
        const uint8_t st = (uint8_t)d[6];
        const bool own = in_slab(s, y);
        s.own[i] = own;
        s.stat[i] = st == ST_DONE ? ST_DONE : (own ? st : ST_RUNNING);
        s.tc[i] = own && st == ST_RUNNING ? (long long)((unsigned long long)(uint32_t)d[7] |
                                                        ((unsigned long long)(uint32_t)d[8] << 32))
                                          : kNever;
        s.np[i] = own && st == ST_RUNNING ? make_int2(d[9], d[10]) : make_int2(x, y);
    }
}

}  // namespace am

using namespace am;

struct am_slab {
    SlabDev s{};
    am_ctx* tr = nullptr;
    cudaStream_t stream = nullptr;
    void* mem = nullptr;
    bool mem_owned = false;
    int32_t* h_flags = nullptr;   // pinned
    uint8_t* tmask = nullptr;     // the tracker's am_ready outputs (PEEK; unused)
    int32_t* torder = nullptr;
    Dev sd{};                     // the order sort's view (keys, ids, control block)
    int32_t* order = nullptr;
    int num_sms = 148;
    bool last_stale = false;      // the last round was a stale round
    // the rank's priority sort runs on a side stream beside commit / exchange / apply;
    // the slab's stream joins it before the next round rewrites its inputs
    cudaStream_t side = nullptr, side2 = nullptr;   // the sort; the merge forest's restore
    cudaEvent_t ev_fork = nullptr, ev_s0 = nullptr, ev_s1 = nullptr, ev_r1 = nullptr;
    bool order_pending = false, order_timed = false, restore_pending = false, last_restore = false;
};

// the slab's stream waits for the last priority sort (an event wait, no host sync)
static void slab_join(am_slab* sl)
{
    if (sl && sl->order_pending) {
        cudaStreamWaitEvent(sl->stream, sl->ev_s1, 0);
        sl->order_pending = false;
    }
    if (sl && sl->restore_pending) {
        cudaStreamWaitEvent(sl->stream, sl->ev_r1, 0);
        sl->restore_pending = false;
    }
}

namespace {
struct SlabLayout {
    size_t total = 0, tracker = 0, trk_bytes = 0;
    size_t gid, pos, tpos, step, stat, own, dirty, ly, traj, tc, np, dig, map, fstack, ftop, mingid, csize, badl, bndl,
        maxd;
    size_t forest, badm, touched, maxdm, glabel, ready, rlist, sctl, rk0, rk1, rv0, rv1, counters, flags, tmask,
        torder, order;
};

int window_rows(const am_slab_geom& g, int& lo, int& hi, int& y0, int& y1)
{
    lo = (int)((long long)g.my_slab * g.map_h / g.n_slabs);
    hi = (int)((long long)(g.my_slab + 1) * g.map_h / g.n_slabs);
    y0 = std::max(0, lo - g.halo);
    y1 = (int)std::min<long long>(g.map_h, (long long)hi + g.halo);
    // the window's tracker packs window rows in 16 bits (one tracker map <= 32768 rows)
    return y1 > y0 && y1 - y0 <= 32768 ? AM_OK : AM_E_ARG;
}

am_config tracker_cfg(const am_slab_geom& g)
{
    am_config c{};
    c.target_step = g.target_step;
    c.n_sims = 1;
    c.cell = 0;
    c.metric = g.metric;
    // mode-3 replica updates ignore AM_VALIDATE (it keeps the incremental round on)
    c.flags = AM_VALIDATE | AM_PEEK | AM_ASYNC | AM_FORCE_BINNED | AM_NO_ORDER | AM_LABELS_ONLY;
    return c;
}

bool geom_ok(const am_slab_geom* g)
{
    return g && g->n_slabs >= 1 && g->my_slab >= 0 && g->my_slab < g->n_slabs && g->n_total > 0 &&
           g->n_total < (1 << 28) && g->target_step > 0 && g->halo >= g->r_p + 2 * g->v_max && g->cap_window > 0 &&
           g->cap_peer > 0 && g->cap_merge > 0 && (g->cap_merge % 2) == 0 && g->map_w >= 1 && g->map_h >= 1 && g->map_w <= 32768 &&
           g->map_h <= (1 << 30) &&   // each window's height is checked by its tracker (<= 32768) g->check_rounds >= 1 && g->n_slabs <= 1024 && g->stale_rounds >= 0 &&
           g->halo >= g->r_p + (std::max(1, g->stale_rounds) + 1) * g->v_max;
}

SlabLayout slab_layout(const am_slab_geom& g)
{
    SlabLayout Ly;
    int lo, hi, y0, y1;
    window_rows(g, lo, hi, y0, y1);
    const size_t L = (size_t)g.cap_window, N = (size_t)g.n_total;
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += (b + 255) & ~size_t(255); return o; };
    am_config c = tracker_cfg(g);
    Ly.trk_bytes = am_workspace_size(g.map_w, std::max(1, y1 - y0), g.r_p, g.v_max, (int32_t)L, &c);
    Ly.tracker = take(Ly.trk_bytes);
    Ly.gid = take(4 * L); Ly.pos = take(8 * L); Ly.tpos = take(8 * L); Ly.step = take(4 * L); Ly.stat = take(L);
    Ly.own = take(L); Ly.dirty = take(L); Ly.ly = take(4 * L);
    Ly.traj = take(8 * L); Ly.tc = take(8 * L); Ly.np = take(8 * L); Ly.dig = take(8 * L);
    Ly.map = take(4 * N); Ly.fstack = take(4 * L); Ly.ftop = take(4);
    Ly.mingid = take(4 * L); Ly.csize = take(4 * L); Ly.badl = take(L); Ly.bndl = take(L); Ly.maxd = take(8 * L);
    Ly.forest = take(4 * N); Ly.badm = take(N); Ly.touched = take(N); Ly.maxdm = take(8 * N);
    Ly.glabel = take(4 * L); Ly.ready = take(L); Ly.rlist = take(4 * L); Ly.sctl = take(sizeof(Ctl));
    Ly.rk0 = take(8 * L); Ly.rk1 = take(8 * L); Ly.rv0 = take(4 * L); Ly.rv1 = take(4 * L);
    Ly.counters = take(8 * 4); Ly.flags = take(4); Ly.tmask = take(L); Ly.torder = take(4 * L); Ly.order = take(4 * L);
    Ly.total = off;
    return Ly;
}

int ck(am_slab* sl, cudaError_t e, const char* where)
{
    if (e == cudaSuccess) return AM_OK;
    fprintf(stderr, "am_slab: %s: %s\n", where, cudaGetErrorString(e));
    (void)sl;
    return AM_E_CUDA;
}
#define SK(call)                                           \
    do {                                                   \
        const int r_ = ck(sl, (call), #call);              \
        if (r_) return r_;                                 \
    } while (0)

unsigned grid_for(const am_slab* sl, long long n, int per = 256)
{
    return (unsigned)std::max(1LL, std::min((n + per - 1) / per, (long long)sl->num_sms * 8));
}
}  // namespace

extern "C" size_t am_slab_workspace_size(const am_slab_geom* g)
{
    if (!geom_ok(g)) return 0;
    int lo, hi, y0, y1;
    if (window_rows(*g, lo, hi, y0, y1) != AM_OK) return 0;
    return slab_layout(*g).total;
}

extern "C" int am_slab_create(am_slab** out, const am_slab_geom* g, const am_synth* synth, int64_t quantum_us,
                              void* workspace, size_t workspace_bytes, void* stream)
{
    if (!out || !geom_ok(g) || !synth) return AM_E_ARG;
    *out = nullptr;
    int lo, hi, y0, y1;
    if (window_rows(*g, lo, hi, y0, y1) != AM_OK) return AM_E_ARG;
    const SlabLayout Ly = slab_layout(*g);
    if (workspace && (workspace_bytes < Ly.total || ((uintptr_t)workspace & 255))) return AM_E_WORKSPACE;
    am_slab* sl = new (std::nothrow) am_slab();
    if (!sl) return AM_E_ARG;
    sl->stream = (cudaStream_t)stream;
    if (workspace) {
        sl->mem = workspace;
    } else {
        if (cudaMalloc(&sl->mem, Ly.total) != cudaSuccess) { delete sl; return AM_E_CUDA; }
        sl->mem_owned = true;
    }
    {
        int dev = 0, sms = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        sl->num_sms = sms > 0 ? sms : 148;
    }
    char* b = (char*)sl->mem;
    // the window's tracker, its workspace inside ours
    am_config c = tracker_cfg(*g);
    c.stream = stream;
    c.workspace = b + Ly.tracker;
    c.workspace_bytes = Ly.trk_bytes;
    int rc = am_init(&sl->tr, g->map_w, y1 - y0, g->r_p, g->v_max, g->cap_window, &c);
    if (rc != AM_OK) {
        if (sl->mem_owned) cudaFree(sl->mem);
        delete sl;
        return rc;
    }
    SlabDev& s = sl->s;
    s.g = *g;
    s.sy = *synth;
    s.Q = quantum_us;
    s.lo = lo; s.hi = hi; s.y0 = y0; s.y1 = y1;
    s.L = g->cap_window;
    s.P = std::max(1, g->stale_rounds);
    {
        int idb = 1;
        while ((1LL << idb) < (long long)g->n_total) idb++;
        s.idb = idb;
    }
    s.gid = (int32_t*)(b + Ly.gid); s.pos = (int2*)(b + Ly.pos); s.tpos = (int2*)(b + Ly.tpos);
    s.step = (int32_t*)(b + Ly.step); s.stat = (uint8_t*)(b + Ly.stat);
    s.own = (uint8_t*)(b + Ly.own); s.dirty = (uint8_t*)(b + Ly.dirty); s.ly = (int32_t*)(b + Ly.ly);
    s.traj = (unsigned long long*)(b + Ly.traj); s.tc = (long long*)(b + Ly.tc); s.np = (int2*)(b + Ly.np);
    s.dig = (unsigned long long*)(b + Ly.dig);
    s.map = (int32_t*)(b + Ly.map); s.fstack = (int32_t*)(b + Ly.fstack); s.ftop = (int32_t*)(b + Ly.ftop);
    s.mingid = (int32_t*)(b + Ly.mingid); s.csize = (int32_t*)(b + Ly.csize); s.badl = (uint8_t*)(b + Ly.badl);
    s.bndl = (uint8_t*)(b + Ly.bndl); s.maxd = (long long*)(b + Ly.maxd);
    s.forest = (uint32_t*)(b + Ly.forest); s.badm = (uint8_t*)(b + Ly.badm); s.touched = (uint8_t*)(b + Ly.touched);
    s.maxdm = (long long*)(b + Ly.maxdm);
    s.glabel = (int32_t*)(b + Ly.glabel); s.ready = (uint8_t*)(b + Ly.ready); s.rlist = (int32_t*)(b + Ly.rlist);
    s.sctl = (Ctl*)(b + Ly.sctl);
    s.rkey[0] = (unsigned long long*)(b + Ly.rk0); s.rkey[1] = (unsigned long long*)(b + Ly.rk1);
    s.rval[0] = (uint32_t*)(b + Ly.rv0); s.rval[1] = (uint32_t*)(b + Ly.rv1);
    s.counters = (long long*)(b + Ly.counters); s.flags = (int32_t*)(b + Ly.flags);
    sl->tmask = (uint8_t*)(b + Ly.tmask); sl->torder = (int32_t*)(b + Ly.torder); sl->order = (int32_t*)(b + Ly.order);
    s.labels = sl->tr->d.labels;
    s.blocked = sl->tr->d.blkid;
    s.tctl = sl->tr->d.ctl;
    // the order sort's view
    sl->sd = sl->tr->d;
    sl->sd.ctl = s.sctl;
    sl->sd.rkey[0] = s.rkey[0]; sl->sd.rkey[1] = s.rkey[1];
    sl->sd.rval[0] = s.rval[0]; sl->sd.rval[1] = s.rval[1];
    cudaStream_t st = sl->stream;
    rc = AM_OK;
    // everything zero except the global-id map (-1) and the forest (identity)
    if (!rc) rc = ck(sl, cudaMemsetAsync(b + Ly.gid, 0, Ly.total - Ly.gid, st), "memset");
    if (!rc) rc = ck(sl, cudaMemsetAsync(s.map, 0xFF, 4 * (size_t)g->n_total, st), "memset map");
    if (!rc) rc = ck(sl, cudaMallocHost((void**)&sl->h_flags, 16), "cudaMallocHost");
    if (!rc) rc = ck(sl, cudaStreamCreateWithFlags(&sl->side, cudaStreamNonBlocking), "side stream");
    if (!rc) rc = ck(sl, cudaEventCreateWithFlags(&sl->ev_fork, cudaEventDisableTiming), "event");
    if (!rc) rc = ck(sl, cudaEventCreate(&sl->ev_s0), "event");
    if (!rc) rc = ck(sl, cudaEventCreate(&sl->ev_s1), "event");
    if (!rc) rc = ck(sl, cudaStreamCreateWithFlags(&sl->side2, cudaStreamNonBlocking), "side stream");
    if (!rc) rc = ck(sl, cudaEventCreate(&sl->ev_r1), "event");
    if (rc) { am_slab_destroy(sl); return rc; }
    // forest = identity: a tiny kernel-free init through the sort's control block is not
    // available, so fill from the host once (n_total words)
    {
        uint32_t* h = (uint32_t*)malloc(4 * (size_t)g->n_total);
        for (int32_t k = 0; k < g->n_total; k++) h[k] = (uint32_t)k;
        rc = ck(sl, cudaMemcpyAsync(s.forest, h, 4 * (size_t)g->n_total, cudaMemcpyHostToDevice, st), "forest");
        if (!rc) rc = ck(sl, cudaStreamSynchronize(st), "sync");
        free(h);
        if (rc) { am_slab_destroy(sl); return rc; }
    }
    *out = sl;
    return AM_OK;
}

extern "C" int am_slab_load(am_slab* sl, int32_t m, const int32_t* gid, const int32_t* pos, const int32_t* steps,
                            const uint8_t* status, const uint64_t* traj, const int64_t* tcommit, const int32_t* newpos,
                            int64_t t)
{
    if (!sl || m < 0 || m > sl->s.L || (m && (!gid || !pos || !steps || !status))) return AM_E_ARG;
    slab_join(sl);
    SK(cudaMemsetAsync(sl->s.map, 0xFF, 4 * (size_t)sl->s.g.n_total, sl->stream));
    SK(launch_k(false, sl->stream, k_sl_load, grid_for(sl, sl->s.L), 256, 0, sl->s, m, gid, (const int2*)pos, steps, status,
                                                             (const unsigned long long*)traj, (const long long*)tcommit,
                                                             (const int2*)newpos, (long long)t));
    SK(cudaGetLastError());
    am_reset(sl->tr);   // the next round recomputes the window from scratch
    return AM_OK;
}

extern "C" int am_slab_round_local(am_slab* sl, int32_t* mbuf)
{
    if (!sl || !mbuf) return AM_E_ARG;
    slab_join(sl);   // the last round's priority sort read the buffers this round rewrites
    SlabDev& s = sl->s;
    const unsigned gr = grid_for(sl, s.L);
    SK(launch_k(sl->tr->pdl, sl->stream, k_sl_prep, gr, 256, 0, s, mbuf));
    SK(cudaGetLastError());
    int rc = am_update_replica(sl->tr, (const int32_t*)s.tpos, s.step, s.stat);
    if (rc) return rc;
    rc = am_ready(sl->tr, sl->tmask, sl->torder, nullptr);   // AM_PEEK | AM_ASYNC
    if (rc) return rc;
    SK(launch_k(sl->tr->pdl, sl->stream, k_sl_clusters, gr, 256, 0, s, 0));
    SK(launch_k(sl->tr->pdl, sl->stream, k_sl_records, gr, 256, 0, s, mbuf));
    SK(cudaGetLastError());
    sl->last_stale = false;
    return AM_OK;
}

// the dispatch of the ready agents of a round (local clusters, or merged through the
// records of `mbufs`): ready bits, dispatch, digests, moves, the rank's order
static int slab_finish(am_slab* sl, const int32_t* mbufs, int32_t* order_out, int32_t* n_order, int64_t* stats);

extern "C" int am_slab_round_stale(am_slab* sl, int32_t* order_out, int32_t* n_order, int64_t* stats)
{
    if (!sl || !order_out || !n_order || !stats) return AM_E_ARG;
    slab_join(sl);   // the last round's priority sort read the buffers this round rewrites
    SlabDev& s = sl->s;
    const unsigned gr = grid_for(sl, s.L);
    SK(launch_k(sl->tr->pdl, sl->stream, k_sl_prep, gr, 256, 0, s, nullptr));
    SK(cudaGetLastError());
    int rc = am_update_replica(sl->tr, (const int32_t*)s.tpos, s.step, s.stat);
    if (rc) return rc;
    rc = am_ready(sl->tr, sl->tmask, sl->torder, nullptr);   // AM_PEEK | AM_ASYNC
    if (rc) return rc;
    SK(launch_k(sl->tr->pdl, sl->stream, k_sl_clusters, gr, 256, 0, s, 1));
    SK(cudaGetLastError());
    sl->last_stale = true;
    return slab_finish(sl, nullptr, order_out, n_order, stats);
}


extern "C" int am_slab_merge(am_slab* sl, const int32_t* mbufs, int32_t* order_out, int32_t* n_order, int64_t* stats)
{
    if (!sl || !mbufs || !order_out || !n_order || !stats) return AM_E_ARG;
    return slab_finish(sl, mbufs, order_out, n_order, stats);
}

static int slab_finish(am_slab* sl, const int32_t* mbufs, int32_t* order_out, int32_t* n_order, int64_t* stats)
{
    SlabDev& s = sl->s;
    // one row of blocks per rank's records (each walks its rank's records up to their count)
    const dim3 gm(std::max(1u, std::min((unsigned)((s.g.cap_merge + 255) / 256), (unsigned)(sl->num_sms * 8) /
                                                                                   (unsigned)s.g.n_slabs)),
                  (unsigned)s.g.n_slabs);
    const unsigned gr = grid_for(sl, s.L);
    if (mbufs) {
        SK(launch_k(sl->tr->pdl, sl->stream, k_sl_unite, gm, 256, 0, s, mbufs));
        SK(launch_k(sl->tr->pdl, sl->stream, k_sl_cbad, gm, 256, 0, s, mbufs, (long long*)stats));
    } else {
        SK(launch_k(sl->tr->pdl, sl->stream, k_sl_stats_init, 1, 32, 0, s, (long long*)stats));
    }
    SK(launch_k(sl->tr->pdl, sl->stream, k_sl_final, gr, 256, 0, s, (long long*)stats));
    SK(cudaGetLastError());
    // perception digests of the dispatched agents (global ids in the terms), their moves
    int rc = am_internal_digest(sl->tr, s.rlist, &s.sctl->n_ready, s.gid, s.dig, s.L, sl->stream);
    if (rc) return rc;
    SK(launch_k(sl->tr->pdl, sl->stream, k_sl_moves, gr, 256, 0, s, n_order));
    SK(cudaGetLastError());
    // on the side stream (nothing in commit / apply reads them; the next round joins it
    // first): the merge forest's restore (reads mbufs: they stay untouched until then)
    // and the rank's priority order -- unique keys (lag, global label, id) -> global ids
    // (two side streams: the restore and the sort touch disjoint buffers and run together)
    SK(cudaEventRecord(sl->ev_fork, sl->stream));
    SK(cudaStreamWaitEvent(sl->side, sl->ev_fork, 0));
    SK(cudaEventRecord(sl->ev_s0, sl->side));
    if (mbufs) {
        SK(cudaStreamWaitEvent(sl->side2, sl->ev_fork, 0));
        SK(launch_k(false, sl->side2, k_sl_restore, gm, 256, 0, s, mbufs));
        SK(cudaEventRecord(sl->ev_r1, sl->side2));
        sl->restore_pending = true;
    }
    sl->last_restore = mbufs != nullptr;
    rc = am_internal_csort(sl->tr, sl->sd, order_out, sl->side);
    if (rc) return rc;
    SK(cudaEventRecord(sl->ev_s1, sl->side));
    sl->order_pending = true;
    sl->order_timed = true;
    return AM_OK;
}

extern "C" int am_slab_wait_order(am_slab* sl)
{
    if (!sl) return AM_E_ARG;
    slab_join(sl);
    return AM_OK;
}

extern "C" int am_slab_order_ms(am_slab* sl, float* ms)
{
    if (!sl || !ms) return AM_E_ARG;
    if (!sl->order_timed) return AM_E_STATE;
    SK(cudaEventSynchronize(sl->ev_s1));
    SK(cudaEventElapsedTime(ms, sl->ev_s0, sl->ev_s1));
    if (sl->last_restore) {   // the restore beside it (same start): the longer of the two
        float mr = 0.0f;
        if (cudaEventSynchronize(sl->ev_r1) == cudaSuccess && cudaEventElapsedTime(&mr, sl->ev_s0, sl->ev_r1) == cudaSuccess)
            *ms = std::max(*ms, mr);
        cudaGetLastError();
    }
    return AM_OK;
}

extern "C" int am_slab_commit(am_slab* sl, const int64_t* stats_global, int32_t* dsend)
{
    if (!sl || !stats_global) return AM_E_ARG;
    SlabDev& s = sl->s;
    SK(launch_k(sl->tr->pdl, sl->stream, k_sl_commit, grid_for(sl, s.L), 256, 0, s, (const long long*)stats_global,
                dsend, sl->last_stale ? 1 : 0));
    if (dsend) SK(launch_k(sl->tr->pdl, sl->stream, k_sl_flush, grid_for(sl, s.L), 256, 0, s, dsend));
    SK(cudaGetLastError());
    return AM_OK;
}

extern "C" int am_slab_apply(am_slab* sl, const int32_t* drecv)
{
    if (!sl || !drecv) return AM_E_ARG;
    SlabDev& s = sl->s;
    const dim3 g(std::max(1u, std::min((unsigned)((s.g.cap_peer + 255) / 256), (unsigned)(sl->num_sms * 4) /
                                                                               (unsigned)s.g.n_slabs)),
                 (unsigned)s.g.n_slabs);
    SK(launch_k(sl->tr->pdl, sl->stream, k_sl_depart, g, 256, 0, s, drecv));
    SK(launch_k(sl->tr->pdl, sl->stream, k_sl_arrive, g, 256, 0, s, drecv));
    SK(cudaGetLastError());
    return AM_OK;
}

extern "C" int am_slab_outputs(am_slab* sl, const int32_t** slot_gid, const int32_t** slot_label,
                               const uint8_t** slot_ready)
{
    if (!sl) return AM_E_ARG;
    if (slot_gid) *slot_gid = sl->s.gid;
    if (slot_label) *slot_label = sl->s.glabel;
    if (slot_ready) *slot_ready = sl->s.ready;
    return AM_OK;
}

extern "C" int am_slab_state(am_slab* sl, const int32_t** pos, const int32_t** steps, const uint8_t** status,
                             const uint64_t** traj, const int64_t** tcommit, const int32_t** newpos,
                             const int64_t** counters)
{
    if (!sl) return AM_E_ARG;
    if (pos) *pos = (const int32_t*)sl->s.pos;
    if (steps) *steps = sl->s.step;
    if (status) *status = sl->s.stat;
    if (traj) *traj = (const uint64_t*)sl->s.traj;
    if (tcommit) *tcommit = (const int64_t*)sl->s.tc;
    if (newpos) *newpos = (const int32_t*)sl->s.np;
    if (counters) *counters = (const int64_t*)sl->s.counters;
    return AM_OK;
}

extern "C" int am_slab_flags(am_slab* sl, int32_t* flags, int32_t* window_used)
{
    if (!sl) return AM_E_ARG;
    SK(cudaMemcpyAsync(sl->h_flags, sl->s.flags, 4, cudaMemcpyDeviceToHost, sl->stream));
    SK(cudaMemcpyAsync(sl->h_flags + 1, sl->s.ftop, 4, cudaMemcpyDeviceToHost, sl->stream));
    SK(cudaMemsetAsync(sl->s.flags, 0, 4, sl->stream));
    SK(cudaStreamSynchronize(sl->stream));
    if (flags) *flags = sl->h_flags[0];
    if (window_used) *window_used = sl->s.L - sl->h_flags[1];
    const int rc = am_sync(sl->tr);   // the window tracker's pending errors
    return rc;
}

extern "C" int am_slab_owned(am_slab* sl, const uint8_t** own)
{
    if (!sl || !own) return AM_E_ARG;
    *own = sl->s.own;
    return AM_OK;
}

extern "C" am_ctx* am_slab_tracker(am_slab* sl) { return sl ? sl->tr : nullptr; }
extern "C" void* am_slab_stream(am_slab* sl) { return sl ? (void*)sl->stream : nullptr; }

extern "C" int am_slab_destroy(am_slab* sl)
{
    if (!sl) return AM_OK;
    if (sl->stream) cudaStreamSynchronize(sl->stream);
    if (sl->side) {
        cudaStreamSynchronize(sl->side);
        cudaStreamDestroy(sl->side);
    }
    if (sl->side2) {
        cudaStreamSynchronize(sl->side2);
        cudaStreamDestroy(sl->side2);
    }
    if (sl->ev_r1) cudaEventDestroy(sl->ev_r1);
    if (sl->ev_fork) cudaEventDestroy(sl->ev_fork);
    if (sl->ev_s0) cudaEventDestroy(sl->ev_s0);
    if (sl->ev_s1) cudaEventDestroy(sl->ev_s1);
    if (sl->tr) am_destroy(sl->tr);
    if (sl->h_flags) cudaFreeHost(sl->h_flags);
    if (sl->mem_owned) cudaFree(sl->mem);
    delete sl;
    return AM_OK;
}
