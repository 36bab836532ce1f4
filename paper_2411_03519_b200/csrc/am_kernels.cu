// am_kernels.cu -- the tracker's kernels for sm_100a.
//
// One scheduling round (Alg. 3 controller l.8-9) on the binned path:
//   k_bin       cell key + slot per agent (counting sort, histogram by atomics)
//   k_cells     chained scan of cell counts -> cell table {start, min step},
//               min-step pyramid (4x4 and 16x16 Morton blocks)
//   k_scatter   agents -> cell-sorted 16-byte records
//   k_scan      time-dilated neighbour scan: blocked bits, coupling
//               unions, perception digests
//   k_finalize  labels = union-find roots (min id), bad[root] |= blocked | RUNNING
//   k_ready     ready mask, dispatch, ordered compaction of the ready set
//   k_sort_*    stable LSD radix sort of the ready set by (step, label) -> order
// and the fused per-simulation path (k_small) for simulations of <= 1024 agents.
#include <climits>

#include "am_internal.cuh"

namespace am {

__device__ __forceinline__ bool round_full(const Dev& d);
__device__ __forceinline__ bool agent_changed(const Dev& d, uint32_t c, uint32_t i);

// ============================================================== am_update: ingest
// mode 0 = commit (update_agents, Alg. 3 l.11), 1 = initial state,
// 2 = full state with statuses (snapshot).  Reads state[cur], writes state[1-cur];
// the last block flips cur iff no error was raised (all-or-nothing update).
__global__ void __launch_bounds__(256) k_ingest(Dev d, const int2* __restrict__ npos,
                                                const int32_t* __restrict__ nstep,
                                                const uint8_t* __restrict__ nstat, int mode, int bin)
{
    pdl_begin();
    Ctl* ctl = d.ctl;
    const uint32_t c = ctl->cur;
    int err = 0, act = 0, run = 0, smin = INT_MAX, smax = INT_MIN, dmax = 0;
    const bool validate = (d.flags & AM_VALIDATE) != 0;
    const uint32_t tag = (ctl->epoch + 1u) & kTagMask;   // the epoch of the round this update feeds
    // every load of the thread's items is issued before any compute or store, so the
    // thread keeps kIngestItems independent load chains in flight (memory-level
    // parallelism; the state buffers and the caller's arrays may not alias)
    int2 p[kIngestItems], op[kIngestItems];
    int s[kIngestItems], os[kIngestItems];
    uint8_t ost[kIngestItems], nst[kIngestItems];
#pragma unroll
    for (int k = 0; k < kIngestItems; k++) {
        const int i = blockIdx.x * (256 * kIngestItems) + k * 256 + threadIdx.x;
        p[k] = make_int2(0, 0); op[k] = make_int2(0, 0); s[k] = 0; os[k] = 0; ost[k] = 0; nst[k] = 0;
        if (i < d.n) {
            p[k] = __ldcs(npos + i);
            s[k] = __ldcs(nstep + i);
            if (mode == 0) {
                os[k] = d.step[c][i];
                ost[k] = d.status[c][i];
                if (validate) op[k] = d.pos[c][i];
            } else if (mode == 2) {
                ost[k] = nstat[i];
            } else if (mode == 3) {   // replica update: the old state to diff against
                os[k] = d.step[c][i];
                ost[k] = d.status[c][i];
                op[k] = d.pos[c][i];
                nst[k] = nstat[i];
            }
        }
    }
#pragma unroll
    for (int k = 0; k < kIngestItems; k++) {
        const int i = blockIdx.x * (256 * kIngestItems) + k * 256 + threadIdx.x;
        if (i >= d.n) break;
        uint8_t st;
        if (p[k].x < 0 || p[k].x >= d.map_w || p[k].y < 0 || p[k].y >= d.map_h) err |= ERR_BOUNDS;
        if (mode == 0) {
            const long long ds = (long long)s[k] - os[k];
            st = ost[k];
            if (ds == 0) {
                if (validate && (op[k].x != p[k].x || op[k].y != p[k].y)) err |= ERR_PROTOCOL;
            } else if (ds == 1) {
                // step changed since the last round (kept even if this update is rejected:
                // that only makes the next round re-scan the agent)
                if (d.chg8) d.chg8[i] = 1;
                // its last-round cluster must be rebuilt by the next round's union-find
                if (d.dirty) {
                    const int lab = d.labels[i];
                    if (lab >= 0) d.dirty[lab] = ctl->epoch + 1u;
                }
                if (ost[k] != ST_RUNNING) {
                    err |= ERR_PROTOCOL;
                } else {
                    if (validate && !within_pts(d, op[k].x, op[k].y, p[k].x, p[k].y, (uint32_t)d.v))
                        err |= ERR_VELOCITY;
                    st = (d.target > 0 && s[k] == d.target) ? ST_DONE : ST_IDLE;
                }
            } else {
                err |= ERR_PROTOCOL;
            }
        } else if (mode == 1) {
            if (s[k] < 0 || (d.target > 0 && s[k] > d.target)) err |= ERR_PROTOCOL;
            st = (d.target > 0 && s[k] == d.target) ? ST_DONE : ST_IDLE;
        } else if (mode == 3) {
            // replica update (spatial-slab window, am_slab.h): statuses are given, DONE marks
            // an absent slot.  An agent CHANGED if it is present and its position or step
            // differs, or it just arrived; it DEPARTED if it was present and is absent now.
            st = nst[k];
            if (st > ST_DONE || s[k] < 0) err |= ERR_PROTOCOL;
            const bool pres = st != ST_DONE, was = ost[k] != ST_DONE;
            const bool moved = pres && (!was || s[k] != os[k] || p[k].x != op[k].x || p[k].y != op[k].y);
            if (moved || (was && !pres)) {
                if (d.chg8) d.chg8[i] = 1;
                if (d.dirty) {
                    const int lab = d.labels[i];
                    if (lab >= 0) d.dirty[lab] = ctl->epoch + 1u;
                }
                if (d.slot) {
                    const uint32_t r = d.slot[i];
                    if (r == kSentinel) {
                        if (pres) atomicOr(&ctl->rebuild_req, 1);   // an arrival has no record yet
                    } else if (pres) {
                        d.rec[r] = make_int4(p[k].x | (p[k].y << 16), s[k], i, (int)st | (int)(tag << kTagShift));
                        int cx, cy;
                        mkey_decode(d, d.key[i], cx, cy);
                        const int x0 = cx << d.clog, y0 = cy << d.clog;
                        const int x1 = x0 + (1 << d.clog) - 1, y1 = y0 + (1 << d.clog) - 1;
                        dmax = max(dmax, max(max(x0 - p[k].x, p[k].x - x1), max(y0 - p[k].y, p[k].y - y1)));
                    } else {
                        // departed: its record stays in its cell until the next rebuild with
                        // a step that no agent's test matches (never behind, never equal)
                        d.rec[r] = make_int4(op[k].x | (op[k].y << 16), INT_MAX, i, (int)ST_DONE);
                    }
                }
            }
        } else {
            st = ost[k];
            if (st > ST_DONE || s[k] < 0) err |= ERR_PROTOCOL;
        }
        d.pos[c ^ 1u][i] = p[k];
        d.step[c ^ 1u][i] = s[k];
        d.status[c ^ 1u][i] = st;
        if (st != ST_DONE) {
            act++;
            smin = min(smin, s[k]);
            smax = max(smax, s[k]);
        }
        run += st == ST_RUNNING;
        if (mode == 0 && s[k] != os[k] && d.slot) {
            // loose cells: a committed agent keeps its record (cell of the last rebuild) and
            // updates it in place; its distance outside that cell's box bounds the drift D
            const uint32_t r = d.slot[i];
            if (r != kSentinel) {
                d.rec[r] = make_int4(p[k].x | (p[k].y << 16), s[k], i, (int)st | (int)(tag << kTagShift));
                int cx, cy;
                mkey_decode(d, d.key[i], cx, cy);
                const int x0 = cx << d.clog, y0 = cy << d.clog;
                const int x1 = x0 + (1 << d.clog) - 1, y1 = y0 + (1 << d.clog) - 1;
                dmax = max(dmax, max(max(x0 - p[k].x, p[k].x - x1), max(y0 - p[k].y, p[k].y - y1)));
            }
        }
    }
    // block reduction, then one atomic per quantity per block
    __shared__ int r_err[8], r_min[8], r_max[8], r_act[8], r_run[8], r_d[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    err = (int)__reduce_or_sync(0xFFFFFFFFu, (unsigned)err);
    smin = __reduce_min_sync(0xFFFFFFFFu, smin);
    smax = __reduce_max_sync(0xFFFFFFFFu, smax);
    act = (int)__reduce_add_sync(0xFFFFFFFFu, (unsigned)act);
    run = (int)__reduce_add_sync(0xFFFFFFFFu, (unsigned)run);
    dmax = __reduce_max_sync(0xFFFFFFFFu, dmax);
    if (lane == 0) { r_err[w] = err; r_min[w] = smin; r_max[w] = smax; r_act[w] = act; r_run[w] = run; r_d[w] = dmax; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < 8; q++) {
            err |= r_err[q]; smin = min(smin, r_min[q]); smax = max(smax, r_max[q]);
            act += r_act[q]; run += r_run[q]; dmax = max(dmax, r_d[q]);
        }
        if (dmax > 0) atomicMax(&ctl->acc_D, dmax);
        if (err) atomicOr(&ctl->err_new, err);
        if (act) {
            atomicMin(&ctl->acc_W, smin);
            atomicMax(&ctl->acc_S, smax);
            atomicAdd(&ctl->acc_active, act);
        }
        if (run) atomicAdd(&ctl->acc_running, run);
    }
}


// k_ingest_done: one thread after k_ingest: flips to the new state buffer iff no agent
// raised an error (all-or-nothing update), publishes W / S / counts, resets the
// accumulators.  (A separate launch instead of a last-block ticket: no per-block fence.)
__global__ void k_ingest_done(Dev d, int mode, int bin)
{
    pdl_begin();
    if (threadIdx.x != 0) return;
    Ctl* ctl = d.ctl;
    const int e = ctl->err_new;
    // a rejected update may have touched records and incremental state: recompute all
    if (e != 0) ctl->full_next = 1;
    ctl->part_valid = 0;                // W / S / counts are this update's
    cstripe_reset(d);
    ctl->D = max(ctl->D, ctl->acc_D);   // (a rejected update is followed by a full rebuild)
    ctl->acc_D = 0;
    if (e == 0) {
        if (mode == 1 || mode == 2) ctl->full = 1;   // modes 0 and 3 are incremental
        ctl->cur ^= 1u;
        ctl->W = ctl->acc_W;
        ctl->S = ctl->acc_S;
        ctl->n_active = ctl->acc_active;
        ctl->n_running = ctl->acc_running;
    } else {
        ctl->err_sticky |= e;
    }
    ctl->err_new = 0;
    ctl->acc_W = INT_MAX;
    ctl->acc_S = INT_MIN;
    ctl->acc_active = 0;
    ctl->acc_running = 0;
    if (bin) round_begin(d);   // replay rounds: the am_ready that follows skips k_round_begin
}

// ============================================================== binned round
// block-aggregated append of the flagged threads' values to queue stripe `stripe` (one
// global atomic per block, in thread order); every thread of the 256-thread block calls it
template <class T>
__device__ __forceinline__ void block_append(T* q, int cap, uint32_t* ctr, int stripe, bool flag, const T& val,
                                             uint32_t* s_w /*[9]*/)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, flag);
    if (lane == 0) s_w[w] = (uint32_t)__popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (int k = 0; k < 8; k++) { const uint32_t v = s_w[k]; s_w[k] = acc; acc += v; }
        s_w[8] = acc ? atomicAdd(ctr + stripe, acc) : 0u;
    }
    __syncthreads();
    if (flag) q[(size_t)stripe * cap + s_w[8] + s_w[w] + (uint32_t)__popc(m & ((1u << lane) - 1u))] = val;
    __syncthreads();   // s_w is reused
}

// k_bin: Morton cell key, slot inside the cell (atomic histogram), per-cell min step;
// also resets the per-root bad flags for this round.
__global__ void __launch_bounds__(256) k_bin(Dev d)
{
    pdl_begin();
    if (!d.ctl->rebuild) return;   // loose cells: the records of the last rebuild serve this round
    const uint32_t c = d.ctl->cur;
    // grid-stride over a resident-sized grid: a loose round's early exit costs one wave
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d.n; i += gridDim.x * blockDim.x) {
        // independent loads first (one round trip), then the atomics
        const uint8_t st = d.status[c][i];
        const int2 p = d.pos[c][i];
        const int s = d.step[c][i];
        uint32_t key = kSentinel;
        if (st != ST_DONE) {
            key = mkey(d, (uint32_t)p.x >> d.clog, (uint32_t)p.y >> d.clog, 0);
            atomicAdd(d.cnt + key, 1u);
            atomicMin(d.cmin + key, s);
        }
        d.key[i] = key;
    }
}

// k_cells: exclusive scan of the cell counts in Morton order -> ctab{start, min};
// lmin1 = min over each 16-cell (4x4) block, lmin2 over each 256-cell (16x16) block;
// resets cmin for the next round (k_scatter counts cnt back to zero).  kCellsThreads threads x 16 cells per tile (small
// tiles: many short look-back chains in parallel).
__global__ void __launch_bounds__(kCellsThreads) k_cells(Dev d)
{
    pdl_begin();
    Ctl* ctl = d.ctl;
    if (!ctl->rebuild) return;        // loose cells: the cell table of the last rebuild serves
    const int kW = blockDim.x >> 5;   // tile = blockDim.x threads x 16 cells (host: <= kCellsThreads)
    __shared__ uint32_t wsum[kCellsThreads / 32];
    __shared__ uint32_t tile_excl;
    const uint32_t tile = take_ticket(&ctl->cells);
    const uint32_t tag = ctl->epoch * 16u + 1u;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const long long base = (long long)tile * (blockDim.x * 16) + t * 16;
    uint4* cnt4 = reinterpret_cast<uint4*>(d.cnt + base);
    int4* min4 = reinterpret_cast<int4*>(d.cmin + base);
    uint32_t cnt[16];
    int mn[16];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        uint4 a = cnt4[k];
        int4 b = min4[k];
        cnt[4 * k] = a.x; cnt[4 * k + 1] = a.y; cnt[4 * k + 2] = a.z; cnt[4 * k + 3] = a.w;
        mn[4 * k] = b.x; mn[4 * k + 1] = b.y; mn[4 * k + 2] = b.z; mn[4 * k + 3] = b.w;
        min4[k] = make_int4(INT_MAX, INT_MAX, INT_MAX, INT_MAX);   // (counts: k_scatter counts them back to 0)
    }
    uint32_t sum = 0;
    int m1 = INT_MAX;
#pragma unroll
    for (int k = 0; k < 16; k++) { sum += cnt[k]; m1 = min(m1, mn[k]); }
    d.lmin1[base >> 4] = m1;
    // 16 consecutive threads = one 256-cell block
    int m2 = m1;
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) m2 = min(m2, __shfl_xor_sync(0xFFFFFFFFu, m2, o));
    if ((lane & 15) == 0) d.lmin2[base >> 8] = m2;
    // block exclusive scan of sum
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
        uint32_t acc = 0;
        for (int k = 0; k < kW; k++) acc += wsum[k];
        const uint32_t ex = gridDim.x <= kScanAllTiles ? chain_scan_all(d.tiles_c, tile, tag, acc)
                                                         : chain_scan_warp(d.tiles_c, tile, tag, acc);
        __syncwarp();   // every lane has read wsum before lane 0 rewrites it
        if (t == 0) {
            tile_excl = ex;
            uint32_t a2 = 0;
            for (int k = 0; k < kW; k++) { uint32_t v = wsum[k]; wsum[k] = a2; a2 += v; }
            if (tile == gridDim.x - 1) d.ctab[d.ncells] = make_int2((int)(ex + acc), INT_MAX);
        }
    }
    __syncthreads();
    uint32_t run = tile_excl + wsum[w] + incl - sum;
    int4* out = reinterpret_cast<int4*>(d.ctab + base);
#pragma unroll
    for (int k = 0; k < 8; k++) {
        int4 v;
        v.x = (int)run; v.y = mn[2 * k]; run += cnt[2 * k];
        v.z = (int)run; v.w = mn[2 * k + 1]; run += cnt[2 * k + 1];
        out[k] = v;
    }
}

// k_scatter: agents -> records sorted by cell (the order inside a cell is arbitrary;
// no output depends on it); the union-find reset, per-agent flags and the scan's work
// queue of this round.
__global__ void __launch_bounds__(256) k_scatter(Dev d)
{
#if !(AM_PDL_EARLY & 4)
    pdl_begin();
#endif
    __shared__ uint32_t s_w[9];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t c = d.ctl->cur;
    const bool rebuild = d.ctl->rebuild != 0;
    const uint32_t ep = d.ctl->epoch & kTagMask;
    bool work = false;
    int4 q = make_int4(0, 0, 0, 0);
    // every read but the binning's (the agent state, last round's labels, witnesses,
    // dirty marks: final before k_bin began) first -- with AM_PDL_EARLY while k_cells
    // still runs; the cell table, the counts and every write after the PDL wait
    int2 p = make_int2(0, 0);
    int s = 0, lab = -1;
    uint8_t st = ST_DONE;
    bool chg = false, dirty = false;
    if (i < d.n) {
        p = d.pos[c][i];
        s = d.step[c][i];
        st = d.status[c][i];
        const bool ch = d.chg8[i] != 0;
        lab = d.labels[i];
        const uint32_t w = d.witness[i];
        const bool full = round_full(d);
        if (st != ST_DONE) {
            chg = full || ch;
            // union-find forest of this round: an agent whose last-round cluster has no
            // changed member keeps that cluster (all its coupling edges are unchanged: it
            // is still connected, and it can only grow through an edge of a changed
            // agent), so it hangs under the old root (= min id = its label); members of
            // dirty clusters start alone
            dirty = full || lab < 0 || d.dirty[lab] == d.ctl->epoch;
            // the scan's work queue (incremental scan): changed
            // agents, and IDLE agents whose recorded blocker (witness) changed
            work = chg || (st == ST_IDLE && w != kSentinel && agent_changed(d, c, w));
        }
    }
#if AM_PDL_EARLY & 4
    pdl_begin();
#endif
    if (i < d.n) {
        d.bad[i] = 0;     // per-root flags of this round (k_finalize)
        d.blkid[i] = 0;
        if (st == ST_DONE) {   // DONE: counts as changed for the carried edges (k_efilter)
            d.agflag[i] = 1;
            if (rebuild) d.slot[i] = kSentinel;
        } else {
            if (rebuild) {
                // slot: the cell's start + its count taken back down (returns the counts to 0)
                const uint32_t key = d.key[i];
                AM_CHECK(key < (uint32_t)d.ncells);
                const uint32_t r = (uint32_t)d.ctab[key].x + (atomicSub(d.cnt + key, 1u) - 1u);
                AM_CHECK(r < (uint32_t)d.n);
                const uint32_t tag = chg ? ep : ((ep + 0x800000u) & kTagMask);   // never this epoch
                d.rec[r] = make_int4(p.x | (p.y << 16), s, i, (int)st | (int)(tag << kTagShift));
                d.slot[i] = r;
            }
            d.parent[i] = dirty ? (uint32_t)i : (uint32_t)lab;
            d.agflag[i] = (uint8_t)((chg ? 1 : 0) | (dirty ? 2 : 0));
            q = make_int4(p.x | (p.y << 16), s, (int)((uint32_t)i | (chg ? 0x80000000u : 0u)), st);
        }
    }
    // stripe = block index mod 64, one atomic per block
    block_append(d.wq, d.wq_cap, d.wq_ctr, (int)(blockIdx.x & (kEdgeStripes - 1)), work, q, s_w);
}

// test every record of cell `key` against agent A; returns true if A got blocked.
template <bool kCouple>
__device__ __forceinline__ bool scan_cell(const Dev& d, uint32_t key, int ax, int ay, int as,
                                          uint32_t aid, bool blocked, uint32_t Rc,
                                          unsigned long long& dig, uint32_t& ncand)
{
    const int beg = d.ctab[key].x, end = d.ctab[key + 1].x;
    ncand += (uint32_t)(end - beg);
    for (int b = beg; b < end; b++) {
        const int4 B = d.rec[b];
        const uint32_t bid = (uint32_t)B.z;
        if (bid == aid) continue;
        const int dx = (B.x & 0xFFFF) - ax, dy = (B.x >> 16) - ay;
        if (kCouple && B.y == as) {
            if (within(dx, dy, Rc, d.metric)) {
                if (aid < bid) uf_unite(d.parent, aid, bid);
                if ((d.flags & AM_DIGEST) && within(dx, dy, (uint32_t)d.r_p, d.metric))
                    dig += digest_term(bid, dx, dy);
            }
        } else if (!blocked && B.y < as) {
            if (within(dx, dy, rb_radius((long long)as - B.y, d.v, d.r_p), d.metric)) {
                blocked = true;
                if (!kCouple) return true;
            }
        }
    }
    return blocked;
}

// k_scan: one thread per sorted record A.
//   phase 1: cells within box distance R_c = r_p + v: coupling unions + blocking tests;
//   phase 2: only if not yet blocked and A is ahead of the watermark: blocking tests
//            over the disk of radius R_b(s_A - W), walking the min-step pyramid:
//            a block with min step m is skipped if m >= s_A or its box distance
//            exceeds R_b(s_A - m) (exact pruning: no agent inside can block A).
__global__ void __launch_bounds__(256) k_scan_thread(Dev d)
{
    pdl_begin();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int nact = d.ctl->n_active;
    const int W = d.ctl->W;
    bool blocked = false;
    uint32_t ncells = 0, ncand = 0, np2 = 0, nb2 = 0, nb1 = 0;
    if (r < nact) {
        const int4 A = d.rec[r];
        const int ax = A.x & 0xFFFF, ay = A.x >> 16, as = A.y;
        const uint32_t aid = (uint32_t)A.z;
        const int cl = d.clog, Gx = 1 << d.gxlog, Gy = 1 << d.gylog;
        const uint32_t Rc = min((uint32_t)(d.r_p + d.v), kRClamp);   // r_p, v <= kRClamp (am_init)
        unsigned long long dig = 0;
        // ---- phase 1
        {
            const int cx0 = max(0, (ax - (int)Rc) >> cl), cx1 = min(Gx - 1, (ax + (int)Rc) >> cl);
            const int cy0 = max(0, (ay - (int)Rc) >> cl), cy1 = min(Gy - 1, (ay + (int)Rc) >> cl);
            for (int cy = cy0; cy <= cy1; cy++)
                for (int cx = cx0; cx <= cx1; cx++) {
                    if (!box_within(ax, ay, cx << cl, cy << cl, ((cx + 1) << cl) - 1,
                                    ((cy + 1) << cl) - 1, Rc, d.metric))
                        continue;
                    const uint32_t key = mkey(d, cx, cy, 0);
                    ncells++;
                    if (d.ctab[key].y > as) continue;
                    blocked = scan_cell<true>(d, key, ax, ay, as, aid, blocked, Rc, dig, ncand);
                }
        }
        if (d.flags & AM_DIGEST) d.digest[aid] = dig;
        // ---- phase 2
        if (!blocked && as > W) {
            np2 = 1;
            const int R = (int)rb_radius((long long)as - W, d.v, d.r_p);
            const int l2 = cl + 4;  // 16 cells per side
            const int G2x = Gx >> 4, G2y = Gy >> 4;
            const int bx0 = max(0, (ax - R) >> l2), bx1 = min(G2x - 1, (ax + R) >> l2);
            const int by0 = max(0, (ay - R) >> l2), by1 = min(G2y - 1, (ay + R) >> l2);
            for (int by = by0; by <= by1 && !blocked; by++)
                for (int bx = bx0; bx <= bx1 && !blocked; bx++) {
                    const int m2 = d.lmin2[mkey(d, bx, by, 4)];
                    nb2++;
                    if (m2 >= as) continue;
                    if (!box_within(ax, ay, bx << l2, by << l2, ((bx + 1) << l2) - 1, ((by + 1) << l2) - 1,
                                    rb_radius((long long)as - m2, d.v, d.r_p), d.metric))
                        continue;
                    for (int sy = 0; sy < 4 && !blocked; sy++)
                        for (int sx = 0; sx < 4 && !blocked; sx++) {
                            const int qx = bx * 4 + sx, qy = by * 4 + sy;  // 4x4-cell block
                            const int l1 = cl + 2;
                            const int m1 = d.lmin1[mkey(d, qx, qy, 2)];
                            nb1++;
                            if (m1 >= as) continue;
                            if (!box_within(ax, ay, qx << l1, qy << l1, ((qx + 1) << l1) - 1,
                                            ((qy + 1) << l1) - 1, rb_radius((long long)as - m1, d.v, d.r_p),
                                            d.metric))
                                continue;
                            for (int ty = 0; ty < 4 && !blocked; ty++)
                                for (int tx = 0; tx < 4 && !blocked; tx++) {
                                    const int cx = qx * 4 + tx, cy = qy * 4 + ty;
                                    const int x0 = cx << cl, y0 = cy << cl;
                                    const int x1 = ((cx + 1) << cl) - 1, y1 = ((cy + 1) << cl) - 1;
                                    // phase-1 cells were tested completely already
                                    if (box_within(ax, ay, x0, y0, x1, y1, Rc, d.metric)) continue;
                                    const uint32_t key = mkey(d, cx, cy, 0);
                                    const int m0 = d.ctab[key].y;
                                    ncells++;
                                    if (m0 >= as) continue;
                                    if (!box_within(ax, ay, x0, y0, x1, y1,
                                                    rb_radius((long long)as - m0, d.v, d.r_p), d.metric))
                                        continue;
                                    blocked = scan_cell<false>(d, key, ax, ay, as, aid, false, Rc, dig, ncand);
                                }
                        }
                }
        }
    }
    const unsigned bits = __ballot_sync(0xFFFFFFFFu, blocked);
    if (r < nact) d.v8[(uint32_t)d.rec[r].z] = blocked;
    if (r == 0) d.ctl->full_next = 1;   // keeps no edge list / witnesses
    if (d.flags & AM_STATS) {
        const unsigned c0 = __reduce_add_sync(0xFFFFFFFFu, ncells), c1 = __reduce_add_sync(0xFFFFFFFFu, ncand);
        const unsigned c2 = __reduce_add_sync(0xFFFFFFFFu, np2), c3 = __reduce_add_sync(0xFFFFFFFFu, nb2);
        const unsigned c4 = __reduce_add_sync(0xFFFFFFFFu, nb1);
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(&d.ctl->st_cells, (unsigned long long)c0);
            atomicAdd(&d.ctl->st_cand, (unsigned long long)c1);
            atomicAdd(&d.ctl->st_p2, (unsigned long long)c2);
            atomicAdd(&d.ctl->st_b2, (unsigned long long)c3);
            atomicAdd(&d.ctl->st_b1, (unsigned long long)c4);
            atomicAdd(&d.ctl->st_blocked, (unsigned long long)__popc(bits));
        }
    }
}

// ---------------------------------------------------------------------------------
// Incremental scan.  Per round only the agents in the WORK QUEUE
// built by k_bin are scanned:
//   * "changed" agents (their step changed since the last round: they committed, or
//     every agent in a full round): new coupling edges and a fresh
//     blocking verdict;
//   * IDLE agents whose recorded blocker (witness) changed: a fresh blocking verdict.
// Coupling edges between two unchanged agents are carried over from the last round's
// edge list by k_efilter (an edge depends only on its two endpoints' states).  An
// IDLE agent whose step did not change keeps "not blocked" (a commit can only remove
// blocking relations of others, App. A) and keeps "blocked" while its
// witness is unchanged.  RUNNING agents need no verdict (their cluster is not ready).
__device__ __forceinline__ uint32_t rb2(int lag, int v, int r_p, int lagcap)
{
    const uint32_t R = min((uint32_t)min(lag, lagcap) * (uint32_t)v + (uint32_t)(v + r_p), kRClamp);
    return R * R;
}

__device__ __forceinline__ bool within2(int dx, int dy, uint32_t R2, uint32_t R, int metric)
{
    if (metric == AM_METRIC_LINF) return (uint32_t)abs(dx) <= R && (uint32_t)abs(dy) <= R;
    return (uint32_t)(dx * dx) + (uint32_t)(dy * dy) <= R2;
}

__device__ __forceinline__ bool round_full(const Dev& d)
{
    // without commit validation positions may change without a step change: no reuse
    return d.ctl->full != 0 || !(d.flags & AM_VALIDATE);
}

__device__ __forceinline__ bool agent_changed(const Dev& d, uint32_t c, uint32_t i)
{
    (void)c;
    return d.chg8[i] != 0;
}

// append one coupling edge (a < b) to the next edge list; a warp stages its edges in
// shared memory and reserves space with one atomic per batch
struct EdgeStage {
    uint2 e[kEdgeStage];
    int ne;
};
__device__ __forceinline__ void stage_edge(const Dev& d, EdgeStage& sm, uint32_t a, uint32_t b)
{
    const int pos = atomicAdd(&sm.ne, 1);
    if (pos < kEdgeStage) {
        sm.e[pos] = make_uint2(a, b);
        return;
    }
    // staging full (dense neighbourhood): append this edge directly
    const uint32_t nxt = d.ctl->ecur ^ 1u;
    const uint32_t k = atomicAdd((uint32_t*)&d.ctl->ncnt[nxt], 1u);
    if ((int)k < d.ecap) {
        d.nedges[(size_t)nxt * d.ecap + k] = make_uint2(a, b);
        if (AM_SCAN_UNITE) uf_unite(d.parent, a, b);
    } else {
        uf_unite(d.parent, a, b);                  // list full: unite now, rebuild next round
        d.ctl->full_next = 1;
    }
}
__device__ __forceinline__ void flush_stage(const Dev& d, EdgeStage& sm, int lane)
{
    __syncwarp();
    const int ne = min(sm.ne, kEdgeStage);
    if (ne) {
        const uint32_t nxt = d.ctl->ecur ^ 1u;
        int base = 0;
        if (lane == 0) base = (int)atomicAdd((uint32_t*)&d.ctl->ncnt[nxt], (uint32_t)ne);
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        for (int k = lane; k < ne; k += 32) {
            const uint2 e = sm.e[k];
            if (base + k < d.ecap) {
                d.nedges[(size_t)nxt * d.ecap + base + k] = e;
                // the union right here (the scan never reads the forest; k_efilter's
                // concurrent unions of carried edges are lock-free hooks too)
                if (AM_SCAN_UNITE) uf_unite(d.parent, e.x, e.y);
            } else {
                uf_unite(d.parent, e.x, e.y);      // list full: unite now, rebuild next round
                d.ctl->full_next = 1;
            }
        }
    }
    __syncwarp();
    if (lane == 0) sm.ne = 0;
    __syncwarp();
}

// exclusive prefix of the kEdgeStripes (= 64) stripe counters into s_pref[0..64],
// computed by warp 0 with two parallel loads per lane (one L2 round trip)
__device__ __forceinline__ void stripe_prefix(const uint32_t* ctr, int cap, int* s_pref)
{
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const int a = min((int)__ldcg(ctr + lane), cap), b = min((int)__ldcg(ctr + 32 + lane), cap);
        int ia = a, ib = b;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int ya = __shfl_up_sync(0xFFFFFFFFu, ia, o), yb = __shfl_up_sync(0xFFFFFFFFu, ib, o);
            if (lane >= o) { ia += ya; ib += yb; }
        }
        const int ta = __shfl_sync(0xFFFFFFFFu, ia, 31);
        s_pref[lane] = ia - a;
        s_pref[32 + lane] = ta + ib - b;
        if (lane == 31) s_pref[64] = ta + ib;
    }
    __syncthreads();
}

// k_efilter: carry over last round's coupling edges (its carried and new lists) whose
// endpoints both kept their state (nothing in a full round) into this round's carried
// list, and unite those of dirty clusters.  Runs on the side stream beside k_scan_hw,
// which writes this round's new list.  One atomic per block.
__global__ void __launch_bounds__(256) k_efilter(Dev d)
{
    pdl_begin();
    const uint32_t cur = d.ctl->ecur, nxt = cur ^ 1u;
    const int nc = min((int)d.ctl->ccnt[cur], d.ecap), ne = nc + min((int)d.ctl->ncnt[cur], d.ecap);
    const bool full = round_full(d);
    __shared__ uint32_t s_w[9];
    for (int base = blockIdx.x * 256; base < ne; base += gridDim.x * 256) {   // block uniform
        const int k = base + threadIdx.x;
        bool keep = false, dirty = false;
        uint2 e = make_uint2(0, 0);
        if (k < ne && !full) {
            e = k < nc ? d.cedges[(size_t)cur * d.ecap + k] : d.nedges[(size_t)cur * d.ecap + (k - nc)];
            // per-endpoint flags of this round (k_scatter): bit 0 changed, bit 1 the
            // endpoint's last-round cluster is dirty (both endpoints share that cluster)
            const uint8_t fx = d.agflag[e.x], fy = d.agflag[e.y];
            keep = !((fx | fy) & 1);
            dirty = (fx & 2) != 0;
        }
        // kept edges are appended in order with one atomic per block
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        const unsigned m = __ballot_sync(0xFFFFFFFFu, keep);
        if (lane == 0) s_w[w] = (uint32_t)__popc(m);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t acc = 0;
            for (int q = 0; q < 8; q++) { const uint32_t v = s_w[q]; s_w[q] = acc; acc += v; }
            s_w[8] = acc ? atomicAdd((uint32_t*)&d.ctl->ccnt[nxt], acc) : 0u;
        }
        __syncthreads();
        if (keep) {
            const uint32_t pos = s_w[8] + s_w[w] + (uint32_t)__popc(m & ((1u << lane) - 1u));
            if ((int)pos < d.ecap) {
                d.cedges[(size_t)nxt * d.ecap + pos] = e;
                // a dirty cluster's forest is rebuilt from its edges (a clean cluster's
                // edges are implied by its members hanging under its root, k_scatter)
                if (dirty) uf_unite(d.parent, e.x, e.y);
            } else {
                uf_unite(d.parent, e.x, e.y);   // list full: unite now, rebuild next round
                d.ctl->full_next = 1;
            }
        }
        __syncthreads();
    }
}

// Morton child k (0..15) of a 4x4 block: offsets (dx, dy) in 0..3
__device__ __forceinline__ void morton_child(int k, int& dx, int& dy)
{
    dx = (k & 1) | ((k >> 1) & 2);
    dy = ((k >> 1) & 1) | ((k >> 2) & 2);
}

// Work counters of the half-warp scan (AM_STATS and the far-item count).
// A counter compiled out (the scan without AM_STATS): adding does nothing, reads give 0,
// so the statistics cost no registers in the kernel that runs every round.
struct StatSink {
    __device__ __forceinline__ StatSink& operator+=(uint32_t) { return *this; }
    __device__ __forceinline__ operator uint32_t() const { return 0u; }
};
template <bool kOn>
struct HwStatsT {
    uint32_t ncells = 0, ncand = 0, nb2 = 0, nb1 = 0, nitems = 0, nblk = 0;
};
template <>
struct HwStatsT<false> {
    StatSink ncells, ncand, nb2, nb1, nblk;
    uint32_t nitems = 0;   // the far-item count is always kept (n_items)
};

// per-warp reduction of the half-warp scan counters, one atomic per warp (no block
// barrier: a warp that is done leaves at once)
template <class HS>
__device__ __forceinline__ void hw_flush_stats(const Dev& d, const HS& hs, int lane)
{
    const unsigned it = __reduce_add_sync(0xFFFFFFFFu, hs.nitems);
    if (lane == 0 && it) atomicAdd(&d.ctl->n_items, (int)it);
    if (d.flags & AM_STATS) {
        const unsigned c0 = __reduce_add_sync(0xFFFFFFFFu, hs.ncells), c1 = __reduce_add_sync(0xFFFFFFFFu, hs.ncand);
        const unsigned c3 = __reduce_add_sync(0xFFFFFFFFu, hs.nb2), c4 = __reduce_add_sync(0xFFFFFFFFu, hs.nb1);
        const unsigned c5 = __reduce_add_sync(0xFFFFFFFFu, hs.nblk);
        if (lane == 0) {
            atomicAdd(&d.ctl->st_blocked, (unsigned long long)c5);
            atomicAdd(&d.ctl->st_cells, (unsigned long long)c0);
            atomicAdd(&d.ctl->st_cand, (unsigned long long)c1);
            atomicAdd(&d.ctl->st_p2, (unsigned long long)it);   // far work items (4x4 blocks)
            atomicAdd(&d.ctl->st_b2, (unsigned long long)c3);
            atomicAdd(&d.ctl->st_b1, (unsigned long long)c4);
        }
    }
}

// The far phase (time-dilated blocking beyond R_c) of one agent A = (ax, ay, as) by the
// 16 lanes of a half-warp (lane l, half h, lane mask hm), walking the Morton min-step
// pyramid with A's own point and step.  The pyramid has a fan-out of 16 at every level,
// so the 16 lanes test the 16 children of a block at once: (level 2) the 16x16-cell
// blocks of A's R_b(s_A - W) box, 16 per step; (level 1) the 4x4-cell children of each
// surviving block; (level 0) the cells of each surviving 4x4 block (one 8-byte table
// entry per lane, next start by shuffle).  A block, 4x4 block or cell with min step m
// is skipped if m >= s_A or its box distance exceeds R_b(s_A - m) (exact pruning:
// nothing inside can block A); cells within R_c of A are tested by the near phase.  The
// records of the surviving cells are flattened over the lanes and tested 16 at a time.
// Returns a blocker's id or kSentinel.
template <class HS>
__device__ __forceinline__ uint32_t hw_far(const Dev& d, int ax, int ay, int as, int W, int D, int l, int h,
                                           unsigned hm, HS& hs)
{
    int ox_l, oy_l;   // lane l's Morton child offsets in a 4x4 block
    morton_child(l, ox_l, oy_l);
    const int cl = d.clog, l1 = cl + 2, l2 = cl + 4, G2x = (1 << d.gxlog) >> 4, G2y = (1 << d.gylog) >> 4;
    const uint32_t Rc = min((uint32_t)(d.r_p + d.v), kRClamp);   // r_p, v <= kRClamp (am_init)
    const int lagcap = d.lagcap;   // host-computed kRClamp / v + 1
    auto& ncells = hs.ncells;
    auto& ncand = hs.ncand;
    auto& nb2 = hs.nb2;
    auto& nb1 = hs.nb1;
    auto& nitems = hs.nitems;
    const int R = (int)rb32(as - W, d.lagcap, d.v, d.r_p);
    const int bx0 = max(0, (ax - R - D) >> l2), bx1 = min(G2x - 1, (ax + R + D) >> l2);
    const int by0 = max(0, (ay - R - D) >> l2), by1 = min(G2y - 1, (ay + R + D) >> l2);
    const int nbx = bx1 - bx0 + 1, nb = nbx * (by1 - by0 + 1);
    uint32_t wit = kSentinel;
    nb2 += l == 0 ? (uint32_t)nb : 0u;
    for (int j0 = 0; j0 < nb && wit == kSentinel; j0 += 16) {
        // level 2: 16 blocks of 16x16 cells per step
        const int j = j0 + l;
        const int bx = bx0 + j % nbx, by = by0 + j / nbx;
        bool ok2 = false;
        if (j < nb) {
            const int m2 = __ldg(d.lmin2 + mkey(d, bx, by, 4));
            ok2 = m2 < as && cell_within(ax, ay, bx, by, l2, D, rb32(as - m2, d.lagcap, d.v, d.r_p), d.metric);
        }
        unsigned mask2 = (__ballot_sync(hm, ok2) >> (16 * h)) & 0xFFFFu;
        while (mask2 && wit == kSentinel) {
            const int jj = __ffs(mask2) - 1;
            mask2 &= mask2 - 1;
            const int bxj = __shfl_sync(hm, bx, jj, 16), byj = __shfl_sync(hm, by, jj, 16);
            const uint32_t k2 = mkey(d, bxj, byj, 4);
            nb1 += l == 0 ? 16u : 0u;
            // level 1: lane l tests child l (4x4 cells)
            const int qx = bxj * 4 + ox_l, qy = byj * 4 + oy_l;
            const int m1 = __ldg(d.lmin1 + k2 * 16 + l);
            const bool ok1 = m1 < as && cell_within(ax, ay, qx, qy, l1, D, rb32(as - m1, d.lagcap, d.v, d.r_p), d.metric);
            unsigned mask1 = (__ballot_sync(hm, ok1) >> (16 * h)) & 0xFFFFu;
            while (mask1 && wit == kSentinel) {
                const int ii = __ffs(mask1) - 1;
                mask1 &= mask1 - 1;
                nitems += l == 0 ? 1u : 0u;
                const uint32_t k1g = k2 * 16 + (uint32_t)ii;
                const int qxi = __shfl_sync(hm, qx, ii, 16), qyi = __shfl_sync(hm, qy, ii, 16);
                // level 0: lane l tests cell l of the 4x4 block
                const int2 e = d.ctab[(size_t)k1g * 16 + l];
                int nx = __shfl_down_sync(hm, e.x, 1, 16);
                if (l == 15) nx = d.ctab[(size_t)k1g * 16 + 16].x;
                const int cx = qxi * 4 + ox_l, cy = qyi * 4 + oy_l;
                // cells within R_c of A (widened boxes) were tested by the near phase
                const bool okc = nx > e.x && e.y < as && !cell_within(ax, ay, cx, cy, cl, D, Rc, d.metric) &&
                                 cell_within(ax, ay, cx, cy, cl, D, rb32(as - e.y, d.lagcap, d.v, d.r_p), d.metric);
                const int cnt = okc ? nx - e.x : 0;
                ncells += nx > e.x ? 1u : 0u;
                // flatten the candidate records over the 16 lanes
                int incl = cnt;
#pragma unroll
                for (int o = 1; o < 16; o <<= 1) {
                    const int y = __shfl_up_sync(hm, incl, o, 16);
                    if (l >= o) incl += y;
                }
                const int excl = incl - cnt;
                const int total = __shfl_sync(hm, incl, 15, 16);
                ncand += l == 0 ? (uint32_t)total : 0u;
                for (int b0 = 0; b0 < total && wit == kSentinel; b0 += 16) {
                    const int tq = b0 + l;
                    // lane holding candidate tq: the last lane with excl <= tq
                    int sl = 0;
#pragma unroll
                    for (int st = 8; st > 0; st >>= 1) {
                        const int ex = __shfl_sync(hm, excl, sl + st, 16);
                        if (ex <= tq) sl += st;
                    }
                    const int rs = __shfl_sync(hm, e.x, sl, 16), rx = __shfl_sync(hm, excl, sl, 16);
                    bool found = false;
                    uint32_t bid = 0;
                    if (tq < total) {
                        AM_CHECK(rs + (tq - rx) >= 0 && rs + (tq - rx) < d.n);
                        const int4 B = d.rec[rs + (tq - rx)];
                        bid = (uint32_t)B.z;
                        if (B.y < as) {
                            const int dx = (B.x & 0xFFFF) - ax, dy = (B.x >> 16) - ay;
                            const uint32_t Rb = min((uint32_t)min(as - B.y, lagcap) * (uint32_t)d.v +
                                                        (uint32_t)(d.v + d.r_p), kRClamp);
                            found = within2(dx, dy, Rb * Rb, Rb, d.metric);
                        }
                    }
                    const unsigned fm = (__ballot_sync(hm, found) >> (16 * h)) & 0xFFFFu;
                    if (fm) wit = __shfl_sync(hm, bid, __ffs(fm) - 1, 16);
                }
            }
        }
    }
    return wit;
}

// k_scan_hw: the whole incremental scan with one HALF-WARP per queued agent A.  The work
// queue (k_scatter) holds A's 16-byte record {x | y<<16, step, id | changed<<31, status}.
//   * the cells of A's query box -- R_c = r_p + v for coupling, plus R_b(s_A - W) when A
//     is IDLE and ahead of the watermark (the far blocking test) -- when the box holds at
//     most kDirect cells: one round trip loads every cell entry {start, min step} (<= 4
//     per lane), and the cells that can matter are compacted into a per-half-warp list,
//     near cells (box distance <= R_c) first.  Near cells: coupling edges for a changed
//     A (once per pair: from the smaller id when both changed) and the
//     blocking test for an IDLE A.  Far cells: blocking only, kept if
//     their min step m < s_A and their box distance <= R_b(s_A - m) (exact pruning);
//   * larger boxes: the near cells the same way, then the Morton min-step pyramid
//     (hw_far) for the far test.
// The records of the listed cells are flattened over the 16 lanes (prefix sum of the
// cell counts, 4-step shuffle search per lane) and tested 16 at a time; the first
// blocker becomes A's witness.
constexpr int kDirect = AM_DIRECT;          // cells of the query box resolved with one table fetch
constexpr int kDirectFull = AM_DIRECT_FULL; // the same for rounds the host knows are full recomputes

// test the records of the cells in `list[0..nl)` (near cells first: nn of them) against
// A; returns (in nblk/wit) the first blocker; stages coupling edges for a changed A
// (list[0, nn) near cells; the far cells follow at list[fgap + nn, fgap + nl): fgap = 0
// when they were appended, the gap to the end of the buffer when they fill it backwards)
template <class HS>
__device__ __forceinline__ void hw_records(const Dev& d, EdgeStage& sm, const int2* list, int nl, int nn, int fgap,
                                           int ax, int ay, int as, uint32_t aid, bool chg, bool idle, uint32_t ep,
                                           int l, int h, unsigned hm, bool& nblk, uint32_t& wit, HS& hs)
{
    const uint32_t Rc = min((uint32_t)(d.r_p + d.v), kRClamp);   // r_p, v <= kRClamp (am_init)
    const uint32_t Rc2 = Rc * Rc;
    const int lagcap = d.lagcap;   // host-computed kRClamp / v + 1
    for (int c0 = 0; c0 < nl; c0 += 16) {
        // nothing left to decide: blocked (or not IDLE) and no coupling in the rest
        if ((nblk || !idle) && (!chg || c0 >= nn)) break;
        const int k = c0 + l;
        int st0 = 0, cnt = 0;
        if (k < nl) {
            AM_CHECK((k < nn ? k : k + fgap) >= 0 && (k < nn ? k : k + fgap) < (AM_DIRECT > AM_DIRECT_FULL ? AM_DIRECT : AM_DIRECT_FULL));
            const int2 e = list[k < nn ? k : k + fgap];
            st0 = e.x;
            cnt = e.y;
        }
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
            const int y = __shfl_up_sync(hm, incl, o, 16);
            if (l >= o) incl += y;
        }
        const int excl = incl - cnt;
        const int total = __shfl_sync(hm, incl, 15, 16);
        // the near cells' records form a prefix [0, near_end) of the flattened range
        const int near_end = nn > c0 ? __shfl_sync(hm, incl, min(nn - c0, 16) - 1, 16) : 0;
        hs.ncand += l == 0 ? (uint32_t)total : 0u;
        for (int b0 = 0; b0 < total; b0 += 16) {
            if ((nblk || !idle) && !(chg && b0 < near_end)) break;   // half-warp uniform
            const int tq = b0 + l;
            int sl = 0;
#pragma unroll
            for (int stp = 8; stp > 0; stp >>= 1) {
                const int ex = __shfl_sync(hm, excl, sl + stp, 16);
                if (ex <= tq) sl += stp;
            }
            const int rs = __shfl_sync(hm, st0, sl, 16), rx = __shfl_sync(hm, excl, sl, 16);
            const bool bnear = tq < near_end;
            bool found = false;
            uint32_t bid = 0;
            if (tq < total) {
                AM_CHECK(rs + (tq - rx) >= 0 && rs + (tq - rx) < d.n);
                        const int4 B = d.rec[rs + (tq - rx)];
                bid = (uint32_t)B.z;
                if (bid != aid) {
                    const int dx = (B.x & 0xFFFF) - ax, dy = (B.x >> 16) - ay;
                    if (B.y == as) {
                        // B's record carries its changed bit (k_scatter)
                        if (chg && bnear && within2(dx, dy, Rc2, Rc, d.metric) && (!rec_changed(B.w, ep) || aid < bid))
                            stage_edge(d, sm, min(aid, bid), max(aid, bid));
                    } else if (idle && !nblk && B.y < as) {
                        const uint32_t R =
                            min((uint32_t)min(as - B.y, lagcap) * (uint32_t)d.v + (uint32_t)(d.v + d.r_p), kRClamp);
                        found = within2(dx, dy, R * R, R, d.metric);
                    }
                }
            }
            const unsigned fm = (__ballot_sync(hm, found) >> (16 * h)) & 0xFFFFu;
            if (fm && !nblk) {
                nblk = true;
                wit = __shfl_sync(hm, bid, __ffs(fm) - 1, 16);
            }
        }
    }
}

// kRec (full-recompute rounds, where the queue holds every binned agent): the agents are
// taken from the cell-sorted records instead of the id-ordered queue, so neighbouring
// half-warps scan neighbouring cells (cell-table and record reads shared in L1/L2)
// ceil(2^32 / n) for box widths n = 2..64 (0 for n <= 1): the scan's row of cell k of a
// box is __umulhi(k, c_rcx[ncx]), without a per-agent division
__constant__ uint32_t c_rcx[65] = {0u, 0u, 2147483648u, 1431655766u, 1073741824u, 858993460u, 715827883u, 613566757u, 536870912u, 477218589u, 429496730u, 390451573u, 357913942u, 330382100u, 306783379u, 286331154u, 268435456u, 252645136u, 238609295u, 226050911u, 214748365u, 204522253u, 195225787u, 186737709u, 178956971u, 171798692u, 165191050u, 159072863u, 153391690u, 148102321u, 143165577u, 138547333u, 134217728u, 130150525u, 126322568u, 122713352u, 119304648u, 116080198u, 113025456u, 110127367u, 107374183u, 104755300u, 102261127u, 99882961u, 97612894u, 95443718u, 93368855u, 91382283u, 89478486u, 87652394u, 85899346u, 84215046u, 82595525u, 81037119u, 79536432u, 78090315u, 76695845u, 75350304u, 74051161u, 72796056u, 71582789u, 70409300u, 69273667u, 68174085u, 67108864u};

template <int KD, bool kRec, bool kStats>
__device__ __forceinline__ void scan_hw(const Dev& d)
{
    pdl_begin();
    __shared__ EdgeStage s_all[8];
    __shared__ int2 s_list[16][KD];
    __shared__ int s_pref[kEdgeStripes + 1];
    const int lane = threadIdx.x & 31, l = lane & 15, h = lane >> 4, hw = threadIdx.x >> 4;
    const unsigned hm = 0xFFFFu << (threadIdx.x & 16);   // this half-warp's lanes
    EdgeStage& sm = s_all[threadIdx.x >> 5];
    int2* list = s_list[hw];
    if (lane == 0) sm.ne = 0;
    if (!kRec) stripe_prefix(d.wq_ctr, 1 << 30, s_pref);
    const int nq = kRec ? d.ctab[d.ncells].x : s_pref[kEdgeStripes];
    if (blockIdx.x == 0 && threadIdx.x == 0) d.ctl->n_work = nq;
    const int W = d.ctl->W;
    const int D = d.ctl->D;                      // loose-cell drift: every cell box widened by D
    const uint32_t ep = d.ctl->epoch & kTagMask;
    const int cl = d.clog, Gx = 1 << d.gxlog, Gy = 1 << d.gylog;
    const uint32_t Rc = min((uint32_t)(d.r_p + d.v), kRClamp);   // r_p, v <= kRClamp (am_init)
    HwStatsT<kStats> hs;
    uint32_t nfar = 0;
#if AM_SCAN_DYN
    // dynamic distribution: each warp takes the next two queue entries (one per half-warp)
    for (;;) {   // warp uniform
        int q0 = 0;
        if (lane == 0) q0 = (int)atomicAdd(&d.ctl->scan_next, 2u);
        q0 = __shfl_sync(0xFFFFFFFFu, q0, 0);
        if (q0 >= nq) break;
        const int q = q0 + h;
#else
    for (int q0 = blockIdx.x * 16; q0 < nq; q0 += gridDim.x * 16) {   // block uniform
        const int q = q0 + hw;
#endif
        if (q < nq) {                                                  // half-warp uniform
            // stripe of queue entry q: the number of stripe starts <= q among stripes
            // 1..63 (prefixes are non-decreasing), counted by the 16 lanes at once
            int4 A;
            if (kRec) {
                A = d.rec[q];
            } else {
                const int lo = (int)__reduce_add_sync(hm, (unsigned)((s_pref[1 + l] <= q) + (s_pref[17 + l] <= q) +
                                                                     (s_pref[33 + l] <= q) + (s_pref[49 + l] <= q)));
                A = d.wq[(size_t)lo * d.wq_cap + (q - s_pref[lo])];
            }
            const int ax = A.x & 0xFFFF, ay = A.x >> 16, as = A.y;
            const uint32_t aid = kRec ? (uint32_t)A.z : ((uint32_t)A.z & 0x7FFFFFFFu);
            const bool chg = kRec ? rec_changed(A.w, ep) : ((uint32_t)A.z >> 31) != 0;
            const bool idle = (A.w & 3) == ST_IDLE;
            const bool far = idle && as > W && !(d.flags & AM_DBG_SKIP_FAR);
            nfar += (far && l == 0) ? 1u : 0u;
            // query box: far radius when the far test is due and the box is small enough
            const int Rf = far ? (int)rb32(as - W, d.lagcap, d.v, d.r_p) : (int)Rc;
            int cx0 = max(0, (ax - Rf - D) >> cl), cx1 = min(Gx - 1, (ax + Rf + D) >> cl);
            int cy0 = max(0, (ay - Rf - D) >> cl), cy1 = min(Gy - 1, (ay + Rf + D) >> cl);
            const bool direct = (cx1 - cx0 + 1) * (cy1 - cy0 + 1) <= KD;
            if (!direct) {   // near cells only; the far test walks the pyramid below
                cx0 = max(0, (ax - (int)Rc - D) >> cl); cx1 = min(Gx - 1, (ax + (int)Rc + D) >> cl);
                cy0 = max(0, (ay - (int)Rc - D) >> cl); cy1 = min(Gy - 1, (ay + (int)Rc + D) >> cl);
            }
            const int ncx = cx1 - cx0 + 1, ncell = ncx * (cy1 - cy0 + 1);
            // row k / ncx of cell k of the box: a multiply-high by ceil(2^32 / ncx), exact
            // for k, ncx < 2^16 (a plain division for the rare larger boxes)
            const uint32_t rcx = ncx <= 64 ? c_rcx[ncx] : 0xFFFFFFFFu / (uint32_t)ncx + 1u;
            const bool mulhi = ncx > 1 && ncell < 65536;
            auto krow = [&](int k) { return ncx == 1 ? k : (mulhi ? (int)__umulhi((uint32_t)k, rcx) : k / ncx); };
            bool nblk = false;
            uint32_t wit = kSentinel;
            for (int cb = 0; cb < ncell; cb += KD) {   // one chunk unless cells are tiny
                if ((nblk || !idle) && !chg) break;
                // one round trip: the entries of the chunk's cells (<= 4 per lane)
                int2 ent[KD / 16];
                int nxt[KD / 16];
                // only the 16-cell groups the box has (half-warp uniform: one agent)
                const int ngrp = min(KD / 16, (ncell - cb + 15) >> 4);
#pragma unroll
                for (int j = 0; j < KD / 16; j++) {
                    const int k = cb + j * 16 + l;
                    ent[j] = make_int2(0, INT_MAX);
                    nxt[j] = 0;
                    if (j < ngrp && k < ncell) {
                        const int ky = krow(k), kx = k - ky * ncx;
                        const uint32_t key = mkey(d, cx0 + kx, cy0 + ky, 0);
                        AM_CHECK(key < (uint32_t)d.ncells);
                        ent[j] = d.ctab[key];
                        nxt[j] = d.ctab[key + 1].x;
                    }
                }
                // classify, compact into the list: near cells first, then far cells
                int nn = 0, nl = 0, fgap = 0;
#if AM_SCAN_1PASS
                // one pass: near cells compacted from the front of the list, far cells
                // from its end (each cell's row / column and box distance computed once)
                {
                    int nf = 0;
#pragma unroll
                    for (int j = 0; j < KD / 16; j++) {
                        if (j >= ngrp) break;                    // half-warp uniform
                        const int k = cb + j * 16 + l;
                        bool okn = false, okf = false;
                        if (k < ncell && nxt[j] > ent[j].x) {
                            const int mn = ent[j].y;
                            const int ky = krow(k);
                            const int cx = cx0 + (k - ky * ncx), cy = cy0 + ky;
                            const bool isnear = cell_within(ax, ay, cx, cy, cl, D, Rc, d.metric);
                            okn = isnear && (chg ? mn <= as : (idle && mn < as));
                            okf = !isnear && far && direct && mn < as &&
                                  cell_within(ax, ay, cx, cy, cl, D, rb32(as - mn, d.lagcap, d.v, d.r_p), d.metric);
                        }
                        const unsigned bn = (__ballot_sync(hm, okn) >> (16 * h)) & 0xFFFFu;
                        const unsigned bf = (__ballot_sync(hm, okf) >> (16 * h)) & 0xFFFFu;
                        const unsigned lt = (1u << l) - 1u;
                        AM_CHECK(!okn || nn + __popc(bn & lt) < KD);
                        AM_CHECK(!okf || (KD - 1 - (nf + __popc(bf & lt)) >= 0 && KD - 1 - (nf + __popc(bf & lt)) >= nn));
                        if (okn) list[nn + __popc(bn & lt)] = make_int2(ent[j].x, nxt[j] - ent[j].x);
                        if (okf) list[KD - 1 - (nf + __popc(bf & lt))] = make_int2(ent[j].x, nxt[j] - ent[j].x);
                        nn += __popc(bn);
                        nf += __popc(bf);
                    }
                    nl = nn + nf;
                    fgap = KD - nl;   // far entry q (0-based) at list[KD - 1 - q] = list[fgap + nn + (nf - 1 - q)]
                }
#else
                unsigned nearbits = 0;
#pragma unroll
                for (int pass = 0; pass < 2; pass++) {
                    if (pass == 1 && !(far && direct)) break;   // no far cells in this box
#pragma unroll
                    for (int j = 0; j < KD / 16; j++) {
                        if (j >= ngrp) break;                    // half-warp uniform
                        const int k = cb + j * 16 + l;
                        bool ok = false;
                        if (k < ncell && nxt[j] > ent[j].x) {
                            const int mn = ent[j].y;
                            if (pass == 0) {
                                const int ky = krow(k);
                                const int cx = cx0 + (k - ky * ncx), cy = cy0 + ky;
                                const bool isnear = cell_within(ax, ay, cx, cy, cl, D, Rc, d.metric);
                                nearbits |= isnear ? 1u << j : 0u;
                                ok = isnear && (chg ? mn <= as : (idle && mn < as));
                            } else if (!((nearbits >> j) & 1u) && far && direct && mn < as) {
                                const int ky = krow(k);
                                const int cx = cx0 + (k - ky * ncx), cy = cy0 + ky;
                                ok = cell_within(ax, ay, cx, cy, cl, D, rb32(as - mn, d.lagcap, d.v, d.r_p), d.metric);
                            }
                        }
                        const unsigned bm = (__ballot_sync(hm, ok) >> (16 * h)) & 0xFFFFu;
                        if (ok) list[nl + __popc(bm & ((1u << l) - 1u))] = make_int2(ent[j].x, nxt[j] - ent[j].x);
                        nl += __popc(bm);
                    }
                    if (pass == 0) nn = nl;
                }
#endif
                hs.ncells += l == 0 ? (uint32_t)nl : 0u;
                __syncwarp(hm);
                hw_records(d, sm, list, nl, nn, fgap, ax, ay, as, aid, chg, idle, ep, l, h, hm, nblk, wit, hs);
                __syncwarp(hm);   // the list is rewritten by the next chunk / agent
            }
            if (idle) {
                if (far && !direct && !nblk) {
                    wit = hw_far(d, ax, ay, as, W, D, l, h, hm, hs);
                    nblk = wit != kSentinel;
                }
                hs.nblk += (l == 0 && nblk) ? 1u : 0u;
                if (l == 0) {
                    d.v8[aid] = nblk ? 1 : 0;
                    d.witness[aid] = nblk ? wit : kSentinel;
                }
            }
        }
        flush_stage(d, sm, lane);   // warp collective: both half-warps
    }
    const unsigned nf = __reduce_add_sync(0xFFFFFFFFu, nfar);
    if (lane == 0 && nf) atomicAdd((unsigned*)&d.ctl->n_far, nf);
    hw_flush_stats(d, hs, lane);
}
// the incremental rounds' scan and the full-recompute rounds' scan (host-selected)
// (the _st instantiations keep the AM_STATS work counters; the host picks them when the
// flag is set)
__global__ void __launch_bounds__(256, AM_SCAN_MINB) k_scan_hw(Dev d) { scan_hw<kDirect, false, false>(d); }
__global__ void __launch_bounds__(256, AM_SCAN_MINB_FULL) k_scan_hw_full(Dev d) { scan_hw<kDirectFull, AM_SCAN_FULL_REC != 0, false>(d); }
__global__ void __launch_bounds__(256, AM_SCAN_MINB) k_scan_hw_st(Dev d) { scan_hw<kDirect, false, true>(d); }
__global__ void __launch_bounds__(256, AM_SCAN_MINB_FULL) k_scan_hw_full_st(Dev d) { scan_hw<kDirectFull, AM_SCAN_FULL_REC != 0, true>(d); }

// k_union: unite this round's coupling edges (carried-over + new), one thread per edge
// (ECL-CC style hooking of the larger root under the smaller, so roots stay the
// minimum id); the last block makes the list current for the next round.
__global__ void __launch_bounds__(256) k_union(Dev d)
{
    pdl_begin();
    const uint32_t nxt = d.ctl->ecur ^ 1u;
    const int ne = min((int)d.ctl->ncnt[nxt], d.ecap);
    if (blockIdx.x == 0 && threadIdx.x == 0) d.ctl->n_edges = ne + min((int)d.ctl->ccnt[nxt], d.ecap);
    // the carried edges were united by k_efilter where their cluster was dirty
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < ne; k += gridDim.x * blockDim.x) {
        const uint2 e = d.nedges[(size_t)nxt * d.ecap + k];
        uf_unite(d.parent, e.x, e.y);
    }
    // the lists of this round become current at the next k_round_begin
}

// k_finalize: label = root of the agent's tree (= min id of its cluster, Q10);
// a blocked or RUNNING member makes its cluster not ready (Q7).
// Id order: status / parent / verdict / label accesses are coalesced; only agents
// whose parent is not themselves chase pointers (singletons are one load).
// early = 1: this kernel's predecessor is k_union, so the statuses and the scan's
// verdicts were final before it began and are loaded before the PDL wait
__global__ void __launch_bounds__(256) k_finalize(Dev d, int early)
{
    early = (AM_PDL_EARLY & 1) ? early : 0;
    if (!early) pdl_begin();
    const int i0 = blockIdx.x * (256 * kFinItems) + threadIdx.x;
    if (i0 == 0 && !early) {
        d.ctl->full = 0;   // every kernel that reads the full-round flag has run
        if (AM_SCAN_UNITE) {   // (k_union's statistic)
            const uint32_t nxt = d.ctl->ecur ^ 1u;
            d.ctl->n_edges = min((int)d.ctl->ncnt[nxt], d.ecap) + min((int)d.ctl->ccnt[nxt], d.ecap);
        }
    }
    const uint32_t c = d.ctl->cur;
    // every item's status / verdict / parent load is issued before any pointer chase
    // (independent chains in flight; one wave of threads covers the agents)
    uint8_t st[kFinItems], vb[kFinItems];
    uint32_t par[kFinItems];
#pragma unroll
    for (int k = 0; k < kFinItems; k++) {
        const int i = i0 + k * 256;
        st[k] = ST_DONE;
        vb[k] = 0;
        par[k] = 0;
        if (i < d.n) {
            st[k] = d.status[c][i];
            vb[k] = d.v8[i];
            if (!early) par[k] = ld_cg(d.parent + i);
        }
    }
    if (early) {   // the forest k_union writes, after the wait
        pdl_begin();
        if (i0 == 0) d.ctl->full = 0;   // every kernel that reads the full-round flag has run
#pragma unroll
        for (int k = 0; k < kFinItems; k++) {
            const int i = i0 + k * 256;
            if (i < d.n) par[k] = ld_cg(d.parent + i);
        }
    }
#pragma unroll
    for (int k = 0; k < kFinItems; k++) {
        const int i = i0 + k * 256;
        if (i < d.n) d.chg8[i] = 0;   // the round consumed this agent's change (nothing after reads it)
        if (st[k] == ST_DONE) {
            if (i < d.n) d.labels[i] = -1;
            continue;
        }
        uint32_t root = par[k];
        if (root != (uint32_t)i) root = uf_find(d.parent, (uint32_t)i);
        d.labels[i] = (int32_t)root;
        const bool blk = st[k] == ST_IDLE && vb[k] == 1;
        d.blkid[i] = blk;
        if (blk || st[k] == ST_RUNNING) d.bad[root] = 1;
    }
}

// k_digest: perception digests ("perceives an area within a radius") of the
// agents dispatched this round, for the replay driver: sum over same-step non-DONE
// agents within r_p of mix64(id<<32 ^ (u16)dx<<16 ^ (u16)dy) (order-independent).
// One HALF-WARP per dispatched agent: lanes take the cells within r_p (one table fetch),
// the records of the cells are flattened over the 16 lanes, partial sums are reduced.
__global__ void __launch_bounds__(256) k_digest(Dev d, const int32_t* __restrict__ ids, const int32_t* count,
                                                const int32_t* __restrict__ gidmap, unsigned long long* out)
{
    pdl_begin();
    // ids: the agents (slots) whose digest is due; count: their number (NULL: this round's
    // ready count); gidmap: slot -> global id of the perceived agents' terms (NULL:
    // identity; the spatial-slab window passes its slot map); out: NULL -> d.digest
    const int nr = count ? *count : d.ctl->n_ready;
    unsigned long long* dst = out ? out : d.digest;
    const uint32_t c = d.ctl->cur;
    const int lane = threadIdx.x & 31, l = lane & 15;
    const unsigned hm = 0xFFFFu << (threadIdx.x & 16);   // this half-warp's lanes
    const int cl = d.clog, Gx = 1 << d.gxlog, Gy = 1 << d.gylog;
    const uint32_t Rp = (uint32_t)d.r_p, Rp2 = Rp * Rp;
    const int D = d.ctl->D;   // loose cells (widened boxes)
    const int hw0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 4, nhw = (gridDim.x * blockDim.x) >> 4;
    for (int k = hw0; k < nr; k += nhw) {   // half-warp uniform
        const uint32_t aid = (uint32_t)ids[k];
        const int2 P = d.pos[c][aid];
        const int ax = P.x, ay = P.y, as = d.step[c][aid];
        const int cx0 = max(0, (ax - (int)Rp - D) >> cl), cx1 = min(Gx - 1, (ax + (int)Rp + D) >> cl);
        const int cy0 = max(0, (ay - (int)Rp - D) >> cl), cy1 = min(Gy - 1, (ay + (int)Rp + D) >> cl);
        const int ncx = cx1 - cx0 + 1, ncell = ncx * (cy1 - cy0 + 1);
        unsigned long long dig = 0;
        for (int cb = 0; cb < ncell; cb += 16) {
            const int q = cb + l;
            int st0 = 0, cnt = 0;
            if (q < ncell) {
                const int cx = cx0 + q % ncx, cy = cy0 + q / ncx;
                if (cell_within(ax, ay, cx, cy, cl, D, Rp, d.metric)) {
                    const uint32_t key = mkey(d, cx, cy, 0);
                    const int2 e = d.ctab[key];
                    if (e.y <= as) {
                        st0 = e.x;
                        cnt = d.ctab[key + 1].x - e.x;
                    }
                }
            }
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) {
                const int y = __shfl_up_sync(hm, incl, o, 16);
                if (l >= o) incl += y;
            }
            const int excl = incl - cnt;
            const int total = __shfl_sync(hm, incl, 15, 16);
            for (int b0 = 0; b0 < total; b0 += 16) {
                const int tq = b0 + l;
                int sl = 0;
#pragma unroll
                for (int stp = 8; stp > 0; stp >>= 1) {
                    const int ex = __shfl_sync(hm, excl, sl + stp, 16);
                    if (ex <= tq) sl += stp;
                }
                const int rs = __shfl_sync(hm, st0, sl, 16), rx = __shfl_sync(hm, excl, sl, 16);
                if (tq < total) {
                    AM_CHECK(rs + (tq - rx) >= 0 && rs + (tq - rx) < d.n);
                        const int4 B = d.rec[rs + (tq - rx)];
                    if (B.y == as && (uint32_t)B.z != aid) {
                        const int dx = (B.x & 0xFFFF) - ax, dy = (B.x >> 16) - ay;
                        if (within2(dx, dy, Rp2, Rp, d.metric))
                            dig += digest_term(gidmap ? (uint32_t)gidmap[B.z] : (uint32_t)B.z, dx, dy);
                    }
                }
            }
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) dig += __shfl_xor_sync(hm, dig, o, 16);
        if (l == 0) dst[aid] = dig;
    }
}

// k_ready: mask, DONE labels, dispatch (IDLE -> RUNNING), and the
// ordered compaction of the ready set: keys ((step - W) << idbits) | label, values id.
// 256 threads x 8 consecutive agents per tile; chained scan keeps id order.
__global__ void __launch_bounds__(kReadyThreads) k_ready(Dev d, uint8_t* __restrict__ mask)
{
    pdl_begin();
    Ctl* ctl = d.ctl;
    constexpr int kW = kReadyThreads / 32;
    __shared__ uint32_t wsum[kW];
    __shared__ uint32_t tile_excl;
    __shared__ uint32_t ncl;
    const uint32_t tile = take_ticket(&ctl->ready);
    const uint32_t tag = ctl->epoch * 16u + 2u;
    const uint32_t c = ctl->cur;
    const int W = ctl->W;
    const bool ok = ctl->err_sticky == 0;
    const bool peek = (d.flags & AM_PEEK) != 0;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (t == 0) ncl = 0;
    const int i0 = tile * kReadyTile + t * kReadyItems;
    uint8_t ready[kReadyItems], st[kReadyItems];
    int lab[kReadyItems];
    uint32_t cnt = 0, mycl = 0;
    // loads in two independent rounds (status + label, then the roots' bad flags),
    // stores after
#pragma unroll
    for (int k = 0; k < kReadyItems; k++) {
        const int i = i0 + k;
        st[k] = ST_DONE;
        lab[k] = -1;
        if (i < d.n) {
            st[k] = d.status[c][i];
            lab[k] = d.labels[i];
        }
    }
#pragma unroll
    for (int k = 0; k < kReadyItems; k++) {
        ready[k] = 0;
        if (st[k] != ST_DONE && ok && st[k] == ST_IDLE) ready[k] = !d.bad[lab[k]];
    }
#pragma unroll
    for (int k = 0; k < kReadyItems; k++) {
        const int i = i0 + k;
        if (i < d.n) {
            if (st[k] == ST_DONE) {
                d.labels[i] = -1;
                lab[k] = -1;
            } else if (ready[k]) {
                if (!peek) d.status[c][i] = ST_RUNNING;
                cnt++;
                mycl += (lab[k] == i);
            }
            mask[i] = ready[k];
        }
    }
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (mycl) atomicAdd(&ncl, mycl);
    if (w == 0) {
        uint32_t acc = 0;
        for (int k = 0; k < kW; k++) acc += wsum[k];
        const uint32_t ex = gridDim.x <= kScanAllTiles ? chain_scan_all(d.tiles_r, tile, tag, acc)
                                                         : chain_scan_warp(d.tiles_r, tile, tag, acc);
        __syncwarp();   // every lane has read wsum before lane 0 rewrites it
        if (t == 0) {
            tile_excl = ex;
            uint32_t a2 = 0;
            for (int k = 0; k < kW; k++) { uint32_t v = wsum[k]; wsum[k] = a2; a2 += v; }
            if (tile == gridDim.x - 1) ctl->n_ready = (int)(ex + acc);
        }
    }
    __syncthreads();
    uint32_t pos = tile_excl + wsum[w] + incl - cnt;
    unsigned long long kor = 0;
#pragma unroll
    for (int k = 0; k < kReadyItems; k++) {
        if (ready[k]) {
            const int i = i0 + k;
            const unsigned long long key =
                ((unsigned long long)(uint32_t)(d.step[c][i] - W) << d.idbits) | (uint32_t)lab[k];
            d.rkey[0][pos] = key;
            d.rval[0][pos] = (uint32_t)i;
            d.rid[pos] = i;
            kor |= key;
            pos++;
        }
    }
    // OR of all keys -> number of radix passes (one atomic per block)
    __shared__ unsigned long long s_or[kW];
    unsigned lo = __reduce_or_sync(0xFFFFFFFFu, (unsigned)kor);
    unsigned hi = __reduce_or_sync(0xFFFFFFFFu, (unsigned)(kor >> 32));
    if (lane == 0) s_or[w] = ((unsigned long long)hi << 32) | lo;
    __syncthreads();
    if (t == 0) {
        unsigned long long o = 0;
        for (int q = 0; q < kW; q++) o |= s_or[q];
        if (o) atomicOr(&ctl->sort_or, o);
        if (ncl) atomicAdd(&ctl->n_clusters, (int)ncl);
    }
    // no last-block epilogue: the sort derives its bit count from sort_or, k_round_begin
    // resets the tile ticket and sort_or, k_finalize consumed the full-round flag
}

// significant bits of this round's ready keys (OR of all keys, k_ready)
__device__ __forceinline__ int ready_key_bits(const Ctl* ctl)
{
    const unsigned long long o = *(volatile const unsigned long long*)&ctl->sort_or;
    return o ? 64 - __clzll((long long)o) : 0;
}
__device__ __forceinline__ int onesweep_passes(const Ctl* ctl)
{
    const int np = (ready_key_bits(ctl) + kRadixBits - 1) / kRadixBits;
    return np < 1 ? 1 : np;
}

// lanes of the warp holding the same digit (and validity), from kRadixBits + 1 ballots
__device__ __forceinline__ unsigned warp_match_digit(int dg, bool valid)
{
    const unsigned vm = __ballot_sync(0xFFFFFFFFu, valid);
    unsigned peers = valid ? vm : ~vm;
#pragma unroll
    for (int b = 0; b < kRadixBits; b++) {
        const bool bit = (dg >> b) & 1;
        const unsigned m = __ballot_sync(0xFFFFFFFFu, bit);
        peers &= bit ? m : ~m;
    }
    return peers;
}

// k_sort_hist: global kRadixBits-bit digit histograms of the ready keys for every pass
// (persistent grid-stride); the last block turns them into exclusive digit offsets.
__global__ void __launch_bounds__(256) k_sort_hist(Dev d, int max_passes)
{
    pdl_begin();
    Ctl* ctl = d.ctl;
    __shared__ uint32_t h[kMaxSortPasses][kRadix];
    const int n = ctl->n_ready;
    const int np = min(onesweep_passes(ctl), max_passes);
    if (blockIdx.x == 0 && threadIdx.x == 0) { ctl->npasses = np; ctl->sort_bits = ready_key_bits(ctl); }
    for (int k = threadIdx.x; k < kMaxSortPasses * kRadix; k += blockDim.x) (&h[0][0])[k] = 0;
    __syncthreads();
    {
        const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
        for (int k0 = blockIdx.x * blockDim.x; k0 < n; k0 += gridDim.x * blockDim.x) {
            const int k = k0 + threadIdx.x;
            const bool valid = k < n;
            const unsigned long long key = valid ? d.rkey[0][k] : 0ull;
            for (int p = 0; p < np; p++) {
                // one shared-memory atomic per distinct digit per warp (skewed high digits)
                const int dg = valid ? (int)((key >> (kRadixBits * p)) & (kRadix - 1)) : kRadix;
                const unsigned peers = warp_match_digit(dg, valid);
                if (valid && (peers & lt) == 0) atomicAdd(&h[p][dg], (uint32_t)__popc(peers));
            }
        }
        __syncthreads();
        for (int k = threadIdx.x; k < np * kRadix; k += blockDim.x) {
            const uint32_t v = (&h[0][0])[k];
            if (v) atomicAdd(d.ghist + k, v);
        }
    }
    if (finish_block(&ctl->hist, gridDim.x)) {
        // last block: thread t owns digits 2t and 2t+1; exclusive scan per pass
        __shared__ uint32_t wtot[8];
        const int t = threadIdx.x, lane = t & 31, w = t >> 5;
        for (int p = 0; p < np; p++) {
            const uint32_t v0 = __ldcg(d.ghist + p * kRadix + 2 * t);
            const uint32_t v1 = __ldcg(d.ghist + p * kRadix + 2 * t + 1);
            const uint32_t v = v0 + v1;
            uint32_t incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) wtot[w] = incl;
            __syncthreads();
            uint32_t base = 0;
            for (int q = 0; q < w; q++) base += wtot[q];
            const uint32_t ex = base + incl - v;
            d.gstart[p * kRadix + 2 * t] = ex;
            d.gstart[p * kRadix + 2 * t + 1] = ex + v0;
            d.ghist[p * kRadix + 2 * t] = 0;
            d.ghist[p * kRadix + 2 * t + 1] = 0;
            __syncthreads();
        }
        __threadfence();
    }
}

// k_sort_pass: one stable LSD pass over kRadixBits bits (onesweep: per-digit decoupled
// look-back across tiles of 8192 keys, 32 warps x 8 keys per lane).  Warp w of a tile
// owns items [256w, 256w+256) and ranks them in index order with __match_any_sync, so
// the pass is stable.  The last pass writes the ids straight into `order`.
// Dynamic shared memory: wcnt[32][kRadix] + goff[kRadix].
__global__ void __launch_bounds__(1024) k_sort_pass(Dev d, int pass, int32_t* __restrict__ order, int ntiles)
{
    pdl_begin();
    Ctl* ctl = d.ctl;
    extern __shared__ uint32_t sort_smem[];
    uint32_t (*wcnt)[kRadix] = reinterpret_cast<uint32_t (*)[kRadix]>(sort_smem);
    uint32_t* goff = sort_smem + 32 * kRadix;
    const int n = ctl->n_ready;
    const int np = onesweep_passes(ctl);
    // persistent: a few CTAs take tiles in ticket order (the look-back only waits on
    // tiles that are being processed, so any grid size is deadlock-free)
    for (;;) {
    const uint32_t tile = take_ticket(&ctl->pass[pass]);
    if (pass >= np || (int)tile * kSortTile >= n) break;
    const uint32_t tag = ctl->epoch * 16u + 4u + (uint32_t)pass;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const unsigned long long* kin = d.rkey[pass & 1];
    const uint32_t* vin = d.rval[pass & 1];
    unsigned long long* kout = d.rkey[(pass + 1) & 1];
    uint32_t* vout = d.rval[(pass + 1) & 1];
    const bool last = pass == np - 1;
    for (int k = t; k < 32 * kRadix; k += 1024) (&wcnt[0][0])[k] = 0;
    __syncthreads();
    const int shift = kRadixBits * pass;
    unsigned long long key[8];
    uint32_t val[8], rnk[8];
    int dig[8];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const int i = tile * kSortTile + w * 256 + k * 32 + lane;
        const bool valid = i < n;
        key[k] = valid ? kin[i] : 0ull;
        val[k] = valid ? vin[i] : 0u;
        dig[k] = valid ? (int)((key[k] >> shift) & (kRadix - 1)) : kRadix;
        const unsigned peers = warp_match_digit(dig[k], valid);
        const uint32_t base = valid ? wcnt[w][dig[k]] : 0u;
        rnk[k] = base + __popc(peers & lt);
        __syncwarp();
        if (valid && (peers & lt) == 0) wcnt[w][dig[k]] = base + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // per digit (thread t = digit): exclusive prefix over warps, tile total, look-back
    if (t < kRadix) {
        uint32_t acc = 0;
#pragma unroll 8
        for (int q = 0; q < 32; q++) { uint32_t v = wcnt[q][t]; wcnt[q][t] = acc; acc += v; }
        unsigned long long* tw = d.tiles_sort + ((size_t)pass * ntiles) * kRadix;
        // column-major tile words: word of (tile, digit) at tw[digit * ntiles + tile]
        unsigned long long* col = tw + (size_t)t * ntiles;
        const uint32_t excl = chain_scan(col, tile, tag, acc);
        goff[t] = d.gstart[pass * kRadix + t] + excl;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 8; k++) {
        if (dig[k] < kRadix) {
            const uint32_t dst = goff[dig[k]] + wcnt[w][dig[k]] + rnk[k];
            if (last) {
                order[dst] = (int32_t)val[k];
            } else {
                kout[dst] = key[k];
                vout[dst] = val[k];
            }
        }
    }
    __syncthreads();   // wcnt / goff are reused by the next tile
    }
    finish_block(&ctl->pass[pass], gridDim.x);
}

// ============================================================== fused small path
// One CTA per simulation (<= 1024 agents): the whole round in shared memory.
// Simulations take tickets in index order; a chained scan over simulations places
// each one's ready agents in `order` (sim-major: order = (sim, step, label, id)).
__global__ void __launch_bounds__(1024) k_small(Dev d, uint8_t* __restrict__ mask,
                                                 int32_t* __restrict__ order)
{
    pdl_begin();
    Ctl* ctl = d.ctl;
    __shared__ int sx[kSmallMax], sy[kSmallMax], ss[kSmallMax];
    __shared__ uint8_t sst[kSmallMax], sbad[kSmallMax], srdy[kSmallMax];
    __shared__ uint32_t par[kSmallMax];
    __shared__ int slab[kSmallMax];
    __shared__ uint32_t s_excl, s_ncl;
    const uint32_t b = take_ticket(&ctl->small_);
    const uint32_t tag = ctl->epoch * 16u + 3u;
    const int lo = (int)((long long)b * d.n / d.n_sims);
    const int hi = (int)((long long)(b + 1) * d.n / d.n_sims);
    const int m = hi - lo;
    const int t = threadIdx.x;
    const uint32_t c = ctl->cur;
    const bool ok = ctl->err_sticky == 0;
    const bool peek = (d.flags & AM_PEEK) != 0;
    if (t == 0) s_ncl = 0;
    if (t < m) {
        const int2 p = d.pos[c][lo + t];
        sx[t] = p.x;
        sy[t] = p.y;
        ss[t] = d.step[c][lo + t];
        sst[t] = d.status[c][lo + t];
        sbad[t] = 0;
        par[t] = (uint32_t)t;
    }
    __syncthreads();
    const uint32_t Rc = min((uint32_t)(d.r_p + d.v), kRClamp);   // r_p, v <= kRClamp (am_init)
    bool blocked = false;
    unsigned long long dig = 0;
    if (t < m && sst[t] != ST_DONE) {
        const int ax = sx[t], ay = sy[t], as = ss[t];
        for (int j = 0; j < m; j++) {
            if (j == t || sst[j] == ST_DONE) continue;
            const int dx = sx[j] - ax, dy = sy[j] - ay, bs = ss[j];
            if (bs == as) {
                if (within_pts(d, ax, ay, sx[j], sy[j], Rc)) {
                    if (t < j) suf_unite(par, (uint32_t)t, (uint32_t)j);
                    if ((d.flags & AM_DIGEST) && within_pts(d, ax, ay, sx[j], sy[j], (uint32_t)d.r_p))
                        dig += digest_term((uint32_t)(lo + j), dx, dy);
                }
            } else if (!blocked && bs < as) {
                blocked = within_pts(d, ax, ay, sx[j], sy[j], rb32(as - bs, d.lagcap, d.v, d.r_p));
            }
        }
    }
    __syncthreads();
    int lab = -1;
    if (t < m && sst[t] != ST_DONE) {
        lab = (int)suf_find(par, (uint32_t)t);
        if (blocked || sst[t] == ST_RUNNING) sbad[lab] = 1;
    }
    __syncthreads();
    bool rdy = false;
    if (t < m) {
        rdy = ok && sst[t] == ST_IDLE && !sbad[lab];
        srdy[t] = rdy;
        slab[t] = lab;
        mask[lo + t] = rdy;
        d.labels[lo + t] = lab < 0 ? -1 : lo + lab;
        d.blkid[lo + t] = blocked && sst[t] == ST_IDLE;
        if (d.flags & AM_DIGEST) d.digest[lo + t] = dig;
        if (rdy && !peek) d.status[c][lo + t] = ST_RUNNING;
        if (rdy && lab == t) atomicAdd(&s_ncl, 1u);
    }
    const int cnt = __syncthreads_count(rdy);
    // rank by (step, label, id) among this simulation's ready agents
    int rank = 0;
    if (rdy) {
        const int as = ss[t];
        for (int j = 0; j < m; j++) {
            if (!srdy[j] || j == t) continue;
            const int bs = ss[j];
            if (bs < as || (bs == as && (slab[j] < lab || (slab[j] == lab && j < t)))) rank++;
        }
    }
    if (t == 0) {
        s_excl = chain_scan(d.tiles_s, b, tag, (uint32_t)cnt);
        if (s_ncl) atomicAdd(&ctl->n_clusters, (int)s_ncl);
        if (b == (uint32_t)d.n_sims - 1) ctl->n_ready = (int)(s_excl + cnt);
    }
    __syncthreads();
    if (rdy) order[s_excl + rank] = lo + t;
    finish_block(&ctl->small_, gridDim.x);
}

__global__ void k_round_begin(Dev d)
{
    pdl_begin();
    round_begin(d);
}

}  // namespace am
