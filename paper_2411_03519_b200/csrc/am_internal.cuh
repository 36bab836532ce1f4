// am_internal.cuh -- context layout and device helpers of libametro (sm_100a).
//
// Product code: shares nothing with oracle/ (the CPU oracle is test-only).
// Citations "P:<line>" refer to /root/reference/PAPER.md.
#pragma once

#include <climits>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "am.h"

namespace am {

constexpr int kSmallMax = 1024;           // agents per simulation for the fused kernel
constexpr int kScanAllTiles = 1024;       // chained scans sum all predecessors up to this many tiles
#ifndef AM_CELLS_THREADS
#define AM_CELLS_THREADS 512
#endif
#ifndef AM_READY_ITEMS
#define AM_READY_ITEMS 4
#endif
#ifndef AM_READY_THREADS
#define AM_READY_THREADS 1024
#endif
#ifndef AM_FIN_ITEMS
#define AM_FIN_ITEMS 2
#endif
#ifndef AM_SCAN_UNITE
#define AM_SCAN_UNITE 0   // 1: the scan unites its new edges as it flushes them, no k_union (A/B: +13 us, rejected)
#endif
#ifndef AM_COMMIT_ITEMS
#define AM_COMMIT_ITEMS 8   // k_commit: agents per thread (commits compacted per warp)
#endif
// Bounds-checked experiment build (-DAM_DEBUG_BOUNDS=1, tools/ab_round.py build dbg=...):
// device asserts on the index of every shared / global access the checks name; the GPU
// suite runs against it with AM_LIB_VARIANT=dbg (compute-sanitizer is closed on the pool)
#ifndef AM_DEBUG_BOUNDS
#define AM_DEBUG_BOUNDS 0
#endif
#if AM_DEBUG_BOUNDS
#include <cassert>
#define AM_CHECK(c) assert(c)
#else
#define AM_CHECK(c) ((void)0)
#endif
#ifndef AM_PDL_EARLY
#define AM_PDL_EARLY 5   // bits: 1 k_finalize, 2 k_commit, 4 k_scatter load what their predecessor does not write before the PDL wait
#endif
#ifndef AM_SCAN_1PASS
#define AM_SCAN_1PASS 1   // scan_hw: near and far cells classified in one pass
#endif
#ifndef AM_SCAN_DYN
#define AM_SCAN_DYN 0
#endif
#ifndef AM_DIRECT
#define AM_DIRECT 64        // direct query box (cells) of the incremental scan
#endif
#ifndef AM_SCAN_MINB
#define AM_SCAN_MINB 4      // k_scan_hw: 4 resident CTAs per SM (64 registers; A/B after the stats registers left: 4 / 5 / 6 CTAs 130.7 / 131.1 / 135.9 us)
#endif
#ifndef AM_SCAN_MINB_FULL
#define AM_SCAN_MINB_FULL 5   // k_scan_hw_full (full-recompute rounds)
#endif
#ifndef AM_SCAN_FULL_REC
#define AM_SCAN_FULL_REC 1   // full rounds take their agents from the cell-sorted records
#endif
#ifndef AM_DIRECT_FULL
#define AM_DIRECT_FULL 32   // ... of full-recompute rounds (C5 snapshot A/B with 16-tile cells: 777 / 649 / 624 us at 64 / 32 / 16; with 32-tile cells: 607 / 597 / 602 us, profiles/r2_sweep_s29)
#endif
#ifndef AM_COMMIT_SPLIT
#define AM_COMMIT_SPLIT 0   // 1: the replay's commit as an O(N) scan + a dense pass over the committing
                            // agents (bit-exact; measured slower: round 166 -> 184 us, commit 28 -> 45 us)
#endif
#ifndef AM_INGEST_ITEMS
#define AM_INGEST_ITEMS 4
#endif
constexpr int kCellsThreads = AM_CELLS_THREADS;   // cell-table scan: threads per tile
constexpr int kReadyItems = AM_READY_ITEMS;   // agents per thread of the ready compaction
constexpr int kReadyThreads = AM_READY_THREADS;   // threads per ready compaction tile
constexpr int kReadyTile = kReadyThreads * kReadyItems;
constexpr int kSortTile = 8192;           // radix pass tile (1024 threads x 8 keys)
constexpr int kMaxSortPasses = 8;
constexpr int kRadixBits = 9;            // radix digit width of the priority sort
constexpr int kRadix = 1 << kRadixBits;
constexpr int kFinItems = AM_FIN_ITEMS;
constexpr int kCommitItems = AM_COMMIT_ITEMS;   // agents per thread in the driver's k_commit         // agents per thread in k_finalize
constexpr int kIngestItems = AM_INGEST_ITEMS;   // agents per thread in k_ingest / k_commit
constexpr int kEdgeStripes = 64;          // striped queues (one atomic counter per stripe)
constexpr int kCommitStripes = 64;        // post-commit reductions (block index mod 64)
constexpr int kEdgeStage = 128;           // coupling edges staged per warp before appending
constexpr uint32_t kSentinel = 0xFFFFFFFFu;
// record word w = status (bits 0-1) | change tag << 8: the 24-bit round epoch in which
// the agent's step last changed ("changed this round" <=> tag == epoch & kTagMask)
constexpr int kTagShift = 8;
constexpr uint32_t kTagMask = 0xFFFFFFu;
#ifndef AM_REBUILD_D
#define AM_REBUILD_D 4      // rebuild the cell binning once an agent drifted this far out of its cell
#endif
#ifndef AM_REBUILD_K
#define AM_REBUILD_K 32     // ... or after this many incremental rounds (cell minima go stale)
#endif
constexpr uint32_t kRClamp = 46340u;      // >= every distance on a 32768^2 map; R^2 < 2^31

enum : int32_t { ERR_BOUNDS = 1, ERR_PROTOCOL = 2, ERR_VELOCITY = 4 };
enum : uint8_t { ST_IDLE = 0, ST_RUNNING = 1, ST_DONE = 2 };

// dynamic tile ticket + "last block" counter of one grid-wide pass; the last block
// to finish resets both, so the next launch starts clean (stream order).
struct Chain {
    unsigned ticket;
    unsigned done;
};

// device control block (one per context, device memory; mirrored to pinned host)
struct Ctl {
    uint32_t cur;          // which of the two state buffers is committed
    uint32_t epoch;        // bumped by every am_ready; tags chained-scan tile words
    int32_t  err_new;      // error bits of the running am_update
    int32_t  err_sticky;   // error bits not yet reported to the host
    int32_t  W, S;         // watermark (min step of non-DONE) and max step
    int32_t  n_active, n_running;
    int32_t  n_ready, n_clusters;
    int32_t  npasses;      // radix passes needed by this round's ready keys (onesweep digits)
    int32_t  sort_bits;    // significant bits of this round's ready keys
    int32_t  full;         // recompute every verdict / coupling edge this round
    int32_t  full_next;    // force a full round next time (edge list overflowed, ablation scan)
    uint32_t ecur;         // which pair of coupling-edge lists is current (ping-pong)
    uint32_t ccnt[2];      // edges in each carried list (k_efilter output)
    uint32_t ncnt[2];      // edges in each new list (k_scan_hw output)
    int32_t  n_work, n_far, n_items, n_edges;   // this round's scan work (stats)
    // incremental binning ("loose cells"): between rebuilds the records stay in their
    // cells and committed agents update their record in place; D = max over agents of
    // the L-inf distance from the agent to its record's cell box (every cell-pruning
    // box is widened by D), acc_D its per-update accumulator
    int32_t  D, acc_D, since_rebuild, rebuild, n_rebuilds;
    int32_t  rebuild_req;  // a replica update brought an agent that has no record (arrival)
    int32_t  part_valid;   // the replay's in-place commit left post-commit partials (k_replay_begin)
    int32_t  n_commit;     // committing agents listed by k_commit_scan (reset by round_begin)
    uint32_t scan_next;    // dynamic work distribution of k_scan_hw (AM_SCAN_DYN)
    // accumulators of am_update (reset by its last block)
    int32_t  acc_W, acc_S, acc_active, acc_running;
    unsigned long long sort_or;   // OR of all ready keys
    // scan statistics (AM_STATS): cells visited, candidate pairs, phase-2 agents,
    // pyramid blocks tested (16x16, 4x4)
    unsigned long long st_cells, st_cand, st_p2, st_b2, st_b1, st_blocked;
    Chain ingest, bin, cells, ready, hist, small_, uni, efil, pass[kMaxSortPasses];
};

// all device pointers of a context, passed by value to kernels
struct Dev {
    Ctl* ctl;
    int32_t n, n_sims, map_w, map_h, r_p, v, target, metric;
    uint32_t flags;
    int32_t clog;          // log2 cell edge
    int32_t gxlog, gylog;  // log2 cells along x / y of the Morton grid (each >= 6)
    int32_t mbits;         // min(gxlog, gylog): interleaved bits per coordinate
    int32_t mxhi;          // 1 if x is the longer side (its extra high bits sit above)
    int32_t ncells;        // 1 << (gxlog + gylog)
    int32_t idbits;        // bits to hold an agent id
    int32_t lagcap;        // step lag beyond which R_b = (lag + 1) v + r_p reaches kRClamp
    // double-buffered state
    int2* pos[2];
    int32_t* step[2];
    uint8_t* status[2];
    // binned round
    uint32_t* key;         // Morton cell key per agent (kSentinel = DONE)
    uint32_t* cnt;         // [ncells] agents per cell (zero between rounds)
    int32_t* cmin;         // [ncells] min step per cell (INT_MAX between rounds)
    int2* ctab;            // [ncells+1] {start, min step}
    int32_t* lmin1;        // [ncells/16]  min step per 4x4-cell block
    int32_t* lmin2;        // [ncells/256] min step per 16x16-cell block
    int4* rec;             // [n] records sorted by cell at the last rebuild {x | y<<16, step, id, w};
                           // positions / steps are kept current (in place) between rebuilds
    uint32_t* slot;        // [n] per id: index of its record (kSentinel: not binned, DONE)
    int32_t* cstripe;      // [64][32] post-commit {min step, max step, active, running} per stripe
                           // (one 128-byte line each; the replay's in-place commits, k_replay_begin)
    int32_t rebuild_d, rebuild_k;   // rebuild policy (drift tiles, incremental rounds)
    const uint16_t* gdist;          // AM_METRIC_GRAPH: [gV][gV] hop distances (0xFFFF: unreachable)
    int32_t gV;
    uint8_t* v8;           // [n] per id: blocking verdict (0 no, 1 yes, 2 far phase pending)
    uint32_t* witness;     // [n] per id: the blocker found last time it was computed
    uint8_t* chg8;         // [n] per id: step changed since the last round (set by am_update)
    uint2* cedges;         // [2][ecap] carried coupling edges (a < b), ping-pong
    uint2* nedges;         // [2][ecap] new coupling edges (a < b), ping-pong
    int32_t ecap;
    int4* wq;              // [kEdgeStripes][wq_cap] work queue of the scan: the agent's record
                           // {x | y<<16, step, id | changed<<31, status}
    uint32_t* wq_ctr;      // [kEdgeStripes]
    int32_t wq_cap;
    uint32_t* parent;      // [n] union-find forest in id space (root = min id)
    uint32_t* dirty;       // [n] per last-round label: epoch of the round its cluster must be rebuilt in
    uint8_t* agflag;       // [n] per agent, this round (k_scatter): bit 0 changed, bit 1 cluster dirty
    uint8_t* bad;          // [n] cluster (root) has a blocked or RUNNING member
    int32_t* labels;       // [n]
    uint8_t* blkid;        // [n] blocked verdict per id (IDLE agents; 0 otherwise)
    unsigned long long* digest;   // [n] perception digests (AM_DIGEST)
    unsigned long long* rkey[2];  // [n] ready keys (ping-pong)
    int32_t* rid;                 // [n] ready ids in id order (k_ready; dispatch and digests read it)
    uint32_t* rval[2];            // [n] ready ids (ping-pong)
    unsigned long long* tiles_c;  // chained-scan tile words: cell table scan
    unsigned long long* tiles_r;  //   ready compaction
    unsigned long long* tiles_s;  //   per-simulation (fused path)
    unsigned long long* tiles_sort;  // [kMaxSortPasses][ntiles_sort][256]
    uint32_t* ghist;              // [kMaxSortPasses][256]
    uint32_t* gstart;             // [kMaxSortPasses][256]
};

}  // namespace am

// per-kernel device timing (am_profile_*): external event records around every
// launch, so they also work inside captured CUDA graphs
namespace am {
enum KernelId : int {
    K_INGEST = 0, K_BIN, K_CELLS, K_SCATTER, K_SCAN, K_FINALIZE, K_READY, K_SORT_HIST, K_SORT_PASS,
    K_SMALL, K_COMMIT, K_DISP_A, K_DISP_B, K_UNION, K_NEAR, K_COUNT
};
struct Prof {
    bool on = false;
    unsigned mask = 0;            // kernels timed (bit = KernelId)
    cudaEvent_t ev[K_COUNT][2] = {};
    unsigned pending = 0;
    double ms[K_COUNT] = {};
    long long cnt[K_COUNT] = {};
};
}  // namespace am

// launch with the programmatic-stream-serialization attribute (pdl) -- the kernel must
// begin with pdl_begin()
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(bool pdl, cudaStream_t s, void (*k)(KArgs...), dim3 g, dim3 b, size_t smem,
                            Args... args)
{
    cudaLaunchConfig_t lc{};
    lc.gridDim = g;
    lc.blockDim = b;
    lc.dynamicSmemBytes = smem;
    lc.stream = s;
    cudaLaunchAttribute at{};
    at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at.val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = &at;
    lc.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&lc, k, static_cast<KArgs>(args)...);
}

struct am_ctx;
void am_prof_begin(am_ctx* c, int id);
void am_prof_end(am_ctx* c, int id);
void am_prof_collect(am_ctx* c);
void am_prof_mark(am_ctx* c, unsigned mask);
void am_join_side(am_ctx* c);
void am_join_digest(am_ctx* c);
int am_update_binned(am_ctx* c, const int32_t* positions, const int32_t* sim_steps);

struct am_ctx {
    am::Prof prof;
    am::Dev d;
    am::Ctl* h_ctl = nullptr;        // pinned host mirror
    cudaStream_t stream = nullptr;
    int path = 0;                    // 0 = fused per-sim kernel, 1 = binned pipeline
    int cell = 0;
    int small_threads = 32;
    int num_sms = 148;
    int scan_blocks = 148 * 4;       // resident blocks of k_scan_hw (occupancy x SMs)
    int scan_blocks_full = 148 * 4;  // ... of k_scan_hw_full
    bool full_hint = true;           // the host knows the next round is a full recompute
    int sort_ctas = 16;              // persistent CTAs of each radix pass
    int sort_passes_max = 1;
    cudaStream_t side = nullptr;     // edge filter (beside the scan) and priority sort (beside
                                     // digest/dispatch) run here
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_efil = nullptr;
    bool join_pending = false;
    cudaStream_t side2 = nullptr;    // perception digests (beside the driver's dispatch part a)
    cudaEvent_t ev_dig = nullptr;
    cudaEvent_t ev_mask = nullptr;   // recorded after k_ready when mask_event is set (am_replay_io)
    bool mask_event = false;
    bool dig_pending = false;
    bool bin_pending = false;        // am_update_binned ran the round's k_bin already
    bool defer_join = false;         // am_ready inside a replay round: the driver joins the sort
    bool pdl = true;                 // programmatic dependent launch between round kernels
    int csort_ctas = 0;              // cluster size of the one-kernel priority sort (0 = onesweep)
    int csort_cap = 0;               // dynamic shared memory bytes per CTA of k_csort
    int ntiles_sort = 1;
    int ntiles_ready = 1;
    int ntiles_cells = 1;
    int cells_threads = 256;   // k_cells block size (16 cells per thread)
    bool first = true;
    bool have_round = false;
    void* ws = nullptr;
    size_t ws_bytes = 0;
    bool ws_owned = false;           // allocated by am_init (no caller workspace in am_config)
    am_round_stats stats{};
    std::string err;
};

// ---------------------------------------------------------------- device helpers
namespace am {

// Programmatic dependent launch: every kernel of the round starts with this.  It waits
// until the preceding kernel of the stream has completed and its memory is visible (a
// no-op without the launch attribute), then lets the next kernel's CTAs be launched, so
// grid launch and CTA rasterisation overlap the tail of the kernel before.
__device__ __forceinline__ void pdl_begin()
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ uint32_t part1by1(uint32_t x)
{
    x &= 0xFFFFu;
    x = (x | (x << 8)) & 0x00FF00FFu;
    x = (x | (x << 4)) & 0x0F0F0F0Fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
}
// inverse of part1by1: the even bits of x packed together
__device__ __forceinline__ uint32_t part_compact(uint32_t x)
{
    x &= 0x55555555u;
    x = (x | (x >> 1)) & 0x33333333u;
    x = (x | (x >> 2)) & 0x0F0F0F0Fu;
    x = (x | (x >> 4)) & 0x00FF00FFu;
    x = (x | (x >> 8)) & 0x0000FFFFu;
    return x;
}
// Morton (Z-order) key of a cell: every aligned 2^k x 2^k block of cells is a
// contiguous key range, so the min-step pyramid is a min over contiguous ranges.
__device__ __forceinline__ uint32_t morton(uint32_t cx, uint32_t cy)
{
    return part1by1(cx) | (part1by1(cy) << 1);
}
// Key of cell (cx, cy) of a rectangular 2^gxlog x 2^gylog grid at pyramid level lv
// (0 = cells, 2 = 4x4-cell blocks, 4 = 16x16-cell blocks; coordinates in units of that
// level): the low mbits - lv bits of both coordinates are interleaved (Z-order inside
// square tiles), the longer side's remaining high bits sit above them.  Aligned 4x4 /
// 16x16 blocks are therefore contiguous key ranges, and key_lv(c) >> 4 = key_{lv+2}(c >> 2)
// (mbits >= 6).  A square grid gives the plain Morton key.
__device__ __forceinline__ uint32_t mkey(const Dev& d, uint32_t cx, uint32_t cy, int lv)
{
    const int m = d.mbits - lv;
    const uint32_t lo = (1u << m) - 1u;
    const uint32_t hi = (d.mxhi ? cx : cy) >> m;
    return part1by1(cx & lo) | (part1by1(cy & lo) << 1) | (hi << (2 * m));
}

__device__ __forceinline__ void mkey_decode(const Dev& d, uint32_t key, int& cx, int& cy)
{
    const int m = d.mbits;
    const uint32_t lo = m >= 16 ? 0xFFFFFFFFu : ((1u << (2 * m)) - 1u);
    const int xl = (int)part_compact(key & lo), yl = (int)part_compact((key & lo) >> 1);
    const int hi = (int)(key >> (2 * m));
    cx = d.mxhi ? (hi << m) | xl : xl;
    cy = d.mxhi ? yl : (hi << m) | yl;
}

// blocking radius clamped so that R^2 fits in 31 bits; exact because the
// clamp exceeds every distance on a <= 32768^2 map.
__device__ __forceinline__ uint32_t rb_radius(long long lag, int v, int r_p)
{
    long long R = (lag + 1) * (long long)v + r_p;
    return R > (long long)kRClamp ? kRClamp : (uint32_t)R;
}

// the same radius for a non-negative int lag in 32-bit arithmetic (d.lagcap host-computed)
__device__ __forceinline__ uint32_t rb32(int lag, int lagcap, int v, int r_p)
{
    return min((uint32_t)min(lag, lagcap) * (uint32_t)v + (uint32_t)(v + r_p), kRClamp);
}

__device__ __forceinline__ bool within(int dx, int dy, uint32_t R, int metric)
{
    if (metric == AM_METRIC_LINF) {
        uint32_t ax = (uint32_t)abs(dx), ay = (uint32_t)abs(dy);
        return ax <= R && ay <= R;
    }
    uint32_t d2 = (uint32_t)(dx * dx) + (uint32_t)(dy * dy);
    return d2 <= R * R;
}

// dist(A, B) <= R for positions A, B under the context's metric (the graph metric looks
// the hop count up; the others use the coordinate differences)
__device__ __forceinline__ bool within(int dx, int dy, uint32_t R, int metric);
__device__ __forceinline__ bool within_pts(const Dev& d, int ax, int ay, int bx, int by, uint32_t R)
{
    if (d.metric == AM_METRIC_GRAPH) {
        const uint32_t h = d.gdist[(size_t)ax * d.gV + bx];
        return h != 0xFFFFu && h <= R;
    }
    return within(bx - ax, by - ay, R, d.metric);
}

// distance between the tile boxes [ax0,ax1]x[ay0,ay1] and [bx0,bx1]x[by0,by1] within R
__device__ __forceinline__ bool box_dist_within(int ax0, int ay0, int ax1, int ay1, int bx0, int by0,
                                                int bx1, int by1, uint32_t R, int metric);

// distance from point (x,y) to the tile box [x0,x1] x [y0,y1] within R
__device__ __forceinline__ bool box_within(int x, int y, int x0, int y0, int x1, int y1,
                                           uint32_t R, int metric)
{
    int dx = x < x0 ? x0 - x : (x > x1 ? x - x1 : 0);
    int dy = y < y0 ? y0 - y : (y > y1 ? y - y1 : 0);
    return within(dx, dy, R, metric);
}

// cell (cx, cy) of edge 2^sh, its tile box widened by D on every side (loose cells:
// every agent recorded in the cell lies inside the widened box), within R of (x, y)
__device__ __forceinline__ bool cell_within(int x, int y, int cx, int cy, int sh, int D, uint32_t R, int metric)
{
    return box_within(x, y, (cx << sh) - D, (cy << sh) - D, ((cx + 1) << sh) - 1 + D, ((cy + 1) << sh) - 1 + D, R,
                      metric);
}

// record word: changed this round (tag == the round's epoch)
__device__ __forceinline__ bool rec_changed(int w, uint32_t ep) { return (((uint32_t)w >> kTagShift) & kTagMask) == ep; }

// inverse of mkey at level 0: the cell coordinates of a key
__device__ __forceinline__ void mkey_decode(const Dev& d, uint32_t key, int& cx, int& cy);

__device__ __forceinline__ bool box_dist_within(int ax0, int ay0, int ax1, int ay1, int bx0, int by0,
                                                int bx1, int by1, uint32_t R, int metric)
{
    const int dx = bx0 > ax1 ? bx0 - ax1 : (ax0 > bx1 ? ax0 - bx1 : 0);
    const int dy = by0 > ay1 ? by0 - ay1 : (ay0 > by1 ? ay0 - by1 : 0);
    return within(dx, dy, R, metric);
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long z)
{
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ unsigned long long key3(unsigned long long s, unsigned long long a,
                                                   unsigned long long b)
{
    return mix64(mix64(mix64(s + a) + b));
}
// one perceived agent's contribution to the perception digest
__device__ __forceinline__ unsigned long long digest_term(uint32_t j, int dx, int dy)
{
    unsigned long long w = ((unsigned long long)j << 32) ^
                           ((unsigned long long)(uint16_t)dx << 16) ^ (unsigned long long)(uint16_t)dy;
    return mix64(w);
}

__device__ __forceinline__ uint32_t ld_cg(const uint32_t* p) { return __ldcg(p); }

// union-find (global, id space): hook the larger root under the smaller, so every
// root is the minimum id of its tree; find uses intermediate pointer jumping.
__device__ __forceinline__ uint32_t uf_find(uint32_t* parent, uint32_t x)
{
    uint32_t cur = ld_cg(parent + x);
    if (cur != x) {
        uint32_t prev = x, next;
        while (cur > (next = ld_cg(parent + cur))) {
            parent[prev] = next;
            prev = cur;
            cur = next;
        }
    }
    return cur;
}
// shared-memory union-find of the fused per-simulation kernels (same hooking rule)
__device__ __forceinline__ uint32_t suf_find(volatile uint32_t* parent, uint32_t x)
{
    uint32_t cur = parent[x];
    if (cur != x) {
        uint32_t prev = x, next;
        while (cur > (next = parent[cur])) {
            // path halving as a shared-memory atomicMin: parent pointers only ever decrease
            // (hooks and halving both move toward the smaller root), so the min keeps the
            // forest valid under concurrent finds and unions without a data race
            atomicMin((uint32_t*)&parent[prev], next);
            prev = cur;
            cur = next;
        }
    }
    return cur;
}
__device__ __forceinline__ void suf_unite(uint32_t* parent, uint32_t a, uint32_t b)
{
    volatile uint32_t* vp = parent;
    uint32_t ra = suf_find(vp, a), rb = suf_find(vp, b);
    while (ra != rb) {
        if (ra < rb) {
            uint32_t old = atomicCAS(parent + rb, rb, ra);
            if (old == rb) break;
            rb = old;
        } else {
            uint32_t old = atomicCAS(parent + ra, ra, rb);
            if (old == ra) break;
            ra = old;
        }
    }
}

__device__ __forceinline__ void uf_unite(uint32_t* parent, uint32_t a, uint32_t b)
{
    uint32_t ra = uf_find(parent, a), rb = uf_find(parent, b);
    while (ra != rb) {
        if (ra < rb) {
            uint32_t old = atomicCAS(parent + rb, rb, ra);
            if (old == rb) break;
            rb = old;
        } else {
            uint32_t old = atomicCAS(parent + ra, ra, rb);
            if (old == ra) break;
            ra = old;
        }
    }
}

// ------------------------------------------------ chained (decoupled look-back) scan
// tile word: [tag:30][flag:2][value:32]; flag 1 = aggregate, 2 = inclusive prefix.
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p)
{
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v)
{
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long tile_word(uint32_t tag, uint32_t flag, uint32_t val)
{
    return ((unsigned long long)(tag & 0x3FFFFFFFu) << 34) | ((unsigned long long)flag << 32) | val;
}
// publish this tile's aggregate, look back, publish the inclusive prefix; returns
// the exclusive prefix.  Called by ONE thread.  tiles[t] for t < tile must be
// published eventually (tickets are handed out in launch order).
__device__ __forceinline__ uint32_t chain_scan(unsigned long long* tiles, uint32_t tile, uint32_t tag,
                                               uint32_t agg)
{
    tag &= 0x3FFFFFFFu;
    if (tile == 0) {
        st_relaxed(tiles, tile_word(tag, 2, agg));
        return 0;
    }
    st_relaxed(tiles + tile, tile_word(tag, 1, agg));
    uint32_t excl = 0;
    int j = (int)tile - 1;
    while (j >= 0) {
        unsigned long long w = ld_relaxed(tiles + j);
        uint32_t wt = (uint32_t)(w >> 34), fl = (uint32_t)(w >> 32) & 3u;
        if (wt != tag || fl == 0) continue;   // not yet published in this epoch
        excl += (uint32_t)w;
        if (fl == 2) break;
        --j;
    }
    st_relaxed(tiles + tile, tile_word(tag, 2, excl + agg));
    return excl;
}

// Warp-parallel decoupled look-back: called by ALL 32 lanes of one warp; lane k reads
// predecessor (j - k), so 32 predecessors are inspected per L2 round trip.  Returns
// the exclusive prefix in every lane.
__device__ __forceinline__ uint32_t chain_scan_warp(unsigned long long* tiles, uint32_t tile, uint32_t tag,
                                                    uint32_t agg)
{
    const int lane = threadIdx.x & 31;
    tag &= 0x3FFFFFFFu;
    if (tile == 0) {
        if (lane == 0) st_relaxed(tiles, tile_word(tag, 2, agg));
        return 0;
    }
    if (lane == 0) st_relaxed(tiles + tile, tile_word(tag, 1, agg));
    uint32_t excl = 0;
    int j = (int)tile - 1;
    for (;;) {
        const int idx = j - lane;
        uint32_t fl = 2, val = 0;
        bool ok = true;
        if (idx >= 0) {
            const unsigned long long w = ld_relaxed(tiles + idx);
            ok = (uint32_t)(w >> 34) == tag && ((uint32_t)(w >> 32) & 3u) != 0;
            fl = (uint32_t)(w >> 32) & 3u;
            val = (uint32_t)w;
        }
        const unsigned incl = __ballot_sync(0xFFFFFFFFu, ok && fl == 2);
        const unsigned bad = __ballot_sync(0xFFFFFFFFu, !ok);
        if (incl) {
            const int f = __ffs(incl) - 1;                 // nearest inclusive predecessor
            if (bad & ((2u << f) - 1u)) continue;          // someone before it not published yet
            excl += __reduce_add_sync(0xFFFFFFFFu, lane <= f ? val : 0u);
            break;
        }
        if (bad) continue;
        excl += __reduce_add_sync(0xFFFFFFFFu, val);
        j -= 32;
    }
    if (lane == 0) st_relaxed(tiles + tile, tile_word(tag, 2, excl + agg));
    return excl;
}

// Reduce-all variant for grids whose tiles are all resident at once: warp 0 publishes
// this tile's aggregate, then sums the aggregates of ALL predecessors in parallel (lane
// k reads tiles k, k+32, ...; one round trip once they are published) instead of
// walking a look-back chain.  Returns the exclusive prefix in every lane.  Only valid
// when every predecessor tile is being processed concurrently (grid <= resident CTAs).
__device__ __forceinline__ uint32_t chain_scan_all(unsigned long long* tiles, uint32_t tile, uint32_t tag,
                                                   uint32_t agg)
{
    const int lane = threadIdx.x & 31;
    tag &= 0x3FFFFFFFu;
    if (lane == 0) st_relaxed(tiles + tile, tile_word(tag, 1, agg));
    uint32_t sum = 0;
    for (int j = lane; j < (int)tile; j += 32) {
        unsigned long long w;
        do {
            w = ld_relaxed(tiles + j);
        } while ((uint32_t)(w >> 34) != tag || ((uint32_t)(w >> 32) & 3u) == 0);
        sum += (uint32_t)w;
    }
    return __reduce_add_sync(0xFFFFFFFFu, sum);
}

__device__ __forceinline__ uint32_t take_ticket(Chain* c)
{
    __shared__ uint32_t t;
    if (threadIdx.x == 0) t = atomicAdd(&c->ticket, 1u);
    __syncthreads();
    uint32_t r = t;
    __syncthreads();
    return r;
}
// returns true in thread 0 of the last block to finish (after a fence)
__device__ __forceinline__ bool finish_block(Chain* c, uint32_t nblocks)
{
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t d = atomicAdd(&c->done, 1u);
        last = (d == nblocks - 1);
        if (last) {
            c->ticket = 0;
            c->done = 0;
            __threadfence();
        }
    }
    __syncthreads();
    return last;
}

}  // namespace am

namespace am {
// reset the per-round counters that the host reads (before the round kernels)
__device__ __forceinline__ void round_begin(const Dev& d)
{
    Ctl* ctl = d.ctl;
    ctl->epoch += 1;
    ctl->n_ready = 0;
    ctl->n_commit = 0;
    ctl->n_clusters = 0;
    ctl->n_items = 0;
    ctl->n_far = 0;
    ctl->scan_next = 0;
    ctl->sort_or = 0;
    ctl->ready.ticket = 0;   // k_ready and k_cells take tile tickets and keep no epilogue
    ctl->cells.ticket = 0;
    ctl->full |= ctl->full_next;
    ctl->full_next = 0;
    if (d.slot) {   // binned path: rebuild the cell binning, or keep the loose cells
        const bool rb = ctl->full != 0 || ctl->D > d.rebuild_d || ctl->since_rebuild >= d.rebuild_k ||
                        ctl->rebuild_req != 0 || !(d.flags & AM_VALIDATE);
        ctl->rebuild_req = 0;
        ctl->rebuild = rb ? 1 : 0;
        if (rb) {
            ctl->D = 0;
            ctl->since_rebuild = 0;
            ctl->n_rebuilds += 1;
        } else {
            ctl->since_rebuild += 1;
        }
    }
    if (ctl->epoch > 1) ctl->ecur ^= 1u;   // last round's edge lists become current
    ctl->ccnt[ctl->ecur ^ 1u] = 0;
    ctl->ncnt[ctl->ecur ^ 1u] = 0;
    if (d.wq_ctr)
        for (int k = 0; k < kEdgeStripes; k++) d.wq_ctr[k] = 0;
}

}  // namespace am

namespace am {
// neutral values of the post-commit reduction stripes (one thread)
__device__ __forceinline__ void cstripe_reset(const Dev& d)
{
    if (!d.cstripe) return;
    for (int k = 0; k < kCommitStripes; k++) {
        int32_t* c = d.cstripe + 32 * k;
        c[0] = INT_MAX; c[1] = INT_MIN; c[2] = 0; c[3] = 0;
    }
}
}  // namespace am
