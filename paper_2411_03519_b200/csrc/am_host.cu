// am_host.cu -- the C ABI (include/am.h): context, workspace, launch sequence.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <new>

#include "am_internal.cuh"

namespace am {
__global__ void k_ingest(Dev d, const int2* npos, const int32_t* nstep, const uint8_t* nstat, int mode, int bin);
__global__ void k_ingest_done(Dev d, int mode, int bin);
__global__ void k_bin(Dev d);
__global__ void k_cells(Dev d);
__global__ void k_scatter(Dev d);
__global__ void k_scan(Dev d);
__global__ void k_scan_thread(Dev d);
__global__ void k_finalize(Dev d, int early);
__global__ void k_union(Dev d);
__global__ void k_scan_hw(Dev d);
__global__ void k_scan_hw_full(Dev d);
__global__ void k_scan_hw_st(Dev d);
__global__ void k_scan_hw_full_st(Dev d);
__global__ void k_ready(Dev d, uint8_t* mask);
__global__ void k_sort_hist(Dev d, int max_passes);
__global__ void k_sort_pass(Dev d, int pass, int32_t* order, int ntiles);
__global__ void k_small(Dev d, uint8_t* mask, int32_t* order);
__global__ void k_round_begin(Dev d);
__global__ void k_efilter(Dev d);
__global__ void k_digest(Dev d, const int32_t* ids, const int32_t* count, const int32_t* gidmap,
                         unsigned long long* out);
__global__ void k_csort(Dev d, int32_t* order, int smem_bytes);
size_t csort_smem_fixed();
size_t csort_smem_need();
int csort_threads();

__global__ void k_copy_status(Dev d, uint8_t* out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < d.n) out[i] = d.status[d.ctl->cur][i];
}
}  // namespace am

using namespace am;

static thread_local std::string g_init_err;
static constexpr int kSortSmem = (32 + 1) * kRadix * 4;   // k_sort_pass dynamic shared memory

static int set_err(am_ctx* c, int code, const char* msg)
{
    if (c) c->err = msg; else g_init_err = msg;
    return code;
}

static int cuda_err(am_ctx* c, cudaError_t e, const char* where)
{
    char buf[256];
    snprintf(buf, sizeof buf, "%s: %s", where, cudaGetErrorString(e));
    return set_err(c, AM_E_CUDA, buf);
}

#define CK(ctx, call)                                         \
    do {                                                      \
        cudaError_t e_ = (call);                              \
        if (e_ != cudaSuccess) return cuda_err(ctx, e_, #call); \
    } while (0)

static int err_code(int bits)
{
    if (bits & ERR_BOUNDS) return AM_E_BOUNDS;
    if (bits & ERR_PROTOCOL) return AM_E_PROTOCOL;
    if (bits & ERR_VELOCITY) return AM_E_VELOCITY;
    return AM_OK;
}

static int ilog2_ceil(long long x)
{
    int l = 0;
    while ((1LL << l) < x) l++;
    return l;
}

static inline unsigned blocks(long long n, int t) { return (unsigned)std::max(1LL, (n + t - 1) / t); }

static const char* kKernelNames[K_COUNT] = {
    "k_ingest", "k_bin", "k_cells", "k_scatter", "k_scan", "k_finalize", "k_ready", "k_sort_hist",
    "k_sort_pass", "k_small", "k_commit", "k_disp_a", "k_disp_b", "k_union", "k_near"};

// inside a stream capture the records become external event nodes of the graph
static void prof_record(am_ctx* c, cudaEvent_t ev)
{
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(c->stream, &cs);
    if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(ev, c->stream, cudaEventRecordExternal);
    else cudaEventRecord(ev, c->stream);
}
void am_prof_begin(am_ctx* c, int id)
{
    if (c->prof.on && (c->prof.mask >> id & 1u)) prof_record(c, c->prof.ev[id][0]);
}
void am_prof_end(am_ctx* c, int id)
{
    if (c->prof.on && (c->prof.mask >> id & 1u)) {
        prof_record(c, c->prof.ev[id][1]);
        c->prof.pending |= 1u << id;
    }
}
// a graph captured with profiling mask `mask` was launched: its events are pending
void am_prof_mark(am_ctx* c, unsigned mask)
{
    if (c->prof.on) c->prof.pending |= mask;
}
// after a synchronisation: accumulate the recorded kernel times
void am_prof_collect(am_ctx* c)
{
    if (!c->prof.on) return;
    for (int k = 0; k < K_COUNT; k++) {
        if (!(c->prof.pending & (1u << k))) continue;
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, c->prof.ev[k][0], c->prof.ev[k][1]) == cudaSuccess) {
            c->prof.ms[k] += ms;
            c->prof.cnt[k] += 1;
        }
    }
    c->prof.pending = 0;
    cudaGetLastError();
}

extern "C" int am_profile_enable(am_ctx* c, uint32_t mask)
{
    if (!c) return set_err(nullptr, AM_E_ARG, "NULL context");
    if (mask && !c->prof.ev[0][0]) {
        for (int k = 0; k < K_COUNT; k++)
            for (int j = 0; j < 2; j++) CK(c, cudaEventCreate(&c->prof.ev[k][j]));
    }
    c->prof.on = mask != 0;
    c->prof.mask = mask;
    c->prof.pending = 0;
    for (int k = 0; k < K_COUNT; k++) { c->prof.ms[k] = 0; c->prof.cnt[k] = 0; }
    return AM_OK;
}

extern "C" int am_profile_read(am_ctx* c, double* ms, int64_t* counts, int32_t max)
{
    if (!c) return set_err(nullptr, AM_E_ARG, "NULL context");
    for (int k = 0; k < K_COUNT && k < max; k++) {
        if (ms) ms[k] = c->prof.ms[k];
        if (counts) counts[k] = c->prof.cnt[k];
    }
    return K_COUNT;
}

extern "C" int am_scan_stats(am_ctx* c, uint64_t* out)
{
    if (!c || !out) return set_err(c, AM_E_ARG, "NULL argument");
    CK(c, cudaMemcpyAsync(c->h_ctl, c->d.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    const Ctl& h = *c->h_ctl;
    out[0] = h.st_cells; out[1] = h.st_cand; out[2] = h.st_p2; out[3] = h.st_b2; out[4] = h.st_b1;
    out[5] = h.st_blocked;
    CK(c, cudaMemsetAsync(&c->d.ctl->st_cells, 0, 6 * sizeof(unsigned long long), c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    return AM_OK;
}

extern "C" int32_t am_launches_per_round(const am_ctx* c)
{
    if (!c) return 0;
    return c->path == 0 ? 3 : 11 - (AM_SCAN_UNITE ? 1 : 0) + (c->csort_ctas ? 1 : 1 + c->sort_passes_max) +
                                  ((c->d.flags & AM_DIGEST) ? 1 : 0);  // all launches of a round
}

extern "C" const char* am_profile_name(int32_t id)
{
    return (id >= 0 && id < K_COUNT) ? kKernelNames[id] : "";
}

extern "C" const char* am_version(void) { return "ametro-b200 0.1 (sm_100a)"; }

// The context's configuration and its device workspace layout -- a pure function of
// the arguments (no CUDA call), shared by am_workspace_size and am_init.
struct Layout {
    size_t total = 0;
    size_t ctl, pos0, pos1, st0, st1, ss0, ss1, labels, digest, blkid, tiles_s;
    size_t key = 0, cnt = 0, cmin = 0, ctab = 0, l1 = 0, l2 = 0, rec = 0, blk = 0, par = 0, bad = 0, rk0 = 0,
           rk1 = 0, rv0 = 0, rv1 = 0, tc = 0, tr = 0, tsort = 0, gh = 0, gs = 0, edges = 0, ectr = 0, wit = 0,
           lrs = 0, wq = 0, dirty = 0, agf = 0, rid = 0, slot = 0, cstripe = 0;
};

static int plan(am_ctx* x, int32_t map_w, int32_t map_h, int32_t radius_p, int32_t v_max, int32_t n_agents,
                const am_config* cfg, Layout& L)
{
    if (map_w < 1 || map_h < 1 || map_w > 32768 || map_h > 32768)
        return set_err(nullptr, AM_E_ARG, "am_init: map dims must be in [1, 32768]");
    if (radius_p < 0 || v_max < 0 || n_agents < 0 || n_agents > (1 << 28))
        return set_err(nullptr, AM_E_ARG, "am_init: negative radius/speed or bad agent count");
    am_config c{};
    c.n_sims = 1;
    c.flags = AM_VALIDATE;
    if (cfg) c = *cfg;
    if (c.n_sims < 1 || (n_agents > 0 && c.n_sims > n_agents))
        return set_err(nullptr, AM_E_ARG, "am_init: n_sims must be in [1, n_agents]");
    if (c.metric != AM_METRIC_L2 && c.metric != AM_METRIC_LINF && c.metric != AM_METRIC_GRAPH)
        return set_err(nullptr, AM_E_ARG, "am_init: unknown metric");
    if (c.metric == AM_METRIC_GRAPH && (map_h != 1 || (c.flags & AM_FORCE_BINNED)))
        return set_err(nullptr, AM_E_ARG, "am_init: the graph metric takes map_h == 1 (x = node) and the fused path");
    if (c.cell < 0 || (c.cell & (c.cell - 1)))
        return set_err(nullptr, AM_E_ARG, "am_init: cell must be 0 or a power of two");
    if (c.target_step < 0) return set_err(nullptr, AM_E_ARG, "am_init: negative target_step");

    const long long n = n_agents;
    const int per_sim_max = (int)((n + c.n_sims - 1) / c.n_sims);
    Dev& d = x->d;
    d.n = n_agents;
    d.n_sims = c.n_sims;
    d.map_w = map_w;
    d.map_h = map_h;
    // radii at or above kRClamp already cover every distance on a <= 32768^2 map (their
    // squares stay < 2^31 and sums like r_p + v cannot wrap): clamping changes no result
    d.r_p = (int32_t)std::min<long long>(radius_p, kRClamp);
    d.v = (int32_t)std::min<long long>(v_max, kRClamp);
    d.target = c.target_step;
    d.metric = c.metric;
    d.flags = c.flags;
    x->stream = (cudaStream_t)c.stream;

    // path selection
    bool small = (c.n_sims > 1) || (n <= kSmallMax);
    if (c.flags & AM_FORCE_BINNED) small = false;
    if (c.flags & AM_FORCE_SMALL) small = true;
    if (small && per_sim_max > kSmallMax)
        return set_err(nullptr, AM_E_ARG, "am_init: fused path needs <= 1024 agents per simulation");
    if (!small && c.n_sims > 1) return set_err(nullptr, AM_E_ARG, "am_init: the binned path takes one simulation");
    if (!small && c.metric == AM_METRIC_GRAPH)
        return set_err(nullptr, AM_E_ARG, "am_init: the graph metric runs on the fused path (<= 1024 agents/sim)");
    x->path = small ? 0 : 1;
    x->small_threads = std::max(32, ((per_sim_max + 31) / 32) * 32);

    // cell size: >= R_c = r_p + v (coupling needs <= 2x2 cells), grown until the Morton
    // grid has at most max(N/2, 4096) cells (>= 2 agents per cell on average) and at most
    // 4096 cells per side.  (A/B on the replay round, tools/ab_round.py AM_CELL: C5 cells
    // of 8 / 16 / 32 / 64 tiles -> 167 / 167 / 146 / 173 us, C4 73 / 67 / 63 / 73 us; the
    // scan's per-cell box work shrinks while the cells stay small enough to prune.)  The grid is
    // rectangular (2^gxlog x 2^gylog cells, each side >= 64 cells, mkey): a long thin map
    // -- e.g. one spatial slab of a wide map -- gets a long thin cell table.
    long long Rc = (long long)d.r_p + d.v;
    auto gl = [&](long long extent, int cl) {
        return ilog2_ceil(std::max(64LL, (extent + (1LL << cl) - 1) >> cl));
    };
    int clog;
    int cell_knob = 0;   // tuning knob (A/B of the grid density): a forced cell edge
    if (!c.cell)
        if (const char* e = getenv("AM_CELL")) cell_knob = std::max(0, atoi(e));
    if (c.cell || cell_knob) {
        clog = ilog2_ceil(c.cell ? c.cell : cell_knob);
    } else {
        clog = ilog2_ceil(std::max(1LL, Rc));
        for (;;) {
            const long long g = 1LL << (gl(map_w, clog) + gl(map_h, clog));
            if (g <= std::max(n / 2, 4096LL) || clog >= 15) break;
            clog++;
        }
    }
    while (std::max(gl(map_w, clog), gl(map_h, clog)) > 12 && clog < 15) clog++;   // <= 4096 cells per side
    d.gxlog = gl(map_w, clog);
    d.gylog = gl(map_h, clog);
    d.mbits = std::min(d.gxlog, d.gylog);
    d.mxhi = d.gxlog > d.gylog ? 1 : 0;
    d.clog = clog;
    d.ncells = 1 << (d.gxlog + d.gylog);
    x->cell = 1 << clog;
    d.idbits = std::max(1, ilog2_ceil(std::max(2LL, n)));
    d.lagcap = (int32_t)(kRClamp / (uint32_t)std::max(1, d.v)) + 1;
    {
        int lagbits = c.target_step > 0 ? ilog2_ceil((long long)c.target_step + 1) : 31;
        int bits = lagbits + d.idbits;
        x->sort_passes_max = std::min(kMaxSortPasses, std::max(1, (bits + kRadixBits - 1) / kRadixBits));
    }
    x->ntiles_sort = (int)blocks(n, kSortTile);
    x->ntiles_ready = (int)blocks(n, kReadyTile);
    x->cells_threads = (int)std::min<long long>(kCellsThreads, d.ncells / 16);
    x->ntiles_cells = (int)(d.ncells / (16LL * x->cells_threads));

    // workspace layout
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
    const size_t N = (size_t)std::max(1LL, n);
    L.ctl = take(sizeof(Ctl));
    L.pos0 = take(8 * N); L.pos1 = take(8 * N);
    L.st0 = take(4 * N); L.st1 = take(4 * N);
    L.ss0 = take(N); L.ss1 = take(N);
    L.labels = take(4 * N); L.digest = take(8 * N); L.blkid = take(N);
    L.tiles_s = take(8 * (size_t)c.n_sims);
    const size_t NC = (size_t)d.ncells;
    if (x->path == 1) {
        L.key = take(4 * N);
        L.cnt = take(4 * NC); L.cmin = take(4 * NC);
        L.ctab = take(8 * (NC + 1)); L.l1 = take(4 * (NC / 16)); L.l2 = take(4 * (NC / 256));
        L.rec = take(16 * N); L.blk = take(N);
        L.par = take(4 * N); L.bad = take(N); L.dirty = take(4 * N); L.agf = take(N);
        L.rk0 = take(8 * N); L.rk1 = take(8 * N); L.rid = take(4 * N); L.rv0 = take(4 * N); L.rv1 = take(4 * N);
        L.tc = take(8 * (size_t)x->ntiles_cells); L.tr = take(8 * (size_t)x->ntiles_ready);
        L.tsort = take(8 * (size_t)kMaxSortPasses * x->ntiles_sort * kRadix);
        L.gh = take(4 * kMaxSortPasses * kRadix); L.gs = take(4 * kMaxSortPasses * kRadix);
        d.ecap = (int)(3 * N + 4096);
        // the scan's work queue: stripes = block index mod 64 of k_scatter (one thread per
        // agent), so a stripe holds at most ceil(blocks / 64) x 256 records
        const long long nbl = blocks(n, 256);
        d.wq_cap = (int)(((nbl + kEdgeStripes - 1) / kEdgeStripes) * 256);
        L.wit = take(4 * N); L.lrs = take(N); L.slot = take(4 * N); L.cstripe = take(4 * 32 * kCommitStripes);
        L.edges = take(8 * 4 * (size_t)d.ecap); L.ectr = take(4 * kEdgeStripes);
        L.wq = take(16 * (size_t)kEdgeStripes * d.wq_cap);
    }
    L.total = off;
    return AM_OK;
}

extern "C" size_t am_workspace_size(int32_t map_w, int32_t map_h, int32_t radius_p, int32_t v_max,
                                    int32_t n_agents, const am_config* cfg)
{
    am_ctx tmp;
    Layout L;
    if (plan(&tmp, map_w, map_h, radius_p, v_max, n_agents, cfg, L) != AM_OK) return 0;
    return L.total;
}

extern "C" int am_init(am_ctx** out, int32_t map_w, int32_t map_h, int32_t radius_p, int32_t v_max,
                       int32_t n_agents, const am_config* cfg)
{
    if (!out) return set_err(nullptr, AM_E_ARG, "am_init: out is NULL");
    *out = nullptr;
    am_ctx* x = new (std::nothrow) am_ctx();
    if (!x) return set_err(nullptr, AM_E_ARG, "am_init: out of host memory");
    Layout L;
    {
        const int rc = plan(x, map_w, map_h, radius_p, v_max, n_agents, cfg, L);
        if (rc != AM_OK) { delete x; return rc; }
    }
    if (cfg && cfg->workspace) {   // caller-owned device workspace (e.g. a torch uint8 tensor)
        if (cfg->workspace_bytes < L.total || ((uintptr_t)cfg->workspace & 255)) {
            delete x;
            return set_err(nullptr, AM_E_WORKSPACE, "am_init: workspace smaller than am_workspace_size() or "
                                                    "not 256-byte aligned");
        }
    }
    Dev& d = x->d;
    const long long n = n_agents;
    cudaFuncSetAttribute(k_sort_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, kSortSmem);
    if (const char* e = getenv("AM_SORT_CTAS")) x->sort_ctas = std::max(1, atoi(e));   // tuning knob
    if (const char* e = getenv("AM_PDL")) x->pdl = atoi(e) != 0;                      // ablation
    // the one-kernel cluster sort: the largest cluster (16, else 8) that can be resident
    {
        const char* e = getenv("AM_SORT");   // "onesweep" = multi-kernel ablation
        if (!(e && !strcmp(e, "onesweep"))) {
            int dev = 0, maxsm = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
            // shared memory: the fixed part + two tile buffers (8192 x 8 or 4096 x 16 bytes)
            const size_t need = csort_smem_need();
            const int cap = (size_t)maxsm >= need ? 1024 : 0;
            if (cap >= 1024 &&
                cudaFuncSetAttribute(k_csort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need) == cudaSuccess) {
                cudaFuncSetAttribute(k_csort, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                int want = 0;
                if (const char* q = getenv("AM_CSORT_CTAS")) want = atoi(q);   // tuning knob
                for (int cs : {16, 8, 4, 2, 1}) {
                    if (want && cs != want) continue;
                    cudaLaunchConfig_t lc{};
                    lc.gridDim = dim3(cs);
                    lc.blockDim = dim3(csort_threads());
                    lc.dynamicSmemBytes = need;
                    cudaLaunchAttribute at{};
                    at.id = cudaLaunchAttributeClusterDimension;
                    at.val.clusterDim.x = cs; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
                    lc.attrs = &at; lc.numAttrs = 1;
                    int ncl = 0;
                    if (cudaOccupancyMaxActiveClusters(&ncl, k_csort, &lc) == cudaSuccess && ncl >= 1) {
                        x->csort_ctas = cs;
                        x->csort_cap = (int)need;   // dynamic shared memory bytes per CTA
                        break;
                    }
                }
            }
            cudaGetLastError();
        }
    }
    {
        int dev = 0, sms = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        x->num_sms = sms > 0 ? sms : 148;
    }
    {   // the scan's persistent grid: exactly the resident blocks (no block waits for a slot)
        int per = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_scan_hw, 256, 0) == cudaSuccess && per > 0)
            x->scan_blocks = per * x->num_sms;
        cudaGetLastError();
        x->scan_blocks_full = x->scan_blocks;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_scan_hw_full, 256, 0) == cudaSuccess && per > 0)
            x->scan_blocks_full = per * x->num_sms;
        cudaGetLastError();
    }

    const size_t off = L.total;
    x->ws_bytes = off;
    cudaError_t e = cudaSuccess;
    if (cfg && cfg->workspace) {
        x->ws = cfg->workspace;
        x->ws_owned = false;
    } else {   // no caller workspace: the context allocates (and frees) its own
        e = cudaMalloc(&x->ws, off);
        if (e != cudaSuccess) { delete x; return cuda_err(nullptr, e, "am_init: cudaMalloc"); }
        x->ws_owned = true;
    }
    auto fail = [&](cudaError_t err, const char* where) {
        if (x->ws_owned) cudaFree(x->ws);
        if (x->h_ctl) cudaFreeHost(x->h_ctl);
        delete x;
        return cuda_err(nullptr, err, where);
    };
    if (x->path == 1) {
        e = cudaStreamCreateWithFlags(&x->side, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x->ev_fork, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x->ev_join, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x->ev_efil, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&x->side2, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x->ev_dig, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x->ev_mask, cudaEventDisableTiming);
        if (e != cudaSuccess) return fail(e, "am_init: side stream");
    }
    e = cudaMallocHost((void**)&x->h_ctl, sizeof(Ctl));
    if (e != cudaSuccess) { x->h_ctl = nullptr; return fail(e, "am_init: cudaMallocHost"); }
    char* b = (char*)x->ws;
    d.ctl = (Ctl*)(b + L.ctl);
    d.pos[0] = (int2*)(b + L.pos0); d.pos[1] = (int2*)(b + L.pos1);
    d.step[0] = (int32_t*)(b + L.st0); d.step[1] = (int32_t*)(b + L.st1);
    d.status[0] = (uint8_t*)(b + L.ss0); d.status[1] = (uint8_t*)(b + L.ss1);
    d.labels = (int32_t*)(b + L.labels);
    d.blkid = (uint8_t*)(b + L.blkid);
    d.digest = (unsigned long long*)(b + L.digest);
    d.tiles_s = (unsigned long long*)(b + L.tiles_s);
    const size_t NC = (size_t)d.ncells;
    const size_t N = (size_t)std::max(1LL, n);
    if (x->path == 1) {
        d.key = (uint32_t*)(b + L.key);
        d.cnt = (uint32_t*)(b + L.cnt); d.cmin = (int32_t*)(b + L.cmin);
        d.ctab = (int2*)(b + L.ctab); d.lmin1 = (int32_t*)(b + L.l1); d.lmin2 = (int32_t*)(b + L.l2);
        d.rec = (int4*)(b + L.rec); d.v8 = (uint8_t*)(b + L.blk);
        d.parent = (uint32_t*)(b + L.par); d.bad = (uint8_t*)(b + L.bad); d.dirty = (uint32_t*)(b + L.dirty); d.agflag = (uint8_t*)(b + L.agf);
        d.rid = (int32_t*)(b + L.rid); d.rkey[0] = (unsigned long long*)(b + L.rk0); d.rkey[1] = (unsigned long long*)(b + L.rk1);
        d.rval[0] = (uint32_t*)(b + L.rv0); d.rval[1] = (uint32_t*)(b + L.rv1);
        d.tiles_c = (unsigned long long*)(b + L.tc); d.tiles_r = (unsigned long long*)(b + L.tr);
        d.tiles_sort = (unsigned long long*)(b + L.tsort);
        d.ghist = (uint32_t*)(b + L.gh); d.gstart = (uint32_t*)(b + L.gs);
        d.cedges = (uint2*)(b + L.edges); d.nedges = d.cedges + 2 * (size_t)d.ecap; d.wq_ctr = (uint32_t*)(b + L.ectr); d.wq = (int4*)(b + L.wq);
        d.witness = (uint32_t*)(b + L.wit); d.chg8 = (uint8_t*)(b + L.lrs);
        d.slot = (uint32_t*)(b + L.slot);
        d.cstripe = (int32_t*)(b + L.cstripe);
        // loose-cell rebuild policy (tuning knobs)
        d.rebuild_d = AM_REBUILD_D;
        d.rebuild_k = AM_REBUILD_K;
        if (const char* q = getenv("AM_REBUILD_D")) d.rebuild_d = atoi(q);
        if (const char* q = getenv("AM_REBUILD_K")) d.rebuild_k = atoi(q);
    }
    // initial contents: everything zero except the min-step table
    e = cudaMemsetAsync(x->ws, 0, off, x->stream);
    if (e == cudaSuccess && x->path == 1) e = cudaMemsetAsync(d.cmin, 0x7F, 4 * NC, x->stream);  // ~INT_MAX
    if (e == cudaSuccess && x->path == 1) e = cudaMemsetAsync(d.witness, 0xFF, 4 * N, x->stream);
    if (e == cudaSuccess && x->path == 1) e = cudaMemsetAsync(d.slot, 0xFF, 4 * N, x->stream);
    int32_t h_stripes[32 * kCommitStripes] = {};
    for (int k = 0; k < kCommitStripes; k++) { h_stripes[32 * k] = INT_MAX; h_stripes[32 * k + 1] = INT_MIN; }
    if (e == cudaSuccess && x->path == 1)
        e = cudaMemcpyAsync(d.cstripe, h_stripes, sizeof h_stripes, cudaMemcpyHostToDevice, x->stream);
    Ctl h{};
    h.acc_W = INT_MAX;
    h.acc_S = INT_MIN;
    h.W = INT_MAX;
    h.S = INT_MIN;
    h.full = 1;
    if (e == cudaSuccess) e = cudaMemcpyAsync(d.ctl, &h, sizeof h, cudaMemcpyHostToDevice, x->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(x->stream);
    if (e != cudaSuccess) return fail(e, "am_init: workspace init");
    x->stats.path = x->path;
    x->stats.cell = x->cell;
    *out = x;
    return AM_OK;
}


static int launch_ingest(am_ctx* c, const int32_t* pos, const int32_t* steps, const uint8_t* st, int mode,
                         bool bin = false)
{
    if (!c) return set_err(nullptr, AM_E_ARG, "NULL context");
    if (c->d.n == 0) return AM_OK;
    if (!pos || !steps || ((mode == 2 || mode == 3) && !st)) return set_err(c, AM_E_ARG, "NULL array");
    if (c->bin_pending) return set_err(c, AM_E_STATE, "update after a binned update without a round");
    if (c->d.metric == AM_METRIC_GRAPH && !c->d.gdist) return set_err(c, AM_E_STATE, "am_set_graph first");
    am_join_side(c);
    if (mode == 1 || mode == 2) c->full_hint = true;   // initial / set state: the next round recomputes everything
    am_prof_begin(c, K_INGEST);
    CK(c, launch_k(c->pdl, c->stream, k_ingest, blocks(c->d.n, 256 * kIngestItems), 256, 0, c->d, (const int2*)pos, steps, st, mode, bin ? 1 : 0));
    CK(c, launch_k(c->pdl, c->stream, k_ingest_done, 1, 1, 0, c->d, mode, bin ? 1 : 0));
    am_prof_end(c, K_INGEST);
    CK(c, cudaGetLastError());
    return AM_OK;
}

extern "C" int am_update(am_ctx* c, const int32_t* positions, const int32_t* sim_steps)
{
    if (!c) return set_err(nullptr, AM_E_ARG, "NULL context");
    const bool first = c->first;
    int rc = launch_ingest(c, positions, sim_steps, nullptr, first ? 1 : 0);
    if (rc) return rc;
    if (first) {
        rc = am_sync(c);  // the initial state is checked synchronously
        if (rc == AM_OK) c->first = false;
    }
    return rc;
}

// Replay rounds (am_driver.cu): the commit update with the cell binning of the round
// fused in (k_bin is skipped by the am_ready that must follow immediately).
int am_update_binned(am_ctx* c, const int32_t* positions, const int32_t* sim_steps)
{
    if (!c) return set_err(nullptr, AM_E_ARG, "NULL context");
    if (c->first || c->path != 1) return am_update(c, positions, sim_steps);
    const int rc = launch_ingest(c, positions, sim_steps, nullptr, 0, true);
    if (rc == AM_OK) c->bin_pending = true;
    return rc;
}

extern "C" int am_set_graph(am_ctx* c, const uint16_t* dist, int32_t n_nodes)
{
    if (!c) return set_err(nullptr, AM_E_ARG, "NULL context");
    if (c->d.metric != AM_METRIC_GRAPH || !dist || n_nodes != c->d.map_w)
        return set_err(c, AM_E_ARG, "am_set_graph: needs AM_METRIC_GRAPH and an n_nodes == map_w distance table");
    c->d.gdist = dist;
    c->d.gV = n_nodes;
    return AM_OK;
}

extern "C" int am_update_replica(am_ctx* c, const int32_t* positions, const int32_t* sim_steps,
                                 const uint8_t* status)
{
    if (!c) return set_err(nullptr, AM_E_ARG, "NULL context");
    if (c->first) return am_set_state(c, positions, sim_steps, status);
    return launch_ingest(c, positions, sim_steps, status, 3);   // stream-ordered; errors at the next sync
}

extern "C" int am_set_state(am_ctx* c, const int32_t* positions, const int32_t* sim_steps,
                            const uint8_t* status)
{
    if (!c) return set_err(nullptr, AM_E_ARG, "NULL context");
    int rc = launch_ingest(c, positions, sim_steps, status, 2);
    if (rc) return rc;
    if (c->d.flags & AM_ASYNC) {   // stream-ordered; a rejected state surfaces at the next sync
        c->first = false;
        return AM_OK;
    }
    rc = am_sync(c);
    if (rc == AM_OK) c->first = false;
    return rc;
}

static void fill_stats(am_ctx* c)
{
    const Ctl& h = *c->h_ctl;
    c->stats.n_ready = h.n_ready;
    c->stats.n_active = h.n_active;
    c->stats.n_running = h.n_running;
    c->stats.watermark = h.W;
    c->stats.max_step = h.S;
    c->stats.n_clusters = h.n_clusters;
    c->stats.n_work = h.n_work;
    c->stats.n_far = h.n_far;
    c->stats.n_items = h.n_items;
    c->stats.n_edges = h.n_edges;
    c->stats.n_passes = h.npasses;
    c->stats.rebuilt = h.rebuild;
    c->stats.drift = h.D;
    c->stats.n_rebuilds = h.n_rebuilds;
}

// the main stream waits for the perception digests of the last round (side2)
void am_join_digest(am_ctx* c)
{
    if (c->dig_pending) {
        cudaStreamWaitEvent(c->stream, c->ev_dig, 0);
        c->dig_pending = false;
    }
}

// the main stream waits for the side-stream sort of the last round
void am_join_side(am_ctx* c)
{
    am_join_digest(c);
    if (c->join_pending) {
        cudaStreamWaitEvent(c->stream, c->ev_join, 0);
        c->join_pending = false;
    }
}

extern "C" int am_sync(am_ctx* c)
{
    if (!c) return set_err(nullptr, AM_E_ARG, "NULL context");
    am_join_side(c);
    CK(c, cudaMemcpyAsync(c->h_ctl, c->d.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    fill_stats(c);
    am_prof_collect(c);
    const int bits = c->h_ctl->err_sticky;
    if (bits) {
        CK(c, cudaMemsetAsync(&c->d.ctl->err_sticky, 0, sizeof(int32_t), c->stream));
        CK(c, cudaStreamSynchronize(c->stream));
        const int code = err_code(bits);
        return set_err(c, code, code == AM_E_BOUNDS ? "update rejected: position out of bounds"
                              : code == AM_E_PROTOCOL ? "update rejected: protocol violation"
                                                      : "update rejected: velocity limit exceeded");
    }
    return AM_OK;
}

extern "C" int am_ready(am_ctx* c, uint8_t* mask, int32_t* order, int32_t* n_ready)
{
    if (!c) return set_err(nullptr, AM_E_ARG, "NULL context");
    if (c->first) return set_err(c, AM_E_STATE, "am_ready before the initial am_update");
    const bool async = (c->d.flags & AM_ASYNC) != 0;
    if (!async && !n_ready) return set_err(c, AM_E_ARG, "n_ready is NULL");
    if (c->d.n == 0) {
        if (n_ready) *n_ready = 0;
        return AM_OK;
    }
    const bool labels_only = c->path == 1 && (c->d.flags & AM_LABELS_ONLY);
    if ((!mask || !order) && !labels_only) return set_err(c, AM_E_ARG, "NULL mask/order");
    am_join_side(c);   // the previous round's sort reads the buffers this round rewrites
    const Dev& d = c->d;
    cudaStream_t s = c->stream;
#define LAUNCH(id, ...)        \
    do {                       \
        am_prof_begin(c, id);  \
        __VA_ARGS__;           \
        am_prof_end(c, id);    \
    } while (0)
    if (!c->bin_pending) CK(c, launch_k(c->pdl, s, k_round_begin, 1, 1, 0, d));   // else done by k_ingest_done
    if (c->path == 0) {
        LAUNCH(K_SMALL, CK(c, launch_k(c->pdl, s, k_small, d.n_sims, c->small_threads, 0, d, mask, order)));
    } else {
        const unsigned nb = blocks(d.n, 256);
        // k_bin / k_cells return at once on loose-cell rounds (the device decides: a rebuild
        // is due after a full recompute, a drift beyond rebuild_d, or rebuild_k rounds)
        LAUNCH(K_BIN, CK(c, launch_k(c->pdl, s, k_bin, std::min(nb, (unsigned)c->num_sms * 8), 256, 0, d)));
        c->bin_pending = false;
        LAUNCH(K_CELLS, CK(c, launch_k(c->pdl, s, k_cells, c->ntiles_cells, c->cells_threads, 0, d)));
        LAUNCH(K_SCATTER, CK(c, launch_k(c->pdl, s, k_scatter, nb, 256, 0, d)));
        if (d.flags & AM_SCAN_THREAD)   // ablation: everything recomputed, no witnesses
            LAUNCH(K_SCAN, CK(c, launch_k(c->pdl, s, k_scan_thread, nb, 256, 0, d)));
        else
        {
            const unsigned pers = (unsigned)c->num_sms * 8;   // persistent grid-stride kernels
            // coupling edges of unchanged pairs carried over; scan of the work queue
            // the carried edges (k_efilter, side stream) beside the scan of the work queue
            // (one half-warp per queued agent: near phase, then far phase; main stream)
            CK(c, cudaEventRecord(c->ev_fork, s));
            CK(c, cudaStreamWaitEvent(c->side, c->ev_fork, 0));
            {
                // the profiling events of k_efilter go on its stream; the context's stream is
                // restored before any error is returned
                cudaStream_t ms = c->stream;
                c->stream = c->side;
                am_prof_begin(c, K_NEAR);
                const cudaError_t le = launch_k(false, c->side, k_efilter, std::min(blocks(2LL * d.ecap, 256), pers), 256, 0, d);
                am_prof_end(c, K_NEAR);
                c->stream = ms;
                if (le != cudaSuccess) return cuda_err(c, le, "k_efilter launch");
            }
            CK(c, cudaEventRecord(c->ev_efil, c->side));
            {
                // a round the host knows is a full recompute (initial / set state, no commit
                // validation) outside a graph capture takes the smaller direct box; every
                // other round (the replay's incremental rounds, device-detected full rounds)
                // the incremental kernel.  Both are exact; only the pruning granularity differs.
                cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
                CK(c, cudaStreamIsCapturing(s, &cs));
                const bool full = (c->full_hint || !(d.flags & AM_VALIDATE)) && cs == cudaStreamCaptureStatusNone;
                const unsigned g = std::min(blocks(d.n, 16), (unsigned)(full ? c->scan_blocks_full : c->scan_blocks));
                const bool st = (d.flags & AM_STATS) != 0;   // the instantiation with work counters
                if (full)
                    LAUNCH(K_SCAN, CK(c, launch_k(c->pdl, s, st ? k_scan_hw_full_st : k_scan_hw_full, g, 256, 0, d)));
                else
                    LAUNCH(K_SCAN, CK(c, launch_k(c->pdl, s, st ? k_scan_hw_st : k_scan_hw, g, 256, 0, d)));
                c->full_hint = false;
            }
            CK(c, cudaStreamWaitEvent(s, c->ev_efil, 0));
            if (!AM_SCAN_UNITE)   // else the scan united its new edges as it flushed them
                LAUNCH(K_UNION, CK(c, launch_k(c->pdl, s, k_union, std::min(blocks(d.ecap, 256), pers), 256, 0, d)));
        }
        {   // early loads when k_union precedes it (not the ablation scan, not AM_SCAN_UNITE)
            const int early = (c->pdl && !(d.flags & AM_SCAN_THREAD) && !AM_SCAN_UNITE) ? 1 : 0;
            LAUNCH(K_FINALIZE, CK(c, launch_k(c->pdl, s, k_finalize, blocks(d.n, 256 * kFinItems), 256, 0, d, early)));
        }
        if (!labels_only) {   // else labels and verdicts are final (AM_LABELS_ONLY)
            LAUNCH(K_READY, CK(c, launch_k(c->pdl, s, k_ready, c->ntiles_ready, kReadyThreads, 0, d, mask)));
            // the mask is final here: a caller may copy it out beside the rest of the round
            if (c->mask_event && c->ev_mask) CK(c, cudaEventRecord(c->ev_mask, s));
            static const bool dbg_nosort = [] { const char* e = getenv("AM_DBG_NOSORT"); return e && atoi(e); }();
            if (dbg_nosort || (d.flags & AM_NO_ORDER)) {
                // PROFILING ONLY (wrong `order`): measures how much of the round the sort holds up
            } else if (c->csort_ctas) {
                // one cluster of csort_ctas CTAs sorts the whole ready set (am_sort.cu), on the
                // side stream: nothing else in the round reads `order` (digests and dispatch
                // take the id-ordered ready list), so it overlaps the rest of the round and
                // joins the main stream at am_join_side (end of a replay round, am_sync)
                CK(c, cudaEventRecord(c->ev_fork, s));
                CK(c, cudaStreamWaitEvent(c->side, c->ev_fork, 0));
                cudaLaunchConfig_t lc{};
                lc.gridDim = dim3(c->csort_ctas);
                lc.blockDim = dim3(csort_threads());
                lc.dynamicSmemBytes = (size_t)c->csort_cap;
                lc.stream = c->side;
                cudaLaunchAttribute at{};
                at.id = cudaLaunchAttributeClusterDimension;
                at.val.clusterDim.x = c->csort_ctas; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
                lc.attrs = &at; lc.numAttrs = 1;
                cudaStream_t ms = c->stream;
                c->stream = c->side;   // profiling events of the sort on its stream
                am_prof_begin(c, K_SORT_PASS);
                const cudaError_t le = cudaLaunchKernelEx(&lc, k_csort, d, order, c->csort_cap);
                am_prof_end(c, K_SORT_PASS);
                c->stream = ms;
                if (le != cudaSuccess) return cuda_err(c, le, "k_csort launch");
                CK(c, cudaEventRecord(c->ev_join, c->side));
                c->join_pending = true;
            } else {
                LAUNCH(K_SORT_HIST, CK(c, launch_k(c->pdl, s, k_sort_hist, std::min(c->ntiles_sort, 32), 256, 0, d, c->sort_passes_max)));
                am_prof_begin(c, K_SORT_PASS);
                for (int p = 0; p < c->sort_passes_max; p++)   // persistent: <= 16 CTAs take tiles
                    CK(c, launch_k(c->pdl, s, k_sort_pass, std::min(c->ntiles_sort, c->sort_ctas), 1024, kSortSmem, d, p, order, c->ntiles_sort));
                am_prof_end(c, K_SORT_PASS);
            }
            // perception digests of the dispatched agents (replay driver), on a second side
            // stream forked after k_ready: they overlap the driver's dispatch part a, which
            // does not read them; the driver joins them (am_join_digest) before part b
            if (d.flags & AM_DIGEST) {
                CK(c, cudaEventRecord(c->ev_fork, s));
                CK(c, cudaStreamWaitEvent(c->side2, c->ev_fork, 0));
                CK(c, launch_k(false, c->side2, k_digest, std::min(blocks(d.n, 16), (unsigned)c->num_sms * 8), 256, 0, d,
                               (const int32_t*)d.rid, (const int32_t*)nullptr, (const int32_t*)nullptr,
                               (unsigned long long*)nullptr));
                CK(c, cudaEventRecord(c->ev_dig, c->side2));
                c->dig_pending = true;
            }
        }
    }
#undef LAUNCH
    CK(c, cudaGetLastError());
    c->have_round = true;
    // the caller's stream waits for the side-stream priority sort (an event wait, no host
    // synchronisation): `order` is complete for any later work on the context's stream.
    // The replay driver's own round (defer_join) joins it after dispatch and commit
    // instead, which do not read `order`, so the sort overlaps them.
    if (!c->defer_join) am_join_side(c);
    if (async) return AM_OK;
    int rc = am_sync(c);
    *n_ready = rc == AM_OK ? c->h_ctl->n_ready : 0;
    return rc;
}

extern "C" int am_clusters(am_ctx* c, int32_t* labels)
{
    if (!c) return set_err(nullptr, AM_E_ARG, "NULL context");
    if (!labels) return set_err(c, AM_E_ARG, "NULL labels");
    if (!c->have_round) return set_err(c, AM_E_STATE, "am_clusters before any am_ready");
    if (c->d.n == 0) return AM_OK;
    CK(c, cudaMemcpyAsync(labels, c->d.labels, 4 * (size_t)c->d.n, cudaMemcpyDeviceToDevice, c->stream));
    return AM_OK;
}

extern "C" int am_blocked(am_ctx* c, uint8_t* blocked)
{
    if (!c) return set_err(nullptr, AM_E_ARG, "NULL context");
    if (!blocked) return set_err(c, AM_E_ARG, "NULL blocked");
    if (!c->have_round) return set_err(c, AM_E_STATE, "am_blocked before any am_ready");
    if (c->d.n == 0) return AM_OK;
    CK(c, cudaMemcpyAsync(blocked, c->d.blkid, (size_t)c->d.n, cudaMemcpyDeviceToDevice, c->stream));
    return AM_OK;
}

extern "C" int am_status(am_ctx* c, uint8_t* status)
{
    if (!c) return set_err(nullptr, AM_E_ARG, "NULL context");
    if (!status) return set_err(c, AM_E_ARG, "NULL status");
    if (c->d.n == 0) return AM_OK;
    k_copy_status<<<blocks(c->d.n, 256), 256, 0, c->stream>>>(c->d, status);
    CK(c, cudaGetLastError());
    return AM_OK;
}

extern "C" int am_stats(const am_ctx* c, am_round_stats* out)
{
    if (!c || !out) return AM_E_ARG;
    *out = c->stats;
    return AM_OK;
}

extern "C" int am_set_flags(am_ctx* c, uint32_t flags)
{
    if (!c) return set_err(nullptr, AM_E_ARG, "NULL context");
    if (c->path == 1 && ((flags ^ c->d.flags) & AM_SCAN_THREAD)) {
        // the ablation scan keeps no blocking witnesses: recompute everything next round
        const int32_t one = 1;
        c->full_hint = true;
        CK(c, cudaMemcpyAsync(&c->d.ctl->full, &one, sizeof one, cudaMemcpyHostToDevice, c->stream));
        CK(c, cudaStreamSynchronize(c->stream));
    }
    c->d.flags = flags;
    return AM_OK;
}

extern "C" int am_set_stream(am_ctx* c, void* stream)
{
    if (!c) return set_err(nullptr, AM_E_ARG, "NULL context");
    c->stream = (cudaStream_t)stream;
    return AM_OK;
}

extern "C" void* am_get_stream(const am_ctx* c) { return c ? (void*)c->stream : nullptr; }

extern "C" int am_reset(am_ctx* c)
{
    if (!c) return set_err(nullptr, AM_E_ARG, "NULL context");
    c->first = true;
    c->have_round = false;
    c->bin_pending = false;   // a replay capture that failed between update and round
    c->full_hint = true;
    return AM_OK;
}

extern "C" size_t am_workspace_bytes(const am_ctx* c) { return c ? c->ws_bytes : 0; }

extern "C" const int32_t* am_ready_count_device(const am_ctx* c) { return c ? &c->d.ctl->n_ready : nullptr; }

extern "C" int am_destroy(am_ctx* c)
{
    if (!c) return AM_OK;
    cudaStreamSynchronize(c->stream);
    if (c->prof.ev[0][0])
        for (int k = 0; k < K_COUNT; k++)
            for (int j = 0; j < 2; j++) cudaEventDestroy(c->prof.ev[k][j]);
    if (c->side) {
        cudaStreamSynchronize(c->side);
        cudaStreamDestroy(c->side);
        cudaEventDestroy(c->ev_fork);
        cudaEventDestroy(c->ev_join);
        cudaEventDestroy(c->ev_efil);
        cudaStreamSynchronize(c->side2);
        cudaStreamDestroy(c->side2);
        cudaEventDestroy(c->ev_dig);
        cudaEventDestroy(c->ev_mask);
    }
    if (c->ws_owned) cudaFree(c->ws);
    cudaFreeHost(c->h_ctl);
    delete c;
    return AM_OK;
}

extern "C" const char* am_last_error(const am_ctx* c) { return c ? c->err.c_str() : g_init_err.c_str(); }

// ---------------------------------------------------------------- for am_slab.cu
// perception digests of the listed agents (ids[0 .. *count)) from the context's last
// round (records, cell table), perceived ids mapped through gidmap; into out[id]
int am_internal_digest(am_ctx* c, const int32_t* ids, const int32_t* count, const int32_t* gidmap,
                       unsigned long long* out, int max_ids, cudaStream_t s)
{
    if (c->path != 1) return set_err(c, AM_E_ARG, "digest list: binned path only");
    CK(c, launch_k(false, s, k_digest, std::min(blocks(std::max(1, max_ids), 16), (unsigned)c->num_sms * 8), 256, 0,
                   c->d, ids, count, gidmap, out));
    return AM_OK;
}

// the context's one-kernel cluster sort on another key set (sd: rkey / rval ping-pong
// buffers and a control block holding n_ready and sort_or): order[k] = rval of the k-th key
int am_internal_csort(am_ctx* c, const Dev& sd, int32_t* order, cudaStream_t s)
{
    if (!c->csort_ctas) return set_err(c, AM_E_ARG, "cluster sort unavailable on this device");
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(c->csort_ctas);
    lc.blockDim = dim3(csort_threads());
    lc.dynamicSmemBytes = (size_t)c->csort_cap;
    lc.stream = s;
    cudaLaunchAttribute at{};
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = c->csort_ctas; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
    lc.attrs = &at; lc.numAttrs = 1;
    CK(c, cudaLaunchKernelEx(&lc, k_csort, sd, order, c->csort_cap));
    return AM_OK;
}
