// am_slab.cu -- spatial-slab decomposition kernels (include/am_slab.h).
#include <algorithm>
#include <climits>
#include <cstdio>

#include "am_internal.cuh"
#include "am_slab.h"

namespace am {

__device__ __forceinline__ int slab_lo(int k, int G, int H) { return (int)((long long)k * H / G); }

__global__ void k_slab_watermark(int n, const int32_t* __restrict__ steps, const uint8_t* __restrict__ status,
                                 int32_t* out)
{
    int mn = INT_MAX, nmx = INT_MAX;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (status[i] == ST_DONE) continue;
        mn = min(mn, steps[i]);
        nmx = min(nmx, -steps[i]);
    }
    mn = __reduce_min_sync(0xFFFFFFFFu, mn);
    nmx = __reduce_min_sync(0xFFFFFFFFu, nmx);
    if ((threadIdx.x & 31) == 0) {
        if (mn != INT_MAX) atomicMin(out, mn);
        if (nmx != INT_MAX) atomicMin(out + 1, nmx);
    }
}

// the local tracker's input: owned agents (slots [0, n)), received ghosts ([n, n + m)),
// DONE padding up to cap; y translated by -y0 (the slab's halo window)
__global__ void k_slab_assemble(int n, const int32_t* __restrict__ gid, const int2* __restrict__ pos,
                                const int32_t* __restrict__ steps, const uint8_t* __restrict__ status, int m,
                                const int4* __restrict__ ghosts, int cap, int y0, int2* __restrict__ lpos,
                                int32_t* __restrict__ lsteps, uint8_t* __restrict__ lstatus,
                                int32_t* __restrict__ lgid)
{
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < cap; k += gridDim.x * blockDim.x) {
        int2 p = make_int2(0, 0);
        int s = 0, g = 0;
        uint8_t st = ST_DONE;
        if (k < n) {
            p = pos[k];
            p.y -= y0;
            s = steps[k];
            st = status[k];
            g = gid[k];
        } else if (k < n + m) {
            const int4 r = ghosts[k - n];
            p = make_int2(r.y & 0xFFFF, (r.y >> 16) - y0);
            s = r.z;
            st = (uint8_t)r.w;
            g = r.x;
        }
        lpos[k] = p;
        lsteps[k] = s;
        lstatus[k] = st;
        lgid[k] = g;
    }
}

__global__ void k_slab_init2(int32_t* out)
{
    out[0] = INT_MAX;
    out[1] = INT_MAX;
}

// owned agent B goes to every other slab whose rows are within R_b(S - s_B)
__global__ void k_slab_halo(am_slab_geom g, int n, const int32_t* __restrict__ gid, const int2* __restrict__ pos,
                            const int32_t* __restrict__ steps, const uint8_t* __restrict__ status,
                            const int32_t* __restrict__ ws, int cap, int4* __restrict__ send,
                            int32_t* __restrict__ counts, uint8_t* __restrict__ sent)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t st = status[i];
    bool any = false;
    if (st != ST_DONE) {
        const int S = -ws[1];
        const int2 p = pos[i];
        const int s = steps[i];
        const uint32_t R = rb_radius((long long)S - s, g.v_max, g.r_p);
        for (int j = 0; j < g.n_slabs; j++) {
            if (j == g.my_slab) continue;
            const int y0 = slab_lo(j, g.n_slabs, g.map_h), y1 = slab_lo(j + 1, g.n_slabs, g.map_h) - 1;
            if (y1 < y0) continue;
            const int dy = p.y < y0 ? y0 - p.y : (p.y > y1 ? p.y - y1 : 0);
            if ((uint32_t)dy > R) continue;   // |dy| <= dist under L2 and L-infinity
            const int k = atomicAdd(counts + j, 1);
            if (k < cap) send[(size_t)j * cap + k] = make_int4(gid[i], p.x | (p.y << 16), s, st);
            any = true;
        }
    }
    sent[i] = any;
}

__global__ void k_slab_zero(int32_t* a, int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = 0;
}

// pass 1: boundary flag and owned-bad flag per local root
__global__ void k_slab_mark(int n_local, int n_owned, const int32_t* __restrict__ labels,
                            const uint8_t* __restrict__ status, const uint8_t* __restrict__ blocked,
                            const uint8_t* __restrict__ sent, uint8_t* badlocal, uint8_t* bnd)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_local) return;
    const int l = labels[i];
    if (l < 0) return;
    const bool owned = i < n_owned;
    if (!owned || sent[i]) bnd[l] = 1;
    if (owned && (status[i] == ST_RUNNING || blocked[i])) badlocal[l] = 1;
}

// pass 2: link records of boundary agents, bad records of bad boundary roots
__global__ void k_slab_emit(int n_local, int n_owned, const int32_t* __restrict__ gid,
                            const int32_t* __restrict__ labels, const uint8_t* __restrict__ sent,
                            const uint8_t* __restrict__ badlocal, const uint8_t* __restrict__ bnd, int cap,
                            int2* __restrict__ links, int32_t* n_links, int32_t* __restrict__ bads,
                            int32_t* n_bads)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_local) return;
    const int l = labels[i];
    if (l < 0) return;
    if (i >= n_owned || sent[i]) {
        const int k = atomicAdd(n_links, 1);
        if (k < cap) links[k] = make_int2(gid[i], gid[l]);
    }
    if (i == l && bnd[i] && badlocal[i]) {
        const int k = atomicAdd(n_bads, 1);
        if (k < cap) bads[k] = gid[i];
    }
}

__global__ void k_slab_unite(const int2* __restrict__ links, int nl, uint32_t* forest, uint8_t* touched)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nl) return;
    const int2 e = links[k];
    touched[e.x] = 1;
    touched[e.y] = 1;
    if (e.x != e.y) uf_unite(forest, (uint32_t)e.x, (uint32_t)e.y);
}

__global__ void k_slab_bad(const int32_t* __restrict__ bads, int nb, uint32_t* forest, uint8_t* badm)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nb) return;
    badm[uf_find(forest, (uint32_t)bads[k])] = 1;
}

__global__ void k_slab_final(am_slab_geom g, int n_owned, const int32_t* __restrict__ gid,
                             const int32_t* __restrict__ steps, const uint8_t* __restrict__ status,
                             const int32_t* __restrict__ labels, const uint8_t* __restrict__ badlocal,
                             const int32_t* __restrict__ ws, uint32_t* forest, const uint8_t* __restrict__ badm,
                             const uint8_t* __restrict__ touched, int32_t* out_label, uint8_t* out_mask,
                             long long* out_key)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_owned) return;
    const uint8_t st = status[i];
    if (st == ST_DONE) {
        out_label[i] = -1;
        out_mask[i] = 0;
        out_key[i] = LLONG_MAX;
        return;
    }
    const int l = labels[i];
    const uint32_t L = (uint32_t)gid[l];
    uint32_t F = L;
    bool bad;
    if (touched[L]) {
        F = uf_find(forest, L);
        bad = badm[F] != 0;
    } else {
        bad = badlocal[l] != 0;
    }
    const bool ready = st == ST_IDLE && !bad;
    out_label[i] = (int32_t)F;
    out_mask[i] = ready;
    out_key[i] = ready ? (((long long)(steps[i] - ws[0]) << 42) | ((long long)F << 21) | (long long)gid[i])
                       : LLONG_MAX;
}

__global__ void k_slab_restore(const int2* __restrict__ links, int nl, uint32_t* forest, uint8_t* badm,
                               uint8_t* touched)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nl) return;
    const int2 e = links[k];
    forest[e.x] = (uint32_t)e.x;
    forest[e.y] = (uint32_t)e.y;
    badm[e.x] = badm[e.y] = 0;
    touched[e.x] = touched[e.y] = 0;
}

}  // namespace am

using namespace am;

static inline unsigned nblk(long long n) { return (unsigned)(n > 0 ? (n + 255) / 256 : 1); }

static int ck(cudaError_t e)
{
    if (e != cudaSuccess) {
        fprintf(stderr, "am_slab: %s\n", cudaGetErrorString(e));
        return AM_E_CUDA;
    }
    return AM_OK;
}

extern "C" int am_slab_watermark(int32_t n, const int32_t* steps, const uint8_t* status, int32_t* out,
                                 void* stream)
{
    if (n < 0 || !out || (n > 0 && (!steps || !status))) return AM_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    k_slab_init2<<<1, 1, 0, s>>>(out);
    if (n > 0) k_slab_watermark<<<std::min(nblk(n), 1184u), 256, 0, s>>>(n, steps, status, out);
    return ck(cudaGetLastError());
}

extern "C" int am_slab_assemble(int32_t n, const int32_t* gid, const int32_t* pos, const int32_t* steps,
                                const uint8_t* status, int32_t m, const int32_t* ghosts, int32_t cap, int32_t y0,
                                int32_t* lpos, int32_t* lsteps, uint8_t* lstatus, int32_t* lgid, void* stream)
{
    if (n < 0 || m < 0 || cap < n + m || (n && (!gid || !pos || !steps || !status)) || (m && !ghosts) ||
        (cap && (!lpos || !lsteps || !lstatus || !lgid)))
        return AM_E_ARG;
    if (cap == 0) return AM_OK;
    k_slab_assemble<<<std::min((cap + 255) / 256, 148 * 8), 256, 0, (cudaStream_t)stream>>>(
        n, gid, (const int2*)pos, steps, status, m, (const int4*)ghosts, cap, y0, (int2*)lpos, lsteps, lstatus, lgid);
    return cudaGetLastError() == cudaSuccess ? AM_OK : AM_E_CUDA;
}

extern "C" int am_slab_halo(const am_slab_geom* g, int32_t n, const int32_t* gid, const int32_t* pos,
                            const int32_t* steps, const uint8_t* status, const int32_t* ws, int32_t cap,
                            int32_t* send, int32_t* counts, uint8_t* sent, void* stream)
{
    if (!g || n < 0 || g->n_slabs < 1 || g->my_slab < 0 || g->my_slab >= g->n_slabs || cap < 0 || !counts)
        return AM_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    k_slab_zero<<<nblk(g->n_slabs), 256, 0, s>>>(counts, g->n_slabs);
    if (n > 0)
        k_slab_halo<<<nblk(n), 256, 0, s>>>(*g, n, gid, (const int2*)pos, steps, status, ws, cap, (int4*)send,
                                            counts, sent);
    return ck(cudaGetLastError());
}

extern "C" int am_slab_links(int32_t n_local, int32_t n_owned, const int32_t* gid, const int32_t* labels,
                             const uint8_t* status, const uint8_t* blocked, const uint8_t* sent, int32_t cap,
                             int32_t* links, int32_t* n_links, int32_t* bads, int32_t* n_bads, uint8_t* badlocal,
                             uint8_t* bnd, void* stream)
{
    if (n_local < 0 || n_owned < 0 || n_owned > n_local || !n_links || !n_bads) return AM_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    k_slab_zero<<<1, 256, 0, s>>>(n_links, 1);
    k_slab_zero<<<1, 256, 0, s>>>(n_bads, 1);
    if (n_local > 0) {
        cudaMemsetAsync(badlocal, 0, (size_t)n_local, s);
        cudaMemsetAsync(bnd, 0, (size_t)n_local, s);
        k_slab_mark<<<nblk(n_local), 256, 0, s>>>(n_local, n_owned, labels, status, blocked, sent, badlocal, bnd);
        k_slab_emit<<<nblk(n_local), 256, 0, s>>>(n_local, n_owned, gid, labels, sent, badlocal, bnd, cap,
                                                  (int2*)links, n_links, bads, n_bads);
    }
    return ck(cudaGetLastError());
}

extern "C" int am_slab_merge(const am_slab_geom* g, int32_t n_owned, const int32_t* gid, const int32_t* steps,
                             const uint8_t* status, const int32_t* labels, const uint8_t* badlocal,
                             const int32_t* links, int32_t n_links_all, const int32_t* bads, int32_t n_bads_all,
                             const int32_t* ws, uint32_t* forest, uint8_t* badm, uint8_t* touched,
                             int32_t* out_label, uint8_t* out_mask, int64_t* out_key, void* stream)
{
    if (!g || n_owned < 0 || n_links_all < 0 || n_bads_all < 0 || g->n_total > (1 << 21)) return AM_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    if (n_links_all > 0) k_slab_unite<<<nblk(n_links_all), 256, 0, s>>>((const int2*)links, n_links_all, forest, touched);
    if (n_bads_all > 0) k_slab_bad<<<nblk(n_bads_all), 256, 0, s>>>(bads, n_bads_all, forest, badm);
    if (n_owned > 0)
        k_slab_final<<<nblk(n_owned), 256, 0, s>>>(*g, n_owned, gid, steps, status, labels, badlocal, ws, forest,
                                                   badm, touched, out_label, out_mask, (long long*)out_key);
    if (n_links_all > 0)
        k_slab_restore<<<nblk(n_links_all), 256, 0, s>>>((const int2*)links, n_links_all, forest, badm, touched);
    return ck(cudaGetLastError());
}
