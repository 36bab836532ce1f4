// am_sort.cu -- the priority order of the ready set (S6) as ONE
// thread-block-cluster kernel.
//
// The ready set arrives compacted in id order with keys ((step - W) << idbits) | label
// (k_ready); a stable LSD radix sort on the key gives order = (step, label, id) (Q9).
// The whole grid is a single cluster of C CTAs (16, non-portable, else 8), so the
// passes are separated by cluster barriers instead of kernel launches, and the per-CTA
// digit histograms are exchanged through distributed shared memory (DSMEM).
//
// CTA r owns the contiguous chunk [r*chunk, (r+1)*chunk) of the sequence.  A pass:
//   (1) digit histogram of the chunk (warp-aggregated shared-memory atomics);
//   (2) cluster barrier; every CTA reads the C histograms over DSMEM -> for each digit
//       the global start of this CTA's run (digit start + the CTAs before it);
//   (3) stable ranking of a tile (per-warp digit counters, each warp owns a consecutive
//       index range, ballot-based peer matching) into a LOCAL staging buffer sorted by
//       digit -- random stores stay in the CTA's own shared memory;
//   (4) copy-out: consecutive staged elements of one digit go to consecutive
//       destinations, so the scatter to the owning CTA's buffer (DSMEM) or to global
//       memory is coalesced;
//   (5) cluster barrier.
// Elements are (key, id) pairs, packed in 8 bytes when the keys have <= 32 significant
// bits (C5: 7 lag bits + 20 id bits), else 16 bytes.  When the ready set fits in the
// cluster's shared memory the pairs stay resident between passes (touching global
// memory once in and once out); larger sets (e.g. the first replay rounds, every agent
// at step 0) stream through the global rkey/rval buffers with the same passes.
#include <cooperative_groups.h>

#include "am_internal.cuh"

namespace cg = cooperative_groups;

namespace am {

constexpr int kCsBits = 8;
constexpr int kCsRadix = 1 << kCsBits;
constexpr int kCsThreads = 1024;
constexpr int kCsItems = 8;                               // per lane per ranking tile (8-byte pairs)
// fixed shared memory: wcnt[32][R] + hist, base, run, tstart, ttot [R] + scan[32]
constexpr size_t kCsFixed = (size_t)(32 * kCsRadix + 5 * kCsRadix + 32) * 4;

struct E32 {
    uint32_t k, v;
};
struct __align__(16) E64 {
    unsigned long long k;
    uint32_t v, pad;
};
__device__ __forceinline__ unsigned long long ekey(const E32& e) { return e.k; }
__device__ __forceinline__ unsigned long long ekey(const E64& e) { return e.k; }
__device__ __forceinline__ void eset(E32& e, unsigned long long k, uint32_t v) { e.k = (uint32_t)k; e.v = v; }
__device__ __forceinline__ void eset(E64& e, unsigned long long k, uint32_t v) { e.k = k; e.v = v; e.pad = 0; }

// lanes of the warp holding the same digit (and validity), from kCsBits + 1 ballots
__device__ __forceinline__ unsigned cs_match(int dg, bool valid)
{
    const unsigned vm = __ballot_sync(0xFFFFFFFFu, valid);
    unsigned peers = valid ? vm : ~vm;
#pragma unroll
    for (int b = 0; b < kCsBits; b++) {
        const bool bit = (dg >> b) & 1;
        const unsigned m = __ballot_sync(0xFFFFFFFFu, bit);
        peers &= bit ? m : ~m;
    }
    return peers;
}

size_t csort_smem_fixed() { return kCsFixed; }

// exclusive scan of v over the kCsRadix digits held by threads 0..kCsRadix-1 (all
// threads of the block call it); returns the exclusive prefix in those threads
__device__ __forceinline__ uint32_t digit_scan(uint32_t v, uint32_t* scan)
{
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (t < kCsRadix && lane == 31) scan[w] = incl;
    __syncthreads();
    uint32_t off = 0;
    if (t < kCsRadix)
        for (int q = 0; q < w; q++) off += scan[q];
    __syncthreads();
    return off + incl - v;
}

template <class E>
__device__ void csort_run(const Dev& d, int32_t* __restrict__ order, unsigned char* smem, size_t smem_bytes,
                          int n, int np)
{
    cg::cluster_group cl = cg::this_cluster();
    const int C = (int)cl.num_blocks();
    const int me = (int)cl.block_rank();
    uint32_t (*wcnt)[kCsRadix] = reinterpret_cast<uint32_t (*)[kCsRadix]>(smem);
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem) + 32 * kCsRadix;
    uint32_t* base = hist + kCsRadix;     // global start of this CTA's run of each digit
    uint32_t* run = base + kCsRadix;      // elements of each digit in earlier tiles
    uint32_t* tstart = run + kCsRadix;    // start of each digit in the staged tile
    uint32_t* ttot = tstart + kCsRadix;   // elements of each digit in the tile
    uint32_t* scan = ttot + kCsRadix;
    const int cap = (int)((smem_bytes - kCsFixed) / (3 * sizeof(E)));
    E* const buf0 = reinterpret_cast<E*>(smem + kCsFixed);   // ping-pong buffers 0 and 1
    E* const stage = buf0 + 2 * cap;

    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int chunk = (n + C - 1) / C;
    const int lo = min(n, me * chunk), m = min(n, lo + chunk) - lo;
    const bool resident = chunk <= cap;
    constexpr int kItems = sizeof(E) == 8 ? kCsItems : kCsItems / 2;   // register budget
    const int tile = min(cap, kCsThreads * kItems);

    for (int p = 0; p < np; p++) {
        const int shift = kCsBits * p;
        const bool last = p == np - 1;
        // source of this pass: the global compaction (pass 0 or streaming), or this CTA's
        // resident buffer
        const bool gsrc = p == 0 || !resident;
        const unsigned long long* gk = d.rkey[p & 1] + lo;
        const uint32_t* gv = d.rval[p & 1] + lo;
        const E* ssrc = buf0 + (p & 1) * cap;
        auto load = [&](int i) {
            E e;
            if (gsrc) eset(e, gk[i], gv[i]); else e = ssrc[i];
            return e;
        };
        // ---- (1) histogram of this CTA's chunk
        for (int k = t; k < kCsRadix; k += kCsThreads) { hist[k] = 0; run[k] = 0; }
        __syncthreads();
        for (int k0 = 0; k0 < m; k0 += kCsThreads) {
            const int k = k0 + t;
            const bool valid = k < m;
            const int dg = valid ? (int)((ekey(load(k)) >> shift) & (kCsRadix - 1)) : 0;
            const unsigned peers = cs_match(dg, valid);
            if (valid && (peers & lt) == 0) atomicAdd(&hist[dg], (uint32_t)__popc(peers));
        }
        // ---- (2) histograms over DSMEM -> base[digit]
        cl.sync();
        {
            uint32_t tot = 0, before = 0;
            if (t < kCsRadix) {
                uint32_t v[16];
#pragma unroll
                for (int r = 0; r < 16; r++) v[r] = r < C ? *cl.map_shared_rank(hist + t, r) : 0u;
#pragma unroll
                for (int r = 0; r < 16; r++) {
                    tot += v[r];
                    before += r < me ? v[r] : 0u;
                }
            }
            const uint32_t ex = digit_scan(tot, scan);
            if (t < kCsRadix) base[t] = ex + before;
        }
        // ---- (3) + (4) tiles: stable ranking into the staging buffer, coalesced copy-out
        for (int tb = 0; tb < m; tb += tile) {
            const int tm = min(tile, m - tb);
            for (int k = t; k < 32 * kCsRadix; k += kCsThreads) (&wcnt[0][0])[k] = 0;
            __syncthreads();
            E el[kItems];
            uint32_t rnk[kItems];
            int dig[kItems];
#pragma unroll
            for (int k = 0; k < kItems; k++) {
                const int i = w * (32 * kItems) + k * 32 + lane;
                const bool valid = i < tm;
                if (valid) el[k] = load(tb + i); else eset(el[k], 0ull, 0u);
                dig[k] = valid ? (int)((ekey(el[k]) >> shift) & (kCsRadix - 1)) : kCsRadix;
                const unsigned peers = cs_match(dig[k] & (kCsRadix - 1), valid);
                const uint32_t b0 = valid ? wcnt[w][dig[k]] : 0u;
                rnk[k] = b0 + __popc(peers & lt);
                __syncwarp();
                if (valid && (peers & lt) == 0) wcnt[w][dig[k]] = b0 + __popc(peers);
                __syncwarp();
            }
            __syncthreads();
            // per digit: exclusive prefix over the warps -> tile totals -> tile starts
            uint32_t acc = 0;
            if (t < kCsRadix) {
#pragma unroll 8
                for (int q = 0; q < 32; q++) { const uint32_t v = wcnt[q][t]; wcnt[q][t] = acc; acc += v; }
                ttot[t] = acc;
            }
            const uint32_t ts = digit_scan(acc, scan);
            if (t < kCsRadix) tstart[t] = ts;
            __syncthreads();
#pragma unroll
            for (int k = 0; k < kItems; k++)
                if (dig[k] < kCsRadix) stage[tstart[dig[k]] + wcnt[w][dig[k]] + rnk[k]] = el[k];
            __syncthreads();
            // copy-out in staged order: destination = run start of the digit + offset
            for (int j = t; j < tm; j += kCsThreads) {
                const E e = stage[j];
                const int dg = (int)((ekey(e) >> shift) & (kCsRadix - 1));
                const uint32_t dst = base[dg] + run[dg] + (uint32_t)j - tstart[dg];
                if (last) {
                    order[dst] = (int32_t)e.v;
                } else if (resident) {
                    const int r = (int)(dst / (uint32_t)chunk);
                    *cl.map_shared_rank(buf0 + ((p + 1) & 1) * cap + (dst - (uint32_t)r * chunk), r) = e;
                } else {
                    d.rkey[(p + 1) & 1][dst] = ekey(e);
                    d.rval[(p + 1) & 1][dst] = e.v;
                }
            }
            __syncthreads();
            if (t < kCsRadix) run[t] += ttot[t];
            __syncthreads();
        }
        // ---- (5) every element of this pass has landed before the next pass reads it
        if (!resident) __threadfence();
        cl.sync();
    }
}

__global__ void __launch_bounds__(kCsThreads, 1) k_csort(Dev d, int32_t* __restrict__ order, int smem_bytes)
{
    extern __shared__ __align__(16) unsigned char cs_smem[];
    const int n = d.ctl->n_ready;
    const int bits = d.ctl->sort_bits;
    const int np = (bits + kCsBits - 1) / kCsBits;
    if (n == 0) return;
    if (np == 0) {   // every key equal: the compaction order (id) is the order
        cg::cluster_group cl = cg::this_cluster();
        const int C = (int)cl.num_blocks(), me = (int)cl.block_rank();
        for (int k = me * kCsThreads + threadIdx.x; k < n; k += C * kCsThreads) order[k] = (int32_t)d.rval[0][k];
        return;
    }
    if (bits <= 32)
        csort_run<E32>(d, order, cs_smem, (size_t)smem_bytes, n, np);
    else
        csort_run<E64>(d, order, cs_smem, (size_t)smem_bytes, n, np);
}

}  // namespace am
