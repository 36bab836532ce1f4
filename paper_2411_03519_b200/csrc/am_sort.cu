// am_sort.cu -- the priority order of the ready set (S6) as ONE
// thread-block-cluster kernel.
//
// The ready set arrives compacted in id order with keys ((step - W) << idbits) | label
// (k_ready); a stable LSD radix sort on the key gives order = (step, label, id) (Q9).
// The whole grid is a single cluster of C CTAs (16, non-portable, else 8), so the
// passes are separated by cluster barriers instead of kernel launches, and the per-CTA
// digit histograms are exchanged through distributed shared memory (DSMEM).
//
// CTA r owns the contiguous chunk [r*chunk, (r+1)*chunk) of the sequence.  A pass over
// one 8-bit digit:
//   (1) digit histogram of the chunk (shared-memory atomics: counts need no order);
//   (2) cluster barrier; every CTA reads the C histograms over DSMEM -> for each digit
//       the global start of this CTA's run (digit start + the CTAs before it);
//   (3) per tile of the chunk: a stable local sort by the digit in shared memory, as
//       two stable 4-bit rank-and-scatter steps.  Ranking uses per-thread counters
//       (thread t owns K consecutive elements and a private column of 16 counters; one
//       block-wide scan over the 16 x 1024 counters in (digit, thread) order gives every
//       element its rank) -- no atomics, no warp matching;
//   (4) copy-out: consecutive sorted elements of one digit go to consecutive global
//       destinations (coalesced; the ping-pong buffers stay L2-resident);
//   (5) global fence + cluster barrier.
// Elements are (key, id) pairs, packed in 8 bytes when the keys have <= 32 significant
// bits (C5: 7 lag bits + 20 id bits), else 16 bytes.
#include <cooperative_groups.h>

#include "am_internal.cuh"

namespace cg = cooperative_groups;

namespace am {

#ifdef CS_TIMING   // tools/micro/csort_bench.cu: globaltimer stamps of CTA 0
__device__ unsigned long long g_cs_t[128];
__device__ __forceinline__ unsigned long long cs_now()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define CS_STAMP(k) \
    if (threadIdx.x == 0 && blockIdx.x == 0) g_cs_t[(k)] = cs_now();
#else
#define CS_STAMP(k)
#endif

#ifndef AM_CS_BITS
#define AM_CS_BITS 9
#endif
#ifndef AM_CS_SUB
#define AM_CS_SUB 3
#endif
constexpr int kCsBits = AM_CS_BITS;          // digit of one global pass
constexpr int kCsRadix = 1 << kCsBits;
constexpr int kCsSub = AM_CS_SUB;            // bits of one local rank step (divides kCsBits)
static_assert(kCsBits % kCsSub == 0, "rank steps must tile the digit");
constexpr int kCsSubR = 1 << kCsSub;
#ifndef AM_CS_THREADS
#define AM_CS_THREADS 1024
#endif
constexpr int kCsThreads = AM_CS_THREADS;    // threads per CTA (power of two, 256..1024)
constexpr int kCsK = 8;                      // max elements per thread per tile
// fixed shared memory: cnt[kCsSubR][kCsThreads] (padded) + hist, base, run, tstart, ttot
// [kCsRadix] + wsum[32].  9-bit digits of three 3-bit rank steps (A/B on the C5 round:
// 197.6 -> 189.4 us against 8-bit digits of two 4-bit steps: C5's 27-bit keys take
// 3 passes instead of 4)
constexpr size_t kCsFixed = (size_t)(kCsSubR * kCsThreads * 33 / 32 + 5 * kCsRadix + 32) * 4;

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

// the ping-pong buffers of the intermediate passes: packed pairs in rkey[b] (E32), or
// keys in rkey[b] and ids in rval[b] (E64)
__device__ __forceinline__ void gload(const Dev& d, int b, int i, E32& e)
{
    e = reinterpret_cast<const E32*>(d.rkey[b])[i];
}
__device__ __forceinline__ void gload(const Dev& d, int b, int i, E64& e)
{
    eset(e, d.rkey[b][i], d.rval[b][i]);
}
__device__ __forceinline__ void gstore(const Dev& d, int b, int i, const E32& e)
{
    reinterpret_cast<E32*>(d.rkey[b])[i] = e;
}
__device__ __forceinline__ void gstore(const Dev& d, int b, int i, const E64& e)
{
    d.rkey[b][i] = e.k;
    d.rval[b][i] = e.v;
}

size_t csort_smem_fixed() { return kCsFixed; }
// dynamic shared memory of k_csort: the fixed part + two tile buffers of 8-byte pairs
// (or half as many 16-byte ones), and its block size
size_t csort_smem_need() { return kCsFixed + 2 * (size_t)kCsThreads * kCsK * 8; }
int csort_threads() { return kCsThreads; }

// block-wide exclusive scan (1024 threads); wsum: 32 words of shared memory
__device__ __forceinline__ uint32_t block_scan(uint32_t v, uint32_t* wsum)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
        const uint32_t x = lane < (kCsThreads >> 5) ? wsum[lane] : 0u;
        uint32_t s = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, s, o);
            if (lane >= o) s += y;
        }
        wsum[lane] = s - x;
    }
    __syncthreads();
    const uint32_t r = wsum[w] + incl - v;
    __syncthreads();
    return r;
}

// Stable local sort step: the tile's elements src[0..tm) by the sub-digit
// (key >> shift) & (kCsSubR - 1) into dst.  Thread t owns elements [t*K, t*K+K) and
// counter column t of a [kCsSubR][kCsThreads] counter array, stored with one pad word
// per 32 (cpad) so that both the per-thread column updates and the scan (thread u owns
// the kCsSubR consecutive counters [kCsSubR u, kCsSubR u + kCsSubR) of the (digit,
// thread) order) are bank-conflict free.
__device__ __forceinline__ int cpad(int i) { return i + (i >> 5); }

template <class E, int K>
__device__ __forceinline__ void rank_step(const E* src, E* dst, int tm, int shift, uint32_t* cnt,
                                          uint32_t* wsum)
{
    const int t = threadIdx.x;
    uint32_t lp[K];   // rank among this thread's earlier elements of the same sub-digit
#pragma unroll
    for (int q = 0; q < kCsSubR; q++) cnt[cpad(q * kCsThreads + t)] = 0;
#pragma unroll
    for (int k = 0; k < K; k++) {
        const int i = t * K + k;
        lp[k] = 0;
        if (i < tm) {
            const int sd = (int)((ekey(src[i]) >> shift) & (kCsSubR - 1));
            uint32_t* c = cnt + cpad(sd * kCsThreads + t);
            lp[k] = *c;
            *c = lp[k] + 1;
        }
    }
    __syncthreads();
    // exclusive scan of the counters in (digit, thread) order: serial over the thread's
    // 16, block-wide over the 1024 per-thread sums
    uint32_t v[kCsSubR], acc = 0;
#pragma unroll
    for (int j = 0; j < kCsSubR; j++) {
        v[j] = cnt[cpad(kCsSubR * t + j)];
        const uint32_t x = v[j];
        v[j] = acc;
        acc += x;
    }
    const uint32_t off = block_scan(acc, wsum);
#pragma unroll
    for (int j = 0; j < kCsSubR; j++) cnt[cpad(kCsSubR * t + j)] = off + v[j];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; k++) {
        const int i = t * K + k;
        if (i < tm) {
            const E e = src[i];
            dst[cnt[cpad((int)((ekey(e) >> shift) & (kCsSubR - 1)) * kCsThreads + t)] + lp[k]] = e;
        }
    }
    __syncthreads();
}

template <class E, int K>
__device__ void csort_run(const Dev& d, int32_t* __restrict__ order, unsigned char* smem, int n, int np, int bits)
{
    cg::cluster_group cl = cg::this_cluster();
    const int C = (int)cl.num_blocks();
    const int me = (int)cl.block_rank();
    uint32_t* cnt = reinterpret_cast<uint32_t*>(smem);
    uint32_t* hist = cnt + kCsSubR * kCsThreads * 33 / 32;
    uint32_t* base = hist + kCsRadix;     // global start of this CTA's run of each digit
    uint32_t* run = base + kCsRadix;      // elements of each digit in earlier tiles
    uint32_t* tstart = run + kCsRadix;    // start of each digit in the sorted tile
    uint32_t* ttot = tstart + kCsRadix;   // elements of each digit in the tile
    uint32_t* wsum = ttot + kCsRadix;
    constexpr int tile = kCsThreads * K;
    E* const sa = reinterpret_cast<E*>(smem + kCsFixed);
    E* const sb = sa + tile;

    const int t = threadIdx.x;
    const int chunk = (n + C - 1) / C;
    const int lo = min(n, me * chunk), m = min(n, lo + chunk) - lo;
    const bool one = m <= tile;

    for (int p = 0; p < np; p++) {
        CS_STAMP(1 + 8 * p);
        const int shift = kCsBits * p;
        const bool last = p == np - 1;
        // pass 0 reads the compaction (rkey[0] keys, rval[0] ids); pass p >= 1 reads
        // ping-pong buffer p & 1 and writes buffer (p + 1) & 1
        auto load = [&](int i) {
            E e;
            if (p == 0) eset(e, d.rkey[0][lo + i], d.rval[0][lo + i]);
            else gload(d, p & 1, lo + i, e);
            return e;
        };
        // ---- (1) histogram of this CTA's chunk.  A chunk that fits one tile (C5: ~2.6k
        // elements per CTA) is loaded once, all of a thread's loads in flight together,
        // straight into the tile buffer: phase (3) sorts it without reloading it
        for (int k = t; k < kCsRadix; k += kCsThreads) { hist[k] = 0; run[k] = 0; }
        __syncthreads();
        if (one) {
            E ev[K];
#pragma unroll
            for (int q = 0; q < K; q++) {
                const int k = t + q * kCsThreads;
                if (k < m) ev[q] = load(k);
            }
#pragma unroll
            for (int q = 0; q < K; q++) {
                const int k = t + q * kCsThreads;
                if (k < m) {
                    sa[k] = ev[q];
                    atomicAdd(&hist[(int)((ekey(ev[q]) >> shift) & (kCsRadix - 1))], 1u);
                }
            }
        } else {
            for (int k = t; k < m; k += kCsThreads)
                atomicAdd(&hist[(int)((ekey(load(k)) >> shift) & (kCsRadix - 1))], 1u);
        }
        // ---- (2) histograms over DSMEM -> base[digit]
        CS_STAMP(2 + 8 * p);
        cl.sync();
        CS_STAMP(3 + 8 * p);
        {
            uint32_t tot = 0, before = 0;
            if (t < kCsRadix) {
                uint32_t xs[16];   // all remote reads in flight together (C <= 16)
#pragma unroll
                for (int r = 0; r < 16; r++) xs[r] = r < C ? *cl.map_shared_rank(hist + t, r) : 0u;
#pragma unroll
                for (int r = 0; r < 16; r++) {
                    tot += xs[r];
                    before += r < me ? xs[r] : 0u;
                }
            }
            const uint32_t ex = block_scan(tot, wsum);
            if (t < kCsRadix) base[t] = ex + before;
        }
        CS_STAMP(4 + 8 * p);
        // ---- (3) + (4) tiles: stable local sort, coalesced copy-out
        for (int tb = 0; tb < m; tb += tile) {
            const int tm = min(tile, m - tb);
            if (one) {   // loaded in phase (1); the tile's digit counts are the histogram
                if (t < kCsRadix) ttot[t] = hist[t];
            } else {
                if (t < kCsRadix) ttot[t] = 0;
                __syncthreads();
                for (int k = t; k < tm; k += kCsThreads) {
                    const E e = load(tb + k);
                    sa[k] = e;
                    atomicAdd(&ttot[(int)((ekey(e) >> shift) & (kCsRadix - 1))], 1u);
                }
            }
            __syncthreads();
            // the digit's sub-digits, low first; a sub-digit of the last pass above the
            // keys' significant bits is all zero, so its stable step is the identity
            E* res = sa;
            E* oth = sb;
#pragma unroll
            for (int ss = 0; ss < kCsBits / kCsSub; ss++) {
                if (shift + ss * kCsSub >= bits) break;
                rank_step<E, K>(res, oth, tm, shift + ss * kCsSub, cnt, wsum);
                E* x = res; res = oth; oth = x;
            }
            CS_STAMP(5 + 8 * p);
            {
                const uint32_t ts = block_scan(t < kCsRadix ? ttot[t] : 0u, wsum);
                if (t < kCsRadix) tstart[t] = ts;
            }
            __syncthreads();
            for (int j = t; j < tm; j += kCsThreads) {
                const E e = res[j];
                const int dg = (int)((ekey(e) >> shift) & (kCsRadix - 1));
                const uint32_t dst = base[dg] + run[dg] + (uint32_t)j - tstart[dg];
                AM_CHECK(dst < (uint32_t)n);
                if (last) order[dst] = (int32_t)e.v;
                else gstore(d, (p + 1) & 1, (int)dst, e);
            }
            __syncthreads();
            if (t < kCsRadix) run[t] += ttot[t];
            __syncthreads();
        }
        // ---- (5) every element of this pass has landed before the next pass reads it
        CS_STAMP(6 + 8 * p);
        __threadfence();
        cl.sync();
        CS_STAMP(7 + 8 * p);
    }
}

__global__ void __launch_bounds__(kCsThreads, 1) k_csort(Dev d, int32_t* __restrict__ order, int smem_bytes)
{
    pdl_begin();
    extern __shared__ __align__(16) unsigned char cs_smem[];
    (void)smem_bytes;
    CS_STAMP(0);
    const int n = d.ctl->n_ready;
    const unsigned long long kor = *(volatile const unsigned long long*)&d.ctl->sort_or;
    const int bits = kor ? 64 - __clzll((long long)kor) : 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) { d.ctl->sort_bits = bits; d.ctl->npasses = (bits + kCsBits - 1) / kCsBits; }
    const int np = (bits + kCsBits - 1) / kCsBits;
    const int C = (int)cg::this_cluster().num_blocks();
    if (n == 0) return;
    if (np == 0) {   // every key equal: the compaction order (id) is the order
        const int me = (int)cg::this_cluster().block_rank();
        for (int k = me * kCsThreads + threadIdx.x; k < n; k += C * kCsThreads) order[k] = (int32_t)d.rval[0][k];
        return;
    }
    // elements per thread per tile: as few as the chunk needs (shorter serial work)
    const int chunk = (n + C - 1) / C;
    if (bits <= 32) {
        if (chunk <= 2 * kCsThreads) csort_run<E32, 2>(d, order, cs_smem, n, np, bits);
        else if (chunk <= 4 * kCsThreads) csort_run<E32, 4>(d, order, cs_smem, n, np, bits);
        else csort_run<E32, kCsK>(d, order, cs_smem, n, np, bits);
    } else {
        if (chunk <= 2 * kCsThreads) csort_run<E64, 2>(d, order, cs_smem, n, np, bits);
        else csort_run<E64, 4>(d, order, cs_smem, n, np, bits);
    }
}

}  // namespace am
