// am_synth.cuh -- the synthetic replay model (include/am_driver.h) on the device: the
// per-agent trajectory hash, the latency draw and the random-walk policy.  Shared by
// the single-GPU driver (am_driver.cu) and the spatial-slab driver (am_slab.cu).
// Product code: the oracle implements the same definitions independently.
#pragma once

#include "am_driver.h"
#include "am_internal.cuh"

namespace am {

__device__ __forceinline__ unsigned long long traj_step(unsigned long long th, int s, int x, int y)
{
    return mix64(th ^ (((unsigned long long)(uint32_t)s << 32) | ((unsigned long long)(uint16_t)x << 16) |
                       (unsigned long long)(uint16_t)y));
}

// duration of agent i's step s in integer microseconds
__device__ __forceinline__ long long duration(const am_synth& sy, int i, int s)
{
    if (sy.dur_table) return sy.dur_table[(long long)i * sy.dur_T + s];
    const unsigned long long u = key3(sy.lat_seed, (uint32_t)i, (uint32_t)s);
    const unsigned long long hi = u >> 32;
    int m = 0;
    while (m < sy.n_vals - 1 && !(hi < sy.cdf32[m])) m++;
    const int K = sy.vals[m];
    long long dsum = sy.base_us;
    for (int k = 0; k < K; k++) {
        const unsigned long long h =
            key3(sy.lat_seed ^ 0xC0FFEEULL, ((unsigned long long)(uint32_t)i << 20) ^ (uint32_t)s, (uint32_t)k);
        dsum += sy.lat[h >> 54];
    }
    return dsum;
}

// within R (R2 = R * R) for the metric
__device__ __forceinline__ bool within2(int dx, int dy, uint32_t R2, uint32_t R, int metric)
{
    if (metric == AM_METRIC_LINF) return (uint32_t)abs(dx) <= R && (uint32_t)abs(dy) <= R;
    return (uint32_t)(dx * dx) + (uint32_t)(dy * dy) <= R2;
}

// the synthetic policy (am_driver.h): random walk on the perception digest; a move into
// a wall or off the map is cancelled.  policy 0: {stay, +x, -x, +y, -y}[h % 5]; 1: stay;
// 2: the 8-connected walk (for the L-infinity metric): the five above, then (+1,+1),
// (-1,+1), (+1,-1), (-1,-1) [h % 9]
__device__ __forceinline__ int2 policy_move_g(const am_synth& sy, int map_w, int map_h, int i, int s, int2 p,
                                              unsigned long long dig)
{
    if (sy.policy == 3) {   // graph walk (AM_METRIC_GRAPH: x = node, one hop <= v)
        const unsigned long long h = mix64(key3(sy.policy_seed, (uint32_t)i, (uint32_t)s) + dig);
        const int deg = sy.graph_off[p.x + 1] - sy.graph_off[p.x];
        const int m = (int)(h % (unsigned long long)(deg + 1));
        return m == 0 ? p : make_int2(sy.graph_adj[sy.graph_off[p.x] + m - 1], p.y);
    }
    int mv = 0;
    if (sy.policy == 0 || sy.policy == 2) {
        const unsigned long long h = mix64(key3(sy.policy_seed, (uint32_t)i, (uint32_t)s) + dig);
        mv = (int)(h % (sy.policy == 2 ? 9ull : 5ull));
    }
    const int qx = p.x + (mv == 1 || mv == 5 || mv == 7) - (mv == 2 || mv == 6 || mv == 8);
    const int qy = p.y + (mv == 3 || mv == 5 || mv == 6) - (mv == 4 || mv == 7 || mv == 8);
    bool ok = qx >= 0 && qx < map_w && qy >= 0 && qy < map_h;
    if (ok && sy.wall && sy.wall[(long long)qy * map_w + qx]) ok = false;
    return ok ? make_int2(qx, qy) : p;
}

}  // namespace am
