/*
 * am_slab.h -- spatial-slab decomposition of the tracker round across GPUs
 * (the paper runs one controller, and scales workers
 * "beyond a single machine", P:194 -- the slab exchange is this repo's design).
 *
 * The map's rows are split into G horizontal slabs; slab k owns rows
 * [k*map_h/G, (k+1)*map_h/G) and every agent whose y lies there.  One distributed
 * round (driven by paper_2411_03519_b200/slabs.py over an exchange: NCCL via
 * torch.distributed, or an in-process loopback for virtual slabs):
 *   1. am_slab_watermark on owned agents; all-reduce min of {W, -S};
 *   2. am_slab_halo: owned agent B is sent to every slab within R_b(S - s_B) rows
 *      (P:406 with the global max step: covers every agent B can block or couple
 *      with, since R_b(0) = r_p + v = R_c); all-to-all of the records;
 *   3. a local tracker round (am_set_state + am_ready, AM_PEEK) over owned agents
 *      (sorted by global id) followed by the received ghosts; am_clusters /
 *      am_blocked;  am_slab_links emits, for every boundary agent (a ghost here, or
 *      owned and sent elsewhere), a link {gid, gid of its local cluster label}, and
 *      for every local cluster with a boundary member whose OWNED members include a
 *      RUNNING or blocked agent, a bad record {gid of the label};  all-gather;
 *   4. am_slab_merge (identical on every rank): union-find over all links in a dense
 *      global-id forest (roots = minimum id), bad flags OR-ed per merged root; final
 *      outputs for the owned agents: global label (min id of the global cluster,
 *      P:139, Q10), ready mask (IDLE and cluster not bad) and a priority
 *      key ((step - W), label, id) (Q9) for the ready ones.
 * Every coupling edge is seen on the owner of one endpoint (the other is within
 * R_c <= the halo radius), every blocker of an owned agent is present as owned or
 * ghost, and every agent is owned once, so the merged result equals the
 * single-GPU round bit for bit (tests/test_gpu_slabs.py).
 *
 * All arrays are DEVICE pointers owned by the caller; counts are device int32.
 * Work is enqueued on `stream`.  Returns AM_OK or AM_E_ARG / AM_E_CUDA.
 */
#ifndef AM_SLAB_H_
#define AM_SLAB_H_

#include <stdint.h>
#include "am.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t map_w, map_h;     /* map (tiles)                                          */
    int32_t r_p, v_max;       /* radius_p, max_vel                            */
    int32_t metric;           /* AM_METRIC_L2 / AM_METRIC_LINF                        */
    int32_t n_slabs;          /* G >= 1                                               */
    int32_t my_slab;          /* this rank's slab                                     */
    int32_t n_total;          /* agents over all slabs (global ids are 0..n_total-1)  */
} am_slab_geom;

/* out[0] = min step over owned non-DONE agents (INT32_MAX if none),
 * out[1] = -(max step) (INT32_MAX if none): ready for an all-reduce MIN. */
int am_slab_watermark(int32_t n, const int32_t* steps, const uint8_t* status, int32_t* out,
                      void* stream);

/* Halo records.  ws: device int32[2] = global {W, -S} after the all-reduce.
 * send: int32 [n_slabs][cap][4] records {gid, x | y<<16, step, status};
 * counts: int32 [n_slabs] (zeroed by the call); sent: uint8 [n] (1 = sent anywhere).
 * Records beyond cap are dropped and counts[j] > cap reports it (caller retries). */
int am_slab_halo(const am_slab_geom* g, int32_t n, const int32_t* gid, const int32_t* pos,
                 const int32_t* steps, const uint8_t* status, const int32_t* ws, int32_t cap,
                 int32_t* send, int32_t* counts, uint8_t* sent, void* stream);

/* The local tracker's input arrays (capacity cap >= n + m): slots [0, n) the owned
 * agents (gid/pos int32[n][2]/steps/status), slots [n, n + m) the received halo
 * records ghosts int32 [m][4] {gid, x | y<<16, step, status}, the rest DONE padding;
 * every y translated by -y0 (the slab's window).  Outputs lpos int32 [cap][2], lsteps
 * int32 [cap], lstatus uint8 [cap], lgid int32 [cap]. */
int am_slab_assemble(int32_t n, const int32_t* gid, const int32_t* pos, const int32_t* steps,
                     const uint8_t* status, int32_t m, const int32_t* ghosts, int32_t cap, int32_t y0,
                     int32_t* lpos, int32_t* lsteps, uint8_t* lstatus, int32_t* lgid, void* stream);

/* Merge records of the local round over n_local agents (owned first, then ghosts).
 * labels/blocked: am_clusters / am_blocked output (local indices); sent: from
 * am_slab_halo (owned part).  links: int32 [cap][2]; bads: int32 [cap];
 * n_links, n_bads: device int32 (zeroed by the call); badlocal: uint8 [n_local]
 * scratch that receives, per local root, "an owned member is RUNNING or blocked";
 * bnd: uint8 [n_local] scratch. */
int am_slab_links(int32_t n_local, int32_t n_owned, const int32_t* gid, const int32_t* labels,
                  const uint8_t* status, const uint8_t* blocked, const uint8_t* sent,
                  int32_t cap, int32_t* links, int32_t* n_links, int32_t* bads, int32_t* n_bads,
                  uint8_t* badlocal, uint8_t* bnd, void* stream);

/* Merge and final outputs for the n_owned owned agents.
 * links [n_links_all][2], bads [n_bads_all]: every rank's records concatenated
 * (host counts).  forest: uint32 [n_total] that must hold the identity (parent[x] =
 * x) and badm/touched: uint8 [n_total] zero on entry; all three are restored on exit.
 * ws: global {W, -S}.  Outputs: out_label int32 [n_owned] (-1 DONE), out_mask uint8
 * [n_owned], out_key int64 [n_owned] = ((step-W) << 42) | (label << 21) | gid for
 * ready agents (n_total <= 2^21), INT64_MAX otherwise. */
int am_slab_merge(const am_slab_geom* g, int32_t n_owned, const int32_t* gid, const int32_t* steps,
                  const uint8_t* status, const int32_t* labels, const uint8_t* badlocal,
                  const int32_t* links, int32_t n_links_all, const int32_t* bads, int32_t n_bads_all,
                  const int32_t* ws, uint32_t* forest, uint8_t* badm, uint8_t* touched,
                  int32_t* out_label, uint8_t* out_mask, int64_t* out_key, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* AM_SLAB_H_ */
