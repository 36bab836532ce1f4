/*
 * oracle/oracle_scale.c -- CPU ORACLE at BASELINE sizes (test infrastructure only).
 *
 * The same definitions as oracle.c (it calls oracle.c's predicates orc_blocked_by,
 * orc_coupled, orc_digest and orc_policy_move; nothing is re-derived here), organised
 * so that the 100k / 1M-agent configurations finish in seconds on the host cores:
 *
 *   orc_round_mt        the brute-force round of oracle.c (orc_round), with the outer
 *                       loop over agents split across threads ("outer loop
 *                       over agents, static chunks").  Every pair is still tested.
 *   orc_labels_steps    the cluster labels alone (Q5/Q6/Q10): all
 *                       pairs of agents AT THE SAME STEP (coupling requires
 *                       Step_A == Step_B, so pairs at different steps can never
 *                       be coupled), brute force per step, then a sequential union-find.
 *   orc_blocked_list    the blocking verdict (strict Step_B < Step_A from
 *                       P:408-417) of listed agents, each by a scan over ALL agents.
 *   orc_lockstep_grid   Algorithm 1 exactly as orc_lockstep, except that the
 *                       perceived set (same-step agents within radius_p) is found
 *                       through a uniform hash grid of cell edge radius_p (perception
 *                       only -- SURVEY 7 hard part 8); the digest sums the same terms.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library; it shares nothing with paper_2411_03519_b200/.
 * Pins (tests/test_oracle.py): each function equals its plain counterpart in oracle.c
 * on random and workload states (orc_round, orc_round_sampled, orc_lockstep), which are
 * themselves pinned by the hand vectors, library routines and closed forms.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { S_IDLE = 0, S_RUNNING = 1, S_DONE = 2 };

/* the parameter / synth structs of oracle.c (same layout) */
typedef struct {
    int32_t map_w, map_h, r_p, v, target, metric, n_sims;
    const uint16_t* gdist;   /* ORC_GRAPH (oracle.c) */
    int32_t gV;
} orc_params;
typedef struct orc_synth orc_synth;

int orc_blocked_by(const orc_params* p, int32_t xa, int32_t ya, int32_t sa, int32_t xb, int32_t yb, int32_t sb);
int orc_coupled(const orc_params* p, int32_t xa, int32_t ya, int32_t sa, int32_t xb, int32_t yb, int32_t sb);
int64_t orc_duration(const orc_synth* sy, int32_t i, int32_t s);
void orc_policy_move(const orc_params* p, const orc_synth* sy, int32_t i, int32_t s, int32_t px, int32_t py,
                     uint64_t digest, int32_t* nx, int32_t* ny);
uint64_t orc_mix64(uint64_t z);

/* ------------------------------------------------------------------ threads */
typedef struct {
    void (*fn)(void* arg, int64_t lo, int64_t hi);
    void* arg;
    int64_t lo, hi;
} chunk_t;

static void* chunk_run(void* a)
{
    chunk_t* c = (chunk_t*)a;
    c->fn(c->arg, c->lo, c->hi);
    return NULL;
}

/* run fn over [0, n) in `nthreads` static chunks of interleaved blocks (the brute
 * force's cost per agent varies with its position in the id order; blocks of 64
 * agents dealt round-robin keep the threads even) */
typedef struct {
    void (*fn)(void* arg, int64_t lo, int64_t hi);
    void* arg;
    int64_t n;
    int nthreads, t;
} rr_t;
static void rr_body(void* a, int64_t lo, int64_t hi)
{
    (void)lo; (void)hi;
    rr_t* r = (rr_t*)a;
    for (int64_t b = (int64_t)r->t * 64; b < r->n; b += (int64_t)r->nthreads * 64)
        r->fn(r->arg, b, b + 64 < r->n ? b + 64 : r->n);
}
static void parallel_for(int nthreads, int64_t n, void (*fn)(void*, int64_t, int64_t), void* arg)
{
    if (nthreads < 1) nthreads = 1;
    if (nthreads == 1 || n < 256) { fn(arg, 0, n); return; }
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
    rr_t* rr = (rr_t*)malloc(sizeof(rr_t) * nthreads);
    chunk_t* ch = (chunk_t*)malloc(sizeof(chunk_t) * nthreads);
    for (int t = 0; t < nthreads; t++) {
        rr[t].fn = fn; rr[t].arg = arg; rr[t].n = n; rr[t].nthreads = nthreads; rr[t].t = t;
        ch[t].fn = rr_body; ch[t].arg = &rr[t]; ch[t].lo = 0; ch[t].hi = 0;
        pthread_create(&th[t], NULL, chunk_run, &ch[t]);
    }
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    free(th); free(rr); free(ch);
}

/* ------------------------------------------------------------------ union-find (root = min id, Q10) */
static int32_t uf_find(int32_t* parent, int32_t i)
{
    while (parent[i] != i) i = parent[i];
    return i;
}
static void uf_union(int32_t* parent, int32_t a, int32_t b)
{
    a = uf_find(parent, a);
    b = uf_find(parent, b);
    if (a == b) return;
    if (a < b) parent[b] = a; else parent[a] = b;
}

typedef struct { int32_t step, label, id; } okey;
static int okey_cmp(const void* pa, const void* pb)
{
    const okey* a = (const okey*)pa;
    const okey* b = (const okey*)pb;
    if (a->step != b->step) return a->step < b->step ? -1 : 1;
    if (a->label != b->label) return a->label < b->label ? -1 : 1;
    return a->id < b->id ? -1 : (a->id > b->id);
}

/* ============================================================ orc_round_mt
 * orc_round (oracle.c) for one simulation, outer loops split across threads:
 *   blocked[i] = act[i] && exists j != i: act[j] && orc_blocked_by(i, j)
 *   edges      = { (i, j), i < j : act both, orc_coupled(i, j) }
 * then (sequentially) union-find over the edges, label = min id, bad, mask, order --
 * exactly orc_round's steps.  Each thread keeps its own edge list. */
typedef struct {
    const orc_params* p;
    int32_t n;
    const int32_t *x, *y, *step;
    const uint8_t* status;
    uint8_t* blk;
    /* per-thread edge lists, indexed by the block's owner: we use one list per block
     * of 64 agents (blocks are disjoint, so no locking) */
    int32_t** eb;
    int64_t* ecount;
    int64_t* ecap;
} rmt_t;

static void rmt_body(void* a, int64_t lo, int64_t hi)
{
    rmt_t* r = (rmt_t*)a;
    const orc_params* p = r->p;
    const int64_t blk_id = lo / 64;
    for (int64_t i = lo; i < hi; i++) {
        r->blk[i] = 0;
        if (r->status[i] == S_DONE) continue;
        for (int32_t j = 0; j < r->n; j++) {
            if (j == i || r->status[j] == S_DONE) continue;
            if (orc_blocked_by(p, r->x[i], r->y[i], r->step[i], r->x[j], r->y[j], r->step[j])) { r->blk[i] = 1; break; }
        }
        for (int32_t j = (int32_t)i + 1; j < r->n; j++) {
            if (r->status[j] == S_DONE) continue;
            if (orc_coupled(p, r->x[i], r->y[i], r->step[i], r->x[j], r->y[j], r->step[j])) {
                if (r->ecount[blk_id] == r->ecap[blk_id]) {
                    r->ecap[blk_id] = r->ecap[blk_id] ? 2 * r->ecap[blk_id] : 64;
                    r->eb[blk_id] = (int32_t*)realloc(r->eb[blk_id], sizeof(int32_t) * 2 * r->ecap[blk_id]);
                }
                r->eb[blk_id][2 * r->ecount[blk_id]] = (int32_t)i;
                r->eb[blk_id][2 * r->ecount[blk_id] + 1] = j;
                r->ecount[blk_id]++;
            }
        }
    }
}

int orc_round_mt(const orc_params* p, int32_t n, const int32_t* x, const int32_t* y, const int32_t* step,
                 uint8_t* status, int32_t peek, uint8_t* blocked, int32_t* label, uint8_t* mask, int32_t* order,
                 int32_t* n_ready, int32_t nthreads)
{
    if (n < 0 || p->n_sims != 1) return -1;
    const int64_t nb = ((int64_t)n + 63) / 64;
    rmt_t r;
    r.p = p; r.n = n; r.x = x; r.y = y; r.step = step; r.status = status;
    r.blk = (uint8_t*)malloc(n ? n : 1);
    r.eb = (int32_t**)calloc(nb ? nb : 1, sizeof(int32_t*));
    r.ecount = (int64_t*)calloc(nb ? nb : 1, sizeof(int64_t));
    r.ecap = (int64_t*)calloc(nb ? nb : 1, sizeof(int64_t));
    parallel_for(nthreads, n, rmt_body, &r);
    int32_t* parent = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    uint8_t* bad = (uint8_t*)calloc(n ? n : 1, 1);
    for (int32_t i = 0; i < n; i++) parent[i] = i;
    for (int64_t b = 0; b < nb; b++)
        for (int64_t k = 0; k < r.ecount[b]; k++) uf_union(parent, r.eb[b][2 * k], r.eb[b][2 * k + 1]);
    for (int32_t i = 0; i < n; i++) {
        if (status[i] == S_DONE) { label[i] = -1; continue; }
        label[i] = uf_find(parent, i);
        if (r.blk[i] || status[i] == S_RUNNING) bad[label[i]] = 1;
    }
    okey* keys = (okey*)malloc(sizeof(okey) * (n ? n : 1));
    int32_t nr = 0;
    for (int32_t i = 0; i < n; i++) {
        mask[i] = (uint8_t)(status[i] == S_IDLE && !bad[label[i]]);
        if (mask[i]) { keys[nr].step = step[i]; keys[nr].label = label[i]; keys[nr].id = i; nr++; }
    }
    qsort(keys, (size_t)nr, sizeof(okey), okey_cmp);
    for (int32_t k = 0; k < nr; k++) order[k] = keys[k].id;
    if (!peek)
        for (int32_t k = 0; k < nr; k++) status[order[k]] = S_RUNNING;
    if (blocked) memcpy(blocked, r.blk, (size_t)n);
    *n_ready = nr;
    for (int64_t b = 0; b < nb; b++) free(r.eb[b]);
    free(r.eb); free(r.ecount); free(r.ecap); free(r.blk); free(parent); free(bad); free(keys);
    return 0;
}

/* ============================================================ orc_labels_steps
 * Cluster labels of every agent: agents grouped by step (a counting of equal steps,
 * qsort of (step, id)); within each group every pair i < j is tested with
 * orc_coupled; sequential union-find; label = min id, -1 for DONE. */
typedef struct { int32_t step, id; } sid_t;
static int sid_cmp(const void* pa, const void* pb)
{
    const sid_t* a = (const sid_t*)pa;
    const sid_t* b = (const sid_t*)pb;
    if (a->step != b->step) return a->step < b->step ? -1 : 1;
    return a->id < b->id ? -1 : (a->id > b->id);
}
typedef struct {
    const orc_params* p;
    const int32_t *x, *y, *step;
    const sid_t* g;          /* active agents sorted by (step, id) */
    const int64_t* gend;     /* per sorted position: end of its step group */
    int64_t m;
    int32_t** eb;
    int64_t *ecount, *ecap;
} lab_t;
static void lab_body(void* a, int64_t lo, int64_t hi)
{
    lab_t* r = (lab_t*)a;
    const int64_t blk_id = lo / 64;
    for (int64_t u = lo; u < hi; u++) {
        const int32_t i = r->g[u].id;
        for (int64_t w = u + 1; w < r->gend[u]; w++) {
            const int32_t j = r->g[w].id;
            if (orc_coupled(r->p, r->x[i], r->y[i], r->step[i], r->x[j], r->y[j], r->step[j])) {
                if (r->ecount[blk_id] == r->ecap[blk_id]) {
                    r->ecap[blk_id] = r->ecap[blk_id] ? 2 * r->ecap[blk_id] : 64;
                    r->eb[blk_id] = (int32_t*)realloc(r->eb[blk_id], sizeof(int32_t) * 2 * r->ecap[blk_id]);
                }
                r->eb[blk_id][2 * r->ecount[blk_id]] = i;
                r->eb[blk_id][2 * r->ecount[blk_id] + 1] = j;
                r->ecount[blk_id]++;
            }
        }
    }
}

int orc_labels_steps(const orc_params* p, int32_t n, const int32_t* x, const int32_t* y, const int32_t* step,
                     const uint8_t* status, int32_t* label, int32_t nthreads)
{
    if (n < 0 || p->n_sims != 1) return -1;
    sid_t* g = (sid_t*)malloc(sizeof(sid_t) * (n ? n : 1));
    int64_t m = 0;
    for (int32_t i = 0; i < n; i++)
        if (status[i] != S_DONE) { g[m].step = step[i]; g[m].id = i; m++; }
    qsort(g, (size_t)m, sizeof(sid_t), sid_cmp);
    int64_t* gend = (int64_t*)malloc(sizeof(int64_t) * (m ? m : 1));
    for (int64_t u = m - 1; u >= 0; u--)
        gend[u] = (u + 1 < m && g[u + 1].step == g[u].step) ? gend[u + 1] : u + 1;
    const int64_t nb = (m + 63) / 64;
    lab_t r;
    r.p = p; r.x = x; r.y = y; r.step = step; r.g = g; r.gend = gend; r.m = m;
    r.eb = (int32_t**)calloc(nb ? nb : 1, sizeof(int32_t*));
    r.ecount = (int64_t*)calloc(nb ? nb : 1, sizeof(int64_t));
    r.ecap = (int64_t*)calloc(nb ? nb : 1, sizeof(int64_t));
    parallel_for(nthreads, m, lab_body, &r);
    int32_t* parent = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    for (int32_t i = 0; i < n; i++) parent[i] = i;
    for (int64_t b = 0; b < nb; b++)
        for (int64_t k = 0; k < r.ecount[b]; k++) uf_union(parent, r.eb[b][2 * k], r.eb[b][2 * k + 1]);
    for (int32_t i = 0; i < n; i++) label[i] = status[i] == S_DONE ? -1 : uf_find(parent, i);
    for (int64_t b = 0; b < nb; b++) free(r.eb[b]);
    free(r.eb); free(r.ecount); free(r.ecap); free(parent); free(g); free(gend);
    return 0;
}

/* ============================================================ orc_blocked_list
 * blocked[k] = agent idx[k] is not DONE and some other non-DONE agent blocks it
 * (orc_blocked_by), each by a scan over all n agents. */
typedef struct {
    const orc_params* p;
    int32_t n;
    const int32_t *x, *y, *step, *idx;
    const uint8_t* status;
    uint8_t* out;
} bl_t;
static void bl_body(void* a, int64_t lo, int64_t hi)
{
    bl_t* r = (bl_t*)a;
    for (int64_t k = lo; k < hi; k++) {
        const int32_t i = r->idx[k];
        uint8_t b = 0;
        if (r->status[i] != S_DONE)
            for (int32_t j = 0; j < r->n; j++) {
                if (j == i || r->status[j] == S_DONE) continue;
                if (orc_blocked_by(r->p, r->x[i], r->y[i], r->step[i], r->x[j], r->y[j], r->step[j])) { b = 1; break; }
            }
        r->out[k] = b;
    }
}
int orc_blocked_list(const orc_params* p, int32_t n, const int32_t* x, const int32_t* y, const int32_t* step,
                     const uint8_t* status, int32_t k, const int32_t* idx, uint8_t* out, int32_t nthreads)
{
    for (int32_t q = 0; q < k; q++)
        if (idx[q] < 0 || idx[q] >= n) return -1;
    bl_t r = {p, n, x, y, step, idx, status, out};
    parallel_for(nthreads, k, bl_body, &r);
    return 0;
}

/* ============================================================ orc_lockstep_grid
 * Algorithm 1 as orc_lockstep (oracle.c; co-occupancy, n_sims == 1): at every
 * step s every agent perceives the agents within radius_p -- all at step s --
 * and moves by orc_policy_move on its perception digest; all moves apply together.
 * The perceived set is gathered from a uniform grid of cell edge max(1, radius_p): the
 * 3x3 cells around the agent's cell contain every agent within radius_p (L2 and L-inf
 * distances are >= the per-axis offset).  The digest is the same sum, mod 2^64, of
 * mix64((j << 32) ^ ((u16)dx << 16) ^ (u16)dy) over perceived j != i (order-independent).
 * traj[i] chains the committed positions as orc_lockstep does; T_sync = sum over steps
 * of the max duration (P:33-46 global barrier). */
static uint64_t traj_step(uint64_t th, int32_t s, int32_t x, int32_t y)
{
    return orc_mix64(th ^ (((uint64_t)(uint32_t)s << 32) | ((uint64_t)(uint16_t)x << 16) | (uint64_t)(uint16_t)y));
}
typedef struct {
    const orc_params* p;
    const orc_synth* sy;
    int32_t n, s, gw, gh, cell;
    const int32_t *x, *y;
    const int32_t *cstart, *cidx;   /* grid: agents of cell c at cidx[cstart[c] .. cstart[c+1]) */
    int32_t *nx, *ny;
    int64_t* dmax;                  /* per 64-agent block */
} lsg_t;
static void lsg_body(void* a, int64_t lo, int64_t hi)
{
    lsg_t* r = (lsg_t*)a;
    const orc_params* p = r->p;
    int64_t mx = 0;
    for (int64_t i = lo; i < hi; i++) {
        const int32_t cx = r->x[i] / r->cell, cy = r->y[i] / r->cell;
        uint64_t dig = 0;
        for (int32_t qy = cy - 1; qy <= cy + 1; qy++)
            for (int32_t qx = cx - 1; qx <= cx + 1; qx++) {
                if (qx < 0 || qy < 0 || qx >= r->gw || qy >= r->gh) continue;
                const int32_t c = qy * r->gw + qx;
                for (int32_t k = r->cstart[c]; k < r->cstart[c + 1]; k++) {
                    const int32_t j = r->cidx[k];
                    if (j == i) continue;
                    const int32_t dx = r->x[j] - r->x[i], dy = r->y[j] - r->y[i];
                    /* within radius_p: the perception radius of P:153 (same rule as orc_digest) */
                    int in;
                    if (p->metric == 1) in = (dx < 0 ? -dx : dx) <= p->r_p && (dy < 0 ? -dy : dy) <= p->r_p;
                    else in = (int64_t)dx * dx + (int64_t)dy * dy <= (int64_t)p->r_p * p->r_p;
                    if (!in) continue;
                    const uint64_t w = ((uint64_t)(uint32_t)j << 32) ^ ((uint64_t)(uint16_t)dx << 16) ^ (uint64_t)(uint16_t)dy;
                    dig += orc_mix64(w);
                }
            }
        orc_policy_move(p, r->sy, (int32_t)i, r->s, r->x[i], r->y[i], dig, &r->nx[i], &r->ny[i]);
        const int64_t d = orc_duration(r->sy, (int32_t)i, r->s);
        if (d > mx) mx = d;
    }
    r->dmax[lo / 64] = mx > r->dmax[lo / 64] ? mx : r->dmax[lo / 64];
}

int orc_lockstep_grid(const orc_params* p, const orc_synth* sy, int32_t n, int32_t T, int32_t* x, int32_t* y,
                      uint64_t* traj, int64_t* T_sync, int32_t nthreads)
{
    if (p->n_sims != 1 || n < 0 || p->metric == 2) return -1;   /* spatial maps only (no graph metric) */
    const int32_t cell = p->r_p > 0 ? p->r_p : 1;
    const int32_t gw = (p->map_w + cell - 1) / cell, gh = (p->map_h + cell - 1) / cell;
    const int64_t nc = (int64_t)gw * gh;
    int32_t* cstart = (int32_t*)malloc(sizeof(int32_t) * (nc + 1));
    int32_t* cidx = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    int32_t* nx = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    int32_t* ny = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    const int64_t nb = ((int64_t)n + 63) / 64;
    int64_t* dmax = (int64_t*)malloc(sizeof(int64_t) * (nb ? nb : 1));
    int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * (nc ? nc : 1));
    for (int32_t i = 0; i < n; i++) traj[i] = 0;
    T_sync[0] = 0;
    for (int32_t s = 0; s < T; s++) {
        /* bucket the agents by grid cell (counting sort): cell c holds
         * cidx[cstart[c] .. cstart[c+1]) */
        memset(cstart, 0, sizeof(int32_t) * (nc + 1));
        for (int32_t i = 0; i < n; i++) cstart[(int64_t)(y[i] / cell) * gw + x[i] / cell + 1]++;
        for (int64_t c = 0; c < nc; c++) cstart[c + 1] += cstart[c];
        memcpy(fill, cstart, sizeof(int32_t) * nc);
        for (int32_t i = 0; i < n; i++) cidx[fill[(int64_t)(y[i] / cell) * gw + x[i] / cell]++] = i;
        for (int64_t b = 0; b < nb; b++) dmax[b] = 0;
        lsg_t r = {p, sy, n, s, gw, gh, cell, x, y, cstart, cidx, nx, ny, dmax};
        parallel_for(nthreads, n, lsg_body, &r);
        int64_t mx = 0;
        for (int64_t b = 0; b < nb; b++) if (dmax[b] > mx) mx = dmax[b];
        T_sync[0] += mx;
        for (int32_t i = 0; i < n; i++) {
            x[i] = nx[i]; y[i] = ny[i];
            traj[i] = traj_step(traj[i], s + 1, x[i], y[i]);
        }
    }
    free(cstart); free(cidx); free(nx); free(ny); free(dmax); free(fill);
    return 0;
}

/* ============================================================ orc_replay_mt
 * orc_replay_cap (oracle.c) with the simulations of a batch (C3) replayed concurrently:
 * each simulation's replay (orc_replay_sim, the loop body of orc_replay_cap) only
 * touches its own slice of the work arrays, so the per-simulation results are those
 * of the sequential loop.  No round log. */
typedef struct {
    uint64_t* qkey;
    int32_t* step;
    uint8_t* status;
    int64_t* tc;
    int32_t *mvx, *mvy;
    int64_t* cmax;
} orc_replay_work;
typedef struct orc_log orc_log;
int orc_replay_sim(const orc_params* p, const orc_synth* sy, int32_t n, int64_t Q, int64_t K, int32_t priority,
                   int32_t b, const orc_replay_work* wk, int32_t* x, int32_t* y, uint64_t* traj, int64_t* T_ooo,
                   int64_t* rounds, orc_log* log);
typedef struct {
    const orc_params* p;
    const orc_synth* sy;
    int32_t n;
    int64_t Q, K;
    int32_t prio;
    const orc_replay_work* wk;
    int32_t *x, *y;
    uint64_t* traj;
    int64_t *T_ooo, *rounds;
    int32_t* rc;
} rp_t;
static void rp_body(void* a, int64_t lo, int64_t hi)
{
    rp_t* r = (rp_t*)a;
    for (int64_t b = lo; b < hi; b++)
        r->rc[b] = orc_replay_sim(r->p, r->sy, r->n, r->Q, r->K, r->prio, (int32_t)b, r->wk, r->x, r->y, r->traj,
                                  r->T_ooo, r->rounds, NULL);
}
int orc_replay_mt(const orc_params* p, const orc_synth* sy, int32_t n, int64_t Q, int64_t K, int32_t priority,
                  int32_t* x, int32_t* y, uint64_t* traj, int64_t* T_ooo, int64_t* rounds, int32_t nthreads)
{
    if (p->target <= 0 || K < 0) return -1;
    orc_replay_work wk;
    wk.qkey = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    wk.step = (int32_t*)calloc(n ? n : 1, sizeof(int32_t));
    wk.status = (uint8_t*)calloc(n ? n : 1, 1);
    wk.tc = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    wk.mvx = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    wk.mvy = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    wk.cmax = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    int32_t* rc = (int32_t*)calloc(p->n_sims, sizeof(int32_t));
    for (int32_t i = 0; i < n; i++) traj[i] = 0;
    rp_t r = {p, sy, n, Q, K, priority, &wk, x, y, traj, T_ooo, rounds, rc};
    parallel_for(nthreads, p->n_sims, rp_body, &r);
    int out = 0;
    for (int32_t b = 0; b < p->n_sims; b++) if (rc[b]) out = rc[b];
    free(wk.step); free(wk.status); free(wk.tc); free(wk.mvx); free(wk.mvy); free(wk.cmax); free(wk.qkey); free(rc);
    return out;
}

/* the replay of simulation b alone, with its round log (infinite capacity) */
int orc_replay_sim_logged(const orc_params* p, const orc_synth* sy, int32_t n, int64_t Q, int32_t b, int32_t* x,
                          int32_t* y, uint64_t* traj, int64_t* T_ooo, int64_t* rounds, orc_log* log)
{
    if (p->target <= 0 || b < 0 || b >= p->n_sims) return -1;
    orc_replay_work wk;
    wk.qkey = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    wk.step = (int32_t*)calloc(n ? n : 1, sizeof(int32_t));
    wk.status = (uint8_t*)calloc(n ? n : 1, 1);
    wk.tc = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    wk.mvx = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    wk.mvy = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    wk.cmax = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    for (int32_t i = 0; i < n; i++) traj[i] = 0;
    const int rc = orc_replay_sim(p, sy, n, Q, 0, 1, b, &wk, x, y, traj, T_ooo, rounds, log);
    free(wk.step); free(wk.status); free(wk.tc); free(wk.mvx); free(wk.mvy); free(wk.cmax); free(wk.qkey);
    return rc;
}
