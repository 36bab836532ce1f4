/*
 * oracle/oracle.c -- CPU ORACLE (test infrastructure only).
 *
 * Plain, slow, obviously-correct C implementation of the AI Metropolis
 * spatio-temporal dependency tracker (arXiv 2411.03519) and of the synthetic
 * trace-replay driver around it.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table generator or constant with the CUDA path under
 * paper_2411_03519_b200/; the two are compared element by element in tests/.
 *
 * Citations: "P:<line>" = /root/reference/PAPER.md line, with its section.
 * Readings of ambiguous passages (Q1..Q21) are listed in DESIGN.md section 3.
 *
 * Everything is integer arithmetic (int64 for squared distances, uint64 mod 2^64
 * for the counter-based hash), so there is no rounding anywhere.
 *
 * Pins (tests/test_oracle.py): hand-worked vectors V1..V14 (tests/golden/),
 * closed-form driver vectors D1..D5, invariants I1..I7, connected components
 * cross-checked against a BFS written independently in the test, brute-force
 * enumeration of tiny maps; orc_validity_violations by exact counts on hand states
 * at the strict P:156 boundary (tests/test_oracle_pins.py).  The synthetic
 * latency/policy functions (mix64, key3, orc_duration, orc_digest, orc_policy_move,
 * the trajectory hash) are our own constructs (the paper is silent, Q16): pinned
 * against an independent Python implementation of SURVEY 8(c.4) built on
 * splitmix64's published outputs, structural cases, and the closed forms D1..D5.
 * oracle_scale.c drives the same predicates at BASELINE sizes (threads, per-step
 * pair enumeration, hash-grid perception for the lock-step run).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { ORC_IDLE = 0, ORC_RUNNING = 1, ORC_DONE = 2 };
enum { ORC_OK = 0, ORC_E_ARG = -1, ORC_E_BOUNDS = -2, ORC_E_PROTOCOL = -3,
       ORC_E_VELOCITY = -4, ORC_E_LIVENESS = -8, ORC_E_INVARIANT = -9, ORC_E_CAPACITY = -10 };
enum { ORC_L2 = 0, ORC_LINF = 1, ORC_GRAPH = 2 };

typedef struct {
    int32_t map_w, map_h;   /* x in [0,map_w), y in [0,map_h)              (Q14) */
    int32_t r_p;            /* radius_p, perception radius in tiles */
    int32_t v;              /* max_vel, tiles per step */
    int32_t target;         /* target_step (Alg. 1/3 P:108); 0 = unbounded      */
    int32_t metric;         /* ORC_L2 (Euclidean, Q1) or ORC_LINF        */
    int32_t n_sims;         /* >=1 independent simulations, agents partitioned  */
    /* ORC_GRAPH ("non-Euclidean spaces such as social networks",
     * P:309): positions are graph nodes (x = node, y = 0) and dist(A,B) is the hop
     * count gdist[x_A * gV + x_B] (0xFFFF = unreachable), the shortest-path metric the
     * App. A derivation needs (triangle inequality + at most v hops per step). */
    const uint16_t* gdist;
    int32_t gV;
} orc_params;

/* agents of simulation b are [b*n/n_sims, (b+1)*n/n_sims) */
static int32_t sim_lo(int64_t n, int64_t n_sims, int64_t b) { return (int32_t)(b * n / n_sims); }

/* dist(A,B) <= R under the metric.  R may exceed any distance on the map
 * (it grows with the step gap); compare in int64 without overflow. */
static int within(const orc_params* p, int64_t dx, int64_t dy, int64_t R)
{
    if (R < 0) return 0;
    if (p->metric == ORC_LINF) {
        int64_t ax = dx < 0 ? -dx : dx, ay = dy < 0 ? -dy : dy;
        return ax <= R && ay <= R;
    }
    if (R > 2000000000LL) return 1;          /* every on-map d^2 < 2^31 < R^2 */
    return dx * dx + dy * dy <= R * R;
}

/* dist(A,B) <= R for the positions of A and B under the metric */
static int within_pts(const orc_params* p, int64_t xa, int64_t ya, int64_t xb, int64_t yb, int64_t R)
{
    if (p->metric == ORC_GRAPH) {
        if (R < 0) return 0;
        const uint16_t d = p->gdist[xa * p->gV + xb];
        return d != 0xFFFF && (int64_t)d <= R;
    }
    return within(p, xa - xb, ya - yb, R);
}

/* P:160 (section 3.2) and App. A: A and B are coupled iff
 * Step_A == Step_B and dist(A,B) <= radius_p + max_vel. */
int orc_coupled(const orc_params* p, int32_t xa, int32_t ya, int32_t sa,
                int32_t xb, int32_t yb, int32_t sb)
{
    return sa == sb && within_pts(p, xa, ya, xb, yb, (int64_t)p->r_p + p->v);
}

/* P:161 (section 3.2; the minus sign is lost there) restated from App. A P:406:
 * A is blocked by B iff dist(A,B) <= (Step_A - Step_B + 1)*max_vel + radius_p.
 * Only agents behind A in time can block it: P:408-417 shows that a future agent
 * (Step_B > Step_A) never blocks, and equal steps are the coupling case
 * (P:380-394), hence the strict Step_B < Step_A (Q3). */
int orc_blocked_by(const orc_params* p, int32_t xa, int32_t ya, int32_t sa,
                   int32_t xb, int32_t yb, int32_t sb)
{
    if (!(sb < sa)) return 0;
    int64_t R = ((int64_t)sa - sb + 1) * p->v + p->r_p;
    return within_pts(p, xa, ya, xb, yb, R);
}

/* ---- sequential union-find; the root of every tree is its minimum id (Q10) ---- */
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

typedef struct { int32_t sim, step, label, id; } ord_key;
static int ord_cmp(const void* pa, const void* pb)
{
    const ord_key* a = (const ord_key*)pa;
    const ord_key* b = (const ord_key*)pb;
    if (a->sim != b->sim) return a->sim < b->sim ? -1 : 1;
    if (a->step != b->step) return a->step < b->step ? -1 : 1;
    if (a->label != b->label) return a->label < b->label ? -1 : 1;
    return a->id < b->id ? -1 : (a->id > b->id);
}

/*
 * One scheduling round = one controller iteration of Alg. 3:
 * geo_clustering (section 3.4) + the cluster-ready rule
 * + priority order by step (section 3.5).
 *
 *   act[i]     = status[i] != DONE                                    (Q8)
 *   blocked[i] = act[i] && exists j: act[j] && orc_blocked_by(i, j)
 *   components of the coupling graph over all act agents             (Q5, Q6)
 *   label[i]   = min id of i's component, -1 if DONE                  (Q10)
 *   bad(C)     = some member blocked or RUNNING                       (Q7)
 *   mask[i]    = status[i]==IDLE && !bad(component of i)
 *   order      = mask agents sorted by (sim, step, label, id)          (Q9)
 *   unless peek: status[i] = RUNNING for every mask agent (dispatch)   (Q12)
 *
 * Every output array has n entries (order: capacity n).  Brute force O(n^2)
 * per simulation.  blocked may be NULL.
 */
int orc_round(const orc_params* p, int32_t n, const int32_t* x, const int32_t* y,
              const int32_t* step, uint8_t* status, int32_t peek,
              uint8_t* blocked, int32_t* label, uint8_t* mask, int32_t* order,
              int32_t* n_ready)
{
    if (n < 0 || p->n_sims < 1) return ORC_E_ARG;
    int32_t* parent = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    uint8_t* blk = (uint8_t*)malloc(n ? n : 1);
    uint8_t* bad = (uint8_t*)calloc(n ? n : 1, 1);
    ord_key* keys = (ord_key*)malloc(sizeof(ord_key) * (n ? n : 1));
    for (int32_t i = 0; i < n; i++) parent[i] = i;

    int32_t nr = 0;
    for (int32_t b = 0; b < p->n_sims; b++) {
        int32_t lo = sim_lo(n, p->n_sims, b), hi = sim_lo(n, p->n_sims, b + 1);
        for (int32_t i = lo; i < hi; i++) {
            blk[i] = 0;
            if (status[i] == ORC_DONE) continue;
            for (int32_t j = lo; j < hi; j++) {
                if (j == i || status[j] == ORC_DONE) continue;
                if (orc_blocked_by(p, x[i], y[i], step[i], x[j], y[j], step[j])) { blk[i] = 1; break; }
            }
        }
        for (int32_t i = lo; i < hi; i++) {
            if (status[i] == ORC_DONE) continue;
            for (int32_t j = i + 1; j < hi; j++) {
                if (status[j] == ORC_DONE) continue;
                if (orc_coupled(p, x[i], y[i], step[i], x[j], y[j], step[j])) uf_union(parent, i, j);
            }
        }
        for (int32_t i = lo; i < hi; i++) {
            if (status[i] == ORC_DONE) { label[i] = -1; continue; }
            label[i] = uf_find(parent, i);
            if (blk[i] || status[i] == ORC_RUNNING) bad[label[i]] = 1;
        }
        for (int32_t i = lo; i < hi; i++) {
            mask[i] = (uint8_t)(status[i] == ORC_IDLE && !bad[label[i]]);
            if (mask[i]) {
                keys[nr].sim = b; keys[nr].step = step[i]; keys[nr].label = label[i]; keys[nr].id = i;
                nr++;
            }
        }
    }
    qsort(keys, (size_t)nr, sizeof(ord_key), ord_cmp);
    for (int32_t k = 0; k < nr; k++) order[k] = keys[k].id;
    if (!peek)
        for (int32_t k = 0; k < nr; k++) status[order[k]] = ORC_RUNNING;
    if (blocked) memcpy(blocked, blk, (size_t)n);
    *n_ready = nr;
    free(parent); free(blk); free(bad); free(keys);
    return ORC_OK;
}

/*
 * Sampled round at sizes where the O(n^2) round is too slow: for each agent i in
 * `sample`, the same three outputs as orc_round but computed one by one:
 *   blocked[i] by scanning all agents; the component of i by a breadth-first
 *   walk of the coupling graph whose every expansion scans all agents;
 *   label[i] = min id in the component; mask[i] = IDLE && no member bad.
 * Pure function of the state (no dispatch).  O(n * |component|) per sample.
 */
int orc_round_sampled(const orc_params* p, int32_t n, const int32_t* x, const int32_t* y,
                      const int32_t* step, const uint8_t* status, int32_t n_sample,
                      const int32_t* sample, uint8_t* blocked, int32_t* label, uint8_t* mask,
                      int32_t* comp_size)
{
    if (p->n_sims != 1) return ORC_E_ARG;
    int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    uint8_t* seen = (uint8_t*)calloc(n ? n : 1, 1);
    for (int32_t k = 0; k < n_sample; k++) {
        int32_t i = sample[k];
        if (i < 0 || i >= n) { free(queue); free(seen); return ORC_E_ARG; }
        if (status[i] == ORC_DONE) { blocked[k] = 0; label[k] = -1; mask[k] = 0; comp_size[k] = 0; continue; }
        int32_t head = 0, tail = 0, minid = i, bad = 0;
        queue[tail++] = i; seen[i] = 1;
        while (head < tail) {
            int32_t a = queue[head++];
            if (a < minid) minid = a;
            int blk = 0;
            for (int32_t j = 0; j < n; j++) {
                if (j == a || status[j] == ORC_DONE) continue;
                if (!blk && orc_blocked_by(p, x[a], y[a], step[a], x[j], y[j], step[j])) blk = 1;
                if (!seen[j] && orc_coupled(p, x[a], y[a], step[a], x[j], y[j], step[j])) {
                    seen[j] = 1; queue[tail++] = j;
                }
            }
            if (a == i) blocked[k] = (uint8_t)blk;
            if (blk || status[a] == ORC_RUNNING) bad = 1;
        }
        label[k] = minid;
        mask[k] = (uint8_t)(status[i] == ORC_IDLE && !bad);
        comp_size[k] = tail;
        for (int32_t q = 0; q < tail; q++) seen[queue[q]] = 0;
    }
    free(queue); free(seen);
    return ORC_OK;
}

/*
 * update_agents (Alg. 3 line 11) with commit validation.
 * first != 0: set the initial state (status IDLE, or DONE at target) -- bounds only.
 * Otherwise per agent, with ds = new_step - step:
 *   ds == 0: position must be unchanged; status unchanged;
 *   ds == 1: agent must be RUNNING (it was dispatched, Alg. 3) and
 *            dist(p', p) <= max_vel (the speed limit of P:153 that App. A P:385 rests
 *            on); status becomes DONE if new_step == target (Q8) else IDLE;
 *   else   : protocol error.
 * All-or-nothing: on any error nothing is changed.  Returns the first error
 * code in the priority BOUNDS > PROTOCOL > VELOCITY (any agent).
 */
int orc_update(const orc_params* p, int32_t n, int32_t first, int32_t* x, int32_t* y,
               int32_t* step, uint8_t* status, const int32_t* nx, const int32_t* ny,
               const int32_t* nstep)
{
    int err_b = 0, err_p = 0, err_v = 0;
    for (int32_t i = 0; i < n; i++) {
        if (nx[i] < 0 || nx[i] >= p->map_w || ny[i] < 0 || ny[i] >= p->map_h) err_b = 1;
        if (first) {
            if (nstep[i] < 0 || (p->target > 0 && nstep[i] > p->target)) err_p = 1;
            continue;
        }
        int64_t ds = (int64_t)nstep[i] - step[i];
        if (ds == 0) {
            if (nx[i] != x[i] || ny[i] != y[i]) err_p = 1;
        } else if (ds == 1) {
            if (status[i] != ORC_RUNNING) err_p = 1;
            else if (!within_pts(p, x[i], y[i], nx[i], ny[i], p->v)) err_v = 1;
        } else {
            err_p = 1;
        }
    }
    if (err_b) return ORC_E_BOUNDS;
    if (err_p) return ORC_E_PROTOCOL;
    if (err_v) return ORC_E_VELOCITY;
    for (int32_t i = 0; i < n; i++) {
        if (first) {
            status[i] = (p->target > 0 && nstep[i] == p->target) ? ORC_DONE : ORC_IDLE;
        } else if (nstep[i] != step[i]) {
            status[i] = (p->target > 0 && nstep[i] == p->target) ? ORC_DONE : ORC_IDLE;
        }
        x[i] = nx[i]; y[i] = ny[i]; step[i] = nstep[i];
    }
    return ORC_OK;
}

/* Validity condition P:156 (section 3.2) = App. A: for all A,B with
 * Step_A != Step_B: dist(A,B) > radius_p + (|Step_A - Step_B| - 1)*max_vel.
 * Returns the number of violating unordered pairs (within each sim). */
int64_t orc_validity_violations(const orc_params* p, int32_t n, const int32_t* x,
                                const int32_t* y, const int32_t* step)
{
    int64_t bad = 0;
    for (int32_t b = 0; b < p->n_sims; b++) {
        int32_t lo = sim_lo(n, p->n_sims, b), hi = sim_lo(n, p->n_sims, b + 1);
        for (int32_t i = lo; i < hi; i++)
            for (int32_t j = i + 1; j < hi; j++) {
                if (step[i] == step[j]) continue;
                int64_t g = (int64_t)step[i] - step[j];
                if (g < 0) g = -g;
                /* dist > R  <=>  !(dist <= R) */
                if (within_pts(p, x[i], y[i], x[j], y[j], (int64_t)p->r_p + (g - 1) * p->v))
                    bad++;
            }
    }
    return bad;
}

/* =========================== synthetic driver ================================
 * The paper replays recorded GenAgent traces; those are not available, so
 * actions come from a deterministic random-walk policy and per-step LLM latencies
 * from integer tables.  The paper is silent on all of
 * this, so SURVEY 8(c.4) defines it; pinned against that definition by independent
 * pure-Python restatements and splitmix64's published outputs
 * (tests/test_oracle_pins.py) and by the D1..D5 closed forms (tests/test_oracle.py). */

/* splitmix64 finalizer (Steele/Lea/Flood 2014), with its golden-gamma increment. */
uint64_t orc_mix64(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
uint64_t orc_key3(uint64_t seed, uint64_t a, uint64_t b)
{
    return orc_mix64(orc_mix64(orc_mix64(seed + a) + b));
}

typedef struct {
    const uint32_t* lat;      /* LAT[1024]: per-call latency quantiles, microseconds */
    const uint64_t* cdf32;    /* cumulative call-count probabilities scaled to 2^32   */
    const int32_t*  vals;     /* call counts K for each CDF bucket                    */
    int32_t n_vals;
    int32_t base_us;          /* fixed per-step cost                                  */
    uint64_t lat_seed;
    uint64_t policy_seed;
    const uint8_t* wall;      /* [map_h*map_w] row-major, 1 = wall; NULL = open map   */
    const int64_t* dur_table; /* optional explicit durations [n][dur_T] (closed forms)  */
    int32_t dur_T;
    int32_t policy;           /* 0 = random walk, 1 = always stay, 2 = 8-connected,    */
                              /* 3 = graph walk (ORC_GRAPH)                             */
    int32_t conflict;         /* 0 = co-occupancy allowed; 1 = exclusive tiles (below)  */
    const int32_t* graph_off; /* policy 3: CSR adjacency of the graph, [gV + 1] offsets  */
    const int32_t* graph_adj; /*           and the neighbour lists                      */
} orc_synth;

/*
 * Exclusive tiles ("write conflicts that must be resolved by
 * developer-specified rules ... two agents might both want to use the bathroom, but
 * only one can step in"; world.resolve_conflict_and_commit, Alg. 3 l.20 P:124):
 * among a group of agents moving together, a proposed move is cancelled if its target
 * tile is occupied now by another agent of the group, or if a lower-id agent of the
 * group proposes the same tile (the lowest id among the proposers gets it).  The group
 * is the whole simulation in lock-step and the cluster in the out-of-order replay:
 * same-step agents that could contest a tile are within 2 v <= r_p + v (coupled), and
 * validity keeps agents at other steps farther than r_p >= 2 v (required).
 * idx[0..k) lists the group; x,y are current positions, px,py the proposals (updated
 * in place: cancelled proposals become the current position).
 */
static void resolve_exclusive(int32_t k, const int32_t* idx, const int32_t* x, const int32_t* y,
                              int32_t* px, int32_t* py)
{
    uint8_t* ok = (uint8_t*)malloc(k ? k : 1);
    for (int32_t a = 0; a < k; a++) {
        int32_t i = idx[a];
        ok[a] = 1;
        if (px[i] == x[i] && py[i] == y[i]) continue;   /* staying never conflicts */
        for (int32_t b = 0; b < k && ok[a]; b++) {
            int32_t j = idx[b];
            if (j == i) continue;
            if (x[j] == px[i] && y[j] == py[i]) ok[a] = 0;               /* occupied now */
            if (j < i && px[j] == px[i] && py[j] == py[i]) ok[a] = 0;    /* lower id wants it */
        }
    }
    for (int32_t a = 0; a < k; a++)
        if (!ok[a]) { px[idx[a]] = x[idx[a]]; py[idx[a]] = y[idx[a]]; }
    free(ok);
}

/* duration of agent i's step s in integer microseconds. */
int64_t orc_duration(const orc_synth* sy, int32_t i, int32_t s)
{
    if (sy->dur_table) return sy->dur_table[(int64_t)i * sy->dur_T + s];
    uint64_t u = orc_key3(sy->lat_seed, (uint64_t)(uint32_t)i, (uint64_t)(uint32_t)s);
    uint64_t hi = u >> 32;
    int32_t m = 0;
    while (m < sy->n_vals - 1 && !(hi < sy->cdf32[m])) m++;
    int32_t K = sy->vals[m];
    int64_t d = sy->base_us;
    for (int32_t k = 0; k < K; k++) {
        uint64_t h = orc_key3(sy->lat_seed ^ 0xC0FFEEULL,
                              ((uint64_t)(uint32_t)i << 20) ^ (uint64_t)(uint32_t)s, (uint64_t)k);
        d += sy->lat[h >> 54];
    }
    return d;
}

/* perception digest of agent i (section 2.1 Alg. 2 line 3 "perceive"; radius_p P:153):
 * sum mod 2^64 over perceived j != i (non-DONE, same step, within radius_p) of
 * mix64((j<<32) ^ ((u16)dx<<16) ^ (u16)dy).  Order independent. */
uint64_t orc_digest(const orc_params* p, int32_t lo, int32_t hi, const int32_t* x,
                    const int32_t* y, const int32_t* step, const uint8_t* status, int32_t i)
{
    uint64_t dig = 0;
    for (int32_t j = lo; j < hi; j++) {
        if (j == i || status[j] == ORC_DONE || step[j] != step[i]) continue;
        int32_t dx = x[j] - x[i], dy = y[j] - y[i];
        if (!within_pts(p, x[i], y[i], x[j], y[j], p->r_p)) continue;
        uint64_t w = ((uint64_t)(uint32_t)j << 32) ^ ((uint64_t)(uint16_t)dx << 16) ^ (uint64_t)(uint16_t)dy;
        dig += orc_mix64(w);
    }
    return dig;
}

/* random-walk policy: one of {stay,+x,-x,+y,-y}; a move into a wall or off the
 * map is replaced by stay (co-occupancy allowed, Q15).  |dp| <= 1 <= max_vel. */
void orc_policy_move(const orc_params* p, const orc_synth* sy, int32_t i, int32_t s,
                     int32_t px, int32_t py, uint64_t digest, int32_t* nx, int32_t* ny)
{
    /* policy 0: 4-connected random walk {stay,+x,-x,+y,-y}[h % 5]; 1: stay;
     * 2: 8-connected random walk (with the L-infinity metric a
     *    diagonal move is within v = 1): {the 5 above, (+1,+1), (-1,+1), (+1,-1), (-1,-1)}[h % 9] */
    static const int32_t MX[9] = {0, 1, -1, 0, 0, 1, -1, 1, -1};
    static const int32_t MY[9] = {0, 0, 0, 1, -1, 1, 1, -1, -1};
    uint64_t h = orc_mix64(orc_key3(sy->policy_seed, (uint64_t)(uint32_t)i, (uint64_t)(uint32_t)s) + digest);
    if (sy->policy == 3) {
        /* graph walk: {stay, neighbour 0, ..., neighbour deg-1}[h % (deg + 1)] -- one hop,
         * within v >= 1 under the hop metric */
        const int32_t deg = sy->graph_off[px + 1] - sy->graph_off[px];
        const int32_t m = (int32_t)(h % (uint64_t)(deg + 1));
        *nx = m == 0 ? px : sy->graph_adj[sy->graph_off[px] + m - 1];
        *ny = py;
        return;
    }
    int32_t m = sy->policy == 1 ? 0 : sy->policy == 2 ? (int32_t)(h % 9) : (int32_t)(h % 5);
    int32_t qx = px + MX[m], qy = py + MY[m];
    int ok = qx >= 0 && qx < p->map_w && qy >= 0 && qy < p->map_h;
    if (ok && sy->wall && sy->wall[(int64_t)qy * p->map_w + qx]) ok = 0;
    *nx = ok ? qx : px;
    *ny = ok ? qy : py;
}

/* per-agent trajectory hash, chained at every committed step */
static uint64_t traj_step(uint64_t th, int32_t s, int32_t x, int32_t y)
{
    return orc_mix64(th ^ (((uint64_t)(uint32_t)s << 32) | ((uint64_t)(uint16_t)x << 16) | (uint64_t)(uint16_t)y));
}

/*
 * Algorithm 1: lock-step simulation for T steps.  Every agent perceives
 * the same-step world (all agents at step s) and all moves are applied together.
 * T_sync[b] = sum_s max_{i in sim b} duration(i, s)  (global barrier per step).
 * x,y are updated in place; traj[i] receives the trajectory hash.
 */
int orc_lockstep(const orc_params* p, const orc_synth* sy, int32_t n, int32_t T,
                 int32_t* x, int32_t* y, uint64_t* traj, int64_t* T_sync)
{
    int32_t* nx = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    int32_t* ny = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    int32_t* st = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    uint8_t* status = (uint8_t*)calloc(n ? n : 1, 1);
    for (int32_t i = 0; i < n; i++) traj[i] = 0;
    for (int32_t b = 0; b < p->n_sims; b++) T_sync[b] = 0;
    for (int32_t s = 0; s < T; s++) {
        for (int32_t i = 0; i < n; i++) st[i] = s;
        for (int32_t b = 0; b < p->n_sims; b++) {
            int32_t lo = sim_lo(n, p->n_sims, b), hi = sim_lo(n, p->n_sims, b + 1);
            int64_t mx = 0;
            for (int32_t i = lo; i < hi; i++) {
                uint64_t dg = orc_digest(p, lo, hi, x, y, st, status, i);
                orc_policy_move(p, sy, i, s, x[i], y[i], dg, &nx[i], &ny[i]);
                int64_t d = orc_duration(sy, i, s);
                if (d > mx) mx = d;
            }
            if (sy->conflict) {   /* the whole simulation moves together */
                int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * (hi - lo ? hi - lo : 1));
                for (int32_t i = lo; i < hi; i++) idx[i - lo] = i;
                resolve_exclusive(hi - lo, idx, x, y, nx, ny);
                free(idx);
            }
            T_sync[b] += mx;
        }
        for (int32_t i = 0; i < n; i++) {
            x[i] = nx[i]; y[i] = ny[i];
            traj[i] = traj_step(traj[i], s + 1, x[i], y[i]);
        }
    }
    free(nx); free(ny); free(st); free(status);
    return ORC_OK;
}

typedef struct {
    /* optional per-round log (all pointers may be NULL).  Entry r of sim b is
     * written in the order rounds happen inside each sim; sims are replayed one
     * after another (they are independent, Alg. 3 per sim). */
    int64_t cap_rounds, cap_entries;
    int64_t* round_t;        /* [cap_rounds]  event time of the round              */
    int32_t* round_sim;      /* [cap_rounds]                                       */
    int32_t* round_nready;   /* [cap_rounds]                                       */
    int32_t* entry_id;       /* [cap_entries] order of each round, concatenated    */
    int32_t* entry_label;    /* [cap_entries] label of each dispatched agent       */
    int64_t n_rounds, n_entries;   /* out */
    int32_t check;           /* check I1 (safety at dispatch) and I2 (validity)    */
    int64_t violations;      /* out: invariant violations seen                     */
    int64_t max_spread;      /* out: max over rounds of S - W                      */
} orc_log;

/*
 * Out-of-order replay (Alg. 3 P:97-126 with infinite LLM capacity):
 * per simulation, t = 0; loop {
 *    commit every RUNNING agent whose cluster completion time <= t (apply the
 *      move computed at dispatch, step += 1; DONE at target)        (Alg. 3 l.20-21, l.11)
 *    round (orc_round with dispatch)                                  (Alg. 3 l.8-9)
 *    every ready cluster C: t_C = t + max_{i in C} duration(i, s_i);
 *      member moves computed now from the current (frozen) perception
 *    if all DONE: T_ooo = t, stop
 *    t = min pending completion (Q = 0) or rounded up to a multiple of Q   (Q11)
 * }
 * x,y in place (start at step 0, all IDLE).  traj[i] as in orc_lockstep.
 */
/*
 * Finite LLM capacity (our model, the paper serves clusters from a
 * priority ready_queue, section 3.5, "no preemption"):
 * capacity K > 0 agent-steps may be in service at once.  A ready cluster is queued
 * (its members become RUNNING, moves computed then) with the key
 *   priority = 1: (step << 32) | label      (earlier steps first)
 *   priority = 0: (round  << 32) | label    (FIFO by the round that queued it)
 * with label the cluster's global min id and round the simulation's round index.
 * After each round's enqueueing, clusters start in key order while they fit
 * (strict order, no bypass; a cluster larger than K starts only when nothing is in
 * service): completion = t + max member duration.  K = 0: infinite capacity, every
 * ready cluster starts at once (orc_replay).
 */
int orc_replay_cap(const orc_params* p, const orc_synth* sy, int32_t n, int64_t Q, int64_t K, int32_t priority,
                   int32_t* x, int32_t* y, uint64_t* traj, int64_t* T_ooo, int64_t* rounds, orc_log* log);

int orc_replay(const orc_params* p, const orc_synth* sy, int32_t n, int64_t Q,
               int32_t* x, int32_t* y, uint64_t* traj, int64_t* T_ooo, int64_t* rounds,
               orc_log* log)
{
    return orc_replay_cap(p, sy, n, Q, 0, 1, x, y, traj, T_ooo, rounds, log);
}

/* work arrays of a replay, indexed by agent id; simulation b only touches its slice
 * [lo, hi), so simulations may be replayed one after another or concurrently */
typedef struct {
    uint64_t* qkey;   /* queued members' keys (finite capacity) */
    int32_t* step;
    uint8_t* status;
    int64_t* tc;      /* completion time of the agent's dispatched step */
    int32_t *mvx, *mvy;   /* move computed at dispatch */
    int64_t* cmax;    /* cluster completion time, by label */
} orc_replay_work;

/* the replay of simulation b (the loop body of orc_replay_cap) */
int orc_replay_sim(const orc_params* p, const orc_synth* sy, int32_t n, int64_t Q, int64_t K, int32_t priority,
                   int32_t b, const orc_replay_work* wk, int32_t* x, int32_t* y, uint64_t* traj, int64_t* T_ooo,
                   int64_t* rounds, orc_log* log)
{
    uint64_t* qkey = wk->qkey;
    int32_t* step = wk->step;
    uint8_t* status = wk->status;
    int64_t* tc = wk->tc;
    int32_t* mvx = wk->mvx;
    int32_t* mvy = wk->mvy;
    int64_t* cmax = wk->cmax;
    int rc = ORC_OK;
    {
        int32_t lo = sim_lo(n, p->n_sims, b), hi = sim_lo(n, p->n_sims, b + 1);
        int32_t m = hi - lo;
        orc_params ps = *p; ps.n_sims = 1;
        int32_t *sx = x + lo, *sy_ = y + lo, *ss = step + lo;
        uint8_t* sst = status + lo;
        int32_t* lab = (int32_t*)malloc(sizeof(int32_t) * (m ? m : 1));
        uint8_t* msk = (uint8_t*)malloc(m ? m : 1);
        int32_t* ord = (int32_t*)malloc(sizeof(int32_t) * (m ? m : 1));
        uint8_t* blk = (uint8_t*)malloc(m ? m : 1);
        int64_t t = 0, nr_b = 0;
        for (int32_t i = 0; i < m; i++) { ss[i] = 0; sst[i] = (p->target == 0) ? ORC_DONE : ORC_IDLE; }
        for (;;) {
            /* commit (Alg. 3 worker l.20 + controller l.11-12) */
            for (int32_t i = 0; i < m; i++) {
                if (sst[i] == ORC_RUNNING && tc[lo + i] <= t) {
                    sx[i] = mvx[lo + i]; sy_[i] = mvy[lo + i]; ss[i] += 1;
                    sst[i] = (ss[i] == p->target) ? ORC_DONE : ORC_IDLE;
                    traj[lo + i] = traj_step(traj[lo + i], ss[i], sx[i], sy_[i]);
                }
            }
            if (log && log->check && orc_validity_violations(&ps, m, sx, sy_, ss) != 0) log->violations++;
            int32_t all_done = 1, any_running = 0, W = INT32_MAX, S = INT32_MIN;
            for (int32_t i = 0; i < m; i++) {
                if (sst[i] != ORC_DONE) {
                    all_done = 0;
                    if (ss[i] < W) W = ss[i];
                    if (ss[i] > S) S = ss[i];
                }
                if (sst[i] == ORC_RUNNING) any_running = 1;
            }
            if (all_done) break;
            if (log && (int64_t)S - W > log->max_spread) log->max_spread = (int64_t)S - W;
            /* round (Alg. 3 controller l.8-9) */
            int32_t nr = 0;
            orc_round(&ps, m, sx, sy_, ss, sst, 0, blk, lab, msk, ord, &nr);
            nr_b++;
            if (log && log->n_rounds < log->cap_rounds) {
                if (log->round_t) log->round_t[log->n_rounds] = t;
                if (log->round_sim) log->round_sim[log->n_rounds] = b;
                if (log->round_nready) log->round_nready[log->n_rounds] = nr;
                log->n_rounds++;
                for (int32_t k = 0; k < nr; k++) {
                    if (log->n_entries < log->cap_entries) {
                        if (log->entry_id) log->entry_id[log->n_entries] = lo + ord[k];
                        if (log->entry_label) log->entry_label[log->n_entries] = lo + lab[ord[k]];
                        log->n_entries++;
                    }
                }
            }
            /* I1 safety at dispatch: nobody behind within the blocking radius */
            if (log && log->check) {
                for (int32_t k = 0; k < nr; k++) {
                    int32_t a = ord[k];
                    for (int32_t j = 0; j < m; j++)
                        if (j != a && sst[j] != ORC_DONE &&
                            orc_blocked_by(&ps, sx[a], sy_[a], ss[a], sx[j], sy_[j], ss[j]))
                            log->violations++;
                }
            }
            /* dispatch: cluster completion time and the members' moves */
            for (int32_t k = 0; k < nr; k++) cmax[lo + lab[ord[k]]] = 0;
            for (int32_t k = 0; k < nr; k++) {
                int32_t a = ord[k];
                int64_t d = orc_duration(sy, lo + a, ss[a]);
                if (d > cmax[lo + lab[a]]) cmax[lo + lab[a]] = d;
            }
            for (int32_t k = 0; k < nr; k++) {
                int32_t a = ord[k];
                tc[lo + a] = t + cmax[lo + lab[a]];
                if (K > 0) {   /* finite capacity: queued, started below */
                    tc[lo + a] = INT64_MAX;
                    qkey[lo + a] = ((uint64_t)(priority ? (uint64_t)ss[a] : (uint64_t)(nr_b - 1)) << 32) |
                                   (uint64_t)(uint32_t)(lo + lab[a]);
                }
                /* digest over the sim, in global ids (perceived agents are cluster-mates) */
                uint64_t dg = orc_digest(p, lo, hi, x, y, step, status, lo + a);
                orc_policy_move(p, sy, lo + a, ss[a], sx[a], sy_[a], dg, &mvx[lo + a], &mvy[lo + a]);
            }
            if (sy->conflict && nr > 0) {   /* per ready cluster (members share a label) */
                int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * nr);
                for (int32_t k = 0; k < nr; k++) {
                    int32_t a = ord[k];
                    int32_t ng = 0;
                    for (int32_t q = 0; q < nr; q++)
                        if (lab[ord[q]] == lab[a]) idx[ng++] = lo + ord[q];
                    if (idx[0] != lo + a) continue;   /* each cluster once: from its lowest member */
                    resolve_exclusive(ng, idx, x, y, mvx, mvy);
                }
                free(idx);
            }
            if (K > 0) {
                /* in service: started members not yet committed */
                int64_t busy = 0;
                for (int32_t i = 0; i < m; i++)
                    if (sst[i] == ORC_RUNNING && tc[lo + i] != INT64_MAX) busy++;
                for (;;) {   /* start queued clusters in key order while they fit */
                    uint64_t best = UINT64_MAX;
                    for (int32_t i = 0; i < m; i++)
                        if (sst[i] == ORC_RUNNING && tc[lo + i] == INT64_MAX && qkey[lo + i] < best) best = qkey[lo + i];
                    if (best == UINT64_MAX) break;
                    int64_t size = 0, dmax = 0;
                    for (int32_t i = 0; i < m; i++)
                        if (sst[i] == ORC_RUNNING && tc[lo + i] == INT64_MAX && qkey[lo + i] == best) {
                            size++;
                            int64_t d = orc_duration(sy, lo + i, ss[i]);
                            if (d > dmax) dmax = d;
                        }
                    if (busy > 0 && busy + size > K) break;
                    for (int32_t i = 0; i < m; i++)
                        if (sst[i] == ORC_RUNNING && tc[lo + i] == INT64_MAX && qkey[lo + i] == best) tc[lo + i] = t + dmax;
                    busy += size;
                }
            }
            /* next event */
            int64_t tn = INT64_MAX;
            for (int32_t i = 0; i < m; i++)
                if (sst[i] == ORC_RUNNING && tc[lo + i] < tn) tn = tc[lo + i];
            if (tn == INT64_MAX) { rc = ORC_E_LIVENESS; break; }
            (void)any_running;
            if (Q > 0) tn = ((tn + Q - 1) / Q) * Q;
            t = tn;
        }
        T_ooo[b] = t;
        rounds[b] = nr_b;
        free(lab); free(msk); free(ord); free(blk);
    }
    return rc;
}

int orc_replay_cap(const orc_params* p, const orc_synth* sy, int32_t n, int64_t Q, int64_t K, int32_t priority,
                   int32_t* x, int32_t* y, uint64_t* traj, int64_t* T_ooo, int64_t* rounds, orc_log* log)
{
    if (p->target <= 0 || K < 0) return ORC_E_ARG;
    orc_replay_work wk;
    wk.qkey = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    wk.step = (int32_t*)calloc(n ? n : 1, sizeof(int32_t));
    wk.status = (uint8_t*)calloc(n ? n : 1, 1);
    wk.tc = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    wk.mvx = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    wk.mvy = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    wk.cmax = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    int rc = ORC_OK;
    if (log) { log->n_rounds = 0; log->n_entries = 0; log->violations = 0; log->max_spread = 0; }
    for (int32_t i = 0; i < n; i++) traj[i] = 0;
    for (int32_t b = 0; b < p->n_sims && rc == ORC_OK; b++)
        rc = orc_replay_sim(p, sy, n, Q, K, priority, b, &wk, x, y, traj, T_ooo, rounds, log);
    free(wk.step); free(wk.status); free(wk.tc); free(wk.mvx); free(wk.mvy); free(wk.cmax); free(wk.qkey);
    return rc;
}

/*
 * Stale-halo replay over G horizontal slabs (derived from App. A:
 * the blocking radius shrinks by exactly the blocker's progress, so a
 * blocker seen at an older step and position still blocks whenever the real one does;
 * the slab exchange itself is this repo's design, include/am_slab.h).  One simulation,
 * infinite capacity, no exclusive tiles.  Slab k owns the rows [k*H/G, (k+1)*H/G).
 * Rounds are counted from 0 while some agent is not DONE; round r is a SYNC round when
 * r % P == 0, else a STALE round.  At the start of every sync round (after its commits)
 * the snapshot (x, y, step, DONE) of every agent is kept and every agent's owner becomes
 * the slab of its row; owners stay fixed until the next sync round.
 *   sync round:  orc_replay's round (global, with dispatch).
 *   stale round: for every slab k, the agents k owns at their current state and every
 *     other agent at its snapshot, as RUNNING unless DONE: orc_round (peek) over that
 *     mixed state; the agents k owns that are ready in it are dispatched, labelled with
 *     their mixed-state label; the round's order is every dispatched agent by
 *     (step, label, id) (Q9).
 * The rest is orc_replay_sim's loop: cluster completion times, moves from the perception
 * digest of the current state, commits, the clock.  A stale round after which nothing is
 * pending leaves the clock where it is (the rounds up to the next sync round may then be
 * idle); only a sync round with nothing pending is a liveness failure.  P = 1 is
 * orc_replay.  That every dispatch is safe and the final state equals lock-step for any P
 * is tested (tests/test_oracle_stale.py), not assumed here.
 */
static int32_t slab_of_row(int32_t yy, int32_t G, int32_t H)
{
    int32_t k = 0;
    while (k + 1 < G && (int64_t)(k + 1) * H / G <= yy) k++;
    return k;
}

int orc_replay_stale(const orc_params* p, const orc_synth* sy, int32_t n, int64_t Q, int32_t G, int32_t P,
                     int32_t* x, int32_t* y, uint64_t* traj, int64_t* T_ooo, int64_t* rounds, orc_log* log)
{
    if (p->target <= 0 || p->n_sims != 1 || G < 1 || P < 1 || sy->conflict || p->metric == ORC_GRAPH) return ORC_E_ARG;
    size_t nn = (size_t)(n ? n : 1);
    int32_t* step = (int32_t*)calloc(nn, sizeof(int32_t));
    uint8_t* status = (uint8_t*)calloc(nn, 1);
    int64_t* tc = (int64_t*)malloc(sizeof(int64_t) * nn);
    int32_t* mvx = (int32_t*)malloc(sizeof(int32_t) * nn);
    int32_t* mvy = (int32_t*)malloc(sizeof(int32_t) * nn);
    int64_t* cmax = (int64_t*)calloc(nn, sizeof(int64_t));
    int32_t* owner = (int32_t*)calloc(nn, sizeof(int32_t));
    int32_t *x0 = (int32_t*)malloc(sizeof(int32_t) * nn), *y0 = (int32_t*)malloc(sizeof(int32_t) * nn);
    int32_t* s0 = (int32_t*)malloc(sizeof(int32_t) * nn);
    uint8_t* d0 = (uint8_t*)malloc(nn);
    int32_t *xm = (int32_t*)malloc(sizeof(int32_t) * nn), *ym = (int32_t*)malloc(sizeof(int32_t) * nn);
    int32_t* sm = (int32_t*)malloc(sizeof(int32_t) * nn);
    uint8_t* stm = (uint8_t*)malloc(nn);
    int32_t* lab = (int32_t*)malloc(sizeof(int32_t) * nn);
    int32_t* labk = (int32_t*)malloc(sizeof(int32_t) * nn);
    uint8_t* msk = (uint8_t*)malloc(nn);
    uint8_t* blk = (uint8_t*)malloc(nn);
    int32_t* ord = (int32_t*)malloc(sizeof(int32_t) * nn);
    ord_key* keys = (ord_key*)malloc(sizeof(ord_key) * nn);
    int rc = ORC_OK;
    int64_t t = 0, r = 0;
    if (log) { log->n_rounds = 0; log->n_entries = 0; log->violations = 0; log->max_spread = 0; }
    for (int32_t i = 0; i < n; i++) { traj[i] = 0; tc[i] = INT64_MAX; }
    for (;;) {
        /* commit (Alg. 3 worker l.20 + controller l.11-12) */
        for (int32_t i = 0; i < n; i++) {
            if (status[i] == ORC_RUNNING && tc[i] <= t) {
                x[i] = mvx[i]; y[i] = mvy[i]; step[i] += 1;
                status[i] = (step[i] == p->target) ? ORC_DONE : ORC_IDLE;
                traj[i] = traj_step(traj[i], step[i], x[i], y[i]);
            }
        }
        if (log && log->check && orc_validity_violations(p, n, x, y, step) != 0) log->violations++;
        int32_t all_done = 1, W = INT32_MAX, S = INT32_MIN;
        for (int32_t i = 0; i < n; i++)
            if (status[i] != ORC_DONE) {
                all_done = 0;
                if (step[i] < W) W = step[i];
                if (step[i] > S) S = step[i];
            }
        if (all_done) break;
        if (log && (int64_t)S - W > log->max_spread) log->max_spread = (int64_t)S - W;
        const int sync = (r % P) == 0;
        int32_t nr = 0;
        if (sync) {
            /* the snapshot and the owners of the rounds up to the next sync round */
            for (int32_t i = 0; i < n; i++) {
                x0[i] = x[i]; y0[i] = y[i]; s0[i] = step[i]; d0[i] = status[i] == ORC_DONE;
                owner[i] = slab_of_row(y[i], G, p->map_h);
            }
            orc_round(p, n, x, y, step, status, 0, blk, lab, msk, ord, &nr);
        } else {
            for (int32_t k = 0; k < G; k++) {
                for (int32_t i = 0; i < n; i++) {
                    if (owner[i] == k) { xm[i] = x[i]; ym[i] = y[i]; sm[i] = step[i]; stm[i] = status[i]; }
                    else { xm[i] = x0[i]; ym[i] = y0[i]; sm[i] = s0[i]; stm[i] = d0[i] ? ORC_DONE : ORC_RUNNING; }
                }
                int32_t nk = 0;
                orc_round(p, n, xm, ym, sm, stm, 1, blk, labk, msk, ord, &nk);
                for (int32_t i = 0; i < n; i++)
                    if (owner[i] == k && msk[i]) {
                        lab[i] = labk[i];
                        keys[nr].sim = 0; keys[nr].step = step[i]; keys[nr].label = labk[i]; keys[nr].id = i;
                        nr++;
                    }
            }
            qsort(keys, (size_t)nr, sizeof(ord_key), ord_cmp);
            for (int32_t q = 0; q < nr; q++) { ord[q] = keys[q].id; status[ord[q]] = ORC_RUNNING; }
        }
        r++;
        if (log && log->n_rounds < log->cap_rounds) {
            if (log->round_t) log->round_t[log->n_rounds] = t;
            if (log->round_sim) log->round_sim[log->n_rounds] = 0;
            if (log->round_nready) log->round_nready[log->n_rounds] = nr;
            log->n_rounds++;
            for (int32_t q = 0; q < nr; q++) {
                if (log->n_entries < log->cap_entries) {
                    if (log->entry_id) log->entry_id[log->n_entries] = ord[q];
                    if (log->entry_label) log->entry_label[log->n_entries] = lab[ord[q]];
                    log->n_entries++;
                }
            }
        }
        /* I1 safety at dispatch, on the real state */
        if (log && log->check) {
            for (int32_t q = 0; q < nr; q++) {
                int32_t a = ord[q];
                for (int32_t j = 0; j < n; j++)
                    if (j != a && status[j] != ORC_DONE &&
                        orc_blocked_by(p, x[a], y[a], step[a], x[j], y[j], step[j]))
                        log->violations++;
            }
        }
        /* dispatch: cluster completion time and the members' moves */
        for (int32_t q = 0; q < nr; q++) cmax[lab[ord[q]]] = 0;
        for (int32_t q = 0; q < nr; q++) {
            int32_t a = ord[q];
            int64_t d = orc_duration(sy, a, step[a]);
            if (d > cmax[lab[a]]) cmax[lab[a]] = d;
        }
        for (int32_t q = 0; q < nr; q++) {
            int32_t a = ord[q];
            tc[a] = t + cmax[lab[a]];
            uint64_t dg = orc_digest(p, 0, n, x, y, step, status, a);
            orc_policy_move(p, sy, a, step[a], x[a], y[a], dg, &mvx[a], &mvy[a]);
        }
        /* next event */
        int64_t tn = INT64_MAX;
        for (int32_t i = 0; i < n; i++)
            if (status[i] == ORC_RUNNING && tc[i] < tn) tn = tc[i];
        if (tn == INT64_MAX) {
            if (sync) { rc = ORC_E_LIVENESS; break; }
            continue;   /* nothing pending after a stale round: the clock stays */
        }
        if (Q > 0) tn = ((tn + Q - 1) / Q) * Q;
        t = tn;
    }
    T_ooo[0] = t;
    rounds[0] = r;
    free(step); free(status); free(tc); free(mvx); free(mvy); free(cmax); free(owner);
    free(x0); free(y0); free(s0); free(d0); free(xm); free(ym); free(sm); free(stm);
    free(lab); free(labk); free(msk); free(blk); free(ord); free(keys);
    return rc;
}
