/*
 * oracle.c -- CPU restatement of the reference hot path, TEST INFRASTRUCTURE.
 *
 * This file is the parity checker for the B200 engine, never the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * it.  It restates trafficsim/engine/world.py (World.step and the queries the
 * engine exports) statement by statement, with the reference's data
 * structures kept literal: per-vehicle records indexed by ascending id
 * (vix), the `_driving` dict as an insertion-ordered array, the per-lane
 * index rebuilt every step, the sequential id-ordered commit, and the
 * collision sweep with its restart-after-every-revert loop.  Float
 * expressions keep CPython's left-to-right association; the file is
 * compiled with -ffp-contract=off so no FMA is introduced.
 *
 * Powers (idm.py:25, idm.py:30): pow_mode 1 calls libm pow() exactly like
 * CPython's float.__pow__ (bit-identical to the reference on the same
 * glibc); pow_mode 0 returns the correctly rounded power for integer
 * exponents, computed independently of the device code via __float128.
 *
 * Pinned against the reference by tests/test_oracle.py (golden fixtures
 * produced by tests/golden/make_golden.py from the reference itself).
 */
#include <float.h>
#include <pthread.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/tsb200.h"

#define OK 0
#define ROADK 0
#define CONNK 1
enum { ST_WAITING = 0, ST_DRIVING = 1, ST_FINISHED = 2, ST_DROPPED = 3 };
enum { GREEN = 0, AMBER = 1, RED = 2 };

static const double EPS_GAP = 1e-6; /* world.py:43 */

static double py_min(double a, double b) { return (b < a) ? b : a; }
static double py_max(double a, double b) { return (b > a) ? b : a; }

typedef struct {
  int32_t* v;
  int32_t n, cap;
} ivec;

static void iv_push(ivec* a, int32_t x) {
  if (a->n == a->cap) {
    a->cap = a->cap ? 2 * a->cap : 8;
    a->v = (int32_t*)realloc(a->v, sizeof(int32_t) * (size_t)a->cap);
  }
  a->v[a->n++] = x;
}

/* Vehicle (world.py:46-69). */
typedef struct {
  int status;
  int32_t lane, ri, rp;
  double s, v;
  int32_t* roads; /* roads_seq as road indices */
  int32_t nroads;
  int routed; /* `veh.route` non-empty */
  double depart, finish, origin_s;
  int32_t origin_lane, dest;
  uint64_t key;
  int32_t snap_lane, snap_ri, snap_rp, idx_pos;
  double snap_s, snap_v;
  int32_t d_lane;
  double d_s, d_v;
  int d_changed, reverted;
} veh_t;

typedef struct {
  int32_t phase;
  double elapsed, since;
} sig_t;

typedef struct {
  int32_t dest;
  double* dist;
  uint64_t stamp;
} dcache_t;

struct orc {
  tsb_params p;
  int32_t nl, nr, nj, nv;
  double *len, *cap;
  int8_t* kind;
  uint8_t* open;
  int32_t *left, *right, *road, *junc, *pred1, *succ1, *succ_off, *succ, *pred_off, *pred;
  int32_t *road_lane_off, *road_lanes;
  uint8_t* jsig;
  int32_t* jph_off;
  double* ph_dur;
  uint64_t* green;
  sig_t* sig;
  int32_t *jc_off, *jc; /* junction -> connectors CSR (junction.connectors) */
  veh_t* V;
  /* _pending: vix sorted by (departure, id); _pend_i; _retry */
  int32_t* pending;
  int32_t pend_i;
  ivec retry;
  /* _driving in insertion order (tombstones compacted at the end of a step) */
  ivec drv;
  int32_t n_driving;
  /* _index: lane -> vix list (CSR rebuilt each step) */
  int32_t *idx_off, *idx;
  /* finished list */
  ivec fin_vix;
  double* fin_t;
  int64_t fin_cap;
  int64_t dropped, vehicle_updates, step_no, injected_now, finished_now, reverts_last, reverts_total;
  int threads; /* update-phase threads (orc_set_threads) */
  double time;
  /* speed accumulators [road][window] */
  int32_t nwin;
  double* acc_sum;
  int64_t* acc_cnt;
  /* router (routing.py) */
  double* w;
  dcache_t cache[256];
  uint64_t stamp;
};
typedef struct orc orc;

/* ---------------------------------------------------------------- powers */

static double pow_cr_int(double x, int n) {
  __float128 r = 1, b = x;
  while (n) {
    if (n & 1) r *= b;
    b *= b;
    n >>= 1;
  }
  return (double)r;
}

/* CPython's float ** float calls libm pow() (it never rewrites x**2 as x*x);
 * the call goes through a volatile pointer so the compiler cannot either. */
static double (*volatile libm_pow)(double, double) = pow;

static double py_pow(const orc* o, double x, double y) {
  if (o->p.pow_mode == 0 && y == floor(y) && y >= 1 && y <= 64) return pow_cr_int(x, (int)y);
  return libm_pow(x, y);
}

/* ---------------------------------------------------------------- rng.py:24-41 */

static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static double keyed_uniform4(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  uint64_t h = 0, k[4] = {a, b, c, d};
  for (int i = 0; i < 4; i++) h = mix64(h + 0x9E3779B97F4A7C15ULL + k[i]);
  return (double)(h >> 11) * 0x1p-53;
}

/* ---------------------------------------------------------------- idm.py:17-31 */

static double idm_accel(const orc* o, double v, double dv, double gap, double v_cap) {
  const tsb_params* p = &o->p;
  double v0_eff = py_min(p->idm_v0, v_cap);
  double fr = py_pow(o, v / v0_eff, p->idm_delta);
  double inter;
  if (isinf(gap)) {
    inter = 0.0;
  } else {
    double s_star = p->idm_s0 + py_max(0.0, v * p->idm_T + v * dv / (2.0 * sqrt(p->idm_a_max * p->idm_b)));
    inter = py_pow(o, s_star / gap, 2.0);
  }
  return p->idm_a_max * (1.0 - fr - inter);
}

/* ---------------------------------------------------------------- mobil.py:26-98 */

typedef struct {
  int ok;
  double s, v, len;
} view_t;

static double gap_to(view_t l, double fs) { return l.ok ? l.s - l.len - fs : INFINITY; }
static double accel_behind(const orc* o, double me_v, view_t l, double gap, double cap) {
  double dv = me_v - (l.ok ? l.v : 0.0);
  return idm_accel(o, me_v, dv, gap, cap);
}

static int evaluate_change(const orc* o, view_t me, view_t cl, view_t cf, view_t tl, view_t tf,
                           double s_t, double cap_cur, double cap_tgt, double* incentive) {
  const tsb_params* p = &o->p;
  double g_tl = gap_to(tl, s_t);
  double g_tf = tf.ok ? s_t - me.len - tf.s : INFINITY;
  if (g_tl <= 0.0 || g_tf <= 0.0) {
    *incentive = -INFINITY;
    return 0;
  }
  double a_me;
  double g_cur = gap_to(cl, me.s);
  if (g_cur <= 0.0)
    a_me = -INFINITY;
  else
    a_me = accel_behind(o, me.v, cl, g_cur, cap_cur);
  double a_me_new = accel_behind(o, me.v, tl, g_tl, cap_tgt);
  double a_nf = 0.0, a_nf_new = 0.0;
  if (tf.ok) {
    double g_nf_old = gap_to(tl, tf.s);
    if (g_nf_old <= 0.0) {
      *incentive = -INFINITY;
      return 0;
    }
    a_nf = accel_behind(o, tf.v, tl, g_nf_old, cap_tgt);
    view_t mev = {1, s_t, me.v, me.len};
    a_nf_new = accel_behind(o, tf.v, mev, g_tf, cap_tgt);
    if (a_nf_new < -p->mobil_b_safe) {
      *incentive = -INFINITY;
      return 0;
    }
  }
  double a_of = 0.0, a_of_new = 0.0;
  if (cf.ok) {
    double g_of_old = me.s - me.len - cf.s;
    double g_of_new = gap_to(cl, cf.s);
    if (g_of_old > 0.0 && g_of_new > 0.0) {
      a_of = accel_behind(o, cf.v, me, g_of_old, cap_cur);
      a_of_new = accel_behind(o, cf.v, cl, g_of_new, cap_cur);
    }
  }
  if (a_me == -INFINITY)
    *incentive = INFINITY;
  else
    *incentive = (a_me_new - a_me) + p->mobil_politeness * ((a_nf_new - a_nf) + (a_of_new - a_of));
  return 1;
}

/* ---------------------------------------------------------------- signals.py:37-61 */

static void advance_fixed(orc* o, int32_t j, double dt) {
  sig_t* st = &o->sig[j];
  int32_t b = o->jph_off[j], n = o->jph_off[j + 1] - b;
  st->elapsed += dt;
  while (st->elapsed >= o->ph_dur[b + st->phase]) {
    st->elapsed -= o->ph_dur[b + st->phase];
    st->phase = (st->phase + 1) % n;
  }
}

/* world.py:247-254 + signals.py:46-61 */
static int connector_aspect(const orc* o, int32_t conn) {
  int32_t j = o->junc[conn];
  if (!o->jsig[j]) return GREEN;
  const sig_t* st = &o->sig[j];
  if (!((o->green[conn] >> st->phase) & 1ULL)) return RED;
  double dur = o->ph_dur[o->jph_off[j] + st->phase];
  int timed = o->p.controller == 0;
  if (timed && o->p.amber > 0.0 && st->elapsed >= dur - o->p.amber) return AMBER;
  return GREEN;
}

/* ---------------------------------------------------------------- network helpers */

/* _conn_from[(lane, road)] (world.py:155-166): smallest successor connector of
 * a road lane whose successor lies on `road`; -1 if none. */
static int32_t conn_from(const orc* o, int32_t lane, int32_t road) {
  for (int32_t k = o->succ_off[lane]; k < o->succ_off[lane + 1]; k++) {
    int32_t c = o->succ[k];
    if (o->kind[c] == CONNK && o->road[o->succ1[c]] == road) return c;
  }
  return -1;
}

/* world.py:256-259 */
static int32_t next_connector(const orc* o, int32_t lane, int32_t rp, const veh_t* vh) {
  if (rp + 1 >= vh->nroads) return -1;
  return conn_from(o, lane, vh->roads[rp + 1]);
}

/* ---------------------------------------------------------------- routing.py */

typedef struct {
  double d;
  int32_t u;
} hitem;

static int hless(hitem a, hitem b) { return a.d < b.d || (a.d == b.d && a.u < b.u); }

static void rebuild_router(orc* o) {
  for (int32_t l = 0; l < o->nl; l++)
    o->w[l] = (o->kind[l] >= 0 && o->open[l]) ? o->len[l] / o->cap[l] : -1.0;
  for (int i = 0; i < 256; i++) {
    free(o->cache[i].dist);
    o->cache[i].dist = NULL;
  }
}

/* Router.dist_to (routing.py:47-68): reverse Dijkstra over open lanes. */
static const double* dist_to(orc* o, int32_t dest) {
  for (int i = 0; i < 256; i++)
    if (o->cache[i].dist && o->cache[i].dest == dest) {
      o->cache[i].stamp = ++o->stamp;
      return o->cache[i].dist;
    }
  double* dist = (double*)malloc(sizeof(double) * (size_t)o->nl);
  for (int32_t l = 0; l < o->nl; l++) dist[l] = -1.0;
  size_t hcap = 1024, hn = 0;
  hitem* h = (hitem*)malloc(sizeof(hitem) * hcap);
  h[hn++] = (hitem){o->w[dest], dest};
  while (hn) {
    hitem top = h[0];
    h[0] = h[--hn];
    for (size_t i = 0;;) { /* sift down */
      size_t a = 2 * i + 1, b = a + 1, m = i;
      if (a < hn && hless(h[a], h[m])) m = a;
      if (b < hn && hless(h[b], h[m])) m = b;
      if (m == i) break;
      hitem t = h[i];
      h[i] = h[m];
      h[m] = t;
      i = m;
    }
    if (dist[top.u] >= 0) continue;
    dist[top.u] = top.d;
    for (int32_t k = o->pred_off[top.u]; k < o->pred_off[top.u + 1]; k++) {
      int32_t pl = o->pred[k];
      if (o->w[pl] < 0 || dist[pl] >= 0) continue;
      if (hn == hcap) {
        hcap *= 2;
        h = (hitem*)realloc(h, sizeof(hitem) * hcap);
      }
      size_t i = hn++;
      h[i] = (hitem){o->w[pl] + top.d, pl};
      while (i && hless(h[i], h[(i - 1) / 2])) { /* sift up */
        hitem t = h[i];
        h[i] = h[(i - 1) / 2];
        h[(i - 1) / 2] = t;
        i = (i - 1) / 2;
      }
    }
  }
  free(h);
  int slot = 0;
  for (int i = 0; i < 256; i++) {
    if (!o->cache[i].dist) {
      slot = i;
      break;
    }
    if (o->cache[i].stamp < o->cache[slot].stamp) slot = i;
  }
  free(o->cache[slot].dist);
  o->cache[slot] = (dcache_t){dest, dist, ++o->stamp};
  return dist;
}

/* Router.route (routing.py:70-101) + roads_of_route (routing.py:110-117).
 * Returns number of roads written to *roads (malloc'd), or -1 if no route. */
static int32_t route_roads(orc* o, int32_t origin, int32_t dest, int32_t** roads) {
  if (o->w[dest] < 0) return -1; /* dest closed: dist_to raises InputError; treated as no route */
  const double* dist = dist_to(o, dest);
  if (dist[origin] < 0) return -1;
  ivec out = {0};
  int32_t u = origin;
  for (;;) {
    if (o->kind[u] == ROADK && (out.n == 0 || out.v[out.n - 1] != o->road[u])) iv_push(&out, o->road[u]);
    if (u == dest) break;
    int32_t nxt = -1;
    for (int32_t k = o->succ_off[u]; k < o->succ_off[u + 1]; k++) {
      int32_t v = o->succ[k];
      if (o->w[v] < 0 || dist[v] < 0) continue;
      if (o->w[u] + dist[v] == dist[u]) {
        nxt = v;
        break;
      }
    }
    if (nxt < 0) {
      free(out.v);
      return -1;
    }
    u = nxt;
  }
  *roads = out.v;
  return out.n;
}

/* ---------------------------------------------------------------- prepare (world.py:227-242) */

static orc* g_sort_ctx;
static int cmp_front_first(const void* a, const void* b) {
  const veh_t* x = &g_sort_ctx->V[*(const int32_t*)a];
  const veh_t* y = &g_sort_ctx->V[*(const int32_t*)b];
  if (x->snap_s != y->snap_s) return (x->snap_s > y->snap_s) ? -1 : 1;
  return (*(const int32_t*)a < *(const int32_t*)b) ? -1 : 1;
}
static int cmp_int(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* sorted(self._driving): ascending vix */
static int32_t sorted_driving(orc* o, int32_t* out) {
  int32_t n = 0;
  for (int32_t k = 0; k < o->drv.n; k++)
    if (o->drv.v[k] >= 0) out[n++] = o->drv.v[k];
  qsort(out, (size_t)n, sizeof(int32_t), cmp_int);
  return n;
}

static void build_index(orc* o, int32_t* order, int32_t n) {
  memset(o->idx_off, 0, sizeof(int32_t) * (size_t)(o->nl + 1));
  for (int32_t k = 0; k < n; k++) {
    veh_t* vh = &o->V[order[k]];
    vh->snap_lane = vh->lane;
    vh->snap_s = vh->s;
    vh->snap_v = vh->v;
    vh->snap_ri = vh->ri;
    vh->snap_rp = vh->rp;
    vh->reverted = 0;
    o->idx_off[vh->lane + 1]++;
  }
  for (int32_t l = 0; l < o->nl; l++) o->idx_off[l + 1] += o->idx_off[l];
  int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * (size_t)(o->nl + 1));
  memcpy(fill, o->idx_off, sizeof(int32_t) * (size_t)(o->nl + 1));
  for (int32_t k = 0; k < n; k++) o->idx[fill[o->V[order[k]].lane]++] = order[k];
  free(fill);
  g_sort_ctx = o;
  for (int32_t l = 0; l < o->nl; l++) {
    int32_t a = o->idx_off[l], b = o->idx_off[l + 1];
    if (b - a > 1) qsort(o->idx + a, (size_t)(b - a), sizeof(int32_t), cmp_front_first);
    for (int32_t k = a; k < b; k++) o->V[o->idx[k]].idx_pos = k - a;
  }
}

#define IDX_N(o, l) ((o)->idx_off[(l) + 1] - (o)->idx_off[(l)])
#define IDX_AT(o, l, k) ((o)->idx[(o)->idx_off[(l)] + (k)])

/* ---------------------------------------------------------------- sensing (world.py:261-332) */

static void sense(orc* o, int32_t vx, int32_t lane, double s, double v, double* gap, double* lead_v) {
  veh_t* vh = &o->V[vx];
  const tsb_params* p = &o->p;
  int32_t n = IDX_N(o, lane);
  if (n > 0) {
    int32_t leader = -1;
    if (lane == vh->snap_lane) {
      if (vh->idx_pos > 0) leader = IDX_AT(o, lane, vh->idx_pos - 1);
    } else {
      for (int32_t k = n - 1; k >= 0; k--) { /* rear-first */
        int32_t c = IDX_AT(o, lane, k);
        if (o->V[c].snap_s > s || (o->V[c].snap_s == s && c < vx)) {
          leader = c;
          break;
        }
      }
    }
    if (leader >= 0) {
      *gap = py_max(o->V[leader].snap_s - p->vehicle_length - s, EPS_GAP);
      *lead_v = o->V[leader].snap_v;
      return;
    }
  }
  double remaining = o->len[lane] - s;
  int32_t rp = vh->snap_rp;
  if (o->kind[lane] == ROADK) {
    if (rp + 1 >= vh->nroads) {
      *gap = INFINITY;
      *lead_v = 0.0;
      return;
    }
    int32_t conn = next_connector(o, lane, rp, vh);
    if (conn < 0 || !o->open[conn] || !o->open[o->succ1[conn]]) {
      *gap = py_max(remaining, EPS_GAP);
      *lead_v = 0.0;
      return;
    }
    int asp = connector_aspect(o, conn);
    if (asp == RED || (asp == AMBER && remaining > v * v / (2.0 * p->idm_b))) {
      *gap = py_max(remaining, EPS_GAP);
      *lead_v = 0.0;
      return;
    }
  }
  int32_t cur = lane, cur_rp = rp;
  double dist = remaining;
  while (dist < p->lookahead) {
    int32_t nxt;
    if (o->kind[cur] == ROADK) {
      nxt = next_connector(o, cur, cur_rp, vh);
      if (nxt < 0 || !o->open[nxt]) break;
    } else {
      nxt = o->succ1[cur];
      cur_rp += 1;
      if (!o->open[nxt]) break;
    }
    int32_t m = IDX_N(o, nxt);
    if (m > 0) {
      veh_t* rear = &o->V[IDX_AT(o, nxt, m - 1)];
      double g = dist + rear->snap_s - p->vehicle_length;
      *gap = py_max(g, EPS_GAP);
      *lead_v = rear->snap_v;
      return;
    }
    dist += o->len[nxt];
    cur = nxt;
  }
  *gap = INFINITY;
  *lead_v = 0.0;
}

static view_t view_of(const orc* o, int32_t vx) {
  if (vx < 0) return (view_t){0, 0, 0, 0};
  return (view_t){1, o->V[vx].snap_s, o->V[vx].snap_v, o->p.vehicle_length};
}

/* world.py:319-332 */
static void neighbor_views(const orc* o, int32_t lane, double s_t, view_t* ld, view_t* fl) {
  int32_t leader = -1, follower = -1, n = IDX_N(o, lane);
  for (int32_t k = 0; k < n; k++) {
    int32_t c = IDX_AT(o, lane, k);
    if (o->V[c].snap_s > s_t)
      leader = c;
    else {
      follower = c;
      break;
    }
  }
  *ld = view_of(o, leader);
  *fl = view_of(o, follower);
}

/* ---------------------------------------------------------------- update (world.py:337-419) */

static int lane_feasible(const orc* o, int32_t lane, int32_t next_road) { return conn_from(o, lane, next_road) >= 0; }

static int consider_change(orc* o, int32_t vx, int32_t* tgt, double* s_tgt) {
  veh_t* vh = &o->V[vx];
  const tsb_params* p = &o->p;
  int32_t lane = vh->snap_lane;
  if (o->kind[lane] != ROADK) return 0;
  int32_t left = o->left[lane], right = o->right[lane];
  if (left < 0 && right < 0) return 0;
  /* _feasible_lanes (world.py:337-342): None when on the arrival road */
  int any = vh->snap_rp + 1 >= vh->nroads;
  int32_t nr = any ? -1 : vh->roads[vh->snap_rp + 1];
  int32_t rd = o->road[lane];
  int mandatory = !any && !lane_feasible(o, lane, nr);
  int32_t sides[2];
  int nsides;
  if (mandatory) {
    int32_t below = -1, above = -1;
    for (int32_t k = o->road_lane_off[rd]; k < o->road_lane_off[rd + 1]; k++) {
      int32_t f = o->road_lanes[k];
      if (!lane_feasible(o, f, nr)) continue;
      if (f < lane && (below < 0 || f > below)) below = f;
      if (f > lane && (above < 0 || f < above)) above = f;
    }
    double d_left = below >= 0 ? (double)(lane - below) : INFINITY;
    double d_right = above >= 0 ? (double)(above - lane) : INFINITY;
    sides[0] = d_left <= d_right ? left : right;
    nsides = 1;
  } else {
    double draw = keyed_uniform4(p->seed, 1, vh->key, (uint64_t)o->step_no);
    if (draw >= p->mobil_eval_prob) return 0;
    sides[0] = left;
    sides[1] = right;
    nsides = 2;
  }
  double s = vh->snap_s;
  int32_t n = IDX_N(o, lane), pos = vh->idx_pos;
  view_t cl = view_of(o, pos > 0 ? IDX_AT(o, lane, pos - 1) : -1);
  view_t cf = view_of(o, pos + 1 < n ? IDX_AT(o, lane, pos + 1) : -1);
  view_t me = {1, s, vh->snap_v, p->vehicle_length};
  int have = 0;
  double best_inc = 0, best_s = 0;
  int32_t best_nb = -1;
  for (int k = 0; k < nsides; k++) {
    int32_t nb = sides[k];
    if (nb < 0 || !o->open[nb]) continue;
    if (!mandatory && !any && !lane_feasible(o, nb, nr)) continue;
    double s_t = s * (o->len[nb] / o->len[lane]);
    view_t tl, tf;
    neighbor_views(o, nb, s_t, &tl, &tf);
    double inc;
    if (!evaluate_change(o, me, cl, cf, tl, tf, s_t, o->cap[lane], o->cap[nb], &inc)) continue;
    if (!mandatory && inc <= p->mobil_threshold) continue;
    if (!have || inc > best_inc || (inc == best_inc && nb < best_nb)) {
      have = 1;
      best_inc = inc;
      best_nb = nb;
      best_s = s_t;
    }
  }
  if (!have) return 0;
  *tgt = best_nb;
  *s_tgt = best_s;
  return 1;
}

static void update_vehicle(orc* o, int32_t vx) {
  veh_t* vh = &o->V[vx];
  const tsb_params* p = &o->p;
  int32_t lane = vh->snap_lane;
  double s = vh->snap_s, v = vh->snap_v;
  int32_t tl;
  double ts;
  int changed = consider_change(o, vx, &tl, &ts);
  if (changed) {
    lane = tl;
    s = ts;
  }
  double gap, lead_v;
  sense(o, vx, lane, s, v, &gap, &lead_v);
  double a = idm_accel(o, v, v - lead_v, gap, o->cap[lane]);
  double dt = p->dt, v_new = v + a * dt, disp;
  if (v_new <= 0.0) {
    v_new = 0.0;
    disp = a < 0.0 ? v * v / (2.0 * -a) : 0.0;
  } else {
    disp = v * dt + 0.5 * a * dt * dt;
    if (disp < 0.0) disp = 0.0;
  }
  vh->d_lane = lane;
  vh->d_s = s + disp;
  vh->d_v = v_new;
  vh->d_changed = changed;
}

/* ---------------------------------------------------------------- commit (world.py:428-499) */

static int reroute(orc* o, veh_t* vh, int32_t lane) {
  int32_t* rs = NULL;
  int32_t n = route_roads(o, lane, vh->dest, &rs);
  if (n < 0) return 0;
  /* roads_seq[:road_pos] + roads_of_route(path) (world.py:439-440) */
  int32_t* nw = (int32_t*)malloc(sizeof(int32_t) * (size_t)(vh->rp + n));
  memcpy(nw, vh->roads, sizeof(int32_t) * (size_t)vh->rp);
  memcpy(nw + vh->rp, rs, sizeof(int32_t) * (size_t)n);
  free(rs);
  free(vh->roads);
  vh->roads = nw;
  vh->nroads = vh->rp + n;
  return 1;
}

static void finish_push(orc* o, int32_t vx, double t) {
  iv_push(&o->fin_vix, vx);
  if (o->fin_vix.n > o->fin_cap) {
    o->fin_cap = o->fin_vix.cap;
    o->fin_t = (double*)realloc(o->fin_t, sizeof(double) * (size_t)o->fin_cap);
  }
  o->fin_t[o->fin_vix.n - 1] = t;
}

static int64_t apply_deltas(orc* o, int32_t* order, int32_t n) {
  int64_t fin = 0;
  double new_time = o->time + o->p.dt;
  for (int32_t k = 0; k < n; k++) {
    int32_t vx = order[k];
    veh_t* vh = &o->V[vx];
    int32_t lane = vh->d_lane, ri = vh->ri;
    double s = vh->d_s, v = vh->d_v;
    int arrived = 0;
    while (s > o->len[lane]) {
      if (o->kind[lane] == ROADK) {
        if (vh->rp + 1 >= vh->nroads) {
          arrived = 1;
          break;
        }
        int32_t conn = next_connector(o, lane, vh->rp, vh);
        if (conn >= 0 && (!o->open[conn] || !o->open[o->succ1[conn]])) {
          if (reroute(o, vh, lane)) {
            if (vh->rp + 1 >= vh->nroads) {
              arrived = 1;
              break;
            }
            conn = next_connector(o, lane, vh->rp, vh);
          } else {
            conn = -1;
          }
        }
        if (conn < 0 || connector_aspect(o, conn) == RED) {
          s = o->len[lane];
          v = 0.0;
          break;
        }
        s -= o->len[lane];
        lane = conn;
        ri += 1;
      } else {
        s -= o->len[lane];
        lane = o->succ1[lane];
        vh->rp += 1;
        ri += 1;
      }
    }
    if (arrived) {
      vh->status = ST_FINISHED;
      vh->finish = new_time;
      finish_push(o, vx, new_time);
      for (int32_t q = 0; q < o->drv.n; q++)
        if (o->drv.v[q] == vx) {
          o->drv.v[q] = -1;
          break;
        }
      o->n_driving--;
      fin++;
      continue;
    }
    vh->lane = lane;
    vh->s = s;
    vh->v = v;
    vh->ri = ri;
  }
  return fin;
}

static void revert(veh_t* vh) {
  vh->lane = vh->snap_lane;
  vh->s = vh->snap_s;
  vh->v = 0.0;
  vh->ri = vh->snap_ri;
  vh->rp = vh->snap_rp;
  vh->reverted = 1;
}

static orc* g_cur;
static int cmp_lane_then_s(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  const veh_t *p = &g_cur->V[x], *q = &g_cur->V[y];
  if (p->lane != q->lane) return p->lane < q->lane ? -1 : 1;
  if (p->s != q->s) return p->s > q->s ? -1 : 1;
  return x < y ? -1 : 1;
}

/* world.py:509-559, including the restart after every revert.
 *
 * Statement for statement the reference's loop: every pass regroups the
 * driving vehicles by lane (world.py:520-522: lanes in id order, members
 * sorted by (-s, id)) and sweeps the lanes in order until the first revert,
 * then starts over from the first lane.  Two bookkeeping shortcuts keep a
 * pass from costing a full sort of the driving set (C4-size parity cases)
 * without changing what any sweep computes:
 *  - the groups are updated incrementally (a pass's groups equal the
 *    previous pass's except for the lanes a revert moved a vehicle between;
 *    a lane whose members' s changed is re-sorted before its next sweep);
 *  - a lane whose last sweep changed nothing, and whose members have not
 *    changed since, is skipped: its sweep is a deterministic function of
 *    exactly that unchanged state, so re-running it would again change
 *    nothing (the reference re-runs it). */
static int cmp_lane_member(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  const veh_t *p = &g_cur->V[x], *q = &g_cur->V[y];
  if (p->s != q->s) return p->s > q->s ? -1 : 1;
  return x < y ? -1 : 1;
}

static int same_bits(double a, double b) { return memcmp(&a, &b, sizeof(double)) == 0; }

static void collision_sweep(orc* o) {
  double floor_gap = o->p.s0_floor, dt = o->p.dt, L = o->p.vehicle_length;
  const int32_t nl = o->nl;
  int32_t* grp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(o->n_driving + 1));
  ivec* lanes = (ivec*)calloc((size_t)nl, sizeof(ivec));
  uint8_t* resort = (uint8_t*)calloc((size_t)nl, 1);
  uint8_t* clean = (uint8_t*)calloc((size_t)nl, 1);
  int32_t n = sorted_driving(o, grp);
  for (int32_t k = 0; k < n; k++) iv_push(&lanes[o->V[grp[k]].lane], grp[k]);
  g_cur = o;
  for (int32_t l = 0; l < nl; l++)
    if (lanes[l].n > 1) qsort(lanes[l].v, (size_t)lanes[l].n, sizeof(int32_t), cmp_lane_member);
  o->reverts_last = 0;
  for (int32_t pass = 0; pass < o->n_driving + 2; pass++) {
    int dirty = 0;
    for (int32_t lane = 0; lane < nl && !dirty; lane++) {
      ivec* g = &lanes[lane];
      if (g->n == 0 || clean[lane]) continue;
      if (resort[lane]) {
        g_cur = o;
        if (g->n > 1) qsort(g->v, (size_t)g->n, sizeof(int32_t), cmp_lane_member);
        resort[lane] = 0;
      }
      int changed = 0;
      veh_t* prev = NULL;
      int32_t prev_k = -1;
      double prev_rear = INFINITY;
      for (int32_t k = 0; k < g->n; k++) {
        veh_t* vh = &o->V[g->v[k]];
        double limit = prev_rear - floor_gap;
        if (vh->s > limit + 1e-12) {
          int entered = vh->lane != vh->snap_lane;
          double floor_s = entered ? 0.0 : vh->snap_s;
          int32_t moved = -1;  /* member index reverted out of this lane */
          const double s_was = vh->s, v_was = vh->v;
          if (limit >= floor_s) {
            vh->v = py_max(0.0, py_min(vh->v, vh->v - (vh->s - limit) / dt));
            vh->s = limit;
          } else if (entered && !vh->reverted) {
            revert(vh);
            moved = k;
          } else if (prev && prev->lane != prev->snap_lane && !prev->reverted) {
            revert(prev);
            moved = prev_k;
          } else {
            vh->v = 0.0;
            vh->s = floor_s;
          }
          if (moved >= 0) {
            const int32_t vx = g->v[moved];
            for (int32_t q = moved; q + 1 < g->n; q++) g->v[q] = g->v[q + 1];
            g->n--;
            const int32_t to = o->V[vx].lane;
            iv_push(&lanes[to], vx);
            resort[to] = 1;
            clean[to] = 0;
            clean[lane] = 0;
            dirty = 1;
            break;
          }
          if (!same_bits(s_was, vh->s) || !same_bits(v_was, vh->v)) {
            changed = 1;
            resort[lane] = 1;
          }
        }
        prev = vh;
        prev_k = k;
        prev_rear = vh->s - L;
      }
      if (!dirty) clean[lane] = changed ? 0 : 1;
    }
    if (dirty) {
      o->reverts_last++;
      o->reverts_total++;
    }
    if (!dirty) break;
  }
  for (int32_t l = 0; l < nl; l++) free(lanes[l].v);
  free(lanes);
  free(resort);
  free(clean);
  free(grp);
}

/* world.py:561-617 */
static int orc_cmp_s_asc(const void* a, const void* b) {
  double x = g_cur->V[*(const int32_t*)a].s, y = g_cur->V[*(const int32_t*)b].s;
  return (x > y) - (x < y);
}

static int64_t inject_due(orc* o) {
  ivec due = o->retry;
  o->retry = (ivec){0};
  while (o->pend_i < o->nv && o->V[o->pending[o->pend_i]].depart <= o->time) iv_push(&due, o->pending[o->pend_i++]);
  if (due.n == 0) {
    free(due.v);
    return 0;
  }
  /* occupants per lane sorted by s (stable sort of _driving order: ties are
   * irrelevant to the gap test) */
  int32_t* cnt = (int32_t*)calloc((size_t)o->nl + 1, sizeof(int32_t));
  for (int32_t k = 0; k < o->drv.n; k++)
    if (o->drv.v[k] >= 0) cnt[o->V[o->drv.v[k]].lane + 1]++;
  for (int32_t l = 0; l < o->nl; l++) cnt[l + 1] += cnt[l];
  ivec* occ = (ivec*)calloc((size_t)o->nl, sizeof(ivec));
  for (int32_t k = 0; k < o->drv.n; k++)
    if (o->drv.v[k] >= 0) iv_push(&occ[o->V[o->drv.v[k]].lane], o->drv.v[k]);
  g_cur = o;
  for (int32_t l = 0; l < o->nl; l++)
    if (occ[l].n > 1) qsort(occ[l].v, (size_t)occ[l].n, sizeof(int32_t), orc_cmp_s_asc);
  int64_t injected = 0;
  double s0 = o->p.idm_s0, L = o->p.vehicle_length;
  for (int32_t q = 0; q < due.n; q++) {
    int32_t vx = due.v[q];
    veh_t* vh = &o->V[vx];
    if (!vh->routed) {
      if (!o->open[vh->origin_lane]) {
        iv_push(&o->retry, vx);
        continue;
      }
      int32_t* rs = NULL;
      int32_t nr = route_roads(o, vh->origin_lane, vh->dest, &rs);
      if (nr < 0) {
        o->dropped++;
        vh->status = ST_DROPPED;
        continue;
      }
      vh->roads = rs;
      vh->nroads = nr;
      vh->routed = 1;
    }
    ivec* lst = &occ[vh->origin_lane];
    double front_gap = INFINITY, rear_gap = INFINITY;
    for (int32_t k = 0; k < lst->n; k++) {
      veh_t* other = &o->V[lst->v[k]];
      if (other->s >= vh->origin_s) {
        front_gap = other->s - L - vh->origin_s;
        break;
      }
      rear_gap = vh->origin_s - L - other->s;
    }
    if (front_gap < s0 + L || rear_gap < s0) {
      iv_push(&o->retry, vx);
      continue;
    }
    vh->status = ST_DRIVING;
    vh->lane = vh->origin_lane; /* route[0] */
    vh->s = vh->origin_s;
    vh->v = 0.0;
    vh->ri = 0;
    vh->rp = 0;
    vh->snap_lane = vh->lane;
    vh->snap_s = vh->s;
    iv_push(&o->drv, vx);
    o->n_driving++;
    int32_t lo = 0;
    while (lo < lst->n && o->V[lst->v[lo]].s < vh->s) lo++;
    iv_push(lst, 0);
    memmove(lst->v + lo + 1, lst->v + lo, sizeof(int32_t) * (size_t)(lst->n - 1 - lo));
    lst->v[lo] = vx;
    injected++;
  }
  for (int32_t l = 0; l < o->nl; l++) free(occ[l].v);
  free(occ);
  free(cnt);
  free(due.v);
  return injected;
}

/* world.py:619-647 */
static void advance_signals(orc* o) {
  const tsb_params* p = &o->p;
  if (p->controller == 0) {
    for (int32_t j = 0; j < o->nj; j++)
      if (o->jsig[j]) advance_fixed(o, j, p->dt);
    return;
  }
  int32_t* counts = NULL;
  for (int32_t j = 0; j < o->nj; j++) {
    if (!o->jsig[j]) continue;
    sig_t* st = &o->sig[j];
    st->elapsed += p->dt;
    st->since += p->dt;
    if (st->since < p->mp_interval || st->elapsed < p->mp_min_green) continue;
    if (!counts) {
      counts = (int32_t*)calloc((size_t)o->nl, sizeof(int32_t));
      for (int32_t k = 0; k < o->drv.n; k++)
        if (o->drv.v[k] >= 0) counts[o->V[o->drv.v[k]].lane]++;
    }
    /* signals.py:64-86 */
    int32_t b = o->jph_off[j], np_ = o->jph_off[j + 1] - b, best = 0;
    int have = 0;
    int64_t best_p = 0;
    for (int32_t ph = 0; ph < np_; ph++) {
      int64_t pr = 0;
      for (int32_t q = o->jc_off[j]; q < o->jc_off[j + 1]; q++) {
        int32_t c = o->jc[q];
        if ((o->green[c] >> ph) & 1ULL) pr += counts[o->pred1[c]] - counts[o->succ1[c]];
      }
      if (!have || pr > best_p) {
        have = 1;
        best_p = pr;
        best = ph;
      }
    }
    if (best != st->phase) {
      st->phase = best;
      st->elapsed = 0.0;
    }
    st->since = 0.0;
  }
  free(counts);
}

static void ensure_windows(orc* o, int32_t wi) {
  if (wi < o->nwin) return;
  int32_t nw = wi + 16;
  double* s = (double*)calloc((size_t)o->nr * (size_t)nw, sizeof(double));
  int64_t* c = (int64_t*)calloc((size_t)o->nr * (size_t)nw, sizeof(int64_t));
  for (int32_t r = 0; r < o->nr; r++)
    for (int32_t w = 0; w < o->nwin; w++) {
      s[(size_t)r * nw + w] = o->acc_sum[(size_t)r * o->nwin + w];
      c[(size_t)r * nw + w] = o->acc_cnt[(size_t)r * o->nwin + w];
    }
  free(o->acc_sum);
  free(o->acc_cnt);
  o->acc_sum = s;
  o->acc_cnt = c;
  o->nwin = nw;
}

/* world.py:649-657, summed in _driving insertion order */
static void accumulate_speeds(orc* o, double new_time) {
  int32_t wi = (int32_t)(new_time / o->p.speed_window);
  ensure_windows(o, wi);
  for (int32_t k = 0; k < o->drv.n; k++) {
    int32_t vx = o->drv.v[k];
    if (vx < 0) continue;
    veh_t* vh = &o->V[vx];
    if (o->kind[vh->lane] != ROADK) continue;
    size_t cell = (size_t)o->road[vh->lane] * o->nwin + wi;
    o->acc_sum[cell] += vh->v;
    o->acc_cnt[cell] += 1;
  }
}

static void compact_driving(orc* o) {
  int32_t m = 0;
  for (int32_t k = 0; k < o->drv.n; k++)
    if (o->drv.v[k] >= 0) o->drv.v[m++] = o->drv.v[k];
  o->drv.n = m;
}

typedef struct {
  orc* o;
  const int32_t* order;
  int32_t lo, hi;
} upd_job;

static void* upd_worker(void* arg) {
  upd_job* j = (upd_job*)arg;
  for (int32_t k = j->lo; k < j->hi; k++) update_vehicle(j->o, j->order[k]);
  return NULL;
}

static void update_parallel(orc* o, const int32_t* order, int32_t n) {
  int t = o->threads;
  if (t <= 1 || n < 256) {
    for (int32_t k = 0; k < n; k++) update_vehicle(o, order[k]);
    return;
  }
  if (t > 256) t = 256;
  pthread_t th[256];
  upd_job jobs[256];
  for (int q = 0; q < t; q++) {
    jobs[q].o = o;
    jobs[q].order = order;
    jobs[q].lo = (int32_t)((int64_t)n * q / t);
    jobs[q].hi = (int32_t)((int64_t)n * (q + 1) / t);
    pthread_create(&th[q], NULL, upd_worker, &jobs[q]);
  }
  for (int q = 0; q < t; q++) pthread_join(th[q], NULL);
}

/* world.py:659-689 */
static void step_once(orc* o) {
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(o->n_driving + 1));
  int32_t n = sorted_driving(o, order);
  build_index(o, order, n);
  o->vehicle_updates += n;
  /* The update phase reads only the snapshot and writes each vehicle's own
   * deltas (world.py:664-669): the reference's thread-pool
   * chunking restated with pthreads.  Results do not depend on the thread count. */
  update_parallel(o, order, n);
  o->finished_now = apply_deltas(o, order, n);
  compact_driving(o);
  collision_sweep(o);
  advance_signals(o);
  o->time += o->p.dt;
  o->step_no += 1;
  o->injected_now = inject_due(o);
  accumulate_speeds(o, o->time);
  free(order);
}

/* ================================================================ C API */

static void* dup(const void* src, size_t bytes) {
  void* d = malloc(bytes ? bytes : 1);
  if (bytes) memcpy(d, src, bytes);
  return d;
}

static orc* g_pend_ctx;
static int cmp_pending(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  double dx = g_pend_ctx->V[x].depart, dy = g_pend_ctx->V[y].depart;
  if (dx != dy) return dx < dy ? -1 : 1;
  return (x > y) - (x < y);
}

int orc_create(const tsb_network* net, const tsb_trips* tr, const tsb_params* p, orc** out) {
  orc* o = (orc*)calloc(1, sizeof(orc));
  o->threads = 1;
  o->p = *p;
  int32_t nl = o->nl = net->n_lanes;
  o->nr = net->n_roads;
  o->nj = net->n_junctions;
  o->nv = tr->n;
  o->len = (double*)dup(net->lane_len, sizeof(double) * nl);
  o->cap = (double*)dup(net->lane_cap, sizeof(double) * nl);
  o->kind = (int8_t*)dup(net->lane_kind, sizeof(int8_t) * nl);
  o->open = (uint8_t*)dup(net->lane_open, sizeof(uint8_t) * nl);
  o->left = (int32_t*)dup(net->lane_left, sizeof(int32_t) * nl);
  o->right = (int32_t*)dup(net->lane_right, sizeof(int32_t) * nl);
  o->road = (int32_t*)dup(net->lane_road, sizeof(int32_t) * nl);
  o->junc = (int32_t*)dup(net->lane_junction, sizeof(int32_t) * nl);
  o->pred1 = (int32_t*)dup(net->lane_pred1, sizeof(int32_t) * nl);
  o->succ1 = (int32_t*)dup(net->lane_succ1, sizeof(int32_t) * nl);
  o->succ_off = (int32_t*)dup(net->succ_off, sizeof(int32_t) * (nl + 1));
  o->succ = (int32_t*)dup(net->succ, sizeof(int32_t) * net->succ_off[nl]);
  o->pred_off = (int32_t*)dup(net->pred_off, sizeof(int32_t) * (nl + 1));
  o->pred = (int32_t*)dup(net->pred, sizeof(int32_t) * net->pred_off[nl]);
  o->road_lane_off = (int32_t*)dup(net->road_lane_off, sizeof(int32_t) * (o->nr + 1));
  o->road_lanes = (int32_t*)dup(net->road_lanes, sizeof(int32_t) * net->road_lane_off[o->nr]);
  o->jsig = (uint8_t*)dup(net->junc_signal, o->nj);
  o->jph_off = (int32_t*)dup(net->junc_phase_off, sizeof(int32_t) * (o->nj + 1));
  o->ph_dur = (double*)dup(net->phase_dur, sizeof(double) * net->junc_phase_off[o->nj]);
  o->green = (uint64_t*)dup(net->lane_green_mask, sizeof(uint64_t) * nl);
  o->sig = (sig_t*)calloc((size_t)o->nj + 1, sizeof(sig_t));
  for (int32_t j = 0; j < o->nj; j++) {
    o->sig[j].phase = net->junc_phase0[j];
    o->sig[j].elapsed = net->junc_elapsed0[j];
  }
  o->jc_off = (int32_t*)calloc((size_t)o->nj + 1, sizeof(int32_t));
  for (int32_t l = 0; l < nl; l++)
    if (o->kind[l] == CONNK) o->jc_off[o->junc[l] + 1]++;
  for (int32_t j = 0; j < o->nj; j++) o->jc_off[j + 1] += o->jc_off[j];
  o->jc = (int32_t*)malloc(sizeof(int32_t) * ((size_t)o->jc_off[o->nj] + 1));
  {
    int32_t* fill = (int32_t*)dup(o->jc_off, sizeof(int32_t) * (o->nj + 1));
    for (int32_t l = 0; l < nl; l++)
      if (o->kind[l] == CONNK) o->jc[fill[o->junc[l]]++] = l;
    free(fill);
  }
  o->V = (veh_t*)calloc((size_t)o->nv + 1, sizeof(veh_t));
  for (int32_t k = 0; k < o->nv; k++) {
    veh_t* vh = &o->V[k];
    vh->status = ST_WAITING;
    vh->lane = tr->origin_lane[k];
    vh->s = tr->origin_s[k];
    vh->depart = tr->departure[k];
    vh->origin_s = tr->origin_s[k];
    vh->origin_lane = tr->origin_lane[k];
    vh->dest = tr->dest_lane[k];
    vh->key = tr->key[k];
    vh->finish = NAN;
  }
  o->pending = (int32_t*)malloc(sizeof(int32_t) * ((size_t)o->nv + 1));
  for (int32_t k = 0; k < o->nv; k++) o->pending[k] = k;
  g_pend_ctx = o;
  qsort(o->pending, (size_t)o->nv, sizeof(int32_t), cmp_pending);
  o->idx_off = (int32_t*)calloc((size_t)nl + 1, sizeof(int32_t));
  o->idx = (int32_t*)malloc(sizeof(int32_t) * ((size_t)o->nv + 1));
  o->w = (double*)malloc(sizeof(double) * ((size_t)nl + 1));
  rebuild_router(o);
  *out = o;
  return OK;
}

void orc_destroy(orc* o) {
  if (!o) return;
  void* ptrs[] = {o->len, o->cap, o->kind, o->open, o->left, o->right, o->road, o->junc, o->pred1,
                  o->succ1, o->succ_off, o->succ, o->pred_off, o->pred, o->road_lane_off, o->road_lanes,
                  o->jsig, o->jph_off, o->ph_dur, o->green, o->sig, o->jc_off, o->jc, o->pending, o->idx_off, o->idx,
                  o->w, o->retry.v, o->drv.v, o->fin_vix.v, o->fin_t, o->acc_sum, o->acc_cnt};
  for (size_t i = 0; i < sizeof(ptrs) / sizeof(ptrs[0]); i++) free(ptrs[i]);
  for (int32_t k = 0; k < o->nv; k++) free(o->V[k].roads);
  free(o->V);
  for (int i = 0; i < 256; i++) free(o->cache[i].dist);
  free(o);
}

static void fill_report(const orc* o, tsb_report* r) {
  r->time = o->time;
  r->step_no = o->step_no;
  r->driving = o->n_driving;
  r->waiting = (o->nv - o->pend_i) + o->retry.n;
  r->finished = o->fin_vix.n;
  r->dropped = o->dropped;
  r->injected_now = o->injected_now;
  r->finished_now = o->finished_now;
  r->vehicle_updates = o->vehicle_updates;
  r->reverts_last = o->reverts_last;
  r->reverts_total = o->reverts_total;
}

int orc_step(orc* o, int32_t n, tsb_report* last) {
  for (int32_t k = 0; k < n; k++) step_once(o);
  if (last) fill_report(o, last);
  return OK;
}

int orc_report(orc* o, tsb_report* r) {
  fill_report(o, r);
  return OK;
}

/* World.prepare() view: lane-sorted (s desc, id asc) snapshot of the current state. */
int orc_state(orc* o, int32_t* n_driving, int32_t* lane_start, int32_t* vix, int32_t* lane, int32_t* road_pos,
              double* s, double* v) {
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * ((size_t)o->n_driving + 1));
  int32_t n = sorted_driving(o, order);
  g_cur = o;
  qsort(order, (size_t)n, sizeof(int32_t), cmp_lane_then_s);
  *n_driving = n;
  if (lane_start) {
    memset(lane_start, 0, sizeof(int32_t) * ((size_t)o->nl + 1));
    for (int32_t k = 0; k < n; k++) lane_start[o->V[order[k]].lane + 1]++;
    for (int32_t l = 0; l < o->nl; l++) lane_start[l + 1] += lane_start[l];
  }
  for (int32_t k = 0; k < n; k++) {
    const veh_t* vh = &o->V[order[k]];
    if (vix) vix[k] = order[k];
    if (lane) lane[k] = vh->lane;
    if (road_pos) road_pos[k] = vh->rp;
    if (s) s[k] = vh->s;
    if (v) v[k] = vh->v;
  }
  free(order);
  return OK;
}

int orc_status(orc* o, uint8_t* status, double* finish, int32_t* route_index) {
  for (int32_t k = 0; k < o->nv; k++) {
    if (status) status[k] = (uint8_t)o->V[k].status;
    if (finish) finish[k] = o->V[k].finish;
    if (route_index) route_index[k] = o->V[k].ri;
  }
  return OK;
}

int orc_finished(orc* o, int64_t since, int64_t cap, int32_t* vix, double* t, int64_t* n_out) {
  int64_t n = 0;
  for (int64_t k = since; k < o->fin_vix.n && n < cap; k++, n++) {
    vix[n] = o->fin_vix.v[k];
    t[n] = o->fin_t[k];
  }
  *n_out = n;
  return OK;
}

int orc_road_acc(orc* o, int32_t nw, double* sum, int64_t* cnt) {
  for (int32_t r = 0; r < o->nr; r++)
    for (int32_t w = 0; w < nw; w++) {
      int in = w < o->nwin;
      sum[(size_t)r * nw + w] = in ? o->acc_sum[(size_t)r * o->nwin + w] : 0.0;
      cnt[(size_t)r * nw + w] = in ? o->acc_cnt[(size_t)r * o->nwin + w] : 0;
    }
  return OK;
}

/* world.py:694-704 */
int orc_min_front_gap(orc* o, double* out) {
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * ((size_t)o->n_driving + 1));
  int32_t n = sorted_driving(o, order);
  g_cur = o;
  qsort(order, (size_t)n, sizeof(int32_t), cmp_lane_then_s);
  double worst = INFINITY;
  for (int32_t k = 0; k + 1 < n; k++) {
    const veh_t *a = &o->V[order[k]], *b = &o->V[order[k + 1]];
    if (a->lane == b->lane) worst = py_min(worst, a->s - o->p.vehicle_length - b->s);
  }
  free(order);
  *out = worst;
  return OK;
}

int orc_set_lane(orc* o, int32_t lane, double max_speed, int32_t open) {
  if (lane < 0 || lane >= o->nl) return TSB_ERANGE;
  o->cap[lane] = max_speed;
  o->open[lane] = (uint8_t)(open != 0);
  rebuild_router(o);
  return OK;
}

int orc_set_signal_phase(orc* o, int32_t j, int32_t phase) {
  if (j < 0 || j >= o->nj || !o->jsig[j]) return TSB_EINVAL;
  if (phase < 0 || phase >= o->jph_off[j + 1] - o->jph_off[j]) return TSB_ERANGE;
  o->sig[j].phase = phase;
  o->sig[j].elapsed = 0.0;
  o->sig[j].since = 0.0;
  return OK;
}

int orc_signal_state(orc* o, int32_t* phase, double* elapsed) {
  for (int32_t j = 0; j < o->nj; j++) {
    phase[j] = o->sig[j].phase;
    elapsed[j] = o->sig[j].elapsed;
  }
  return OK;
}

/* Router.route for tests: lane path length and cost; *n = 0 if unroutable. */
int orc_route_cost(orc* o, int32_t origin, int32_t dest, double* cost, int32_t* n_roads) {
  int32_t* rs = NULL;
  int32_t n = route_roads(o, origin, dest, &rs);
  free(rs);
  *n_roads = n < 0 ? 0 : n;
  *cost = n < 0 ? -1.0 : dist_to(o, dest)[origin];
  return OK;
}

/* Router.dist_to(dest) key sets for n destinations (routing.py:47-68: an
 * origin can reach dest iff it is a key of dist_to(dest)); out is n x lanes. */
int orc_reach(orc* o, int32_t n, const int32_t* dests, uint8_t* out) {
  for (int32_t i = 0; i < n; i++) {
    uint8_t* row = out + (size_t)i * (size_t)o->nl;
    if (o->w[dests[i]] < 0) {
      memset(row, 0, (size_t)o->nl);
      continue;
    }
    const double* dist = dist_to(o, dests[i]);
    for (int32_t l = 0; l < o->nl; l++) row[l] = dist[l] >= 0;
  }
  return OK;
}

/* Threads for the update phase (EngineConfig.threads, params.py:48-83). */
int orc_set_threads(orc* o, int32_t n) {
  o->threads = n < 1 ? 1 : n;
  return OK;
}

/* the IDM law alone (idm.py:17-31) for formula tests */
double orc_idm_accel(orc* o, double v, double dv, double gap, double v_cap) { return idm_accel(o, v, dv, gap, v_cap); }
double orc_keyed_uniform4(uint64_t a, uint64_t b, uint64_t c, uint64_t d) { return keyed_uniform4(a, b, c, d); }
double orc_pow_cr(double x, int32_t n) { return pow_cr_int(x, n); }
