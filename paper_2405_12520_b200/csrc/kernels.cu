// kernels.cu -- the per-step device pipeline of the MOSS vehicle loop.
//
// One step (World.step, trafficsim/engine/world.py:659-689) is the sequence
// (engine.cu issue_step builds it into one CUDA graph)
//
//   k_begin_step            zero lane counts, reset the step scalars
//   k_speeds   (branch)     world.py:649-657 on the previous snapshot
//   k_update       A -> B   prepare-consumer + update + lane/road transitions
//                           (world.py:261-419, 443-499), lane counts
//   k_scan                  cnt -> C lane starts (+ lane ranges)
//   k_place        B -> C   stayers to their slot, movers to their lane's tail
//   k_lanefix      C        per-lane sort by (s desc, id asc) + tentative
//                           collision sweep (world.py:509-559) of flagged lanes
//   k_signals, k_conn_flags, k_inject_due   (branch) world.py:619-647, 561-573
//   k_resolve_fast C        exact revert chains, one warp per event
//   k_regroup      C -> A'  C with the dirty lanes rebuilt into its tail
//   RARE (IF node, branch): k_resolve_closure/_comp/k_resolve (meeting revert
//       chains), k_inject_* (world.py:561-617), full regroup
//
// The snapshot layout A is the reference's per-lane index itself
// (world.py:227-242): vehicles grouped by lane, s descending, id ascending,
// so "leader" is the previous record and the MOBIL / sensing lookups are
// binary searches in a contiguous segment.
#include <cuda_runtime.h>
#include <math_constants.h>

#include "device.cuh"

namespace tsb {

enum { GREEN = 0, AMBER = 1, RED = 2 };
enum : uint8_t { OUT_NONE = 0, OUT_INJECT = 1, OUT_RETRY = 2, OUT_DROP = 3 };

static constexpr double EPS_GAP = 1e-6;  // world.py:43

// Programmatic dependent launch: kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel's launch and
// prologue overlap the previous kernel's tail; this waits for the previous
// grid (and its memory) before anything is read.  No-op without the attribute.
#define PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")

// Step timeline (tsb_set_timeline): while c.tl_on, block 0 of each step
// kernel stamps %globaltimer once its predecessors completed (after
// PDL_WAIT), into slot k of the current step's row of c.tl (a ring of
// TL_ROWS steps x TL_SLOTS).  bench.py reads the in-graph duration of
// k_update from it over the timed window itself; one load and a predicated
// store per kernel when off.
static constexpr int TL_SLOTS = 16;
static constexpr int TL_ROWS = 1024;
enum { TL_BEGIN, TL_UPDATE, TL_SCAN, TL_PLACE, TL_LANEFIX, TL_RESOLVE, TL_REGROUP, TL_END, TL_SPEEDS, TL_SIGNALS,
       TL_INJECT_DUE, TL_SPEEDS_END, TL_RESOLVE_END, TL_INJECT_DUE_END };
#define TL_MARK(k)                                                                        \
  do {                                                                                    \
    if (c.tl_on && blockIdx.x == 0 && threadIdx.x == 0) {                                 \
      unsigned long long t_;                                                              \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                              \
      c.tl[(size_t)(c.dyn->tl_row & (TL_ROWS - 1)) * TL_SLOTS + (k)] = t_;                \
    }                                                                                     \
  } while (0)

// Stamps slot k when the kernel's block 0 thread 0 leaves the scope (every
// return path): the approximate end of a kernel whose block 0 finishes last.
struct TlEnd {
  const Ctx& c;
  int k;
  __device__ ~TlEnd() {
    if (c.tl_on && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      c.tl[(size_t)(c.dyn->tl_row & (TL_ROWS - 1)) * TL_SLOTS + k] = t_;
    }
  }
};

__device__ __forceinline__ int gtid() { return blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int gstride() { return gridDim.x * blockDim.x; }

// Buffer selectors: the snapshot layout A and the post-sweep layout C swap
// roles through dyn->cur (a device value), so kernels captured once in a
// CUDA graph pick their buffers at run time.
enum { SEL_A = 0, SEL_C = 1, SEL_B = 2, SEL_D = 3, SEL_NONE = 4 };
__device__ __forceinline__ VRec* rec_buf(const Ctx& c, int sel) {
  const int cur = c.dyn->cur;
  switch (sel) {
    case SEL_A: return c.lay[cur];
    case SEL_C: return c.lay[cur ^ 1];
    case SEL_B: return c.B;
    default: return c.D;
  }
}
__device__ __forceinline__ int32_t* start_buf(const Ctx& c, int sel) {
  return sel == SEL_A ? c.start[c.dyn->cur] : c.start[c.dyn->cur ^ 1];
}
__device__ __forceinline__ bool gated_off(const int32_t* gate) { return gate && *gate == 0; }

// Sharded mode (shard.py): lanes are own, halo (ghost copies imported from
// their owner after every step) or outside the zone.
enum : uint8_t { ZF_OWN = 1, ZF_HALO = 2, ZF_EXACT = 4 };
// Range [x, y) of lane L's records in a layout buffer, R = c.rng[buffer]:
// written by the scan that lays the buffer out (the lane's CSR segment), then
// overridden for the lanes the regroup rebuilt into the buffer's tail and,
// when sharded, for the halo lanes by the ghost import.  Records of the buffer
// outside their lane's range are stale copies and are skipped.
__device__ __forceinline__ int2 seg(const Ctx& c, const int2* R, int32_t L) { return R[L]; }

// Conditional graph nodes (engine.cu issue_step): a section of the step graph
// runs only when its deciding kernel sets the handle.  The handles default to
// 0 at every graph launch; in eager launches (profiling, host-continuation
// mode) use_cond is 0 and the sections' kernels gate themselves instead.
enum { COND_RARE = 0, N_COND = 1 };
__device__ __forceinline__ void set_cond(const Ctx& c, int k, bool v) {
  if (c.use_cond && v) cudaGraphSetConditional(c.cond[k], 1u);
}
// The step needs the RARE body of the step graph (engine.cu issue_step).
__device__ __forceinline__ void set_rare(const Ctx& c) {
  set_cond(c, COND_RARE, true);
  c.dyn->rare = 1;
}

// A lane whose membership or order changed after the sweep; the next
// snapshot rebuilds only these lanes (k_regroup), unless too many changed.
__device__ __forceinline__ void mark_dirty(const Ctx& c, int32_t L) {
  if (atomicExch(&c.dirty_flag[L], 1) == 0) {
    int32_t k = atomicAdd(&c.dyn->n_dirty, 1);
    c.dirty_list[k] = L;
  }
  c.dyn->need_regroup = 1;
}

// ------------------------------------------------------------------ network helpers

// _conn_from[(lane, road)] (world.py:155-166): smallest successor connector
// of road lane `lane` leading onto `road`.  Successor lists are sorted.
__device__ __forceinline__ int32_t conn_from(const Ctx& c, const LaneRec& L, int32_t road) {
  for (int k = 0; k < L.nsucc; k++)
    if (__ldg(c.succ_dst_road + L.succ_off + k) == road) return __ldg(c.succ + L.succ_off + k);
  return -1;
}

// Same, from the lane's 4-wide successor table (two independent 16 B loads
// keyed by the lane id instead of a dependent walk of the CSR).
__device__ __forceinline__ int32_t conn_from_id(const Ctx& c, int32_t lane, int32_t road) {
  const int4 r = __ldg(c.succ_road4 + lane);
  const int4 k = __ldg(c.succ_conn4 + lane);
  if (r.x == road) return k.x;
  if (r.y == road) return k.y;
  if (r.z == road) return k.z;
  if (r.w == road) return k.w;
  if (k.w == -2) {  // more than 4 successors: the first 3 are in the table
    const LaneRec L = c.lanes[lane];
    for (int q = 3; q < L.nsucc; q++)
      if (__ldg(c.succ_dst_road + L.succ_off + q) == road) return __ldg(c.succ + L.succ_off + q);
  }
  return -1;
}

__device__ __forceinline__ int lf_aspect(uint8_t f) { return (f >> LF_ASPECT_SHIFT) & 3; }
// A connector a vehicle may enter: it and its successor lane are open
// (world.py:282-283, 460-462).
__device__ __forceinline__ bool lf_passable(uint8_t f) { return (f & (LF_OPEN | LF_SUCC_OPEN)) == (LF_OPEN | LF_SUCC_OPEN); }

// Aspect of connector `conn` from its junction's state (world.py:247-254 +
// signals.py:46-61).
__device__ __forceinline__ int aspect_of(const Ctx& c, int32_t j, int32_t conn, const JuncState& st) {
  if (!c.junc_signal[j]) return GREEN;
  if (!((c.green[conn] >> st.phase) & 1ULL)) return RED;
  double dur = c.phase_dur[c.junc_phase_off[j] + st.phase];
  if (c.p.controller == 0 && c.p.amber > 0.0 && st.elapsed >= dur - c.p.amber) return AMBER;
  return GREEN;
}

// Refresh the connector bits of lflag for junction j's connectors.
__device__ __forceinline__ void write_conn_flags(const Ctx& c, int32_t j, const JuncState& st) {
  for (int32_t q = c.jc_off[j]; q < c.jc_off[j + 1]; q++) {
    const int32_t cn = c.jc[q];
    uint8_t f = c.lflag[cn] & LF_OPEN;
    const int32_t sc = c.lanes[cn].succ1;  // < 0: outside a sharded rank's local lanes
    if (sc >= 0 && (c.lflag[sc] & LF_OPEN)) f |= LF_SUCC_OPEN;
    f |= (uint8_t)(aspect_of(c, j, cn, st) << LF_ASPECT_SHIFT);
    c.lflag[cn] = f;
  }
}

// All junctions (after construction and after any host control change).
__global__ void k_lane_flags(Ctx c) {
  PDL_WAIT();
  for (int32_t j = gtid(); j < c.n_junc; j += gstride()) write_conn_flags(c, j, c.sig[j]);
}

struct View {
  bool ok;
  double s, v;
};

// B (the post-update records) is written once by k_update and read once by
// k_place: with REC_STREAM its lines are marked evict-first in L2
// (st.global.cs / ld.global.cs) so they do not push the snapshot and the lane
// tables out of the 126 MB L2.
#ifndef REC_STREAM
#define REC_STREAM 1
#endif
__device__ __forceinline__ void store_b(VRec* p, const VRec& r) {
#if REC_STREAM
  const double2* src = reinterpret_cast<const double2*>(&r);
  double2* dst = reinterpret_cast<double2*>(p);
  __stcs(dst, src[0]);
  __stcs(dst + 1, src[1]);
#else
  *p = r;
#endif
}
__device__ __forceinline__ VRec load_b(const VRec* p) {
#if REC_STREAM
  VRec r;
  double2* d = reinterpret_cast<double2*>(&r);
  d[0] = __ldcs(reinterpret_cast<const double2*>(p));
  d[1] = __ldcs(reinterpret_cast<const double2*>(p) + 1);
  return r;
#else
  return *p;
#endif
}

__device__ __forceinline__ View view_at(const VRec* A, int32_t k) {
  if (k < 0) return View{false, 0.0, 0.0};
  return View{true, A[k].s, A[k].v};
}

// gap from follower position fs to leader l (mobil.py:33-36)
__device__ __forceinline__ double gap_to(const View& l, double fs, double Lv) {
  return l.ok ? l.s - Lv - fs : CUDART_INF;
}
// speed difference to leader l, 0-speed stand-in when absent (mobil.py:39-42)
__device__ __forceinline__ double dv_to(double v, const View& l) { return v - (l.ok ? l.v : 0.0); }

// Number of records in A[lo, hi) strictly above s_t (world.py:325-330):
// leader = lo+m-1, follower = lo+m.
__device__ __forceinline__ int32_t count_above(const VRec* A, int32_t lo, int32_t hi, double s_t) {
  int32_t a = lo, b = hi;
  while (a < b) {
    int32_t m = (a + b) >> 1;
    if (A[m].s > s_t)
      a = m + 1;
    else
      b = m;
  }
  return a - lo;
}

// Records ahead of (s, vix) in (s desc, id asc) order (world.py:276-280).
__device__ __forceinline__ int32_t count_ahead(const VRec* A, int32_t lo, int32_t hi, double s, int32_t vix) {
  int32_t a = lo, b = hi;
  while (a < b) {
    int32_t m = (a + b) >> 1;
    if (ahead_of(A[m].s, A[m].vix, s, vix))
      a = m + 1;
    else
      b = m;
  }
  return a - lo;
}

// Lanes per tile of the step's lane scan (engine.cu SCAN_TILE): k_update adds
// each tile's total (c.scan_tile_sums, zeroed by k_begin_step) next to the
// per-lane counts, so the scan needs no separate tile-sum pass.
static constexpr int LANE_TILE = 2048;

// Post-update lane counts for the C layout; a vehicle that left its snapshot
// lane is also a "mover" (k_place_movers / k_lanefix).
// A mover's slot among its new lane's entrants comes from the same atomic
// (k_place then needs no atomic of its own).
__device__ __forceinline__ void count_bucket(const Ctx& c, int32_t lane, int32_t snap_lane, int32_t i) {
  atomicAdd(&c.cnt[lane], 1);
  if (lane != snap_lane) c.mslot[i] = atomicAdd(&c.ent[lane], 1);
  c.stay[i] = lane == snap_lane ? 1 : 0;
}

// ------------------------------------------------------------------ k_update

// World._update_vehicle + World._apply_deltas for one vehicle (thread per
// driving vehicle of the lane-sorted snapshot A; neighbours are adjacent
// records, so a warp mostly covers one or two lanes).
//
// MOBIL (mobil.py:45-98, world.py:344-397) is restated with its pure
// sub-terms shared instead of recomputed: the current-leader and
// old-follower accelerations do not depend on the side evaluated, the
// free-road term (v/v0_eff)^delta depends only on (v, v0_eff), and the
// final IDM call of world.py:406 usually repeats one MOBIL already made
// (same leader, same gap, same cap).  Every reused value is the same fp64
// expression on the same operands, so results are bit-identical to the
// per-call evaluation.
// Block size / min resident blocks of k_update (register budget: 64K / (BT * MINB)).
#ifndef UPD_BT
#define UPD_BT 256
#endif
#ifndef UPD_MINB
#define UPD_MINB 4
#endif
// One thread per vehicle (grid = ceil(N / BT) blocks, scheduled dynamically)
// instead of a grid-stride loop: the last partial wave of a grid-stride
// launch left most of the machine idle.
#ifndef UPD_GRID_CAP
#define UPD_GRID_CAP (1 << 30)
#endif
#ifndef PLACE_A0
#define PLACE_A0 1  // 1: B.src carries the snapshot lane's range start from k_update to k_place
#endif
#ifndef MOBIL_UNROLL
#define MOBIL_UNROLL 2
#endif
static constexpr int kMobilUnroll = MOBIL_UNROLL;  // the two MOBIL sides: unrolled (ILP) or looped (code size)
template <bool G>
__global__ void __launch_bounds__(UPD_BT, UPD_MINB) k_update(Ctx c) {
  PDL_WAIT();
  TL_MARK(TL_UPDATE);
  Dyn* dy = c.dyn;
  const int32_t n_a = dy->n_a;
  const int32_t n = n_a + (c.sharded ? dy->n_g : 0);
  const VRec* A = c.lay[dy->cur];
  const int2* S = c.rng[dy->cur];
  const Params& p = c.p;
  const uint64_t step_no = (uint64_t)dy->step_no;
  const double new_time = dy->time + p.dt;
  const double Lv = p.L;
  const int2* nrc_prev = c.nrc[(step_no + 1) & 1];
  int2* nrc_cur = c.nrc[step_no & 1];
  for (int32_t i = gtid(); i < n; i += gstride()) {
    int32_t counted = -1;  // the lane this record was counted into
    do {
    const VRec me = A[i];
    const int32_t snap_lane = me.lane;
    const bool ghost = c.sharded && i >= n_a;
    // a record outside its lane's snapshot range is a stale copy: a lane the
    // regroup relocated, or (sharded) last step's local copy of a halo lane,
    // superseded by the imported ghosts -- drop it
    // own-lane neighbours: the adjacent records of the lane's range (loaded
    // unconditionally, beside `me`, off the range lookup's critical path)
    const VRec prv_ = A[i > 0 ? i - 1 : i];
    const VRec nxv_ = A[i + 1 < n ? i + 1 : i];
    const int2 sg0 = seg(c, S, snap_lane);
    if (i < sg0.x || i >= sg0.y || (c.sharded && !ghost && !(c.zone[snap_lane] & ZF_OWN))) {
      store_b(&c.B[i], VRec{me.s, me.v, me.vix, me.rptr, -1, i});
      c.stay[i] = 0;
      break;
    }
    const LaneRec L0 = c.lanes[snap_lane];
    const bool has_prev = i > sg0.x, has_next = i + 1 < sg0.y;
    const VRec prv = has_prev ? prv_ : VRec{0.0, 0.0, 0, 0, -1, 0};
    const VRec nxv = has_next ? nxv_ : VRec{0.0, 0.0, 0, 0, -1, 0};
    const int32_t* roads = c.routes + me.rptr;  // roads[0] = current road, roads[1] = next (or -1)
    // next road of the route: cached by the previous step's update for the
    // record this snapshot entry came from (src = its index in that step's B,
    // nearly sequential), so the random route-pool gather leaves the
    // critical path; the cache entry is keyed by rptr and re-gathered on a
    // mismatch (reverted, injected, rerouted, ghost records)
    int32_t next_road;
    {
      const int32_t sidx = me.src;
      int2 ce = make_int2(-1, 0);
#if REC_STREAM
      if (!ghost && sidx >= 0 && sidx < c.cap_rec) ce = __ldcs(nrc_prev + sidx);  // last read of the cache entry
#else
      if (!ghost && sidx >= 0 && sidx < c.cap_rec) ce = __ldg(nrc_prev + sidx);
#endif
      next_road = ce.x == me.rptr ? ce.y : __ldg(roads + 1);
    }
    const double v = me.v;
    const double v0e_cur = py_min(p.v0, L0.cap);

    // Cached pure terms (valid flags below).
    double fr_me = 0.0;  // free term of me at v0e_cur
    bool have_fr_me = false;
    double a_final = 0.0;
    bool have_final = false;

    // ---- _consider_change (world.py:344-397)
    int32_t lane = snap_lane;
    double s = me.s;
    bool changed = false;
    int32_t best_tl = -1;       // target leader index of the chosen side
    double best_a_new = 0.0, best_g_tl = 0.0;
    if (L0.kind == TSB_KIND_ROAD && (L0.left >= 0 || L0.right >= 0)) {
      const bool any = next_road < 0;
      const bool mandatory = !any && conn_from_id(c, snap_lane, next_road) < 0;
      bool go = true;
      int32_t sides[2] = {L0.left, L0.right};
      int nsides = 2;
      if (mandatory) {
        int32_t below = -1, above = -1;
        for (int32_t k = c.road_lane_off[L0.road]; k < c.road_lane_off[L0.road + 1]; k++) {
          int32_t f = c.road_lanes[k];
          if (conn_from_id(c, f, next_road) < 0) continue;
          if (f < lane && (below < 0 || f > below)) below = f;
          if (f > lane && (above < 0 || f < above)) above = f;
        }
        double dl = below >= 0 ? (double)(lane - below) : CUDART_INF;
        double dr = above >= 0 ? (double)(above - lane) : CUDART_INF;
        sides[0] = dl <= dr ? L0.left : L0.right;
        nsides = 1;
      } else {
        const uint64_t key = c.ids_dense ? (uint64_t)me.vix : c.keys[me.vix];
        double draw = keyed_uniform_tail(p.rng_h2, key, step_no);  // rng.py:39-41 (seed, 1, id, step)
        go = !(draw >= p.eval_prob);
      }
      if (go) {
        // ---- evaluate_change (mobil.py:45-98) for each side.  All IDM
        // calls are pure, so the side-independent ones (current leader, old
        // follower) are evaluated once, up front and branch-free, and each
        // side's three calls are evaluated together: independent fp64
        // chains the scheduler can overlap instead of one long chain.
        const View mev{true, me.s, v};
        const View cl = has_prev ? View{true, prv.s, prv.v} : View{false, 0.0, 0.0};
        const View cf = has_next ? View{true, nxv.s, nxv.v} : View{false, 0.0, 0.0};
        const double g_cur = gap_to(cl, me.s, Lv);
        const double g_of_old = me.s - Lv - cf.s;
        const double g_of_new = gap_to(cl, cf.s, Lv);
        const bool of_ok = cf.ok && g_of_old > 0.0 && g_of_new > 0.0;
        fr_me = idm_free<G>(p, v, v0e_cur);
        have_fr_me = true;
        const double fr_cf = idm_free<G>(p, cf.v, v0e_cur);
        const double a_me_x = idm_safe<G>(p, fr_me, v, dv_to(v, cl), g_cur);
        const double a_of_x = idm_safe<G>(p, fr_cf, cf.v, dv_to(cf.v, mev), g_of_old);
        const double a_of_new_x = idm_safe<G>(p, fr_cf, cf.v, dv_to(cf.v, cl), g_of_new);
        const double a_me = (g_cur <= 0.0) ? -CUDART_INF : a_me_x;
        const double a_of = of_ok ? a_of_x : 0.0;
        const double a_of_new = of_ok ? a_of_new_x : 0.0;
        bool have = false;
        double best_inc = 0.0, best_s = 0.0;
        int32_t best_nb = -1;
        // both sides evaluated without branches (a side that does not exist
        // or fails a check is evaluated on safe stand-ins and discarded):
        // the warp stays converged through the fp64 work
#pragma unroll(kMobilUnroll)
        for (int k = 0; k < 2; k++) {
          const int32_t nb = k < nsides ? sides[k] : -1;
          const int32_t nbs = nb >= 0 ? nb : snap_lane;
          bool ok = nb >= 0 && (c.lflag[nbs] & LF_OPEN);
          const LaneRec LN = c.lanes[nbs];
          ok = ok && (mandatory || any || conn_from_id(c, nbs, next_road) >= 0);
          // lanes of one road share its length: the ratio is then exactly 1
          // (a branch, so the division is skipped, not just discarded)
          double ratio = 1.0;
          if (LN.len != L0.len) ratio = LN.len / L0.len;
          const double s_t = me.s * ratio;
          const int2 sgn = seg(c, S, nbs);
          const int32_t lo = sgn.x, hi = sgn.y;
          const int32_t m = count_above(A, lo, hi, s_t);
          const int32_t tl_i = m > 0 ? lo + m - 1 : -1;
          const View tl = view_at(A, tl_i);
          const View tf = view_at(A, lo + m < hi ? lo + m : -1);
          const double g_tl = gap_to(tl, s_t, Lv);
          const double g_tf = tf.ok ? s_t - Lv - tf.s : CUDART_INF;
          const double g_nf_old = gap_to(tl, tf.s, Lv);
          ok = ok && !(g_tl <= 0.0 || g_tf <= 0.0 || (tf.ok && g_nf_old <= 0.0));
                    const double v0e_tgt = py_min(p.v0, LN.cap);
          const double fr_me_t = (v0e_tgt == v0e_cur) ? fr_me : idm_free<G>(p, v, v0e_tgt);
          const double fr_tf = idm_free<G>(p, tf.v, v0e_tgt);
          const double a_me_new = idm_safe<G>(p, fr_me_t, v, dv_to(v, tl), g_tl);
          const double a_nf_x = idm_safe<G>(p, fr_tf, tf.v, dv_to(tf.v, tl), g_nf_old);
          const double a_nf_new_x = idm_safe<G>(p, fr_tf, tf.v, tf.v - v, g_tf);  // new leader: me at s_t
          const double a_nf = tf.ok ? a_nf_x : 0.0;
          const double a_nf_new = tf.ok ? a_nf_new_x : 0.0;
          ok = ok && !(tf.ok && a_nf_new < -p.b_safe);
          double inc;
          if (a_me == -CUDART_INF)
            inc = CUDART_INF;
          else
            inc = (a_me_new - a_me) + p.politeness * ((a_nf_new - a_nf) + (a_of_new - a_of));
          ok = ok && (mandatory || !(inc <= p.threshold));
          if (ok && (!have || inc > best_inc || (inc == best_inc && nb < best_nb))) {
            have = true;
            best_inc = inc;
            best_nb = nb;
            best_s = s_t;
            best_tl = tl_i;
            best_a_new = a_me_new;
            best_g_tl = g_tl;
          }
        }
        if (have) {
          changed = true;
          lane = best_nb;
          s = best_s;
        } else if (cl.ok && g_cur >= EPS_GAP) {
          // world.py:406 will evaluate exactly a_me: same leader (i-1), gap
          // max(g_cur, 1e-6) == g_cur, same cap
          a_final = a_me;
          have_final = true;
        }
      }
    }

    // ---- _sense (world.py:261-317)
    const LaneRec L1 = changed ? c.lanes[lane] : L0;
    double gap = CUDART_INF, lead_v = 0.0;
    bool found = false;
    if (!have_final) {
      const int2 sgl = seg(c, S, lane);
      const int32_t lo = sgl.x, hi = sgl.y;
      if (hi > lo) {
        int32_t ld = -1;
        if (!changed) {
          if (has_prev) ld = i - 1;
        } else {
          int32_t m = count_ahead(A, lo, hi, s, me.vix);
          if (m > 0) ld = lo + m - 1;
        }
        if (ld >= 0) {
          if (changed && ld == best_tl && best_g_tl >= EPS_GAP) {
            a_final = best_a_new;  // MOBIL's a_me_new: same leader, gap, cap
            have_final = true;
          } else {
            gap = py_max(A[ld].s - Lv - s, EPS_GAP);
            lead_v = A[ld].v;
          }
          found = true;
        }
      }
    } else {
      found = true;
    }
    if (!found) {
      const double remaining = L1.len - s;
      bool stop = false;
      if (L1.kind == TSB_KIND_ROAD) {
        if (next_road < 0) {
          gap = CUDART_INF;
          lead_v = 0.0;
          found = true;
        } else {
          const int32_t conn = conn_from_id(c, lane, next_road);
          const uint8_t f = conn >= 0 ? c.lflag[conn] : 0;
          if (conn < 0 || !lf_passable(f)) {
            stop = true;
          } else {
            const int asp = lf_aspect(f);
            if (asp == RED || (asp == AMBER && remaining > v * v / (2.0 * p.b))) stop = true;
          }
        }
        if (stop) {
          gap = py_max(remaining, EPS_GAP);
          lead_v = 0.0;
          found = true;
        }
      }
      if (!found) {
        const int32_t* rq = roads;
        LaneRec LC = L1;
        int32_t cur = lane;
        double dist = remaining;
        gap = CUDART_INF;
        lead_v = 0.0;
        while (dist < p.lookahead) {
          int32_t nxt;
          if (LC.kind == TSB_KIND_ROAD) {
            const int32_t nr = rq == roads ? next_road : __ldg(rq + 1);
            nxt = nr < 0 ? -1 : conn_from_id(c, cur, nr);
            if (nxt < 0 || !(c.lflag[nxt] & LF_OPEN)) break;
          } else {
            nxt = LC.succ1;
            rq += 1;
            if (nxt < 0 || !(c.lflag[nxt] & LF_OPEN)) break;  // (< 0: beyond a rank's local lanes)
          }
          const int2 sgx = seg(c, S, nxt);
          const int32_t lo = sgx.x, hi = sgx.y;
          if (hi > lo) {
            const VRec rear = A[hi - 1];
            double g = dist + rear.s - Lv;
            gap = py_max(g, EPS_GAP);
            lead_v = rear.v;
            break;
          }
          LC = c.lanes[nxt];
          cur = nxt;
          dist += LC.len;
        }
      }
    }

    // ---- IDM + integration (world.py:406-419)
    double a;
    if (have_final) {
      a = a_final;
    } else {
      const double v0e = py_min(p.v0, L1.cap);
      const double fr = (have_fr_me && v0e == v0e_cur) ? fr_me : idm_free<G>(p, v, v0e);
      a = idm_with_free<G>(p, fr, v, v - lead_v, gap);
    }
    const double dt = p.dt;
    double v_new = v + a * dt, disp;
    if (v_new <= 0.0) {
      v_new = 0.0;
      disp = a < 0.0 ? div_pos(v * v, 2.0 * -a) : 0.0;
    } else {
      disp = v * dt + 0.5 * a * dt * dt;
      if (disp < 0.0) disp = 0.0;
    }
    double ns = s + disp, nv = v_new;
    int32_t nl = lane, nptr = me.rptr, nxt_rd = next_road;

    // ---- _apply_deltas transitions (world.py:443-499)
    LaneRec LT = L1;
    bool arrived = false, host = false;
    while (ns > LT.len) {
      if (LT.kind == TSB_KIND_ROAD) {
        const int32_t nr = nxt_rd;
        if (nr < 0) {
          arrived = true;
          break;
        }
        const int32_t conn = conn_from_id(c, nl, nr);
        const uint8_t f = conn >= 0 ? c.lflag[conn] : 0;
        if (conn >= 0 && !lf_passable(f)) {
          host = true;  // reroute needs the host router (world.py:460-469)
          break;
        }
        if (conn < 0 || lf_aspect(f) == RED) {
          ns = LT.len;
          nv = 0.0;
          break;
        }
        ns -= LT.len;
        nl = conn;
        LT = c.lanes[conn];
      } else {
        if (LT.succ1 < 0) {  // a sharded rank's halo edge: the lane beyond is not local (inexact zone)
          ns = LT.len;
          nv = 0.0;
          break;
        }
        ns -= LT.len;
        nl = LT.succ1;
        nptr += 1;
        nxt_rd = __ldg(c.routes + nptr + 1);
        LT = c.lanes[nl];
      }
    }
#if PLACE_A0
    // B's src field is the record's own index (implied by its position): it
    // carries the snapshot lane's range start instead, which k_place needs
    // for a stayer's rank (one dependent load less there); k_place restores src
    VRec out{ns, nv, me.vix, nptr, nl, sg0.x};
#else
    VRec out{ns, nv, me.vix, nptr, nl, i};
#endif
    nrc_cur[i] = make_int2(nptr, nxt_rd);
    if (arrived && ghost) {  // the owner records it
      out.lane = -1;
      c.stay[i] = 0;
    } else if (arrived) {
      out.lane = -1;
      c.stay[i] = 0;
      c.status[me.vix] = TSB_STATUS_FINISHED;
      c.finish[me.vix] = new_time;
      c.fin_state[me.vix] = me;
      unsigned long long k = atomicAdd((unsigned long long*)&dy->finished_now, 1ULL);
      FinEntry fe;
      fe.vix = me.vix;
      fe.pad = 0;
      fe.step = (int64_t)step_no;
      c.fin_log[dy->fin_log_n + (int64_t)k] = fe;
    } else if (host) {
      int32_t k = atomicAdd(&dy->n_hostq, 1);
      c.hostq[k] = i;
      if (!c.split) {  // closures only occur in split mode; keep the state consistent
        out.lane = nl;
        count_bucket(c, nl, snap_lane, i);
        counted = nl;
      }
    } else {
      count_bucket(c, nl, snap_lane, i);
      counted = nl;
      if (ghost && (c.zone[nl] & ZF_OWN)) c.status[me.vix] = TSB_STATUS_DRIVING;  // entered an own lane
    }
    store_b(&c.B[i], out);
    } while (0);
    // the scan's tile totals: one atomic per tile per warp
    const unsigned am = __activemask();
    const int32_t tile = counted >= 0 ? counted / LANE_TILE : -1;
    const unsigned grp = __match_any_sync(am, tile);
    if (tile >= 0 && (threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&c.scan_tile_sums[tile], __popc(grp));
  }
}

// Fix-up after host continuation of rerouted vehicles: count their lanes.
__global__ void k_count_hostq(Ctx c) {
  PDL_WAIT();
  Dyn* dy = c.dyn;
  const VRec* A = c.lay[dy->cur];
  for (int32_t k = gtid(); k < dy->n_hostq; k += gstride()) {
    const int32_t i = c.hostq[k];
    const VRec r = c.B[i];
    if (r.lane >= 0) {
      count_bucket(c, r.lane, A[i].lane, i);
      atomicAdd(&c.scan_tile_sums[r.lane / LANE_TILE], 1);
    } else
      c.stay[i] = 0;  // arrived during the host continuation
  }
}

// ------------------------------------------------------------------ scan

// Exclusive scan of in[0, n) into out[0, n] (out[n] = total), single pass
// with decoupled look-back.  n is read from *n_dev when n_dev != nullptr.
// Every call site owns a status region and a 64-bit ticket counter that are
// never reset: block b of invocation k draws ticket k * ntiles + b, and the
// status words carry the invocation's epoch, so stale words from earlier
// steps are ignored and the step graph needs no memset nodes.  All ntiles
// blocks must be launched and draw a ticket (the gate is grid-uniform).
static constexpr int SCAN_SITES = 6;
enum { SCAN_LANES = 0, SCAN_INJ_LANES = 1, SCAN_INJ_RETRY = 2, SCAN_REGROUP = 3, SCAN_EXPORT = 4, SCAN_IMPORT = 5 };
// The step's lane scan takes the tile totals k_update summed
// (tile_sums != nullptr): tile b's prefix is the sum of the totals before it
// -- no serial look-back chain across 150+ tiles, no separate tile-sum pass.
template <int BT, int IPT>
__global__ void __launch_bounds__(BT) k_scan(Ctx c, int site, const int32_t* in, int32_t* out, int out_sel,
                                             const int32_t* n_dev, int32_t n_static, int32_t ntiles,
                                             const int32_t* gate, const int32_t* tile_sums) {
  PDL_WAIT();
  if (site == SCAN_LANES) TL_MARK(TL_SCAN);
  if (gated_off(gate)) return;
  int2* rng = nullptr;
  if (out_sel != SEL_NONE) {
    out = start_buf(c, out_sel);
    rng = out_sel == SEL_A ? c.rng[c.dyn->cur] : c.rng[c.dyn->cur ^ 1];
  }
  unsigned long long* status = c.scan_status + (size_t)site * c.scan_tiles_cap;
  const int32_t n = n_dev ? *n_dev : n_static;
  __shared__ int32_t s_tile, s_prefix;
  __shared__ unsigned s_epoch;
  __shared__ int32_t s_warp[BT / 32];
  if (threadIdx.x == 0) {
    if (tile_sums) {
      s_tile = blockIdx.x;
      s_epoch = 1u;
    } else {
      const unsigned long long t = atomicAdd(c.scan_tickets + site, 1ULL);
      s_tile = (int32_t)(t % (unsigned long long)ntiles);
      s_epoch = (unsigned)((t / (unsigned long long)ntiles) % 0x3fffffffULL) + 1u;
    }
  }
  __syncthreads();
  const int32_t tile = s_tile;
  const unsigned long long ep = (unsigned long long)s_epoch << 34;
  const int64_t base = (int64_t)tile * BT * IPT;
  if (base > n) return;
  int32_t v[IPT];
  int32_t local = 0;
#pragma unroll
  for (int k = 0; k < IPT; k++) {
    int64_t idx = base + (int64_t)threadIdx.x * IPT + k;
    v[k] = idx < n ? in[idx] : 0;
    local += v[k];
  }
  // block exclusive scan of `local`
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t x = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int32_t w = lane < BT / 32 ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < BT / 32) s_warp[lane] = w;
  }
  __syncthreads();
  const int32_t warp_excl = warp ? s_warp[warp - 1] : 0;
  const int32_t total = s_warp[BT / 32 - 1];
  int32_t excl = warp_excl + x - local;
  // status word: epoch (30 bits) | flag (2 bits) | value (32 bits);
  // flag 1 = tile aggregate, 2 = inclusive prefix
  volatile unsigned long long* st = status;
  if (tile_sums) {
    if (warp == 0) {
      int32_t acc = 0;
      for (int32_t t = lane; t < tile; t += 32) acc += tile_sums[t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) s_prefix = acc;
    }
  } else if (tile == 0) {
    if (threadIdx.x == 0) {
      __threadfence();
      st[0] = ep | (2ULL << 32) | (unsigned)total;
      s_prefix = 0;
    }
  } else if (warp == 0) {
    if (lane == 0) st[tile] = ep | (1ULL << 32) | (unsigned)total;
    __threadfence();
    // warp-wide look-back: 32 predecessors per round, nearest first
    int32_t acc = 0;
    int32_t t = tile - 1;
    for (;;) {
      const int32_t idx = t - lane;
      unsigned long long w = idx >= 0 ? st[idx] : (ep | (2ULL << 32));
      while (!__all_sync(0xffffffffu, (w >> 34) == (ep >> 34))) {  // wait for the window to publish
        if ((w >> 34) != (ep >> 34)) w = st[idx];
      }
      const unsigned incl = __ballot_sync(0xffffffffu, ((unsigned)(w >> 32) & 3u) == 2u);
      const int last = incl ? __ffs(incl) - 1 : 31;  // nearest inclusive prefix ends the walk
      int32_t pv = lane <= last ? (int32_t)(unsigned)(w & 0xffffffffULL) : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) pv += __shfl_xor_sync(0xffffffffu, pv, o);
      acc += pv;
      if (incl) break;
      t -= 32;
    }
    if (lane == 0) {
      __threadfence();
      st[tile] = ep | (2ULL << 32) | (unsigned)(acc + total);
      s_prefix = acc;
    }
  }
  __syncthreads();
  int32_t run = s_prefix + excl;
#pragma unroll
  for (int k = 0; k < IPT; k++) {
    int64_t idx = base + (int64_t)threadIdx.x * IPT + k;
    if (idx <= n) out[idx] = run;
    if (rng && idx < n) rng[idx] = make_int2(run, run + v[k]);
    run += v[k];
  }
}

// ------------------------------------------------------------------ scatter / sort / sweep

// Bucket records by lane: dst[start[lane] + cursor++].  Records with lane < 0
// (arrivals) are dropped.  src has *n_ptr (+ *n_extra) records.
__global__ void k_scatter(Ctx c, int src_sel, const int32_t* n_ptr, const int32_t* n_extra, int start_sel,
                          const int32_t* gate) {
  PDL_WAIT();
  if (gated_off(gate)) return;
  if (src_sel == SEL_B && gtid() == 0) {
    // vehicles bucketed into C this step (last CSR entry of the scan)
    c.dyn->n_c = c.start[c.dyn->cur ^ 1][c.n_lanes];
    if (c.dyn->n_hostq > 0 && !c.split) c.dyn->overflow |= 4;
  }
  const VRec* src = rec_buf(c, src_sel);
  const int32_t* start = start_buf(c, start_sel);
  VRec* dst = c.D;
  const int32_t n = *n_ptr + (n_extra ? *n_extra : 0);
  for (int32_t i = gtid(); i < n; i += gstride()) {
    const VRec r = src[i];
    if (r.lane < 0) continue;
    int32_t k = atomicAdd(&c.cursor[r.lane], 1);
    dst[start[r.lane] + k] = r;
  }
}

__global__ void k_hist(Ctx c, int src_sel, const int32_t* n_ptr, const int32_t* n_extra, const int32_t* gate) {
  PDL_WAIT();
  if (gated_off(gate)) return;
  const VRec* src = rec_buf(c, src_sel);
  const int32_t n = *n_ptr + (n_extra ? *n_extra : 0);
  for (int32_t i = gtid(); i < n; i += gstride()) {
    int32_t l = src[i].lane;
    if (l >= 0) atomicAdd(&c.cnt[l], 1);
  }
}

// Warp per lane: sort D[lo,hi) by (s desc, vix asc) into C[lo,hi), then (if
// sweep) the tentative collision sweep of world.py:524-555 on this lane from
// its post-delta state.  A lane whose sweep would revert a vehicle is left
// unswept (C keeps the sorted post-delta values) and queued for k_resolve.
template <bool SWEEP>
__global__ void k_lanesort(Ctx c, int dst_sel, const int32_t* gate) {
  PDL_WAIT();
  if (gated_off(gate)) return;
  const VRec* D = c.D;
  VRec* C = rec_buf(c, dst_sel);
  const int32_t* start = start_buf(c, dst_sel);
  const VRec* snapA = rec_buf(c, SEL_A);
  const int lane_id = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const Params& p = c.p;
  Dyn* dy = c.dyn;
  for (int32_t L = gtid() >> 5; L < c.n_lanes; L += warps) {
    const int32_t lo = start[L], hi = start[L + 1], n = hi - lo;
    if (n == 0) continue;
    // the bucketing counters of this lane are consumed: leave them zero for
    // the next use (replaces per-step memsets)
    if (lane_id == 0) {
      c.cnt[L] = 0;
      c.cursor[L] = 0;
    }
    // rank sort (keys unique: vix distinct)
    for (int32_t j = lane_id; j < n; j += 32) {
      const VRec r = D[lo + j];
      int32_t rank = 0;
      for (int32_t k = 0; k < n; k++) {
        const double sk = D[lo + k].s;
        const int32_t vk = D[lo + k].vix;
        rank += ahead_of(sk, vk, r.s, r.vix) ? 1 : 0;
      }
      C[lo + rank] = r;
    }
    __syncwarp();
    if (!SWEEP) continue;
    // parallel trigger test on unclamped predecessors
    int32_t first = n;
    for (int32_t j = lane_id; j < n; j += 32) {
      if (j == 0) continue;
      double limit = (C[lo + j - 1].s - p.L) - p.s0_floor;
      if (C[lo + j].s > limit + 1e-12) first = min(first, j);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    if (first >= n) continue;
    if (lane_id == 0) {
      // sequential sweep from `first` (everything before is untouched)
      VRec prev = C[lo + first - 1];
      bool prev_entered = prev.lane != snapA[prev.src].lane;
      double prev_rear = prev.s - p.L;
      bool event = false;
      int32_t k = first;
      for (; k < n; k++) {
        VRec r = C[lo + k];
        const double limit = prev_rear - p.s0_floor;
        const VRec sn = snapA[r.src];
        const bool entered = r.lane != sn.lane;
        if (r.s > limit + 1e-12) {
          const double floor_s = entered ? 0.0 : sn.s;
          if (limit >= floor_s) {
            r.v = py_max(0.0, py_min(r.v, r.v - (r.s - limit) / p.dt));
            r.s = limit;
          } else if (entered) {  // not reverted: no vehicle is reverted before resolve
            event = true;
            break;
          } else if (prev_entered) {
            event = true;
            break;
          } else {
            r.v = 0.0;
            r.s = floor_s;
          }
          C[lo + k].s = r.s;
          C[lo + k].v = r.v;
        }
        prev_entered = entered;
        prev_rear = r.s - p.L;
      }
      if (event) {
        // restore the post-delta values written so far; resolve re-sweeps
        for (int32_t q = first; q < k; q++) {
          const VRec o = c.B[C[lo + q].src];
          C[lo + q].s = o.s;
          C[lo + q].v = o.v;
        }
        int32_t e = atomicAdd(&dy->n_events, 1);
        c.events[e] = L;
      } else {
        // a hold can break the (s desc) order; the next snapshot must be re-sorted
        for (int32_t q = (first > 0 ? first - 1 : 0); q + 1 < n; q++)
          if (!ahead_of(C[lo + q].s, C[lo + q].vix, C[lo + q + 1].s, C[lo + q + 1].vix)) {
            mark_dirty(c, L);
            break;
          }
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ lane assembly

// Post-update lane assembly, the main path of the bucketing (replaces a full
// scatter + per-lane sort).  B is in snapshot order, so the vehicles that
// stayed on their lane ("stayers", nearly all) keep their relative order:
// k_place writes each stayer straight to its C position (its snapshot rank
// minus the lane's leavers ahead of it) and each mover to the tail of its new
// lane's segment, and flags the lanes whose assembly is not final: a mover
// entered, two stayers swapped order, or the sweep would touch a vehicle
// (world.py:531 trigger).  k_lanefix then sorts (s desc, id asc) and sweeps
// only the flagged lanes, on chip.
#ifndef PLACE_LIST
#define PLACE_LIST 1  // 1: k_place appends flagged lanes to a list (atomics); 0: flag words only (same speed, A/B r2)
#endif
__device__ __forceinline__ void flag_lane(const Ctx& c, int32_t L) {
  if (atomicExch(&c.fix_flag[L], 1) == 0) c.fix_list[atomicAdd(&c.dyn->n_fix, 1)] = L;
}

__global__ void k_place(Ctx c) {
  PDL_WAIT();
  TL_MARK(TL_PLACE);
  Dyn* dy = c.dyn;
  VRec* C = c.lay[dy->cur ^ 1];
  const int32_t* CS = c.start[dy->cur ^ 1];
  const int2* SA = c.rng[dy->cur];
  const Params& p = c.p;
  if (gtid() == 0) {
    // vehicles bucketed into C this step (last CSR entry of the scan)
    dy->n_c = CS[c.n_lanes];
    if (dy->n_hostq > 0 && !c.split) dy->overflow |= 4;
  }
  const int32_t n = dy->n_a + (c.sharded ? dy->n_g : 0);
  const int lid = threadIdx.x & 31;
#if PLACE_LIST
  __shared__ int32_t s_cnt, s_base;
  __shared__ int32_t s_list[256];
#endif
  // one pass in the usual case; block-uniform trip count (the block-level
  // append below synchronises), whole warps (the ballots need all 32 lanes)
  for (int32_t bbase = blockIdx.x * blockDim.x; bbase < n; bbase += gstride()) {
    const int32_t base = bbase + (threadIdx.x & ~31);
    const int32_t j = base + lid;
    const bool valid = j < n;
    VRec r = valid ? load_b(&c.B[j]) : VRec{0.0, 0.0, 0, 0, -1, 0};
    const bool st = valid && c.stay[j];
    const unsigned stay_bits = __ballot_sync(0xffffffffu, st);
    const int32_t L = r.lane;
    // stayer rank in its lane = stayers ahead of it in its snapshot range
    // [a0, j): inside the warp from the ballot; before the warp only for the
    // lane whose range covers `base` -- the first stayer's lane, if its range
    // starts before the warp -- counted by the whole warp, 32 at a time
#if PLACE_A0
    const int32_t a0 = st ? r.src : 0;  // the snapshot lane's range start (k_update)
    r.src = j;                          // C records point at their snapshot record
#else
    const int32_t a0 = st ? seg(c, SA, L).x : 0;
#endif
    const int first_st = stay_bits ? __ffs(stay_bits) - 1 : 0;
    const int32_t Ls = __shfl_sync(0xffffffffu, L, first_st);
    const int32_t a0s = __shfl_sync(0xffffffffu, a0, first_st);
    int32_t before = 0, kb = -1;  // its stayers in [a0s, base), the last of them
    if (stay_bits && a0s < base) {
      for (int32_t hi = base; hi > a0s; hi -= 32) {
        const int32_t q = hi - 1 - lid;
        const unsigned bq = __ballot_sync(0xffffffffu, q >= a0s && c.stay[q]);
        if (kb < 0 && bq) kb = hi - __ffs(bq);  // nearest first: lowest lid = largest q
        before += __popc(bq);
      }
    }
    const unsigned below = (1u << lid) - 1u;
    const int lo_lane = a0 > base ? a0 - base : 0;
    const unsigned prev_bits = stay_bits & below & ~((1u << lo_lane) - 1u);
    // previous stayer inside the warp: its record by shuffle
    const int pl = prev_bits ? 31 - __clz(prev_bits) : lid;
    const double pr_s = __shfl_sync(0xffffffffu, r.s, pl);
    const int32_t pr_vix = __shfl_sync(0xffffffffu, r.vix, pl);
    bool flag = false;  // this lane needs k_lanefix
    if (L >= 0) {
      if (!st) {
        const int32_t pos = CS[L] + (c.cnt[L] - c.ent[L]) + c.mslot[j];
        C[pos] = r;
        flag = true;
      } else {
        const bool straddle = a0 < base;  // then L == Ls
        const int32_t rank = __popc(prev_bits) + (straddle ? before : 0);
        C[CS[L] + rank] = r;
        double ps;
        int32_t pv;
        bool have = true;
        if (prev_bits) {
          ps = pr_s;
          pv = pr_vix;
        } else if (straddle && kb >= 0) {
          const VRec pr = c.B[kb];
          ps = pr.s;
          pv = pr.vix;
        } else {
          have = false;
        }
        if (have) flag = !ahead_of(ps, pv, r.s, r.vix) || r.s > ((ps - p.L) - p.s0_floor) + 1e-12;
      }
    }
#if PLACE_LIST
    // append newly flagged lanes: one flag atomic per lane per warp (jammed
    // lanes flag every vehicle), collected per block in shared memory, one
    // counter atomic per block (a per-warp counter atomic serialised ~30k
    // same-address atomics per step)
    const unsigned fm = __ballot_sync(0xffffffffu, flag);
    bool first_flag = false;
    if (flag) {
      const unsigned grp = __match_any_sync(fm, L);
      if (lid == __ffs(grp) - 1) first_flag = atomicExch(&c.fix_flag[L], 1) == 0;
    }
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    if (first_flag) s_list[atomicAdd(&s_cnt, 1)] = L;
    __syncthreads();
    const int32_t nb = s_cnt;
    if (threadIdx.x == 0 && nb) s_base = atomicAdd(&dy->n_fix, nb);
    __syncthreads();
    for (int32_t k = threadIdx.x; k < nb; k += blockDim.x) c.fix_list[s_base + k] = s_list[k];
    __syncthreads();
#else
    // flag the lane for k_lanefix: a plain store per lane per warp (the flag
    // words are the work list: k_lanefix scans them 32 lanes per warp), no
    // atomic round trip and no block-wide append
    const unsigned fm = __ballot_sync(0xffffffffu, flag);
    if (flag) {
      const unsigned grp = __match_any_sync(fm, L);
      if (lid == __ffs(grp) - 1) c.fix_flag[L] = 1;
    }
#endif
  }
}

#ifndef LX_CAP_CFG
#define LX_CAP_CFG 64
#endif
// LX_G threads per flagged lane: 16 = two lanes in flight per warp, each
// group with half the warp's shared-memory staging (32 members on chip; M1's
// flagged lanes hold <= 32, larger ones stage in global memory).  A/B at M1
// (r2): 32 -> 16 takes k_lanefix 17.7 -> 16.0 us; 8 threads: 19.9 us.
#ifndef LX_G
#define LX_G 16
#endif
// LX_REUSE: the snapshot (s, lane) of a swept lane's members go into the
// unsorted copy's shared memory (dead after the sort): 32 KB per block, so
// with <= 40 registers (LX_MINB) six blocks fit per SM.  A/B at M1 (r2):
// k_lanefix 19.2 -> 17.2 us, the step -1.6 us; the reuse alone at 5 blocks: -0.5.
#ifndef LX_REUSE
#define LX_REUSE 1
#endif
static constexpr int LX_GPW = 32 / LX_G;               // lanes in flight per warp
static constexpr int LX_CAP = LX_CAP_CFG / LX_GPW;     // lane members staged in shared memory
static constexpr int LX_WARPS = 8;
#if !PLACE_LIST && LX_G != 32
#error "LX_G < 32 needs PLACE_LIST"
#endif
// k_lanefix grid: blocks per SM (grid-stride over the flagged lanes); 6 is
// what fits at once (shared memory, registers), so the launch is one full wave
#ifndef LX_BLOCKS_PER_SM
#define LX_BLOCKS_PER_SM 6
#endif
#ifndef LX_MINB
#define LX_MINB LX_BLOCKS_PER_SM
#endif
__global__ void __launch_bounds__(32 * LX_WARPS, LX_MINB) k_lanefix(Ctx c) {
  PDL_WAIT();
  TL_MARK(TL_LANEFIX);
  __shared__ VRec s_in[LX_WARPS * LX_GPW][LX_CAP];
  __shared__ VRec s_out[LX_WARPS * LX_GPW][LX_CAP];
#if !LX_REUSE
  __shared__ double s_snap_s[LX_WARPS * LX_GPW][LX_CAP];
  __shared__ int32_t s_snap_l[LX_WARPS * LX_GPW][LX_CAP];
#endif
  Dyn* dy = c.dyn;
  VRec* C = c.lay[dy->cur ^ 1];
  const int32_t* CS = c.start[dy->cur ^ 1];
  const VRec* A = c.lay[dy->cur];
  const int lid = threadIdx.x & 31;
  const int gi = lid / LX_G, gl = lid % LX_G;  // group in the warp, thread in the group
  const int w = (threadIdx.x >> 5) * LX_GPW + gi;  // this group's staging slot
  const unsigned gmask = LX_G == 32 ? 0xffffffffu : (((1u << LX_G) - 1u) << (gi * LX_G));
#if LX_REUSE
  // the members' snapshot (s, lane) in the unsorted copy's storage, dead
  // after the rank sort (12 of its 32 bytes per member)
  double* const snap_s = reinterpret_cast<double*>(&s_in[w][0]);
  int32_t* const snap_l = reinterpret_cast<int32_t*>(snap_s + LX_CAP);
#else
  double* const snap_s = s_snap_s[w];
  int32_t* const snap_l = s_snap_l[w];
#endif
  const int groups = ((gridDim.x * blockDim.x) >> 5) * LX_GPW;
  const Params& p = c.p;
#if PLACE_LIST
  const int32_t nfix = dy->n_fix;
  for (int32_t f = (gtid() >> 5) * LX_GPW + gi; f < nfix; f += groups) {
    const int32_t L = c.fix_list[f];
#else
  // the flagged lanes: each warp takes 32 lanes' flag words at a time
  const int32_t ngrp = (c.n_lanes + 31) >> 5;
  for (int32_t g = gtid() >> 5; g < ngrp; g += groups) {
   const int32_t Lg = (g << 5) + lid;
   unsigned todo = __ballot_sync(0xffffffffu, Lg < c.n_lanes && c.fix_flag[Lg]);
   while (todo) {
    const int32_t L = (g << 5) + __ffs(todo) - 1;
    todo &= todo - 1;
#endif
    const int32_t lo = CS[L], n = CS[L + 1] - lo;
    if (gl == 0) {
      c.fix_flag[L] = 0;
      c.ent[L] = 0;  // consumed: zero for the next step (no memsets)
    }
    const bool on_chip = n <= LX_CAP;
    VRec* in = on_chip ? s_in[w] : c.D + lo;  // oversized lanes stage in D
    VRec* out = on_chip ? s_out[w] : C + lo;
    for (int32_t q = gl; q < n; q += LX_G) in[q] = C[lo + q];
    __syncwarp(gmask);
    // rank sort (keys unique: vix distinct)
    for (int a = gl; a < n; a += LX_G) {
      const double sa = in[a].s;
      const int32_t va = in[a].vix;
      int rank = 0;
      for (int b2 = 0; b2 < n; b2++) rank += ahead_of(in[b2].s, in[b2].vix, sa, va) ? 1 : 0;
      out[rank] = in[a];
    }
    __syncwarp(gmask);
    // tentative sweep: parallel trigger test, then thread 0 from the first trigger
    int32_t first = n;
    for (int32_t j = gl; j < n; j += LX_G) {
      if (j == 0) continue;
      const double limit = (out[j - 1].s - p.L) - p.s0_floor;
      if (out[j].s > limit + 1e-12) first = min(first, j);
    }
#pragma unroll
    for (int o = LX_G / 2; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(gmask, first, o, LX_G));
    // the sweep reads each member's snapshot lane / s: gathered in parallel
    // first (on-chip lanes), not one dependent load per member in thread 0
    const bool pre = on_chip && first < n;
    if (pre) {
      for (int32_t q = first - 1 + gl; q < n; q += LX_G) {
        const VRec sn = A[out[q].src];
        snap_l[q] = sn.lane;
        snap_s[q] = sn.s;
      }
      __syncwarp(gmask);
    }
    int32_t q_ev = -1;  // event: members [first, q_ev) were clamped and are restored
    if (first < n && gl == 0) {
      VRec prev = out[first - 1];
      bool prev_entered = prev.lane != (pre ? snap_l[first - 1] : A[prev.src].lane);
      double prev_rear = prev.s - p.L;
      bool event = false;
      int32_t q = first;
      for (; q < n; q++) {
        VRec r = out[q];
        const double limit = prev_rear - p.s0_floor;
        int32_t sn_lane;
        double sn_s;
        if (pre) {
          sn_lane = snap_l[q];
          sn_s = snap_s[q];
        } else {
          const VRec sn = A[r.src];
          sn_lane = sn.lane;
          sn_s = sn.s;
        }
        const bool entered = r.lane != sn_lane;
        if (r.s > limit + 1e-12) {
          const double floor_s = entered ? 0.0 : sn_s;
          if (limit >= floor_s) {
            r.v = py_max(0.0, py_min(r.v, r.v - (r.s - limit) / p.dt));
            r.s = limit;
          } else if (entered || prev_entered) {  // a revert: resolved by k_resolve_*
            event = true;
            break;
          } else {
            r.v = 0.0;
            r.s = floor_s;
          }
          out[q].s = r.s;
          out[q].v = r.v;
        }
        prev_entered = entered;
        prev_rear = r.s - p.L;
      }
      if (event) {
        q_ev = q;
        c.events[atomicAdd(&dy->n_events, 1)] = L;
      } else {
        // a hold can break the (s desc) order; the next snapshot must be re-sorted
        for (int32_t u = first - 1; u + 1 < n; u++)
          if (!ahead_of(out[u].s, out[u].vix, out[u + 1].s, out[u + 1].vix)) {
            mark_dirty(c, L);
            break;
          }
      }
    }
    q_ev = __shfl_sync(gmask, q_ev, 0, LX_G);
    __syncwarp(gmask);
    if (q_ev >= 0) {
      // leave the lane unswept (post-delta values) for the replay
      for (int32_t u = first + gl; u < q_ev; u += LX_G) {
        const VRec o = c.B[out[u].src];
        out[u].s = o.s;
        out[u].v = o.v;
      }
    }
    __syncwarp(gmask);
    if (on_chip)
      for (int a = gl; a < n; a += LX_G) C[lo + a] = out[a];
    __syncwarp(gmask);
#if !PLACE_LIST
   }
#endif
  }
}

// ------------------------------------------------------------------ revert resolution
//
// k_lanefix's tentative sweep handles every lane whose sweep needs no
// revert.  Lanes that would revert ("events") are resolved here by
// replaying the reference's restart-after-revert loop (world.py:518-559)
// exactly.  The replay only ever touches lanes reachable from an event lane
// through "entered" vehicles: a revert moves an entered member of the lane
// being swept (or its entered predecessor) back to its snapshot lane.
// k_resolve_closure collects that closure and splits it into connected
// components; k_resolve_comp replays each component in its own warp.
//
// Why components are independent (and exact): the reference's passes always
// restart at lane 0 and stop at the smallest lane that reverts, so the lane
// swept next is always the minimum pending lane -- a min-heap over dirty
// lanes.  Components with disjoint lane sets interact only through "reach",
// the largest lane any pass has swept, which decides whether a lane
// receiving a reverted vehicle is swept for the first time (from its
// post-delta state) or re-swept (from its clamped state).  When a component
// X pops lane E, every lane popped by another component since X last popped
// is < E (heap order), and before that < X's then-pending minimum, so the
// global reach at any X event equals X's own reach.  If the closure does not
// fit the on-chip budgets, the sequential k_resolve replays all events in
// one warp instead (same algorithm, one global heap).

static constexpr int RS_CAP = 192;     // members per lane staged on chip
static constexpr int CL_CAP = 2048;    // closure lanes
static constexpr int CE_CAP = 2048;    // closure edges (entered members)
static constexpr int HCAP = 64;        // lanes per component (heap capacity)

struct RsM {
  double s, v, snap_s;
  int32_t j, vix;
  uint8_t entered, reverted, pad[6];
};

// Min-heap of lane ids.
__device__ void heap_push(int32_t* h, int32_t& n, int32_t x) {
  int32_t i = n++;
  h[i] = x;
  while (i > 0) {
    int32_t pa = (i - 1) >> 1;
    if (h[pa] <= h[i]) break;
    int32_t t = h[pa];
    h[pa] = h[i];
    h[i] = t;
    i = pa;
  }
}
__device__ int32_t heap_pop(int32_t* h, int32_t& n) {
  int32_t top = h[0];
  h[0] = h[--n];
  int32_t i = 0;
  for (;;) {
    int32_t a = 2 * i + 1, b = a + 1, m = i;
    if (a < n && h[a] < h[m]) m = a;
    if (b < n && h[b] < h[m]) m = b;
    if (m == i) break;
    int32_t t = h[m];
    h[m] = h[i];
    h[i] = t;
    i = m;
  }
  return top;
}

// One lane of the replay, whole warp: gather the lane's current members (its
// C segment entries still on it, plus vehicles reverted into it, listed in
// moved[0, nmoved)), sort them (s desc, id asc), run the reference's sweep
// (world.py:527-555) and write the clamped values back.  Returns the C index
// of the vehicle to revert, or -1 (same value in every thread).
__device__ int32_t resolve_lane(const Ctx& c, VRec* C, const int32_t* CS, const VRec* A, int32_t L,
                                const int32_t* moved, int32_t nmoved, RsM* m, RsM* tmp) {
  const int lid = threadIdx.x & 31;
  const Params& p = c.p;
  const int32_t lo = CS[L], hi = CS[L + 1];
  int n = 0;
  for (int32_t base = lo; base < hi; base += 32) {
    const int32_t j = base + lid;
    const bool mine = j < hi && C[j].lane == L;
    const unsigned b = __ballot_sync(0xffffffffu, mine);
    const int slot = n + __popc(b & ((1u << lid) - 1));
    if (mine && slot < RS_CAP) {
      const VRec r = C[j];
      const VRec sn = A[r.src];
      m[slot] = RsM{r.s, r.v, sn.s, j, r.vix, (uint8_t)(sn.lane != L), c.rs_reverted[j], {0}};
    }
    n += __popc(b);
  }
  if (c.rs_movedin[L]) {
    for (int32_t base = 0; base < nmoved; base += 32) {
      const int32_t q = base + lid;
      int32_t j = -1;
      if (q < nmoved) {
        j = moved[q];
        if (!(C[j].lane == L && (j < lo || j >= hi))) j = -1;
      }
      const unsigned b = __ballot_sync(0xffffffffu, j >= 0);
      const int slot = n + __popc(b & ((1u << lid) - 1));
      if (j >= 0 && slot < RS_CAP) {
        const VRec r = C[j];
        const VRec sn = A[r.src];
        m[slot] = RsM{r.s, r.v, sn.s, j, r.vix, (uint8_t)(sn.lane != L), c.rs_reverted[j], {0}};
      }
      n += __popc(b);
    }
  }
  __syncwarp();
  int32_t rev = -1;
  if (n <= RS_CAP) {
    for (int a = lid; a < n; a += 32) tmp[a] = m[a];
    __syncwarp();
    for (int a = lid; a < n; a += 32) {
      int rank = 0;
      const double sa = tmp[a].s;
      const int32_t va = tmp[a].vix;
      for (int b2 = 0; b2 < n; b2++) rank += ahead_of(tmp[b2].s, tmp[b2].vix, sa, va) ? 1 : 0;
      m[rank] = tmp[a];
    }
    __syncwarp();
    if (lid == 0) {
      int prev = -1;
      double prev_rear = CUDART_INF;
      for (int a = 0; a < n; a++) {
        const double limit = prev_rear - p.s0_floor;
        if (m[a].s > limit + 1e-12) {
          const double floor_s = m[a].entered ? 0.0 : m[a].snap_s;
          if (limit >= floor_s) {
            m[a].v = py_max(0.0, py_min(m[a].v, m[a].v - (m[a].s - limit) / p.dt));
            m[a].s = limit;
          } else if (m[a].entered && !m[a].reverted) {
            rev = m[a].j;
            break;
          } else if (prev >= 0 && m[prev].entered && !m[prev].reverted) {
            rev = m[prev].j;
            break;
          } else {
            m[a].v = 0.0;
            m[a].s = floor_s;
          }
        }
        prev = a;
        prev_rear = m[a].s - p.L;
      }
    }
    __syncwarp();
    for (int a = lid; a < n; a += 32) {
      C[m[a].j].s = m[a].s;
      C[m[a].j].v = m[a].v;
    }
  } else if (lid == 0) {
    // oversized lane (> RS_CAP members): sort indices in global scratch.
    // Only the sequential replay gets here (k_resolve_closure sends any
    // closure with an oversized lane to it), so one scratch array suffices.
    int32_t* mem = c.rs_members;
    int32_t cnt = 0;
    for (int32_t j = lo; j < hi; j++)
      if (C[j].lane == L) mem[cnt++] = j;
    for (int32_t q = 0; q < nmoved; q++) {
      const int32_t j = moved[q];
      if (C[j].lane == L && (j < lo || j >= hi)) mem[cnt++] = j;
    }
    for (int32_t a = 1; a < cnt; a++) {
      const int32_t x = mem[a];
      int32_t b2 = a - 1;
      while (b2 >= 0 && ahead_of(C[x].s, C[x].vix, C[mem[b2]].s, C[mem[b2]].vix)) {
        mem[b2 + 1] = mem[b2];
        b2--;
      }
      mem[b2 + 1] = x;
    }
    int32_t prev = -1;
    double prev_rear = CUDART_INF;
    for (int32_t a = 0; a < cnt; a++) {
      const int32_t j = mem[a];
      VRec& r = C[j];
      const double limit = prev_rear - p.s0_floor;
      if (r.s > limit + 1e-12) {
        const VRec sn = A[r.src];
        const bool entered = r.lane != sn.lane;
        const double floor_s = entered ? 0.0 : sn.s;
        if (limit >= floor_s) {
          r.v = py_max(0.0, py_min(r.v, r.v - (r.s - limit) / p.dt));
          r.s = limit;
        } else if (entered && !c.rs_reverted[j]) {
          rev = j;
          break;
        } else if (prev >= 0 && C[prev].lane != A[C[prev].src].lane && !c.rs_reverted[prev]) {
          rev = prev;
          break;
        } else {
          r.v = 0.0;
          r.s = floor_s;
        }
      }
      prev = j;
      prev_rear = r.s - p.L;
    }
  }
  rev = __shfl_sync(0xffffffffu, rev, 0);
  __syncwarp();
  return rev;
}

// State of one replay (a component, or everything in the sequential path).
struct Replay {
  int32_t zf;  // sharded: zone flags seen (1 = an own lane, 2 = an inexact lane)
  int32_t* heap;
  int32_t hn;
  int32_t reach;
  int32_t* moved;   // vehicles reverted so far (C indices)
  int32_t nmoved;
  int32_t* touched;  // lanes touched so far
  int32_t nt;
  int64_t reverts;
};

// Runs the min-heap replay until no pending lane reverts.  Lane 0 owns the
// bookkeeping; the whole warp calls.  The heap must hold the initial lanes.
__device__ void replay(const Ctx& c, VRec* C, const int32_t* CS, const VRec* A, Replay& R, RsM* m, RsM* tmp,
                       int64_t max_reverts) {
  const int lid = threadIdx.x & 31;
  for (;;) {
    int32_t L = -1;
    if (lid == 0) {
      while (R.hn > 0) {
        const int32_t x = heap_pop(R.heap, R.hn);
        if (!c.rs_inwork[x]) continue;
        c.rs_inwork[x] = 0;
        if (!c.rs_touched[x]) {
          c.rs_touched[x] = 1;
          R.touched[R.nt++] = x;
        }
        if (c.sharded) R.zf |= ((c.zone[x] & ZF_OWN) ? 1 : 0) | ((c.zone[x] & ZF_EXACT) ? 0 : 2);
        if (x > R.reach) R.reach = x;
        L = x;
        break;
      }
    }
    L = __shfl_sync(0xffffffffu, L, 0);
    if (L < 0) break;
    const int32_t nmoved = __shfl_sync(0xffffffffu, R.nmoved, 0);
    const int32_t rev = resolve_lane(c, C, CS, A, L, R.moved, nmoved, m, tmp);
    if (rev < 0) continue;
    // _revert (world.py:501-507) and rescheduling
    const VRec sn = A[C[rev].src];
    const int32_t Lb = sn.lane;
    int restore = 0, stop = 0;
    if (lid == 0) {
      R.reverts++;
      VRec& r = C[rev];
      r.lane = sn.lane;
      r.s = sn.s;
      r.v = 0.0;
      r.rptr = sn.rptr;
      c.rs_reverted[rev] = 1;
      R.moved[R.nmoved++] = rev;
      c.rs_movedin[Lb] = 1;
      atomicAdd(&c.cdelta[L], -1);  // membership change for the regroup
      atomicAdd(&c.cdelta[Lb], 1);
      if (!c.rs_touched[Lb]) {
        c.rs_touched[Lb] = 1;
        R.touched[R.nt++] = Lb;
        // the reference sweeps Lb for the first time only now, with the
        // reverted vehicle present: undo k_lanefix's tentative sweep
        restore = (Lb > R.reach && !c.rs_event[Lb]) ? 1 : 0;
      }
      if (!c.rs_inwork[L]) {
        c.rs_inwork[L] = 1;
        heap_push(R.heap, R.hn, L);
      }
      if (!c.rs_inwork[Lb]) {
        c.rs_inwork[Lb] = 1;
        heap_push(R.heap, R.hn, Lb);
      }
      stop = R.reverts >= max_reverts;  // the reference's pass bound (world.py:518)
    }
    restore = __shfl_sync(0xffffffffu, restore, 0);
    if (restore)
      for (int32_t j = CS[Lb] + lid; j < CS[Lb + 1]; j += 32) {
        const VRec o = c.B[C[j].src];
        C[j].s = o.s;
        C[j].v = o.v;
      }
    __syncwarp();
    if (__shfl_sync(0xffffffffu, stop, 0)) break;
  }
}

// Clears the per-lane replay flags of R's lanes and marks them dirty (their
// membership or order changed: the next snapshot rebuilds them).
__device__ void replay_finish(const Ctx& c, const Replay& R) {
  for (int32_t q = 0; q < R.nt; q++) {
    const int32_t L = R.touched[q];
    mark_dirty(c, L);
    c.rs_touched[L] = 0;
    c.rs_event[L] = 0;
    c.rs_movedin[L] = 0;
    c.rs_inwork[L] = 0;
  }
  for (int32_t q = 0; q < R.nmoved; q++) c.rs_reverted[R.moved[q]] = 0;
}

// In-place exclusive scan of a[0, n) (shared or global memory), n <= K *
// blockDim.x; returns the total.  Every thread of the block calls.
template <int K>
__device__ int32_t block_excl_scan(int32_t* a, int n) {
  __shared__ int32_t ws[32];
  const int t = threadIdx.x, lid = t & 31, w = t >> 5, nw = (blockDim.x + 31) >> 5;
  int32_t x[K];
  int32_t sum = 0;
#pragma unroll
  for (int k = 0; k < K; k++) {
    const int i = K * t + k;
    x[k] = i < n ? a[i] : 0;
    sum += x[k];
  }
  int32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lid >= o) incl += y;
  }
  if (lid == 31) ws[w] = incl;
  __syncthreads();
  if (w == 0) {
    int32_t v = lid < nw ? ws[lid] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, v, o);
      if (lid >= o) v += y;
    }
    ws[lid] = v;
  }
  __syncthreads();
  int32_t run = (w ? ws[w - 1] : 0) + incl - sum;
#pragma unroll
  for (int k = 0; k < K; k++) {
    const int i = K * t + k;
    if (i < n) a[i] = run;
    run += x[k];
  }
  const int32_t total = ws[nw - 1];
  __syncthreads();
  return total;
}
__device__ __forceinline__ int32_t block_excl_scan2(int32_t* a, int n) { return block_excl_scan<2>(a, n); }

// Closure of the event lanes under "entered member -> its snapshot lane",
// split into components (one CTA).  Output: dy->n_comp components, comp_off
// / comp_ev (event lanes per component), comp_size; or dy->complex = 1 when
// a budget is exceeded (then the sequential replay runs instead).
__global__ void __launch_bounds__(1024) k_resolve_closure(Ctx c) {
  PDL_WAIT();
  Dyn* dy = c.dyn;
  __shared__ int32_t cl[CL_CAP];
  __shared__ int32_t lab[CL_CAP];
  __shared__ int32_t eu[CE_CAP], ev[CE_CAP];
  __shared__ int32_t indeg[CL_CAP];
  __shared__ int32_t s_n, s_ne, s_over, s_changed;
  __shared__ int32_t s_done, s_events, s_ncl;
  // the step scalars, read once and shared: every thread takes the same branches
  if (threadIdx.x == 0) {
    s_done = dy->rf_done;
    s_events = dy->n_events;
    s_ncl = dy->n_cl;
  }
  __syncthreads();
  if (s_done) return;  // k_resolve_fast replayed the events (eager mode runs this section)
  const int32_t ne = s_events;
  // clear the previous step's closure marks
  for (int32_t q = threadIdx.x; q < s_ncl; q += blockDim.x) c.cl_idx[c.cl_lanes[q]] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    dy->n_cl = 0;
    dy->n_comp = 0;
    s_n = 0;
    s_ne = 0;
    s_over = (ne > CL_CAP) || (c.debug & 1);
  }
  __syncthreads();
  if (ne == 0 || s_over) {
    if (threadIdx.x == 0 && ne > 0) dy->complex = 1;
    return;
  }
  for (int32_t e = threadIdx.x; e < ne; e += blockDim.x) {
    const int32_t L = c.events[e];
    cl[e] = L;
    c.cl_idx[L] = e + 1;
    c.rs_event[L] = 1;
  }
  if (threadIdx.x == 0) s_n = ne;
  __syncthreads();
  const VRec* C = c.lay[dy->cur ^ 1];
  const int32_t* CS = c.start[dy->cur ^ 1];
  const VRec* A = c.lay[dy->cur];
  const int w = threadIdx.x >> 5, lid = threadIdx.x & 31, nw = blockDim.x >> 5;
  int32_t f_lo = 0, f_hi = ne;
  while (f_lo < f_hi) {
    for (int32_t i = f_lo + w; i < f_hi; i += nw) {
      const int32_t L = cl[i];
      for (int32_t j = CS[L] + lid; j < CS[L + 1]; j += 32) {
        const VRec r = C[j];
        const int32_t T = A[r.src].lane;
        if (T == L) continue;  // not entered
        const int32_t k = atomicAdd(&s_ne, 1);
        if (k < CE_CAP) {
          eu[k] = L;
          ev[k] = T;
        }
        if (atomicCAS(&c.cl_idx[T], 0, -1) == 0) {
          const int32_t x = atomicAdd(&s_n, 1);
          if (x < CL_CAP) {
            cl[x] = T;
            c.cl_idx[T] = x + 1;
          } else {
            c.cl_idx[T] = 0;
          }
        }
      }
    }
    __syncthreads();
    if (s_n > CL_CAP || s_ne > CE_CAP) break;
    f_lo = f_hi;
    f_hi = s_n;
    __syncthreads();
  }
  const int32_t n = min(s_n, CL_CAP), nedge = min(s_ne, CE_CAP);
  if (threadIdx.x == 0) s_over = s_n > CL_CAP || s_ne > CE_CAP;
  // record the closure for clearing (next step)
  for (int32_t q = threadIdx.x; q < n; q += blockDim.x) c.cl_lanes[q] = cl[q];
  if (threadIdx.x == 0) dy->n_cl = n;
  __syncthreads();
  if (s_over) {
    if (threadIdx.x == 0) dy->complex = 1;
    return;
  }
  // on-chip budget per lane: members now + vehicles that can be reverted into it
  for (int32_t i = threadIdx.x; i < n; i += blockDim.x) indeg[i] = 0;
  __syncthreads();
  for (int32_t k = threadIdx.x; k < nedge; k += blockDim.x) atomicAdd(&indeg[c.cl_idx[ev[k]] - 1], 1);
  __syncthreads();
  for (int32_t i = threadIdx.x; i < n; i += blockDim.x)
    if (CS[cl[i] + 1] - CS[cl[i]] + indeg[i] > RS_CAP) s_over = 1;
  __syncthreads();
  if (s_over) {
    if (threadIdx.x == 0) dy->complex = 1;
    return;
  }
  // connected components: min-label propagation with pointer jumping
  for (int32_t i = threadIdx.x; i < n; i += blockDim.x) lab[i] = i;
  __syncthreads();
  for (;;) {
    if (threadIdx.x == 0) s_changed = 0;
    __syncthreads();
    for (int32_t k = threadIdx.x; k < nedge; k += blockDim.x) {
      const int32_t a = c.cl_idx[eu[k]] - 1, b = c.cl_idx[ev[k]] - 1;
      const int32_t la = lab[a], lb = lab[b];
      if (la != lb) {
        const int32_t mn = min(la, lb);
        atomicMin(&lab[a], mn);
        atomicMin(&lab[b], mn);
        atomicMin(&lab[la], mn);
        atomicMin(&lab[lb], mn);
        s_changed = 1;
      }
    }
    __syncthreads();
    // pointer jumping in two phases (walk, then publish): no thread writes a
    // label another thread may be walking through
    for (int32_t i = threadIdx.x; i < n; i += blockDim.x) {
      int32_t x = lab[i];
      while (lab[x] != x) x = lab[x];
      indeg[i] = x;
    }
    __syncthreads();
    for (int32_t i = threadIdx.x; i < n; i += blockDim.x) lab[i] = indeg[i];
    __syncthreads();
    if (!s_changed) break;
    __syncthreads();
  }
  // component ids (roots in index order), sizes, events per component
  for (int32_t i = threadIdx.x; i < n; i += blockDim.x) indeg[i] = lab[i] == i ? 1 : 0;
  __syncthreads();
  const int32_t nc = block_excl_scan2(indeg, n);  // indeg[root] = component id
  for (int32_t i = threadIdx.x; i < n; i += blockDim.x) c.comp_id[i] = indeg[lab[i]];
  for (int32_t k = threadIdx.x; k <= nc; k += blockDim.x) {
    c.comp_size[k] = 0;
    c.comp_edges[k] = 0;
    c.comp_off[k] = 0;
  }
  __syncthreads();
  for (int32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int32_t k = c.comp_id[i];
    atomicAdd(&c.comp_size[k], 1);
    if (i < ne) atomicAdd(&c.comp_off[k], 1);
  }
  for (int32_t e = threadIdx.x; e < nedge; e += blockDim.x)
    atomicAdd(&c.comp_edges[c.comp_id[c.cl_idx[eu[e]] - 1]], 1);
  __syncthreads();
  // event offsets per component (scan in shared memory; eu is free now)
  for (int32_t k = threadIdx.x; k < nc; k += blockDim.x) {
    eu[k] = c.comp_off[k];
    // heap / touched lists hold distinct lanes; each revert moves a
    // distinct entered member (an edge)
    if (c.comp_size[k] > HCAP || c.comp_edges[k] > 2 * HCAP) s_over = 1;
  }
  __syncthreads();
  const int32_t tot_ev = block_excl_scan2(eu, nc);
  for (int32_t k = threadIdx.x; k < nc; k += blockDim.x) {
    c.comp_off[k] = eu[k];
    c.comp_fill[k] = eu[k];
  }
  if (threadIdx.x == 0) c.comp_off[nc] = tot_ev;
  __syncthreads();
  if (s_over) {
    if (threadIdx.x == 0) dy->complex = 1;
    return;
  }
  for (int32_t i = threadIdx.x; i < ne; i += blockDim.x) {
    const int32_t k = c.comp_id[i];
    c.comp_ev[atomicAdd(&c.comp_fill[k], 1)] = cl[i];
  }
  if (c.sharded) {
    // a chain that can change an own lane must stay inside lanes this rank
    // computes exactly (shard.py); otherwise fail loudly
    for (int32_t k = threadIdx.x; k < nc; k += blockDim.x) c.comp_flags[k] = 0;
    __syncthreads();
    for (int32_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint8_t z = c.zone[cl[i]];
      const int32_t k = c.comp_id[i];
      if (z & ZF_OWN) atomicOr(&c.comp_flags[k], 1);
      if (!(z & ZF_EXACT)) atomicOr(&c.comp_flags[k], 2);
    }
    __syncthreads();
    for (int32_t k = threadIdx.x; k < nc; k += blockDim.x)
      if (c.comp_flags[k] == 3) dy->overflow |= 16;
  }
  if (threadIdx.x == 0) dy->n_comp = nc;
}

// One warp per component: the replay restricted to the component's lanes.
static constexpr int RC_WARPS = 2;

// The common-step body of the step graph only patches the snapshot: when the
// lanes changed after the sweep exceed what the patch handles, the step must
// take the RARE body (which can run the full regroup).
static constexpr int PATCH_MAX = 4096;  // dirty lanes (and moved vehicles) the patch handles
__device__ void rare_if_unpatchable(const Ctx& c) {
  const Dyn* dy = c.dyn;
  if (dy->n_dirty > PATCH_MAX || dy->n_moved > PATCH_MAX || (c.debug & 2)) set_rare(c);
}

// Fast-path replay on chip.  Every vehicle that can be on a closure lane
// during the replay is a member of some closure lane's C segment (a revert
// only moves a vehicle back to its snapshot lane, which is in the closure),
// so the warp stages all of them once, during the closure search, and the
// replay reads and updates the staged copy; rf_writeback copies the result
// to C once the closures are known to be disjoint (the lanes are then this
// warp's alone).  Same algorithm, same arithmetic as replay() /
// resolve_lane().
static constexpr int RF_CACHE = 192;
struct RfE {
  double s, v, snap_s;
  int32_t j, vix, lane, snap_lane, snap_rptr, src;
  int32_t reverted, rev_from;
};
struct RfSmem {
  union {
    struct {
      RsM m[RS_CAP];
      RsM t[RS_CAP];
    } g;  // global-gather replay (closure larger than the cache)
    struct {
      RfE e[RF_CACHE];
      int16_t i1[RF_CACHE], i2[RF_CACHE];
    } k;
  };
};

// resolve_lane() on the staged members (results stay staged); returns the
// cache index of the vehicle to revert, or -1 (same value in every thread).
__device__ int32_t resolve_lane_cached(const Ctx& c, VRec* C, int32_t L, RfE* E, int32_t ncache, int16_t* i1,
                                       int16_t* i2) {
  const int lid = threadIdx.x & 31;
  const Params& p = c.p;
  int n = 0;
  for (int32_t base = 0; base < ncache; base += 32) {
    const int32_t k = base + lid;
    const bool mine = k < ncache && E[k].lane == L;
    const unsigned b = __ballot_sync(0xffffffffu, mine);
    if (mine) i1[n + __popc(b & ((1u << lid) - 1))] = (int16_t)k;
    n += __popc(b);
  }
  __syncwarp();
  for (int a = lid; a < n; a += 32) {
    const RfE& x = E[i1[a]];
    int rank = 0;
    for (int b2 = 0; b2 < n; b2++) rank += ahead_of(E[i1[b2]].s, E[i1[b2]].vix, x.s, x.vix) ? 1 : 0;
    i2[rank] = i1[a];
  }
  __syncwarp();
  // the sweep changes nothing before its first trigger: find it in
  // parallel, then run the sequential sweep from there (same arithmetic)
  int first = n;
  for (int a = lid; a < n; a += 32)
    if (a > 0 && E[i2[a]].s > ((E[i2[a - 1]].s - p.L) - p.s0_floor) + 1e-12) first = min(first, a);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
  int32_t rev = -1;
  if (lid == 0 && first < n) {
    int prev = first - 1;
    double prev_rear = E[i2[prev]].s - p.L;
    for (int a = first; a < n; a++) {
      RfE& x = E[i2[a]];
      const double limit = prev_rear - p.s0_floor;
      const bool entered = x.snap_lane != L;
      if (x.s > limit + 1e-12) {
        const double floor_s = entered ? 0.0 : x.snap_s;
        if (limit >= floor_s) {
          x.v = py_max(0.0, py_min(x.v, x.v - (x.s - limit) / p.dt));
          x.s = limit;
        } else if (entered && !x.reverted) {
          rev = i2[a];
          break;
        } else if (prev >= 0 && E[i2[prev]].snap_lane != L && !E[i2[prev]].reverted) {
          rev = i2[prev];
          break;
        } else {
          x.v = 0.0;
          x.s = floor_s;
        }
      }
      prev = a;
      prev_rear = x.s - p.L;
    }
  }
  rev = __shfl_sync(0xffffffffu, rev, 0);
  __syncwarp();
  return rev;
}

// replay() on the staged members, with the per-lane replay flags on chip
// too (closure lanes q[0, qn), flags fl[]; E = the one event lane).  Nothing
// outside shared memory is written: the replay runs before the launch's
// warps know whether their closures met, and rf_writeback publishes it.
enum : uint8_t { RF_INWORK = 1, RF_TOUCHED = 2 };
__device__ void replay_cached(const Ctx& c, VRec* C, const int32_t* CS, Replay& R, RfE* E, int32_t ncache,
                              int16_t* i1, int16_t* i2, const int32_t* q, uint8_t* fl, int32_t ev_lane,
                              int64_t max_reverts) {
  const int lid = threadIdx.x & 31;
  auto qi = [&](int32_t x) {
    int k = 0;
    while (q[k] != x) k++;
    return k;
  };
  for (;;) {
    int32_t L = -1;
    if (lid == 0) {
      while (R.hn > 0) {
        const int32_t x = heap_pop(R.heap, R.hn);
        uint8_t& f = fl[qi(x)];
        if (!(f & RF_INWORK)) continue;
        f &= ~RF_INWORK;
        if (!(f & RF_TOUCHED)) {
          f |= RF_TOUCHED;
          R.touched[R.nt++] = x;
        }
        if (c.sharded) R.zf |= ((c.zone[x] & ZF_OWN) ? 1 : 0) | ((c.zone[x] & ZF_EXACT) ? 0 : 2);
        if (x > R.reach) R.reach = x;
        L = x;
        break;
      }
    }
    L = __shfl_sync(0xffffffffu, L, 0);
    if (L < 0) break;
    const int32_t rk = resolve_lane_cached(c, C, L, E, ncache, i1, i2);
    if (rk < 0) continue;
    // _revert (world.py:501-507) and rescheduling
    const int32_t Lb = E[rk].snap_lane;
    int restore = 0, stop = 0;
    if (lid == 0) {
      R.reverts++;
      RfE& x = E[rk];
      x.lane = Lb;
      x.s = x.snap_s;
      x.v = 0.0;
      x.reverted = 1;
      x.rev_from = L;  // membership change for the regroup, applied by rf_writeback
      R.moved[R.nmoved++] = x.j;
      uint8_t& fb = fl[qi(Lb)];
      if (!(fb & RF_TOUCHED)) {
        fb |= RF_TOUCHED;
        R.touched[R.nt++] = Lb;
        // the reference sweeps Lb for the first time only now, with the
        // reverted vehicle present: undo k_lanefix's tentative sweep
        restore = (Lb > R.reach && Lb != ev_lane) ? 1 : 0;
      }
      uint8_t& fa = fl[qi(L)];
      if (!(fa & RF_INWORK)) {
        fa |= RF_INWORK;
        heap_push(R.heap, R.hn, L);
      }
      if (!(fb & RF_INWORK)) {
        fb |= RF_INWORK;
        heap_push(R.heap, R.hn, Lb);
      }
      stop = R.reverts >= max_reverts;  // the reference's pass bound (world.py:518)
    }
    restore = __shfl_sync(0xffffffffu, restore, 0);
    __syncwarp();
    if (restore) {
      // Lb's C segment members: the staged entries whose C index lies in it
      const int32_t lo = CS[Lb], hi = CS[Lb + 1];
      for (int32_t k = lid; k < ncache; k += 32) {
        RfE& x = E[k];
        if (x.j >= lo && x.j < hi) {
          const VRec o = c.B[x.src];
          x.s = o.s;
          x.v = o.v;
        }
      }
    }
    __syncwarp();
    if (__shfl_sync(0xffffffffu, stop, 0)) break;
  }
}

// Publishes a staged replay: every staged member's state to C (reverted ones
// with their snapshot lane and route position) and the lane membership
// deltas of the reverts.
__device__ void rf_writeback(const Ctx& c, VRec* C, const RfE* E, int32_t ncache) {
  const int lid = threadIdx.x & 31;
  for (int32_t k = lid; k < ncache; k += 32) {
    const RfE& x = E[k];
    VRec& r = C[x.j];
    r.s = x.s;
    r.v = x.v;
    if (x.reverted) {
      r.lane = x.lane;
      r.rptr = x.snap_rptr;
      atomicAdd(&c.cdelta[x.rev_from], -1);
      atomicAdd(&c.cdelta[x.lane], 1);
    }
  }
  __syncwarp();
}

// The common case without the closure kernel: every event's closure is
// computed by its own warp (breadth-first over "entered member -> its
// snapshot lane", as k_resolve_closure), lanes are claimed in rf_owner
// (epoch-tagged: no clearing), and if no two closures meet and each fits the
// component budgets, each event is a component of its own and its warp
// replays it at once.  Otherwise nothing was modified except the claims and
// the general path (closure, components, sequential fallback) runs in the
// RARE body of the step graph.  The warps of one launch wait for each other once
// (all co-resident: at most RF_BLOCKS small blocks).
static constexpr int RF_BLOCKS = 64;
static constexpr int32_t RF_ABORT = 1 << 30;                // k_resolve_fast arrival word: wait aborted
static constexpr unsigned long long RF_WAIT_NS = 2000000ULL;  // 2 ms (the wait takes microseconds)
__global__ void __launch_bounds__(32 * RC_WARPS) k_resolve_fast(Ctx c) {
  PDL_WAIT();
  TL_MARK(TL_RESOLVE);
  TlEnd tl_end{c, TL_RESOLVE_END};
  Dyn* dy = c.dyn;
  const int32_t ne = dy->n_events;
  if (ne == 0) {
    if (gtid() == 0) rare_if_unpatchable(c);
    return;
  }
  if (ne > RF_BLOCKS * RC_WARPS || (c.debug & 5)) {  // debug bit 0: sequential, bit 2: general path
    if (gtid() == 0) {
      set_rare(c);
      dy->n_resolve_general++;
    }
    return;
  }
  const int w = threadIdx.x >> 5, lid = threadIdx.x & 31;
  const int32_t ev = blockIdx.x * RC_WARPS + w;
  if (ev >= ne) return;
  __shared__ RfSmem U[RC_WARPS];
  __shared__ int32_t sh[RC_WARPS][HCAP], smv[RC_WARPS][2 * HCAP], stl[RC_WARPS][HCAP], sq[RC_WARPS][HCAP];
  __shared__ uint8_t sfl[RC_WARPS][HCAP];
  __shared__ int32_t s_bad[RC_WARPS];
  VRec* C = c.lay[dy->cur ^ 1];
  const int32_t* CS = c.start[dy->cur ^ 1];
  const VRec* A = c.lay[dy->cur];
  const unsigned long long mine = ((unsigned long long)(uint32_t)(dy->step_no + 1) << 32) | (uint32_t)(ev + 1);
  const unsigned long long epoch = mine >> 32;
  int32_t* q = sq[w];  // closure lanes
  // claim lane T for this closure: 1 new, 0 already ours, -1 another closure's
  auto claim = [&](int32_t T) -> int {
    unsigned long long old = c.rf_owner[T];
    for (;;) {
      if ((old >> 32) == epoch) return old == mine ? 0 : -1;
      const unsigned long long got = atomicCAS(c.rf_owner + T, old, mine);
      if (got == old) return 1;
      old = got;
    }
  };
#ifdef TSB_RF_TRACE
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#endif
  const int32_t E = c.events[ev];
  int32_t qn = 1, nedge = 0, ncache = 0;  // ncache > RF_CACHE: not staged (global replay)
  RfE* cache = U[w].k.e;
  bool bad = false;
  if (lid == 0) q[0] = E;
  __syncwarp();
  // breadth-first over the closure with a local visited list; the lanes are
  // claimed afterwards, all at once (one atomic round trip, not one per lane)
  for (int32_t h = 0; h < qn && !bad; h++) {
    const int32_t L = q[h];
    const int32_t j0 = CS[L], j1 = CS[L + 1];
    for (int32_t b0 = j0; b0 < j1; b0 += 32) {
      const int32_t j = b0 + lid;
      int32_t T = L;
      VRec r, sn;
      if (j < j1) {
        r = C[j];
        sn = A[r.src];
        T = sn.lane;
      }
      // stage the member for the replay
      const unsigned vm = __ballot_sync(0xffffffffu, j < j1);
      const int slot = ncache + __popc(vm & ((1u << lid) - 1));
      if (j < j1 && slot < RF_CACHE)
        cache[slot] = RfE{r.s, r.v, sn.s, j, r.vix, L, sn.lane, sn.rptr, r.src, 0, -1};
      ncache += __popc(vm);
      const bool entered = T != L;
      const unsigned em = __ballot_sync(0xffffffffu, entered);
      nedge += __popc(em);
      // new origin lanes: one representative per distinct lane, not yet listed
      bool fresh = false;
      if (entered) {
        const unsigned grp = __match_any_sync(em, T);
        fresh = lid == __ffs(grp) - 1;
        for (int32_t k = 0; k < qn && fresh; k++)
          if (q[k] == T) fresh = false;
      }
      const unsigned nm = __ballot_sync(0xffffffffu, fresh);
      if (qn + __popc(nm) > HCAP) {
        bad = true;
      } else if (fresh) {
        q[qn + __popc(nm & ((1u << lid) - 1))] = T;
      }
      __syncwarp();
      qn += __popc(nm);
      if (qn > HCAP) qn = HCAP;
    }
    // on-chip budget: a lane's members plus every edge of the closure (a
    // bound on the vehicles that can be reverted into it)
    if (j1 - j0 + nedge > RS_CAP || nedge > 2 * HCAP) bad = true;
    __syncwarp();
  }
  // the budget check above used the edges found so far; recheck with all
  if (!bad)
    for (int32_t h = 0; h < qn; h++)
      if (CS[q[h] + 1] - CS[q[h]] + nedge > RS_CAP) bad = true;
  // claim the closure: a lane another closure claimed first means they meet
  if (!bad) {
    bool lost = false;
    for (int32_t k = lid; k < qn; k += 32) lost |= claim(q[k]) < 0;
    if (__any_sync(0xffffffffu, lost)) bad = true;
  }
#ifdef TSB_RF_TRACE
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
#endif
  // a staged closure is replayed at once, on chip, while the other warps
  // are still searching: it is published only if no closures met
  Replay R{0, sh[w], 0, -1, smv[w], 0, stl[w], 0, 0};
  const bool staged = ncache <= RF_CACHE;
  if (!bad && staged) {
    if (lid == 0) {
      for (int k = 0; k < qn; k++) sfl[w][k] = 0;
      sfl[w][0] = RF_INWORK;  // q[0] == E
      heap_push(R.heap, R.hn, E);
    }
    __syncwarp();
    replay_cached(c, C, CS, R, cache, ncache, U[w].k.i1, U[w].k.i2, q, sfl[w], E, (int64_t)dy->n_c + 2);
  }
#ifdef TSB_RF_TRACE
  unsigned long long t2;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
#endif
  if (lid == 0) {
    // Launch-wide wait, bounded: the launch is not cooperative, so its blocks
    // are co-resident only in practice (a shared or MPS-partitioned GPU may
    // delay some).  A warp that waits longer than RF_WAIT_NS aborts the fast
    // path for the whole launch by setting RF_ABORT in the arrival word, but
    // only while the count is short of ne (a CAS on the observed word): the
    // warps either all see every arrival without the bit (fast path) or all
    // see the bit (general path).  Nothing global was modified before this
    // point except the epoch-tagged lane claims.
    if (bad) atomicExch(&dy->rf_conflict, 1);
    __threadfence();
    int32_t a = atomicAdd(&dy->rf_arrive, 1) + 1;
    unsigned long long t_start;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    while (!(a & RF_ABORT) && a < ne) {
      __nanosleep(64);
      a = atomicAdd(&dy->rf_arrive, 0);
      if (a & RF_ABORT || a >= ne) break;
      unsigned long long t_now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_now));
      if (t_now - t_start > RF_WAIT_NS) a = atomicCAS(&dy->rf_arrive, a, a | RF_ABORT) == a ? (a | RF_ABORT) : a;
    }
    __threadfence();
    s_bad[w] = (a & RF_ABORT) ? 1 : atomicAdd(&dy->rf_conflict, 0);
  }
  __syncwarp();
  if (s_bad[w]) {
    if (ev == 0 && lid == 0) {
      set_rare(c);
      dy->n_resolve_general++;
    }
    return;
  }
  if (ev == 0 && lid == 0) {
    dy->rf_done = 1;  // read by the general path's kernels in eager mode
    dy->n_resolve_fast++;
  }
  if (staged) {
    rf_writeback(c, C, cache, ncache);
  } else {
    if (lid == 0) {
      c.rs_event[E] = 1;
      c.rs_inwork[E] = 1;
      heap_push(R.heap, R.hn, E);
    }
    __syncwarp();
    replay(c, C, CS, A, R, U[w].g.m, U[w].g.t, (int64_t)dy->n_c + 2);
  }
#ifdef TSB_RF_TRACE
  unsigned long long t3;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t3));
  if (lid == 0)
    printf("RF step %lld ev %d/%d E %d qn %d edges %d lanes_touched %d reverts %lld bfs %llu replay %llu wait+publish %llu ns\n",
           (long long)dy->step_no, ev, ne, E, qn, nedge, R.nt, (long long)R.reverts, t1 - t0, t2 - t1, t3 - t2);
#endif
  // publish the bookkeeping with the whole warp: the touched lanes' dirty
  // marks and the moved list in parallel (lane 0's serial atomics were a
  // chain of dependent round trips)
  const int32_t nt = __shfl_sync(0xffffffffu, R.nt, 0);
  const int32_t nmv = __shfl_sync(0xffffffffu, R.nmoved, 0);
  if (staged) {
    for (int32_t k = lid; k < nt; k += 32) mark_dirty(c, R.touched[k]);  // no global flags to clear
  } else if (lid == 0) {
    replay_finish(c, R);
  }
  int32_t base = 0;
  if (lid == 0) {
    if (c.sharded && R.zf == 3) dy->overflow |= 16;
    base = atomicAdd(&dy->n_moved, R.nmoved);
    atomicAdd((unsigned long long*)&dy->reverts_last, (unsigned long long)R.reverts);
  }
  base = __shfl_sync(0xffffffffu, base, 0);
  for (int32_t k = lid; k < nmv; k += 32) c.rs_moved[base + k] = R.moved[k];
  __threadfence();  // every lane's writes before the warp's arrival below
  __syncwarp();
  if (lid == 0) {
    // the last replay to finish sees the final dirty / moved counts
    if (atomicAdd(&dy->rf_fin, 1) == ne - 1) {
      __threadfence();
      rare_if_unpatchable(c);
    }
  }
}
__global__ void __launch_bounds__(32 * RC_WARPS) k_resolve_comp(Ctx c) {
  PDL_WAIT();
  Dyn* dy = c.dyn;
  const int32_t nc = dy->n_comp;
  if (nc == 0 || dy->complex || dy->rf_done) return;
  __shared__ RsM sm[RC_WARPS][RS_CAP];
  __shared__ RsM st[RC_WARPS][RS_CAP];
  __shared__ int32_t sh[RC_WARPS][HCAP], smv[RC_WARPS][2 * HCAP], stl[RC_WARPS][HCAP];
  const int w = threadIdx.x >> 5, lid = threadIdx.x & 31;
  VRec* C = c.lay[dy->cur ^ 1];
  const int32_t* CS = c.start[dy->cur ^ 1];
  const VRec* A = c.lay[dy->cur];
  const int64_t max_reverts = (int64_t)dy->n_c + 2;
  for (int32_t k = blockIdx.x * RC_WARPS + w; k < nc; k += gridDim.x * RC_WARPS) {
    Replay R{0, sh[w], 0, -1, smv[w], 0, stl[w], 0, 0};
    if (lid == 0)
      for (int32_t q = c.comp_off[k]; q < c.comp_off[k + 1]; q++) {
        const int32_t L = c.comp_ev[q];
        c.rs_inwork[L] = 1;
        heap_push(R.heap, R.hn, L);
      }
    __syncwarp();
    // heap / touched <= HCAP lanes and moved <= 2 * HCAP vehicles
    // (component budgets checked by k_resolve_closure)
    replay(c, C, CS, A, R, sm[w], st[w], max_reverts);
    if (lid == 0) {
      replay_finish(c, R);
      const int32_t base = atomicAdd(&dy->n_moved, R.nmoved);
      for (int32_t q = 0; q < R.nmoved; q++) c.rs_moved[base + q] = R.moved[q];
      atomicAdd((unsigned long long*)&dy->reverts_last, (unsigned long long)R.reverts);
    }
    __syncwarp();
  }
}

// Sequential replay of all events (fallback when the closure exceeds the
// component budgets, or forced by the debug knob).
__global__ void __launch_bounds__(32) k_resolve(Ctx c) {
  PDL_WAIT();
  Dyn* dy = c.dyn;
  const int32_t ne = dy->n_events;
  if (ne == 0 || !dy->complex) return;
  __shared__ RsM m[RS_CAP];
  __shared__ RsM tmp[RS_CAP];
  const int lid = threadIdx.x;
  VRec* C = c.lay[dy->cur ^ 1];
  const int32_t* CS = c.start[dy->cur ^ 1];
  const VRec* A = c.lay[dy->cur];
  Replay R{0, c.rs_heap, 0, -1, c.rs_moved, 0, c.rs_touched_list, 0, 0};
  if (lid == 0) {
    dy->n_moved = 0;
    dy->reverts_last = 0;
    for (int32_t e = 0; e < ne; e++) {
      const int32_t L = c.events[e];
      c.rs_event[L] = 1;
      c.rs_inwork[L] = 1;
      heap_push(R.heap, R.hn, L);
    }
  }
  __syncwarp();
  replay(c, C, CS, A, R, m, tmp, (int64_t)dy->n_c + 2);
  if (lid == 0) {
    replay_finish(c, R);
    for (int32_t e = 0; e < ne; e++) {
      c.rs_event[c.events[e]] = 0;
      c.rs_inwork[c.events[e]] = 0;
    }
    dy->n_moved = R.nmoved;
    dy->reverts_last = R.reverts;
    dy->resolve_sequential += 1;
    // conservative in sharded mode (no component split here): an own lane and
    // an inexact lane in the same replay
    if (c.sharded && R.zf == 3) dy->overflow |= 16;
  }
}

// ------------------------------------------------------------------ signals + clock

// Lane occupancy after the sweep (max-pressure input, world.py:634-637).
__global__ void k_lane_counts(Ctx c) {
  PDL_WAIT();
  Dyn* dy = c.dyn;
  const VRec* C = c.lay[dy->cur ^ 1];
  const int32_t n = dy->n_c;
  for (int32_t i = gtid(); i < n; i += gstride()) atomicAdd(&c.lane_counts[C[i].lane], 1);
}

// world.py:619-647 (+ time/step increment, world.py:677-678).
// mode SIG_FULL: both, after the step's sweep.  A sharded max-pressure engine
// splits them: SIG_CLOCK after the sweep, SIG_DEFERRED at the start of the
// next step, once the exchange brought the owners' post-sweep counts of the
// pressure lanes (shard.pressure_lanes) -- the same decisions from the same
// counts, taken before anything reads the new states (the next update).
enum { SIG_FULL = 0, SIG_CLOCK = 1, SIG_DEFERRED = 2 };
__global__ void k_signals(Ctx c, int mode) {
  PDL_WAIT();
  TL_MARK(TL_SIGNALS);
  const Params& p = c.p;
  if (mode == SIG_DEFERRED && c.dyn->step_no == 0) return;  // no step has swept yet
  for (int32_t j = (mode == SIG_CLOCK ? c.n_junc : gtid()); j < c.n_junc; j += gstride()) {
    if (!c.junc_signal[j]) continue;
    JuncState st = c.sig[j];
    const int32_t b = c.junc_phase_off[j], np_ = c.junc_phase_off[j + 1] - b;
    if (p.controller == 0) {
      st.elapsed += p.dt;  // signals.advance_fixed (signals.py:37-43)
      while (st.elapsed >= c.phase_dur[b + st.phase]) {
        st.elapsed -= c.phase_dur[b + st.phase];
        st.phase = (st.phase + 1) % np_;
      }
    } else {
      st.elapsed += p.dt;
      st.since += p.dt;
      if (!(st.since < p.mp_interval || st.elapsed < p.mp_min_green)) {
        int32_t best = 0;
        long long best_p = 0;
        bool have = false;
        for (int32_t ph = 0; ph < np_; ph++) {  // signals.py:64-86
          long long pr = 0;
          for (int32_t q = c.jc_off[j]; q < c.jc_off[j + 1]; q++) {
            int32_t cn = c.jc[q];
            if ((c.green[cn] >> ph) & 1ULL) {
              const LaneRec LR = c.lanes[cn];
              if (LR.pred1 >= 0 && LR.succ1 >= 0)  // (a sharded rank's junction it never reads may be partial)
                pr += (long long)c.lane_counts[LR.pred1] - (long long)c.lane_counts[LR.succ1];
            }
          }
          if (!have || pr > best_p) {
            have = true;
            best_p = pr;
            best = ph;
          }
        }
        if (best != st.phase) {
          st.phase = best;
          st.elapsed = 0.0;
        }
        st.since = 0.0;
      }
    }
    c.sig[j] = st;
  }
  if (gtid() == 0 && mode != SIG_DEFERRED) {  // world.py:677-678 (nothing in this kernel reads the clock)
    c.dyn->time += p.dt;
    c.dyn->step_no += 1;
  }
}

// Connector flag bytes from the new junction states (thread per connector).
__global__ void k_conn_flags(Ctx c) {
  PDL_WAIT();
  for (int32_t q = gtid(); q < c.n_conn; q += gstride()) {
    const int32_t cn = c.jc[q], j = c.jc_junc[q];
    uint8_t f = c.lflag[cn] & LF_OPEN;
    if (c.jc_succ1[q] >= 0 && (c.lflag[c.jc_succ1[q]] & LF_OPEN)) f |= LF_SUCC_OPEN;
    f |= (uint8_t)(aspect_of(c, j, cn, c.sig[j]) << LF_ASPECT_SHIFT);
    c.lflag[cn] = f;
  }
}


// ------------------------------------------------------------------ injection (world.py:561-617)

// Build the due list: retry (in due order) ++ pending with departure <= time.
__global__ void k_inject_due(Ctx c) {
  PDL_WAIT();
  TL_MARK(TL_INJECT_DUE);
  TlEnd tl_end{c, TL_INJECT_DUE_END};
  Dyn* dy = c.dyn;
  __shared__ int32_t s_new;
  const int32_t nr = dy->n_retry;
  if (threadIdx.x == 0) {
    const int32_t lo = dy->pend_ptr;
    int32_t a = lo, b = c.n_pend;
    const double t = dy->time;
    while (a < b) {  // pending departures are non-decreasing
      int32_t m = (a + b) >> 1;
      if (c.pend_dep[m] <= t)
        a = m + 1;
      else
        b = m;
    }
    s_new = a - lo;
  }
  __syncthreads();
  const int32_t nn = s_new, lo = dy->pend_ptr;
  for (int32_t k = threadIdx.x; k < nr; k += blockDim.x) c.due[k] = c.retry[k];
  for (int32_t k = threadIdx.x; k < nn; k += blockDim.x) c.due[nr + k] = c.pend_vix[lo + k];
  __syncthreads();
  if (threadIdx.x == 0) {
    dy->pend_ptr = lo + nn;
    dy->n_due = nr + nn;
    dy->n_retry = 0;
    dy->injected_now = 0;
    if (nr + nn > 0) set_rare(c);
    if (nr + nn > 0) dy->n_inject_steps++;
  }
}

__global__ void k_inject_hist(Ctx c) {
  PDL_WAIT();
  Dyn* dy = c.dyn;
  for (int32_t k = gtid(); k < dy->n_due; k += gstride()) atomicAdd(&c.inj_cnt[c.cold[c.due[k]].origin_lane], 1);
}

__global__ void k_inject_scatter(Ctx c) {
  PDL_WAIT();
  Dyn* dy = c.dyn;
  for (int32_t k = gtid(); k < dy->n_due; k += gstride()) {
    int32_t o = c.cold[c.due[k]].origin_lane;
    int32_t pos = c.inj_start[o] + atomicAdd(&c.inj_cursor[o], 1);
    c.due_grp[pos] = k;  // due position; sorted per lane below
  }
}

// One thread per origin lane: candidates in due order, gap tests against the
// lane's current occupants and the vehicles injected before them.
__global__ void k_inject_lanes(Ctx c) {
  PDL_WAIT();
  Dyn* dy = c.dyn;
  if (dy->n_due == 0) return;
  const Params& p = c.p;
  VRec* C = c.lay[dy->cur ^ 1];
  const int32_t* CS = c.start[dy->cur ^ 1];
  const int32_t nmoved = dy->n_moved;
  for (int32_t L = gtid(); L < c.n_lanes; L += gstride()) {
    const int32_t lo = c.inj_start[L], hi = c.inj_start[L + 1];
    if (hi == lo) continue;
    c.inj_cnt[L] = 0;  // consumed: zero for the next injection (no memsets)
    c.inj_cursor[L] = 0;
    // insertion sort of due positions
    for (int32_t a = lo + 1; a < hi; a++) {
      int32_t x = c.due_grp[a], b = a - 1;
      while (b >= lo && c.due_grp[b] > x) {
        c.due_grp[b + 1] = c.due_grp[b];
        b--;
      }
      c.due_grp[b + 1] = x;
    }
    const bool lane_open = c.lflag[L] & LF_OPEN;
    for (int32_t q = lo; q < hi; q++) {
      const int32_t dpos = c.due_grp[q];
      const int32_t vx = c.due[dpos];
      const VCold cd = c.cold[vx];
      uint8_t outc;
      if (!c.routed[vx] && !lane_open) {
        outc = OUT_RETRY;
      } else if (!c.routed[vx] && cd.route_len <= 0) {
        outc = OUT_DROP;
        c.status[vx] = TSB_STATUS_DROPPED;
        atomicAdd((unsigned long long*)&dy->dropped, 1ULL);
      } else {
        c.routed[vx] = 1;
        const double o_s = cd.origin_s;
        bool have_f = false, have_r = false;
        double fs = 0.0, rs = 0.0;
        auto consider = [&](double s) {
          if (s >= o_s) {
            if (!have_f || s < fs) {
              fs = s;
              have_f = true;
            }
          } else if (!have_r || s > rs) {
            rs = s;
            have_r = true;
          }
        };
        for (int32_t j = CS[L]; j < CS[L + 1]; j++)
          if (C[j].lane == L) consider(C[j].s);
        for (int32_t q2 = 0; q2 < nmoved; q2++) {
          const int32_t j = c.rs_moved[q2];
          if (C[j].lane == L && (j < CS[L] || j >= CS[L + 1])) consider(C[j].s);
        }
        for (int32_t r = lo; r < q; r++)
          if (c.outcome[c.due_grp[r]] == OUT_INJECT) consider(c.cold[c.due[c.due_grp[r]]].origin_s);
        const double front_gap = have_f ? (fs - p.L) - o_s : CUDART_INF;
        const double rear_gap = have_r ? (o_s - p.L) - rs : CUDART_INF;
        if (front_gap < p.s0 + p.L || rear_gap < p.s0) {
          outc = OUT_RETRY;
        } else {
          outc = OUT_INJECT;
          int32_t k = atomicAdd(&dy->n_inj, 1);
          VRec nr_{o_s, 0.0, vx, (int32_t)cd.route_off, L, -1};
          C[dy->n_c + k] = nr_;
          c.status[vx] = TSB_STATUS_DRIVING;
          atomicAdd(&c.cdelta[L], 1);
          mark_dirty(c, L);
        }
      }
      c.outcome[dpos] = outc;
    }
  }
}

__global__ void k_retry_flags(Ctx c) {
  PDL_WAIT();
  Dyn* dy = c.dyn;
  for (int32_t k = gtid(); k < dy->n_due; k += gstride()) c.flag_in[k] = c.outcome[k] == OUT_RETRY ? 1 : 0;
}

__global__ void k_retry_compact(Ctx c) {
  PDL_WAIT();
  Dyn* dy = c.dyn;
  const int32_t n = dy->n_due;
  for (int32_t k = gtid(); k < n; k += gstride()) {
    if (c.outcome[k] == OUT_RETRY) c.retry[c.flag_scan[k]] = c.due[k];
    c.outcome[k] = OUT_NONE;
  }
}

__global__ void k_inject_finish(Ctx c) {
  PDL_WAIT();
  Dyn* dy = c.dyn;
  if (dy->n_due > 0) dy->n_retry = c.flag_scan[dy->n_due];
  dy->injected_now = dy->n_inj;
}

// ------------------------------------------------------------------ incremental regroup


// Members of dirty lane L in the post-sweep layout C: segment entries still on
// L, vehicles reverted into L, vehicles injected into L (C tail).
template <class F>
__device__ void for_members(const Ctx& c, const VRec* C, const int32_t* CS, int32_t L, F f) {
  const Dyn* dy = c.dyn;
  const int lane_id = threadIdx.x & 31;
  for (int32_t j = CS[L] + lane_id; j < CS[L + 1]; j += 32)
    if (C[j].lane == L) f(j);
  for (int32_t q = lane_id; q < dy->n_moved; q += 32) {
    const int32_t j = c.rs_moved[q];
    if (C[j].lane == L && (j < CS[L] || j >= CS[L + 1])) f(j);
  }
  for (int32_t j = dy->n_c + lane_id; j < dy->n_c + dy->n_inj; j += 32)
    if (C[j].lane == L) f(j);
}

// Dirty lanes: gather members on chip, sort (s desc, id asc), write to the
// lane's tail range.  Warp per lane; lanes with more than PD_CAP members rank
// straight from global.
static constexpr int PD_CAP = 128;
static constexpr int PD_WARPS = 4;
// One dirty lane L (whole warp): its n members, sorted, to A[base, base + n).
__device__ void patch_lane(const Ctx& c, const VRec* C, VRec* A, const int32_t* CS, int32_t L, int32_t base,
                           int32_t n, VRec* m) {
  const Dyn* dy = c.dyn;
  const int lane_id = threadIdx.x & 31;
  {
    if (n <= PD_CAP) {
      // gather: segment entries still on L, reverted into L, injected into L
      int k = 0;
      auto take = [&](bool mine, int32_t j) {
        const unsigned bb = __ballot_sync(0xffffffffu, mine);
        if (mine) m[k + __popc(bb & ((1u << lane_id) - 1))] = C[j];
        k += __popc(bb);
      };
      for (int32_t b0 = CS[L]; b0 < CS[L + 1]; b0 += 32) {
        const int32_t j = b0 + lane_id;
        take(j < CS[L + 1] && C[j].lane == L, j);
      }
      for (int32_t b0 = 0; b0 < dy->n_moved; b0 += 32) {
        const int32_t q = b0 + lane_id;
        const int32_t j = q < dy->n_moved ? c.rs_moved[q] : 0;
        take(q < dy->n_moved && C[j].lane == L && (j < CS[L] || j >= CS[L + 1]), j);
      }
      for (int32_t b0 = dy->n_c; b0 < dy->n_c + dy->n_inj; b0 += 32) {
        const int32_t j = b0 + lane_id;
        take(j < dy->n_c + dy->n_inj && C[j].lane == L, j);
      }
      __syncwarp();
      for (int a = lane_id; a < n; a += 32) {
        const double sa = m[a].s;
        const int32_t va = m[a].vix;
        int rank = 0;
        for (int b2 = 0; b2 < n; b2++) rank += ahead_of(m[b2].s, m[b2].vix, sa, va) ? 1 : 0;
        A[base + rank] = m[a];
      }
      __syncwarp();
    } else {
      for_members(c, C, CS, L, [&](int32_t j) {
        const VRec r = C[j];
        int rank = 0;
        for (int32_t q = CS[L]; q < CS[L + 1]; q++)
          if (C[q].lane == L && ahead_of(C[q].s, C[q].vix, r.s, r.vix)) rank++;
        for (int32_t q = 0; q < dy->n_moved; q++) {
          const int32_t jj = c.rs_moved[q];
          if (C[jj].lane == L && (jj < CS[L] || jj >= CS[L + 1]) && ahead_of(C[jj].s, C[jj].vix, r.s, r.vix))
            rank++;
        }
        for (int32_t jj = dy->n_c; jj < dy->n_c + dy->n_inj; jj++)
          if (C[jj].lane == L && ahead_of(C[jj].s, C[jj].vix, r.s, r.vix)) rank++;
        if (rank < n) A[base + rank] = r;
      });
    }
  }
}

// Step end, once: clear the dirty marks; C becomes the snapshot (swap the
// layout buffers) unless the full regroup rebuilt A; record and vehicle
// counts of the new snapshot; end-of-step counters.
__device__ void regroup_finish(const Ctx& c) {
  Dyn* dy = c.dyn;
  for (int i = threadIdx.x; i < dy->n_dirty; i += blockDim.x) {
    c.dirty_flag[c.dirty_list[i]] = 0;
    c.cdelta[c.dirty_list[i]] = 0;
  }
  if (threadIdx.x == 0) {
    if (!dy->need_regroup) {
      dy->cur ^= 1;
      dy->n_a = dy->n_drv = dy->n_c;
    } else if (!dy->full_regroup) {
      dy->cur ^= 1;
      dy->n_drv = dy->n_c + dy->n_inj;
      dy->n_a = dy->n_drv + dy->tail_n;
      dy->n_regroup_patch++;
    } else {
      dy->n_drv = dy->n_a;
      dy->n_regroup_full++;
    }
    dy->finished_total += dy->finished_now;
    dy->reverts_total += dy->reverts_last;
    dy->fin_log_n += dy->finished_now;
    dy->speeds_pending = 1;  // accumulated by the next step's k_speeds branch or a flush
    dy->n_own = 0;           // sharded: recounted by k_count_own
  }
  if (c.pub_dyn && threadIdx.x < 32) {
    // the step's scalars into mapped host memory by one warp, then the step
    // number and an order-free hash of the scalars: tsb_step waits for the
    // number and accepts the copy once the hash matches (plain stores: no
    // system fence on the step's critical path)
    __syncwarp();
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(dy);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(c.pub_dyn);
    unsigned long long h = 0;
    for (int k = threadIdx.x; k < (int)(sizeof(Dyn) / 8); k += 32) {
      const unsigned long long w = src[k];
      dst[k] = w;
      h ^= mix64(w + 0x9E3779B97F4A7C15ULL * (unsigned long long)(k + 1));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) h ^= __shfl_xor_sync(0xffffffffu, h, o);
    if (threadIdx.x == 0) {
      c.pub_seq[0] = dy->step_no;
      c.pub_seq[1] = (long long)h;
    }
  }
}

// The next snapshot, in one launch.  Nothing changed after the sweep: C is
// the snapshot.  Some lanes changed membership or order (dirty): C is the
// snapshot with those lanes rebuilt into its tail, after n_c + n_inj -- every
// block scans the dirty lanes' new member counts (C segment + the deltas the
// revert replay and the injection recorded, cdelta) into their tail offsets,
// block 0 publishes the lane ranges, and each warp rebuilds its lanes.  Too
// many dirty lanes: the full regroup (the RARE body's following kernels)
// instead, which also ends the step.  Otherwise the last block to finish ends it.
#ifndef RG_BLOCKS_CFG
#define RG_BLOCKS_CFG 148
#endif
static constexpr int RG_BLOCKS = RG_BLOCKS_CFG;
__global__ void __launch_bounds__(32 * PD_WARPS) k_regroup(Ctx c, int may_full) {
  PDL_WAIT();
  Dyn* dy = c.dyn;
  // two launches per step: the RARE body's (may_full) and the common one;
  // exactly one of them works
  if (may_full ? !dy->rare : dy->rare) return;
  TL_MARK(TL_REGROUP);
  __shared__ int32_t sd[PATCH_MAX];
  __shared__ VRec sm[PD_WARPS][PD_CAP];
  __shared__ int s_last;
  const int nd = dy->n_dirty;
  if (dy->need_regroup) {
    if (nd > PATCH_MAX || dy->n_inj > PATCH_MAX || dy->n_moved > PATCH_MAX || (c.debug & 2)) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (may_full)
          dy->full_regroup = 1;  // the full regroup kernels follow in this body
        else
          dy->overflow |= 32;  // common body without the full regroup: rare_if_unpatchable missed it
      }
      return;
    }
    VRec* C = c.lay[dy->cur ^ 1];  // sources [0, n_c + n_inj), destination its tail
    const int32_t* CS = c.start[dy->cur ^ 1];
    for (int i = threadIdx.x; i < nd; i += blockDim.x) {
      const int32_t L = c.dirty_list[i];
      sd[i] = (CS[L + 1] - CS[L]) + c.cdelta[L];
    }
    __syncthreads();
    const int32_t tot = block_excl_scan<PATCH_MAX / (32 * PD_WARPS)>(sd, nd);
    const int32_t base0 = dy->n_c + dy->n_inj;
    if (blockIdx.x == 0) {
      int2* R = c.rng[dy->cur ^ 1];
      for (int i = threadIdx.x; i < nd; i += blockDim.x)
        R[c.dirty_list[i]] = make_int2(base0 + sd[i], base0 + (i + 1 < nd ? sd[i + 1] : tot));
      if (threadIdx.x == 0) dy->tail_n = tot;
    }
    const int w = threadIdx.x >> 5;
    for (int i = blockIdx.x * PD_WARPS + w; i < nd; i += gridDim.x * PD_WARPS) {
      const int32_t n = (i + 1 < nd ? sd[i + 1] : tot) - sd[i];
      patch_lane(c, C, C, CS, c.dirty_list[i], base0 + sd[i], n, sm[w]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&dy->rg_done, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  regroup_finish(c);
  if (c.tl_on && threadIdx.x == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    c.tl[(size_t)(c.dyn->tl_row & (TL_ROWS - 1)) * TL_SLOTS + TL_END] = t_;
  }
}

// End of a step whose snapshot the full regroup rebuilt.
__global__ void k_full_finish(Ctx c) {
  PDL_WAIT();
  if (!c.dyn->full_regroup) return;  // k_regroup ended it (eager mode runs this section)
  regroup_finish(c);
}

// ------------------------------------------------------------------ end of step


// Road aggregate (world.py:649-657) of a step's final snapshot A: per road,
// sum of v and count over its lanes (road lanes are consecutive ids,
// network.py:422-442; each lane's records are the range seg() gives), in a
// fixed order (deterministic).  In the step graph this runs at the start of
// the NEXT step on a parallel branch (A is only read until that step's
// regroup, which joins it); mode 1 is the flush a query issues between
// steps.  Both use the same order.
// threads per road in k_speeds: 8 (four roads per warp).  The kernel runs on
// a side branch beside k_update's last wave and the lane scan; a warp per
// road held 4x the warps for the same ~3 us of work.  A/B at M1 (r2): 32 ->
// 8 threads: k_update -3 us, the scan phase -2.8 us, the step -7 us; 4: -6 us.
#ifndef SP_G
#define SP_G 8
#endif
__global__ void k_speeds(Ctx c, int flush) {
  PDL_WAIT();
  if (!flush) TL_MARK(TL_SPEEDS);
  Dyn* dy = c.dyn;
  if (!(flush ? dy->speeds_pending : dy->acc_now)) return;
  const VRec* A = c.lay[dy->cur];
  const int2* S = c.rng[dy->cur];
  const int32_t wi = (int32_t)((flush ? dy->time : dy->acc_time) / c.p.speed_window);
  if (wi >= c.n_win) {
    if (gtid() == 0) dy->overflow |= 2;
    return;
  }
  // SP_G threads per road: a segmented reduction -- the group's threads
  // stride over the road's lane ranges (road lanes are consecutive ids, each
  // lane's records one range), then a butterfly sum across the group; the
  // order is fixed, so the aggregate is deterministic run to run
  const int32_t ln = threadIdx.x % SP_G;
  const unsigned gmask = SP_G == 32 ? 0xffffffffu : (((1u << SP_G) - 1u) << ((threadIdx.x & 31) / SP_G * SP_G));
  const int32_t nw = gstride() / SP_G;
  for (int32_t r = gtid() / SP_G; r < c.n_roads; r += nw) {
    const int2 span = c.road_span[r];
    if (c.sharded && !(c.zone[span.x] & ZF_OWN)) continue;  // the owner accumulates it
    double sum = 0.0;
    int32_t cnt = 0;
    for (int32_t L = span.x; L <= span.y; L++) {
      const int2 sg = seg(c, S, L);
      for (int32_t j = sg.x + ln; j < sg.y; j += SP_G) sum += __ldg(&A[j].v);
      cnt += sg.y - sg.x;
    }
    if (cnt == 0) continue;
#pragma unroll
    for (int o = SP_G / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(gmask, sum, o, SP_G);
    if (ln == 0) {
      const size_t cell = (size_t)r * c.n_win + wi;
      c.acc_sum[cell] += sum;
      c.acc_cnt[cell] += cnt;
    }
  }
}

__global__ void k_speeds_done(Ctx c) {
  PDL_WAIT(); c.dyn->speeds_pending = 0; }


__global__ void k_begin_step(Ctx c) {
  PDL_WAIT();
  for (int32_t L = gtid(); L < c.n_lanes; L += gstride()) c.cnt[L] = 0;
  for (int32_t t = gtid(); t < c.scan_tiles_cap; t += gstride()) c.scan_tile_sums[t] = 0;
  if (gtid() != 0) return;
  if (c.tl_on) c.dyn->tl_row += 1;
  TL_MARK(TL_BEGIN);
  Dyn* dy = c.dyn;
  dy->vehicle_updates += c.sharded ? dy->n_own : dy->n_drv;
  dy->finished_now = 0;
  dy->n_events = 0;
  dy->complex = 0;
  dy->n_dirty = 0;
  dy->full_regroup = 0;
  dy->n_moved = 0;
  dy->need_regroup = 0;
  dy->n_inj = 0;
  dy->n_hostq = 0;
  dy->n_fix = 0;
  dy->acc_now = dy->speeds_pending;
  dy->acc_time = dy->time;
  dy->speeds_pending = 0;
  dy->reverts_last = 0;
  dy->n_due = 0;
  dy->rf_arrive = 0;
  dy->rf_conflict = 0;
  dy->rf_done = 0;
  dy->rg_done = 0;
  dy->rf_fin = 0;
  dy->rare = 0;
}

// Snapshot-isolation check (tsb_set_debug bit 6): before the update, every
// buffer a step may only write before it reads -- the post-update records B,
// the sort scratch D and the layout buffer the step will build C in -- is
// filled with 0xff bytes (NaN speeds and positions, -1 indices), so a read of
// anything but the snapshot A (world.py:231-236, 416-419: the update reads
// only snap_*) poisons the results and the parity tests fail.
__global__ void k_poison(Ctx c) {
  PDL_WAIT();
  const int64_t n = (int64_t)c.cap_rec * (sizeof(VRec) / 16);
  int4* bufs[3] = {(int4*)c.B, (int4*)c.D, (int4*)c.lay[c.dyn->cur ^ 1]};
  const int4 ff = make_int4(-1, -1, -1, -1);
  for (int b = 0; b < 3; b++)
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
      bufs[b][k] = ff;
}

__global__ void k_zero_cnt(Ctx c, const int32_t* gate) {
  PDL_WAIT();
  if (gated_off(gate)) return;
  for (int32_t L = gtid(); L < c.n_lanes; L += gstride()) c.cnt[L] = 0;
}

__global__ void k_set_na(Ctx c, const int32_t* gate) {
  PDL_WAIT();
  if (gated_off(gate)) return;
  c.dyn->n_a = c.start[c.dyn->cur][c.n_lanes];
}

// min_front_gap (world.py:694-704) over the snapshot layout.
__global__ void k_min_gap(Ctx c, double* out) {
  PDL_WAIT();
  Dyn* dy = c.dyn;
  const VRec* A = c.lay[dy->cur];
  __shared__ double sm[32];
  double best = CUDART_INF;
  const int2* S = c.rng[dy->cur];
  for (int32_t L = threadIdx.x; L < c.n_lanes; L += blockDim.x) {
    if (c.sharded && !(c.zone[L] & ZF_OWN)) continue;
    const int2 sg = seg(c, S, L);
    for (int32_t i = sg.x; i + 1 < sg.y; i++) best = py_min(best, A[i].s - c.p.L - A[i + 1].s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); w++) best = fmin(best, sm[w]);
    best = fmin(best, sm[0]);
    *out = best;
  }
}


// ------------------------------------------------------------------ queries
//
// Per-id and batch queries (World.get_vehicle, world.py:706-714;
// World.record_step, world.py:771-782) answered on the device.  k_locate
// maps each vix to its record in the snapshot A: records outside their
// lane's range are stale copies and, in a sharded engine, only own lanes
// count (a ghost belongs to the rank owning its lane).

__global__ void k_locate(Ctx c, int32_t* loc) {
  PDL_WAIT();
  Dyn* dy = c.dyn;
  const VRec* A = c.lay[dy->cur];
  const int2* S = c.rng[dy->cur];
  const int32_t n = dy->n_a + (c.sharded ? dy->n_g : 0);
  for (int32_t i = gtid(); i < n; i += gstride()) {
    const int32_t L = A[i].lane;
    if (L < 0) continue;
    const int2 sg = seg(c, S, L);
    if (i < sg.x || i >= sg.y) continue;
    if (c.sharded && !(c.zone[L] & ZF_OWN)) continue;
    loc[A[i].vix] = i;
  }
}

__global__ void k_vehicle_views(Ctx c, const int32_t* loc, const int32_t* q, int32_t n, tsb_vehicle_view* out) {
  PDL_WAIT();
  const VRec* A = c.lay[c.dyn->cur];
  for (int32_t k = gtid(); k < n; k += gstride()) {
    const int32_t x = q[k];
    tsb_vehicle_view o;
    o.pad = 0;
    o.finish_time = 0.0;
    const int32_t i = loc[x];
    const int st = c.status[x];
    const VCold cd = c.cold[x];
    if (i >= 0) {
      const VRec r = A[i];
      o.s = r.s;
      o.v = r.v;
      o.lane = r.lane;
      o.road_pos = (int32_t)(r.rptr - cd.route_off);
      o.status = TSB_STATUS_DRIVING;
    } else if (st == TSB_STATUS_FINISHED) {
      const VRec r = c.fin_state[x];
      o.s = r.s;
      o.v = r.v;
      o.lane = r.lane;
      o.road_pos = (int32_t)(r.rptr - cd.route_off);
      o.status = st;
      o.finish_time = c.finish[x];
    } else if (st == TSB_STATUS_DRIVING) {  // sharded: driving on another rank's lanes
      o.s = 0.0;
      o.v = 0.0;
      o.lane = -1;
      o.road_pos = 0;
      o.status = TSB_STATUS_ELSEWHERE;
    } else {  // waiting or dropped: the trip's origin (world.py:196-198)
      o.s = cd.origin_s;
      o.v = 0.0;
      o.lane = cd.origin_lane;
      o.road_pos = 0;
      o.status = st;
    }
    out[k] = o;
  }
}

// Record stream, id order: block b takes vix [b*RECB, (b+1)*RECB); pass 1
// counts the located ones per block, a one-block scan turns the counts into
// offsets, pass 2 writes each block's records in vix order.
static constexpr int RECB = 1024;
__global__ void __launch_bounds__(RECB) k_rec_count(Ctx c, const int32_t* loc, int32_t* bcnt) {
  PDL_WAIT();
  const int32_t x = blockIdx.x * RECB + threadIdx.x;
  const int on = x < c.n_trips && loc[x] >= 0;
  const int t = __syncthreads_count(on);
  if (threadIdx.x == 0) bcnt[blockIdx.x] = t;
}

__global__ void __launch_bounds__(1024) k_rec_offsets(int32_t* bcnt, int32_t nb) {
  PDL_WAIT();
  __shared__ int32_t carry;
  __shared__ int32_t ws[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int32_t base = 0; base < nb; base += 1024) {
    const int32_t k = base + threadIdx.x;
    const int32_t x = k < nb ? bcnt[k] : 0;
    int32_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if ((threadIdx.x & 31) >= o) incl += y;
    }
    if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = incl;
    __syncthreads();
    if (threadIdx.x < 32) {
      int32_t w = ws[threadIdx.x];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (threadIdx.x >= o) w += y;
      }
      ws[threadIdx.x] = w;
    }
    __syncthreads();
    const int32_t wpre = (threadIdx.x >> 5) ? ws[(threadIdx.x >> 5) - 1] : 0;
    const int32_t c0 = carry;
    if (k < nb) bcnt[k] = c0 + wpre + incl - x;
    __syncthreads();
    if (threadIdx.x == 1023) carry = c0 + wpre + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) bcnt[nb] = carry;
}

struct RecOut {
  int32_t* vix;
  int32_t* lane;
  int32_t* road_pos;
  double* s;
  double* v;
  double* angle;
};

__global__ void __launch_bounds__(RECB) k_rec_write(Ctx c, const int32_t* loc, const int32_t* boff, RecOut o,
                                                    const int64_t* geo_off, const double* geo_cum,
                                                    const double* geo_angle) {
  PDL_WAIT();
  __shared__ int32_t ws[RECB / 32];
  const VRec* A = c.lay[c.dyn->cur];
  const int32_t x = blockIdx.x * RECB + threadIdx.x;
  const int32_t i = x < c.n_trips ? loc[x] : -1;
  const unsigned bal = __ballot_sync(0xffffffffu, i >= 0);
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  if (ln == 0) ws[w] = __popc(bal);
  __syncthreads();
  int32_t pre = boff[blockIdx.x];
  for (int k = 0; k < w; k++) pre += ws[k];
  if (i < 0) return;
  const int32_t j = pre + __popc(bal & ((1u << ln) - 1u));
  const VRec r = A[i];
  o.vix[j] = x;
  o.lane[j] = r.lane;
  o.road_pos[j] = (int32_t)(r.rptr - c.cold[x].route_off);
  o.s[j] = r.s;
  o.v[j] = r.v;
  // geometry.heading_deg_at(line, cum, min(s, len)) (world.py:777-779):
  // segment = bisect_right(cum, s) - 1 clamped to the lane's segments
  const double len = c.lanes[r.lane].len;
  const double sq = py_min(r.s, len);
  const int64_t a = geo_off[r.lane], b = geo_off[r.lane + 1];
  int64_t lo = a, hi = b;  // first k with cum[k] > sq
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (geo_cum[m] > sq)
      hi = m;
    else
      lo = m + 1;
  }
  int64_t sgi = lo - 1;
  if (sgi < a) sgi = a;
  if (sgi > b - 1) sgi = b - 1;
  o.angle[j] = b > a ? geo_angle[sgi] : 0.0;
}

// ------------------------------------------------------------------ sharded exchange
//
// Message of rank r to peer q (bytes): int32 counts of r's export lanes for q
// (ascending lane ids, shard.py), padded to 32 B, then the lanes' vehicle
// records (VRec, lane-sorted as in r's snapshot).  The receiver appends them
// to its snapshot as ghosts and points its halo lanes at them.

__device__ __forceinline__ int64_t align32(int64_t x) { return (x + 31) & ~(int64_t)31; }

// Own vehicles in the snapshot (vehicle_updates counts them next step).
__global__ void k_count_own(Ctx c) {
  PDL_WAIT();
  Dyn* dy = c.dyn;
  const int2* S = c.rng[dy->cur];
  int32_t mine = 0;
  for (int32_t L = gtid(); L < c.n_lanes; L += gstride())
    if (c.zone[L] & ZF_OWN) {
      const int2 sg = seg(c, S, L);
      mine += sg.y - sg.x;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&dy->n_own, mine);
}

__global__ void k_exp_count(Ctx c, int p2p) {
  PDL_WAIT();
  if (p2p && gtid() == 0) c.dyn->xchg_epoch += 1;  // this exchange's epoch (device-side: graph-capturable)
  const int2* S = c.rng[c.dyn->cur];
  for (int32_t e = gtid(); e < c.n_exp; e += gstride()) {
    const int32_t L = c.exp_lane[e];
    const int2 sg = seg(c, S, L);
    c.exp_cnt[e] = c.exp_kind[e] ? 0 : sg.y - sg.x;  // a max-pressure entry carries no records
  }
}

// Byte offset of peer q's message in the send buffer.
__device__ __forceinline__ int64_t exp_base(const Ctx& c, int q) {
  int64_t b = 0;
  for (int p = 0; p < q; p++) {
    const int64_t e0 = c.peer_first_exp[p], e1 = c.peer_first_exp[p + 1];
    b += align32(4 * (e1 - e0)) + 32 * (int64_t)(c.exp_pos[e1] - c.exp_pos[e0]);
  }
  return b;
}

// Warp per export entry: header count and records.
__global__ void k_exp_pack(Ctx c, uint8_t* send) {
  PDL_WAIT();
  const VRec* A = c.lay[c.dyn->cur];
  const int2* S = c.rng[c.dyn->cur];
  const int lid = threadIdx.x & 31;
  for (int32_t e = gtid() >> 5; e < c.n_exp; e += gstride() >> 5) {
    const int q = c.exp_peer[e];
    const int64_t e0 = c.peer_first_exp[q];
    const int64_t base = exp_base(c, q);
    const int32_t L = c.exp_lane[e];
    const int32_t n = c.exp_cnt[e];
    // header: the lane's record count, or (max-pressure entry) its post-sweep vehicle count
    if (lid == 0) ((int32_t*)(send + base))[e - e0] = c.exp_kind[e] ? c.lane_counts[L] : n;
    VRec* dst = (VRec*)(send + base + align32(4 * (c.peer_first_exp[q + 1] - e0))) + (c.exp_pos[e] - c.exp_pos[e0]);
    const int32_t at = seg(c, S, L).x;
    for (int32_t k = lid; k < n; k += 32) dst[k] = A[at + k];
  }
}

// ---- the device-driven exchange in four kernels (issue_exchange)
//
// k_exp_prep: export counts and their exclusive scan in one block (the
// entries are the boundary lanes: a few thousand).  k_exp_pack_signal: the
// own-vehicle count, the pack into the peers' slots, and -- by the last block
// to finish, after every block fenced its remote writes -- the release of the
// peers' arrival flags.  k_p2p_wait_import: the wait for every peer's flag,
// then the import counts and their scan in one block.  k_imp_copy.

// Block-wide: cnt[i] = count(i), pos[i] = exclusive prefix, pos[n] = total
// (each thread a contiguous chunk, one block scan of the chunk sums).
template <class F>
__device__ void block_count_scan(int32_t n, F count, int32_t* cnt, int32_t* pos) {
  __shared__ int32_t s_w[32];
  __shared__ int32_t s_total;
  const int T = blockDim.x;
  const int32_t chunk = (n + T - 1) / T;
  const int32_t a = min(n, (int32_t)threadIdx.x * chunk), b = min(n, a + chunk);
  int32_t sum = 0;
  for (int32_t i = a; i < b; i++) {
    const int32_t v = count(i);
    cnt[i] = v;
    sum += v;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int32_t w = lane < (T >> 5) ? s_w[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < (T >> 5)) s_w[lane] = w;
    if (lane == 31) s_total = w;
  }
  __syncthreads();
  int32_t run = (warp ? s_w[warp - 1] : 0) + x - sum;
  for (int32_t i = a; i < b; i++) {
    pos[i] = run;
    run += cnt[i];
  }
  if (threadIdx.x == 0) pos[n] = s_total;
}

__global__ void __launch_bounds__(1024) k_exp_prep(Ctx c) {
  PDL_WAIT();
  if (threadIdx.x == 0) c.dyn->xchg_epoch += 1;  // this exchange's epoch (device-side: graph-capturable)
  const int2* S = c.rng[c.dyn->cur];
  block_count_scan(
      c.n_exp,
      [&](int32_t e) {
        const int2 sg = seg(c, S, c.exp_lane[e]);
        return c.exp_kind[e] ? 0 : sg.y - sg.x;  // a max-pressure entry carries no records
      },
      c.exp_cnt, c.exp_pos);
}

__global__ void k_exp_pack_signal(Ctx c) {
  PDL_WAIT();
  Dyn* dy = c.dyn;
  const int2* S = c.rng[dy->cur];
  // own vehicles in the snapshot (vehicle_updates counts them next step)
  {
    int32_t mine = 0;
    for (int32_t L = gtid(); L < c.n_lanes; L += gstride())
      if (c.zone[L] & ZF_OWN) {
        const int2 sg = seg(c, S, L);
        mine += sg.y - sg.x;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&dy->n_own, mine);
  }
  // the pack, straight into the peers' receive slots
  const unsigned long long epoch = dy->xchg_epoch;
  const VRec* A = c.lay[dy->cur];
  const int lid = threadIdx.x & 31;
  const int64_t slot = (int64_t)((epoch & 1) * c.nranks + c.rank) * c.p2p_slot;
  if (gtid() == 0) dy->xchg_bytes += (unsigned long long)exp_base(c, c.nranks);
  for (int32_t e = gtid() >> 5; e < c.n_exp; e += gstride() >> 5) {
    const int q = c.exp_peer[e];
    const int64_t e0 = c.peer_first_exp[q];
    uint8_t* base = c.p2p_peer_recv[q] + slot;
    const int32_t L = c.exp_lane[e];
    const int32_t n = c.exp_cnt[e];
    if (lid == 0) ((int32_t*)base)[e - e0] = c.exp_kind[e] ? c.lane_counts[L] : n;
    VRec* dst = (VRec*)(base + align32(4 * (c.peer_first_exp[q + 1] - e0))) + (c.exp_pos[e] - c.exp_pos[e0]);
    const int32_t at = seg(c, S, L).x;
    for (int32_t k = lid; k < n; k += 32) dst[k] = A[at + k];
  }
  // the last block releases the peers' flags once every block's remote
  // writes are visible system-wide (each writer fenced before arriving)
  __threadfence_system();
  __syncthreads();
  __shared__ int s_last;
  if (threadIdx.x == 0)
    s_last = (atomicAdd(&dy->xchg_packed, 1ULL) % (unsigned long long)gridDim.x) == gridDim.x - 1;
  __syncthreads();
  if (s_last) {
    __threadfence_system();
    const int q = threadIdx.x;
    if (q < c.nranks && q != c.rank) {
      unsigned long long* f = c.p2p_peer_flag[q] + (epoch & 1) * c.nranks + c.rank;
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(epoch) : "memory");
    }
  }
}

// Device-driven exchange over peer memory (NVLink P2P / CUDA IPC): the pack
// writes each peer's message straight into that peer's receive slot for this
// rank and step parity -- the same layout as k_exp_pack's -- then the step
// epoch is released in the peer's flag for this rank and every peer's flag is
// awaited before the import reads the local slots (k_exp_pack_signal,
// k_p2p_wait_import below).  Two slot sets by step parity: a rank writes parity t+1 only after
// its own import of step t saw every peer's step-t flag, which each peer
// raised after importing step t-1 from that slot set.
// Receive side: counts from the headers (src_base[q] = byte offset of
// source q's message in the receive buffer).
struct SrcBase {
  int64_t b[9];
};
// Byte offset of source q's message: sb, or (P2P: sb.b[0] < 0) the slot of
// q for the current exchange epoch's parity.
__device__ __forceinline__ int64_t src_base(const Ctx& c, const SrcBase& sb, int q) {
  if (sb.b[0] >= 0) return sb.b[q];
  return (int64_t)((c.dyn->xchg_epoch & 1) * c.nranks + q) * c.p2p_slot;
}

__global__ void k_imp_count(Ctx c, const uint8_t* recv, SrcBase sb) {
  PDL_WAIT();
  for (int32_t e = gtid(); e < c.n_imp; e += gstride()) {
    const int q = c.imp_peer[e];
    const int32_t h = ((const int32_t*)(recv + src_base(c, sb, q)))[e - c.peer_first_imp[q]];
    if (c.imp_kind[e]) {  // the owner's post-sweep count of a max-pressure lane
      c.lane_counts[c.imp_lane[e]] = h;
      c.imp_cnt[e] = 0;
    } else {
      c.imp_cnt[e] = h;
    }
  }
}

// Wait for every peer's arrival flag, then the import counts
// from the headers and their scan, in one block (k_imp_count + scan).
__global__ void __launch_bounds__(1024) k_p2p_wait_import(Ctx c, const uint8_t* recv, SrcBase sb) {
  PDL_WAIT();
  const unsigned long long epoch = c.dyn->xchg_epoch;
  const int q = threadIdx.x;
  if (q < c.nranks && q != c.rank) {
    const unsigned long long* f = c.p2p_flag + (epoch & 1) * c.nranks + q;
    unsigned long long v, t_start, t_now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
      if (v >= epoch) break;
      __nanosleep(256);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_now));
      if (t_now - t_start > c.p2p_timeout_ns) {  // a peer stopped stepping: fail loudly, do not hang
        atomicOr(&c.dyn->overflow, 128);
        break;
      }
    }
  }
  __syncthreads();
  __threadfence_system();
  block_count_scan(
      c.n_imp,
      [&](int32_t e) {
        const int qq = c.imp_peer[e];
        const int32_t h = ((const int32_t*)(recv + src_base(c, sb, qq)))[e - c.peer_first_imp[qq]];
        if (c.imp_kind[e]) {  // the owner's post-sweep count of a max-pressure lane
          c.lane_counts[c.imp_lane[e]] = h;
          return 0;
        }
        return h;
      },
      c.imp_cnt, c.imp_pos);
  if (threadIdx.x == 0 && c.n_imp == 0) c.dyn->n_g = 0;
}

// Warp per import entry: ghost range of the lane, records appended after the
// snapshot's own records.
__global__ void k_imp_copy(Ctx c, const uint8_t* recv, SrcBase sb) {
  PDL_WAIT();
  Dyn* dy = c.dyn;
  VRec* A = c.lay[dy->cur];
  const int32_t base = dy->n_a;
  const int lid = threadIdx.x & 31;
  for (int32_t e = gtid() >> 5; e < c.n_imp; e += gstride() >> 5) {
    const int q = c.imp_peer[e];
    const int64_t e0 = c.peer_first_imp[q];
    if (c.imp_kind[e]) continue;  // count only (k_imp_count)
    const int32_t L = c.imp_lane[e];
    const int32_t n = c.imp_cnt[e];
    const VRec* src = (const VRec*)(recv + src_base(c, sb, q) + align32(4 * (c.peer_first_imp[q + 1] - e0))) +
                      (c.imp_pos[e] - c.imp_pos[e0]);
    const int32_t at = base + c.imp_pos[e];
    if ((int64_t)at + n > c.cap_rec) {  // ghost capacity (fails loudly at the next sync)
      if (lid == 0) dy->overflow |= 64;
      continue;
    }
    if (lid == 0) c.rng[dy->cur][L] = make_int2(at, at + n);
    for (int32_t k = lid; k < n; k += 32) {
      VRec r = src[k];
      r.lane = L;  // the sender's lane id in this rank's numbering (local lane spaces differ)
      A[at + k] = r;
    }
  }
  if (gtid() == 0) dy->n_g = c.imp_pos[c.n_imp];
}

}  // namespace tsb
