// device.cuh -- device data layout and the per-vehicle model arithmetic.
//
// Every floating-point expression keeps CPython's evaluation order and
// rounding (the reference is trafficsim/engine/*.py); the library is built
// with --fmad=false so nvcc never contracts a*b+c into an FMA.  The only FMA
// calls below are explicit, inside the double-double power, where they are
// exact error-free transforms.
#pragma once
#include <cstdint>

#include "../../include/tsb200.h"
#include "pow_glibc.cuh"

namespace tsb {

// ---------------------------------------------------------------- layout

// One driving vehicle in a lane-sorted layout (32 B, two 16 B vectors).
// `lane` is explicit (the CSR position implies it, but the update kernel
// needs it without a search); `src` is the index of the vehicle in the
// step's snapshot layout A, which carries the snapshot lane/s/rptr needed by
// the collision sweep and by reverts (world.py:501-507).
// `rptr` replaces the reference's road_pos: it is the absolute index in the
// route pool of roads_seq[road_pos].  Every route in the pool is followed by
// a -1 sentinel, so "on the final road" (world.py:276, 455) is
// routes[rptr + 1] < 0 and the update never gathers per-vehicle route
// metadata; road_pos = rptr - route_off[vix] is recovered on the host.
struct __align__(16) VRec {
  double s;
  double v;
  int32_t vix;
  int32_t rptr;
  int32_t lane;
  int32_t src;
};

// Per-lane flag byte (lflag[]), read by the update instead of chains of
// LaneRec / signal-state gathers.  Bit 0 (OPEN) is the lane's own
// restriction (host-maintained); for connectors, bit 1 (SUCC_OPEN) is the
// restriction of its successor road lane and bits 2-3 its signal aspect
// (world.py:247-254, signals.py:46-61), refreshed by k_signals each step and
// by k_lane_flags after a control change.
enum : uint8_t { LF_OPEN = 1, LF_SUCC_OPEN = 2, LF_ASPECT_SHIFT = 2 };

// Static per-lane record (48 B) gathered by the update kernel.
struct __align__(16) LaneRec {
  double len;
  double cap;
  int32_t road;      // road index (road lane) or -1
  int32_t junc;      // junction index (connector) or -1
  int32_t left, right;
  int32_t succ1;     // connector: successor road lane
  int32_t pred1;     // connector: predecessor road lane
  int32_t succ_off;  // CSR into succ / succ_dst_road
  int16_t nsucc;
  int8_t kind;
  uint8_t open;
};

// Per-vehicle cold data, indexed by vix.
struct __align__(16) VCold {
  uint64_t key;       // id & (2^64-1)
  int64_t route_off;  // into the road-index route pool
  int32_t route_len;  // roads in roads_seq; 0 = unroutable; -1 = not computed
  int32_t origin_lane;
  double origin_s;
  double depart;
};

struct JuncState {
  int32_t phase;
  int32_t pad;
  double elapsed;
  double since;
};

struct FinEntry {
  int32_t vix;
  int32_t pad;
  int64_t step;
};

// Scalars that change every step (device resident so a whole step is a
// CUDA graph with no host round trip).
struct Dyn {
  double time;
  int64_t step_no;
  int64_t vehicle_updates;
  int64_t finished_total;
  int64_t dropped;
  int64_t injected_now;
  int64_t finished_now;
  int64_t reverts_last;
  int32_t cur;          // which layout buffer holds the snapshot A
  int32_t n_a;          // vehicles in A
  int32_t n_c;          // vehicles scattered into C (post-update, excl. arrivals)
  int32_t n_inj;        // injected this step (appended after n_c in C)
  int32_t n_events;     // lanes whose tentative sweep hit a revert
  int32_t n_moved;      // vehicles moved by resolve (reverted into another lane)
  int32_t need_regroup; // membership or order changed after the sweep
  int32_t complex;      // some revert event is not simple: sequential resolve
  int32_t n_dirty;      // lanes rebuilt by the incremental regroup
  int32_t full_regroup; // too many dirty lanes: full regroup instead
  int64_t resolve_sequential;  // steps that needed the sequential resolver
  int32_t pend_ptr;
  int32_t n_retry;
  int32_t n_due;
  int32_t n_hostq;      // vehicles needing a host reroute (closures only)
  int32_t overflow;     // sticky error flag
  int64_t fin_log_n;
  int64_t reverts_total;
  int32_t n_cl;    // lanes in the revert closure (cleared at the next step)
  int32_t n_comp;  // closure components replayed in parallel
  int32_t n_fix;   // lanes k_lanefix must sort / sweep this step
  int32_t n_g;     // sharded: ghost records appended to the snapshot at [n_a, n_a + n_g)
  int32_t n_own;   // sharded: vehicles on own lanes in the snapshot
  int32_t speeds_pending;  // the snapshot's road aggregate is not yet accumulated
  int32_t acc_now;         // this step's k_speeds branch accumulates it
  double acc_time;         // the time of that snapshot
  int32_t n_drv;    // driving vehicles in the snapshot (n_a minus its stale copies)
  int32_t tail_n;   // records of the lanes the regroup rebuilt into the snapshot's tail
  int32_t rf_arrive;    // k_resolve_fast: warps past the claim phase
  int32_t rf_conflict;  // k_resolve_fast: closures overlap or exceed a budget (general path)
  int32_t rf_done;      // k_resolve_fast replayed every event
  int32_t rg_done;      // k_regroup: blocks finished (the last one ends the step)
  int32_t rf_fin;       // k_resolve_fast: replays finished
  int32_t tl_row;       // the step's row in the timeline ring (while the timeline is on)
  int32_t rare;         // the step takes the RARE body (set_rare)
  int32_t pad4_;
  unsigned long long xchg_epoch;  // sharded P2P exchanges so far (k_exp_count)
  unsigned long long xchg_bytes;  // sharded P2P: bytes this rank wrote into peer slots so far
  unsigned long long xchg_packed; // sharded P2P: blocks of k_exp_pack_signal finished so far (all launches)
  // cumulative step-path counters (tsb_path_counters)
  int64_t n_resolve_fast, n_resolve_general, n_regroup_patch, n_regroup_full, n_inject_steps;
};

struct Params {
  double dt, lookahead;
  double v0, T, a_max, b, delta, s0;
  double politeness, threshold, b_safe, eval_prob;
  double L, speed_window, amber, s0_floor, mp_interval, mp_min_green;
  double sqrt_ab2;   // 2.0 * sqrt(a_max * b), evaluated as in idm.py:29
  double inv_ab2;    // 1 / sqrt_ab2 when sqrt_ab2 is a power of two (then x / sqrt_ab2 == x * inv_ab2 exactly)
  int32_t ab2_pow2;
  double rcp_ab2;    // RN(1 / sqrt_ab2): x / sqrt_ab2 by div_rcp()
  double rcp_v0;     // RN(1 / v0): v / v0 by div_rcp() (0: plain division)
  uint64_t rng_h2;   // keyed-RNG fold state after (seed, STREAM_MOBIL): constant for the run
  int32_t controller;
  int32_t delta_int; // delta as an integer power if integral in [1, 64], else 0
  int32_t pow_glibc; // 1: powers exactly as glibc's pow (CPython `**`); 0: correctly rounded
  uint64_t seed;
};

// All device pointers of one engine (passed by value to every kernel).
struct Ctx {
  Params p;
  int32_t n_lanes, n_roads, n_junc, n_trips;
  int32_t n_pend;  // trips in the pending list (all, or a shard's own)
  int32_t split;  // 1 when lane closures exist: host continuation of reroutes
  int32_t debug;  // test knobs: 1 = always sequential resolve, 2 = always full regroup
  const LaneRec* lanes;
  const int32_t* succ;
  const int32_t* succ_dst_road;
  const int4* succ_road4;  // per lane: roads of its first 4 successors (-5 = none)
  const int4* succ_conn4;  // per lane: those successors (w = -2: more than 4; slots 3.. in the CSR)
  const int32_t* road_lane_off;
  const int2* road_span;  // per road: first and last lane id (consecutive ids)
  const int32_t* road_lanes;
  const int32_t* junc_phase_off;
  const double* phase_dur;
  const uint64_t* green;
  const uint8_t* junc_signal;
  const int32_t* jc_off;  // junction -> connectors CSR
  const int32_t* jc;
  JuncState* sig;
  const VCold* cold;
  const uint64_t* keys;  // RNG key per vix (id & (2^64-1)); unused when ids_dense
  int32_t ids_dense;     // 1 when id == vix for every trip: key = vix
  uint8_t* lflag;
  const int32_t* routes;
  uint8_t* status;
  uint8_t* routed;
  double* finish;
  VRec* fin_state;  // last committed state of finished vehicles (by vix)
  VRec* lay[2];
  int32_t* start[2];
  VRec* B;
  VRec* D;
  int32_t* cnt;
  int32_t* cursor;
  int32_t* ent;      // per lane: movers entering it this step
  int32_t* mslot;    // per B record (movers): slot among the new lane's entrants
  uint8_t* stay;     // per B record: still on its snapshot lane
  int2* nrc[2];      // per B record, by step parity: {rptr, next road} of its post-update state
  int32_t cap_rec;   // capacity of the record layouts
  int32_t* fix_flag;
  int32_t* fix_list;
  unsigned long long* scan_status;   // SCAN_SITES regions of scan_tiles_cap words
  unsigned long long* scan_tickets;  // per scan site, never reset
  int32_t* scan_tile_sums;           // per tile totals of the two-pass lane scan
  int32_t scan_tiles_cap;
  // sharded mode (shard.py): per-lane zone flags, ghost ranges, export/import lists
  int32_t sharded;
  const uint8_t* zone;  // ZF_OWN | ZF_HALO, ZF_EXACT

  int32_t n_exp, n_imp;
  const int32_t* exp_lane;  // export entries (peer-major, ascending lanes)
  const int32_t* exp_peer;
  const int32_t* imp_lane;  // import entries (source-major, ascending lanes)
  const int32_t* imp_peer;
  const uint8_t* exp_kind;  // per entry: 0 halo lane (records), 1 max-pressure lane (count only)
  const uint8_t* imp_kind;
  int32_t* exp_cnt;
  int32_t* exp_pos;  // exclusive scan of exp_cnt (n_exp + 1)
  int32_t* imp_cnt;
  int32_t* imp_pos;
  int64_t peer_first_exp[9], peer_first_imp[9];  // entry index ranges per peer (nranks <= 8)
  int32_t nranks, rank;
  // device-driven exchange over peer memory (tsb_shard_p2p_*): each rank's
  // receive slots [parity][source rank] and arrival flags, mapped in every peer
  uint8_t* p2p_peer_recv[8];
  unsigned long long* p2p_peer_flag[8];
  unsigned long long* p2p_flag;  // own flags [parity][source rank]
  int64_t p2p_slot;               // bytes per slot
  uint64_t p2p_timeout_ns;        // k_p2p_wait gives up after this long (overflow bit 0x80)
  int32_t* comp_flags;  // per component: bit 0 has an own lane, bit 1 has an inexact lane
  // conditional sections of the step graph (kernels.cu set_cond)
  unsigned long long cond[4];
  int32_t use_cond;
  // connectors in junction order (jc) with their junction / successor lane
  int32_t n_conn;
  const int32_t* jc_junc;
  const int32_t* jc_succ1;
  int32_t* stage;  // scan staging (n_lanes + 1)
  int32_t* events;
  // revert closure / components (k_resolve_closure)
  int32_t* cl_idx;    // per lane: 1 + index in the closure, 0 = outside
  int32_t* cl_lanes;  // closure lanes of the current step
  int32_t* comp_id;
  int32_t* comp_off;
  int32_t* comp_size;
  int32_t* comp_edges;
  int32_t* comp_fill;
  int32_t* comp_ev;
  int32_t* dirty_flag;
  int32_t* cdelta;  // per lane: membership change this step (reverts, injections)
  int32_t* dirty_list;
  int2* rng[2];         // per layout buffer and lane: [start, end) of the lane's records (see seg())
  // resolve scratch
  int32_t* rs_heap;
  uint8_t* rs_inwork;
  uint8_t* rs_touched;
  uint8_t* rs_event;
  uint8_t* rs_movedin;
  int32_t* rs_moved;
  uint8_t* rs_reverted;
  unsigned long long* rf_owner;  // per lane: (step epoch << 32) | (event + 1) of the closure that claimed it
  int32_t* rs_members;
  int32_t* rs_touched_list;
  // injection
  const int32_t* pend_vix;
  const double* pend_dep;
  int32_t* retry;
  int32_t* retry2;
  int32_t* due;
  int32_t* due_grp;
  int32_t* inj_cnt;
  int32_t* inj_start;
  int32_t* inj_cursor;
  uint8_t* outcome;
  int32_t* flag_in;
  int32_t* flag_scan;
  int32_t* lane_counts;  // max-pressure lane occupancy
  // output
  FinEntry* fin_log;
  double* acc_sum;
  long long* acc_cnt;
  int32_t n_win;
  int32_t* hostq;
  Dyn* dyn;
  unsigned long long* tl;  // step timestamps, TL_ROWS x TL_SLOTS (kernels.cu TL_MARK)
  // end-of-step report published into mapped (zero-copy) host memory by the
  // block that ends the step: the step scalars, then the step number
  Dyn* pub_dyn;
  volatile long long* pub_seq;
  int32_t tl_on;           // tsb_set_timeline
  double* scratch_d;
};

// ---------------------------------------------------------------- arithmetic

__device__ __forceinline__ double py_min(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double py_max(double a, double b) { return (b > a) ? b : a; }

// x**n for integer n >= 1, correctly rounded: binary powering in
// double-double (error-free products via explicit FMA), one final rounding.
__device__ __forceinline__ void dd_mul(double ah, double al, double bh, double bl, double& rh, double& rl) {
  double p = ah * bh;
  double e = fma(ah, bh, -p);
  e = e + (ah * bl + al * bh);
  rh = p + e;
  rl = e - (rh - p);
}

__device__ __forceinline__ double pow_int_cr(double x, int n) {
  double rh = 1.0, rl = 0.0, bh = x, bl = 0.0;
  bool first = true;
  while (n) {
    if (n & 1) {
      if (first) {
        rh = bh;
        rl = bl;
        first = false;
      } else {
        dd_mul(rh, rl, bh, bl, rh, rl);
      }
    }
    n >>= 1;
    if (n) dd_mul(bh, bl, bh, bl, bh, bl);
  }
  return rh + rl;
}

// x / y for y > 0 (finite, nonzero).  IEEE gives x exactly (signed zero
// kept) when x == 0.  A zero numerator sends the inline division to its
// out-of-line slow path (stopped vehicles, v == 0, are the common case in
// queues: that call dominated the update kernel, profiles/r1a_*), and a
// plain `x == 0 ? x : x / y` does not help because the compiler speculates
// the division.  Dividing an opaque copy of (z ? 1.0 : x) -- the asm
// barrier stops the compiler from folding the select back into x -- keeps
// every division on the fast path.
__device__ __forceinline__ double div_pos(double x, double y) {
  const bool z = (x == 0.0);
  double n = z ? 1.0 : x;
  asm("mov.b64 %0, %0;" : "+d"(n));
  const double q = n / y;
  return z ? x : q;
}

// x**4 correctly rounded: pow_int_cr(x, 4) with the loop unrolled (the same
// operations in the same order, so the same bits).
__device__ __forceinline__ double pow4_cr(double x) {
  double h, l;
  dd_mul(x, 0.0, x, 0.0, h, l);
  dd_mul(h, l, h, l, h, l);
  return h + l;
}

#ifndef UPD_RCPV0
#define UPD_RCPV0 0  // 1: v / v0 by reciprocal + Markstein correction (exact, but measured 17% slower in k_update, r2)
#endif

// x / b for a divisor fixed for the run, given y = RN(1/b): q = RN(x*y) is
// within one ulp of x/b, the residual x - b*q is exact (FMA), and
// RN(q + r*y) is the correctly rounded quotient (Markstein's theorem) as
// long as nothing under- or overflows -- x outside [2^-900, 2^900] takes the
// division (never on the model's data: vdv is a product of speeds); zero
// keeps its sign.
__device__ __forceinline__ double div_rcp(double x, double b, double y) {
  const double q = x * y;
  const double r = fma(-b, q, x);
  double out = fma(r, y, q);
  const int ex = (__double2hiint(x) >> 20) & 0x7ff;
  if (ex < 1023 - 900 || ex > 1023 + 900) out = x / b;
  return x == 0.0 ? x : out;
}

// Free-road term (v / v0_eff)**delta (idm.py:24-25).
// G: glibc-pow arithmetic (compile-time, so each k_update instantiation only
// carries the code of its own mode).
template <bool G>
__device__ __forceinline__ double idm_free(const Params& p, double v, double v0_eff) {
#if UPD_RCPV0
  // v0_eff == v0 (the lane's cap is not lower): the correctly rounded
  // quotient by the run constant's reciprocal (div_rcp), else the division
  const double x = (v0_eff == p.v0 && p.rcp_v0 != 0.0) ? div_rcp(v, p.v0, p.rcp_v0) : div_pos(v, v0_eff);
#else
  const double x = div_pos(v, v0_eff);
#endif
  if (G) return glibc_pow::pow(x, p.delta);
  if (p.delta_int == 4) return pow4_cr(x);  // the default delta (params.py)
  return p.delta_int ? pow_int_cr(x, p.delta_int) : pow(x, p.delta);
}

// idm.py:26-31 given the free term.  (s*/gap)**2 is the correctly rounded
// square, i.e. q*q.
// The interaction division is evaluated with a dummy divisor on a free road
// (gap == inf): the compiler speculates it past the branch, and s*/inf == 0
// would take the division slow path for every leaderless vehicle.
template <bool G>
__device__ __forceinline__ double idm_with_free(const Params& p, double fr, double v, double dv, double gap) {
  const bool free_road = isinf(gap);
  const double vdv = v * dv;
  const double s_star = p.s0 + py_max(0.0, v * p.T + (p.ab2_pow2 ? vdv * p.inv_ab2
                                                      : p.rcp_ab2 != 0.0 ? div_rcp(vdv, p.sqrt_ab2, p.rcp_ab2)
                                                                         : div_pos(vdv, p.sqrt_ab2)));
  double g = free_road ? 1.0 : gap;
  asm("mov.b64 %0, %0;" : "+d"(g));
  const double q = div_pos(s_star, g);
  const double inter = free_road ? 0.0 : (G ? glibc_pow::pow(q, 2.0) : q * q);
  return p.a_max * (1.0 - fr - inter);
}

// idm_with_free for a gap that may be <= 0 where the caller discards the
// result (branch-free MOBIL evaluation): a safe divisor keeps the division
// on its fast path; for gap > 0 it is the same expression, bit for bit.
template <bool G>
__device__ __forceinline__ double idm_safe(const Params& p, double fr, double v, double dv, double gap) {
  return idm_with_free<G>(p, fr, v, dv, gap > 0.0 ? gap : 1.0);
}

// idm.py:17-31.
template <bool G>
__device__ __forceinline__ double idm_accel(const Params& p, double v, double dv, double gap, double v_cap) {
  return idm_with_free<G>(p, idm_free<G>(p, v, py_min(p.v0, v_cap)), v, dv, gap);
}

// rng.py:24-41: splitmix64 finaliser fold over (seed, stream, id, step).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
// The last two folds of keyed_uniform4(seed, 1, key, step) from the state
// after the first two (a run constant, Params::rng_h2).
__device__ __forceinline__ double keyed_uniform_tail(uint64_t h2, uint64_t key, uint64_t step) {
  const uint64_t G = 0x9E3779B97F4A7C15ULL;
  uint64_t h = mix64(h2 + G + key);
  h = mix64(h + G + step);
  return (double)(h >> 11) * 0x1p-53;
}
__device__ __forceinline__ double keyed_uniform4(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  const uint64_t G = 0x9E3779B97F4A7C15ULL;
  uint64_t h = mix64(0 + G + a);
  h = mix64(h + G + b);
  h = mix64(h + G + c);
  h = mix64(h + G + d);
  return (double)(h >> 11) * 0x1p-53;
}

// (s desc, vix asc): true if (sa, va) sorts before (sb, vb) in a lane.
__device__ __forceinline__ bool ahead_of(double sa, int32_t va, double sb, int32_t vb) {
  return sa > sb || (sa == sb && va < vb);
}

}  // namespace tsb
