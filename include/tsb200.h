/*
 * tsb200.h -- C-ABI of the B200-native MOSS per-step vehicle loop.
 *
 * The reference (trafficsim, pure Python) has no FFI: the hot path sits behind
 * the Python class trafficsim.engine.world.World (engine/world.py:111-834,
 * re-exported at engine/__init__.py:18-27).  This header is the boundary that
 * replaces it: paper_2405_12520_b200.world.World (the drop-in Python class)
 * binds these symbols with ctypes.  Each entry point names the reference
 * interface it replaces.  All calls are synchronous with respect to the
 * engine's CUDA stream unless stated; an engine is single-threaded (one
 * caller, control calls only between steps).
 *
 * Inputs are plain host pointers and sizes; they are copied on create.
 * Outputs go to caller-allocated buffers.  No torch types cross this line.
 *
 * Return codes: TSB_OK (0) or a negative code; tsb_last_error() gives the
 * thread-local message.  TSB_EINVAL / TSB_ERANGE map to InputError,
 * everything else to EngineError (a TrafficSimError).
 */
#ifndef TSB200_H
#define TSB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSB_OK 0
#define TSB_EINVAL (-1) /* bad argument            -> InputError  */
#define TSB_ERANGE (-2) /* index out of range      -> InputError  */
#define TSB_ECUDA (-3)  /* CUDA runtime failure    -> EngineError */
#define TSB_ECAP (-4)   /* device capacity exceeded -> EngineError */
#define TSB_EHOST (-5)  /* host-side failure (alloc, internal) */

#define TSB_KIND_ROAD 0
#define TSB_KIND_CONNECTOR 1
#define TSB_KIND_NONE (-1)

#define TSB_STATUS_WAITING 0
#define TSB_STATUS_DRIVING 1
#define TSB_STATUS_FINISHED 2
#define TSB_STATUS_DROPPED 3

/* Lane-level network, SoA; lane index == reference lane id.
 * Replaces the per-lane tables of World.__init__ (world.py:127-179). */
typedef struct tsb_network {
  int32_t n_lanes;
  const double* lane_len;
  const double* lane_cap;        /* max_speed */
  const int8_t* lane_kind;       /* TSB_KIND_* */
  const uint8_t* lane_open;      /* restriction == "open" */
  const int32_t* lane_left;      /* -1 = none */
  const int32_t* lane_right;
  const int32_t* lane_road;      /* road index of a road lane, -1 for connectors */
  const int32_t* lane_junction;  /* junction index of a connector, -1 for road lanes */
  const int32_t* lane_pred1;     /* connector: its single predecessor road lane */
  const int32_t* lane_succ1;     /* connector: its single successor road lane */
  const int32_t* succ_off;       /* [n_lanes+1] CSR of lane.successors (sorted) */
  const int32_t* succ;
  const int32_t* pred_off;       /* [n_lanes+1] CSR of lane.predecessors (sorted) */
  const int32_t* pred;
  int32_t n_roads;
  const int32_t* road_lane_off;  /* [n_roads+1] CSR of net.roads[rid] (leftmost first) */
  const int32_t* road_lanes;
  int32_t n_junctions;
  const uint8_t* junc_signal;    /* 1 = has a signal program */
  const int32_t* junc_phase_off; /* [n_junctions+1] CSR into phase_dur */
  const double* phase_dur;
  const uint64_t* lane_green_mask; /* connector: bit p set iff green in phase p */
  const int32_t* junc_phase0;      /* initial state (signals.initial_state) */
  const double* junc_elapsed0;
} tsb_network;

/* Trips in ascending-id order: index == vix (dense vehicle index).
 * Replaces list[Trip] (demand.py:47-53) as consumed by World (world.py:181-198). */
typedef struct tsb_trips {
  int32_t n;
  const uint64_t* key;  /* id & (2^64-1): the keyed-RNG vehicle key (rng.py:35) */
  const int32_t* origin_lane;
  const double* origin_s;
  const int32_t* dest_lane;
  const double* departure;
} tsb_trips;

/* EngineConfig (params.py:48-83) flattened; seed = World seed & (2^64-1). */
typedef struct tsb_params {
  double dt, lookahead;
  double idm_v0, idm_T, idm_a_max, idm_b, idm_delta, idm_s0;
  double mobil_politeness, mobil_threshold, mobil_b_safe, mobil_eval_prob;
  double vehicle_length, speed_window, amber, s0_floor, mp_interval, mp_min_green;
  int32_t controller; /* 0 = fixed, 1 = max_pressure */
  int32_t pow_mode;   /* 1 = glibc pow() bit for bit, as CPython's `**` (default);
                       * 0 = correctly rounded powers.  See DESIGN.md. */
  uint64_t seed;
} tsb_params;

/* StepReport (world.py:72-80) plus engine counters. */
typedef struct tsb_report {
  double time;
  int64_t step_no;
  int64_t driving, waiting, finished, dropped, injected_now, finished_now;
  int64_t vehicle_updates; /* cumulative, world.py:663 */
  int64_t reverts_last;    /* collision-sweep reverts in the last step */
  int64_t resolve_sequential; /* steps whose revert chains needed the sequential replay */
  int64_t reverts_total;      /* collision-sweep reverts, cumulative */
} tsb_report;

typedef struct tsb_engine tsb_engine;

/* World.__init__ (world.py:112-206): upload network/trips, compute routes on
 * the host router (routing.py:19-107), build the step graph. */
int tsb_create(const tsb_network* net, const tsb_trips* trips, const tsb_params* p,
               int32_t device, tsb_engine** out);
void tsb_destroy(tsb_engine* e); /* World.close (world.py:827-830) */
const char* tsb_last_error(void);

/* Sharded (multi-GPU) engine: lanes partitioned into spatial
 * bands, each rank simulating its own lanes plus a halo of ghost lanes
 * (paper_2405_12520_b200/shard.py computes the plan).  No reference
 * counterpart: the reference is single-process (world.py:664-669 threads). */
typedef struct tsb_shard {
  int32_t rank, nranks;        /* 1 <= nranks <= 8 */
  const uint8_t* zone;         /* per lane: 1 own, 2 halo (ghost), | 4 computed exactly; 0 outside */
  const int32_t* export_off;   /* [nranks+1] CSR over export_lanes, by destination rank */
  const int32_t* export_lanes; /* own lanes in each peer's halo, ascending */
  const int32_t* import_off;   /* [nranks+1] CSR over import_lanes, by source rank */
  const int32_t* import_lanes; /* each peer's lanes in my halo, ascending */
  /* Per export / import entry (NULL = all 0): 0 = a halo lane (its vehicles
   * travel as ghosts); 1 = a max-pressure lane: only its post-sweep vehicle
   * count travels (signals.py:64-86 reads it for a junction the receiver
   * computes).  Kind-1 entries follow the kind-0 entries of their peer. */
  const uint8_t* export_kind;
  const uint8_t* import_kind;
} tsb_shard;
int tsb_create_sharded(const tsb_network* net, const tsb_trips* trips, const tsb_params* p, int32_t device,
                       const tsb_shard* shard, tsb_engine** out);
/* The same with the rank's zone renumbered into a compact local lane space
 * (shard.local_network): `local_net` holds only the rank's lanes (own, halo,
 * max-pressure lanes) with local ids, local_to_global[local] = global id
 * (ascending, so every lane-id order and tie-break is unchanged), `shard`
 * uses local ids, the trips global ids; routes are computed on `global_net`
 * (the road ids of a route are global in both).  Every lane-proportional
 * buffer and kernel of the rank shrinks to its zone. */
int tsb_create_sharded_local(const tsb_network* global_net, const tsb_network* local_net,
                             const int32_t* local_to_global, const tsb_trips* trips, const tsb_params* p,
                             int32_t device, const tsb_shard* shard, tsb_engine** out);
/* After a step: pack the boundary lanes for every peer into `send` (device
 * memory of `cap` bytes); bytes[q] = size of the message to rank q. */
int tsb_shard_export(tsb_engine* e, void* send, int64_t cap, int64_t* bytes);
/* Before the next step: ghosts from `recv` (device memory, the peers'
 * messages concatenated in rank order, bytes[q] each). */
int tsb_shard_import(tsb_engine* e, const void* recv, const int64_t* bytes);

/* Device-driven exchange over peer memory (replaces export + the host's
 * all-to-all + import; NVLink P2P between GPUs, CUDA IPC between processes):
 * tsb_shard_p2p_alloc returns this rank's receive slots (2 x nranks slots of
 * *slot_bytes) and arrival flags (2 x nranks u64), both cudaMalloc bases, so
 * tsb_ipc_handle can export them; every rank opens its peers' with
 * tsb_ipc_open and passes them (rank order, own entry ignored) to
 * tsb_shard_p2p_set_peers.  From then on every step (tsb_step, in the step
 * graph) ends with the exchange: the pack written straight into each peer's
 * slot, a release of the peer's flag, the wait for every peer's flag and the
 * ghost import -- on the engine stream, no host synchronisation.
 * tsb_shard_p2p_exchange enqueues one exchange on its own (the initial
 * ghosts, before the first step). */
int tsb_shard_p2p_alloc(tsb_engine* e, void** recv, void** flags, int64_t* slot_bytes);
int tsb_shard_p2p_set_peers(tsb_engine* e, void* const* peer_recv, void* const* peer_flags);
int tsb_shard_p2p_exchange(tsb_engine* e);
/* The device-side wait for a peer's arrival flag is bounded (default 60 s):
 * on expiry the step completes with garbage ghosts and the next synchronising
 * call returns TSB_ECUDA ("peer stopped stepping") instead of hanging. */
int tsb_set_p2p_timeout(tsb_engine* e, double seconds);
/* Bytes this rank's device-driven exchange wrote into its peers' receive
 * slots since creation (per-lane count headers + 32 B records). */
int tsb_exchange_bytes(tsb_engine* e, int64_t* out);
/* cudaIpcGetMemHandle / cudaIpcOpenMemHandle / cudaIpcCloseMemHandle
 * (64-byte handles). */
#define TSB_IPC_HANDLE_BYTES 64
int tsb_ipc_handle(const void* dev_ptr, uint8_t* handle);
int tsb_ipc_open(const uint8_t* handle, void** dev_ptr);
int tsb_ipc_close(void* dev_ptr);

/* World.step() x n (world.py:659-689); report of the last step (may be NULL). */
int tsb_step(tsb_engine* e, int32_t n_steps, tsb_report* last);
/* tsb_step without the final synchronisation (errors surface at the next
 * synchronising call); for pipelines such as the sharded P2P loop. */
int tsb_step_async(tsb_engine* e, int32_t n_steps);
/* Current counters without stepping. */
int tsb_report_get(tsb_engine* e, tsb_report* out);

/* World.prepare() (world.py:211-242): the per-lane index.  Fills the
 * lane-sorted snapshot (lane asc, s desc, id asc): lane_start[n_lanes+1] and
 * per-vehicle vix/lane/road_pos/s/v arrays of capacity >= n_driving
 * (n_trips suffices; a sharded engine also lists its halo lanes' ghosts:
 * capacity 2 * n_trips, filter by the shard's zone). */
int tsb_state(tsb_engine* e, int32_t* n_driving, int32_t* lane_start, int32_t* vix,
              int32_t* lane, int32_t* road_pos, double* s, double* v);
/* Per-vix status (TSB_STATUS_*), finish time, and for finished vehicles the
 * last committed state (lane, s, v, road_pos) before the arrival step, which
 * is what World.get_vehicle reports for them (world.py:488-494, 706-714).
 * Any output pointer may be NULL. */
int tsb_status(tsb_engine* e, uint8_t* status, double* finish_time, int32_t* last_lane, double* last_s,
               double* last_v, int32_t* last_rp);
/* World.finished (world.py:199, 491): arrivals appended since index `since`
 * in reference order (step, then id).  *n_out = number written. */
int tsb_finished(tsb_engine* e, int64_t since, int64_t cap, int32_t* vix, double* finish_time,
                 int64_t* n_out);
/* Road aggregate (world.py:649-657): per (road, window) speed sum and count,
 * row-major [n_roads][n_windows]; windows beyond the engine's range are 0. */
int tsb_road_acc(tsb_engine* e, int32_t n_windows, double* sum, int64_t* count);
/* World.min_front_gap (world.py:694-704), computed on device. */
int tsb_min_front_gap(tsb_engine* e, double* out);

/* Per-id query: World.get_vehicle -> StatusView (world.py:83-92, 706-714),
 * answered on the device for just the requested vehicles (a locator kernel
 * maps vix -> snapshot record, then one gather per query).
 * status: TSB_STATUS_*; driving: the snapshot state (world.py:712); finished:
 * the last committed state before arrival (world.py:488-494) and finish_time;
 * waiting/dropped: origin lane and s, v = 0, road_pos = 0.  A sharded engine
 * reports TSB_STATUS_ELSEWHERE for a vehicle driving on another rank's lanes. */
#define TSB_STATUS_ELSEWHERE (-1)
typedef struct tsb_vehicle_view {
  double s, v;
  double finish_time; /* finished vehicles only */
  int32_t lane;
  int32_t road_pos;   /* roads_seq index; route_index = 2*road_pos + (lane is a connector) */
  int32_t status;
  int32_t pad;
} tsb_vehicle_view;
int tsb_get_vehicles(tsb_engine* e, const int32_t* vix, int32_t n, tsb_vehicle_view* out);

/* Lane geometry for record angles (geometry.py:22-52): per lane, the
 * centerline segments [geo_off[l], geo_off[l+1]), each with its start arc
 * position geo_cum[k] and its heading geo_angle[k] in degrees (evaluated on
 * the host with the reference's own expression: math.degrees(atan2(dx, dy))
 * % 360).  Copied to the device; required before tsb_records. */
int tsb_set_geometry(tsb_engine* e, const int64_t* geo_off, int64_t n_segments, const double* geo_cum,
                     const double* geo_angle);
/* World.record_step (world.py:771-782) as a batch: every driving vehicle of
 * the snapshot (a sharded engine: of its own lanes) in ascending id (vix)
 * order, with its heading at min(s, lane length) (geometry.py:30-52: the
 * segment by bisect_right on the cumulative lengths), gathered and ordered
 * on the device.  Arrays of capacity `cap`; *n = records written.  Any
 * output pointer may be NULL. */
int tsb_records(tsb_engine* e, int32_t cap, int32_t* vix, int32_t* lane, int32_t* road_pos, double* s,
                double* v, double* angle_deg, int32_t* n);

/* Control surface, between steps only (world.py:716-740). */
int tsb_set_lane(tsb_engine* e, int32_t lane, double max_speed, int32_t open);
int tsb_set_signal_phase(tsb_engine* e, int32_t junction, int32_t phase);
/* Signal state per junction: phase, elapsed (signals.py:22-26). */
int tsb_signal_state(tsb_engine* e, int32_t* phase, double* elapsed);

/* Host router (routing.py:70-107): lane path origin -> dest on the engine's
 * current lane state.  Returns TSB_OK and *n = 0 when unroutable. */
int tsb_route(tsb_engine* e, int32_t origin, int32_t dest, int32_t cap, int32_t* lanes,
              int32_t* n, double* cost);

/* Native grid builder (host only, no device): the flattened arrays of
 * trafficsim's generate_grid(rows, cols, block_length, lanes_per_direction,
 * max_speed) compiled by build_network (network.py:367-560) -- the same lane
 * numbering, geometry and signal programs -- without Python objects.
 * tsb_grid_sizes: sizes[0..9] = lanes, successors, predecessors, roads, road
 * lanes, junctions, phases, geometry segments, bytes of the '\n'-joined road
 * ids, bytes of the junction ids.  tsb_grid_export copies into 28 caller
 * buffers, in this order (NULL skips one): lane_len, lane_cap, lane_kind,
 * lane_open, lane_left, lane_right, lane_road, lane_junction, lane_pred1,
 * lane_succ1, succ_off, succ, pred_off, pred, road_lane_off, road_lanes,
 * junc_signal, junc_phase_off, phase_dur, lane_green_mask, junc_phase0,
 * junc_elapsed0, geo_off (int64), geo_cum, geo_angle, junction positions
 * (x, y per junction), road ids, junction ids. */
typedef struct tsb_grid tsb_grid;
int tsb_grid_build(int32_t rows, int32_t cols, double block_length, int32_t lanes_per_direction,
                   double max_speed, int32_t controller, tsb_grid** out);
int tsb_grid_sizes(const tsb_grid* g, int64_t* sizes);
int tsb_grid_export(const tsb_grid* g, void* const* dst);
void tsb_grid_destroy(tsb_grid* g);
/* CPython's math.dist for two points (the grid builder's lengths; test hook). */
double tsb_py_dist(double ax, double ay, double bx, double by);

/* Standalone router (no device): used by demand generators and tests. */
typedef struct tsb_router tsb_router;
int tsb_router_create(const tsb_network* net, tsb_router** out);
void tsb_router_destroy(tsb_router* r);
int tsb_router_route(tsb_router* r, int32_t origin, int32_t dest, int32_t cap, int32_t* lanes,
                     int32_t* n, double* cost);
/* reach[k*n_lanes + l] = 1 iff lane l reaches dests[k] (dist_to keys). */
int tsb_router_reach(tsb_router* r, int32_t n_dests, const int32_t* dests, uint8_t* reach);

/* Measurement hooks for bench.py: run n steps launching each kernel with
 * CUDA events on the engine stream; kernel_ms[k] = mean per-step duration of
 * kernel class k, names via tsb_kernel_name(k). Returns number of classes. */
int tsb_profile_steps(tsb_engine* e, int32_t n_steps, int32_t cap, double* kernel_ms);
const char* tsb_kernel_name(int32_t k);
/* Device time (ms) of n graph-replayed steps bracketed by CUDA events. */
int tsb_time_steps(tsb_engine* e, int32_t n_steps, double* ms);
/* Switch the power arithmetic between steps (tsb_params.pow_mode). */
int tsb_set_pow_mode(tsb_engine* e, int32_t pow_mode);
/* Timing marks on the engine stream (slots 0..7): record, then elapsed ms
 * between two recorded marks (waits for the later one). */
int tsb_mark(tsb_engine* e, int32_t slot);
int tsb_marks_elapsed(tsb_engine* e, int32_t a, int32_t b, double* ms);
/* Test knobs: bit 0 forces the sequential revert-chain resolver, bit 1 the
 * full (non-incremental) regroup, bit 2 the general (closure + components)
 * resolver instead of the per-event fast path, bit 3 a step graph without
 * conditional nodes (every section's kernels launched, gating themselves),
 * bit 4 the parallel branches at default (not highest) priority, bit 5
 * one graph replay per step (no multi-step batch graph), bit 6 the
 * snapshot-isolation check: before each update the step's write-before-read
 * buffers (post-update records, sort scratch, the next layout) are filled
 * with 0xff bytes (NaN / -1), so any read outside the snapshot shows.
 * Results must not change. */
int tsb_set_debug(tsb_engine* e, int32_t flags);
/* Which step paths ran so far (measurement hook): out[0] steps whose revert
 * events were all replayed by the per-event fast path, out[1] steps that
 * needed the general resolver, out[2] incremental (patch) regroups, out[3]
 * full regroups, out[4] steps that ran the injection section. */
#define TSB_PATH_COUNTERS 5
int tsb_path_counters(tsb_engine* e, int64_t* out);
/* Step timeline.  While on (tsb_set_timeline; turning it on clears the
 * ring), every step kernel's block 0 stamps %globaltimer when it passed its
 * dependency wait: out[TSB_TL_ROWS * TSB_TL_SLOTS] = stamps (ns) of the last
 * TSB_TL_ROWS steps, a ring of rows, slot = phase (kernels.cu TL_*; 0 =
 * step begin, 1 = k_update, 2 = lane scan, 7 = step end).  Used by bench.py
 * for the in-graph kernel durations of the timed window. */
#define TSB_TL_ROWS 1024
#define TSB_TL_SLOTS 16
int tsb_set_timeline(tsb_engine* e, int32_t on);
int tsb_timeline(tsb_engine* e, uint64_t* out);
/* Kernel launches every step issues (for the bench's gpu_launches claim):
 * the step graph's kernels outside its conditional (RARE) body. */
int tsb_launches_per_step(tsb_engine* e, int32_t* n);
/* Bytes a synchronising call (tsb_step, tsb_report_get) reads back from the
 * device: the step scalars (StepReport counters, error flags). */
int tsb_step_sync_bytes(int64_t* n);
/* Measured fp64 FMA throughput of a device (TFLOP/s, 2 flops per DFMA):
 * the denominator bench.py reports k_update's fp64 rate against. */
int tsb_fp64_peak(int32_t device, double* tflops);

#ifdef __cplusplus
}
#endif
#endif
