"""Flatten a ``RoadNetwork`` + trips + ``EngineConfig`` into struct-of-arrays.

This is the upload format for the C-ABI (``include/tsb200.h``: tsb_network,
tsb_trips, tsb_params).  It restates the per-lane tables that
``World.__init__`` builds (trafficsim/engine/world.py:127-179) and the trip
validation it performs (world.py:181-198):

* lane ids are kept verbatim (index = reference lane id); holes get kind -1;
* ``lane_road`` maps a road lane to the index of its parent road in
  ``net.roads`` order, connectors to -1; ``lane_junction`` maps a connector
  to its junction index (sorted junction ids);
* successor / predecessor lists are CSR, in the reference's sorted order, so
  "first successor connector whose target lies on road R" is the reference's
  ``_conn_from`` smallest-id rule (world.py:155-166);
* signal programs become per-junction phase durations plus one 64-bit green
  mask per connector; the initial fixed-time state (offset pre-advance,
  signals.py:29-43) is computed here in Python so it is bit-identical;
* vehicles get a dense index ``vix`` in ascending-id order: every id
  tie-break in the reference is then a ``vix`` comparison, and the RNG key is
  ``id & (2**64-1)`` (rng.py:35).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InputError
from .network import CONNECTOR, OPEN, ROAD, heading_at, vertex_arclengths
from .params import FIXED

MASK64 = (1 << 64) - 1
KIND_ROAD, KIND_CONNECTOR, KIND_NONE = 0, 1, -1


@dataclass
class FlatNet:
    n_lanes: int
    lane_len: np.ndarray
    lane_cap: np.ndarray
    lane_kind: np.ndarray
    lane_open: np.ndarray
    lane_left: np.ndarray
    lane_right: np.ndarray
    lane_road: np.ndarray
    lane_junction: np.ndarray
    lane_pred1: np.ndarray
    lane_succ1: np.ndarray
    succ_off: np.ndarray
    succ: np.ndarray
    pred_off: np.ndarray
    pred: np.ndarray
    road_ids: list
    road_lane_off: np.ndarray
    road_lanes: np.ndarray
    junction_ids: list
    junc_signal: np.ndarray
    junc_phase_off: np.ndarray
    phase_dur: np.ndarray
    lane_green_mask: np.ndarray
    junc_phase0: np.ndarray
    junc_elapsed0: np.ndarray
    # host-only geometry for the record angle (geometry.py:45-52)
    geo_off: np.ndarray
    geo_cum: np.ndarray
    geo_angle: np.ndarray


@dataclass
class FlatTrips:
    ids: list            # python ints, ascending (index = vix)
    key: np.ndarray      # uint64
    origin_lane: np.ndarray
    origin_s: np.ndarray
    dest_lane: np.ndarray
    departure: np.ndarray


def _advance_fixed(phase: int, elapsed: float, durs: list[float], dt: float):
    elapsed += dt
    while elapsed >= durs[phase]:
        elapsed -= durs[phase]
        phase = (phase + 1) % len(durs)
    return phase, elapsed


def flatten_network(net, controller: str = FIXED) -> FlatNet:
    n = (max(net.lanes) + 1) if net.lanes else 0
    f64 = lambda v=0.0: np.full(n, v, dtype=np.float64)
    i32 = lambda v=-1: np.full(n, v, dtype=np.int32)
    lane_len, lane_cap = f64(0.0), f64(1.0)
    lane_kind = np.full(n, KIND_NONE, dtype=np.int8)
    lane_open = np.zeros(n, dtype=np.uint8)
    lane_left, lane_right, lane_road, lane_junc = i32(), i32(), i32(), i32()
    lane_pred1, lane_succ1 = i32(), i32()
    road_ids = list(net.roads)
    road_index = {rid: k for k, rid in enumerate(road_ids)}
    junction_ids = sorted(net.junctions)
    junc_index = {jid: k for k, jid in enumerate(junction_ids)}
    succ_lists = [[] for _ in range(n)]
    pred_lists = [[] for _ in range(n)]
    geo_off = np.zeros(n + 1, dtype=np.int64)
    cums, angs = [], []
    for lid in range(n):
        lane = net.lanes.get(lid)
        if lane is not None:
            lane_len[lid] = lane.length
            lane_cap[lid] = lane.max_speed
            lane_open[lid] = 1 if lane.restriction == OPEN else 0
            lane_left[lid] = -1 if lane.left is None else lane.left
            lane_right[lid] = -1 if lane.right is None else lane.right
            succ_lists[lid] = list(lane.successors)
            pred_lists[lid] = list(lane.predecessors)
            if lane.kind == ROAD:
                lane_kind[lid] = KIND_ROAD
                lane_road[lid] = road_index[lane.parent]
            elif lane.kind == CONNECTOR:
                lane_kind[lid] = KIND_CONNECTOR
                lane_junc[lid] = junc_index[lane.parent]
                lane_succ1[lid] = lane.successors[0]
                lane_pred1[lid] = lane.predecessors[0]
            pts = lane.centerline
            cum = vertex_arclengths(pts)
            cums.extend(cum[:-1])
            angs.extend(heading_at(pts, cum, cum[k]) for k in range(len(pts) - 1))
            geo_off[lid + 1] = geo_off[lid] + len(pts) - 1
        else:
            geo_off[lid + 1] = geo_off[lid]
    succ_off = np.zeros(n + 1, dtype=np.int32)
    pred_off = np.zeros(n + 1, dtype=np.int32)
    succ_off[1:] = np.cumsum([len(x) for x in succ_lists]) if n else []
    pred_off[1:] = np.cumsum([len(x) for x in pred_lists]) if n else []
    succ = np.array([x for xs in succ_lists for x in xs], dtype=np.int32)
    pred = np.array([x for xs in pred_lists for x in xs], dtype=np.int32)

    road_lane_off = np.zeros(len(road_ids) + 1, dtype=np.int32)
    road_lane_off[1:] = np.cumsum([len(net.roads[r]) for r in road_ids]) if road_ids else []
    road_lanes = np.array([l for r in road_ids for l in net.roads[r]], dtype=np.int32)

    nj = len(junction_ids)
    junc_signal = np.zeros(nj, dtype=np.uint8)
    junc_phase_off = np.zeros(nj + 1, dtype=np.int32)
    phase_dur: list[float] = []
    green = np.zeros(n, dtype=np.uint64)
    phase0 = np.zeros(nj, dtype=np.int32)
    elapsed0 = np.zeros(nj, dtype=np.float64)
    for k, jid in enumerate(junction_ids):
        prog = net.junctions[jid].signal
        if prog is not None:
            junc_signal[k] = 1
            if len(prog.phases) > 64:
                raise InputError(f"junction {jid}: more than 64 signal phases")
            durs = [p.duration for p in prog.phases]
            for pi, ph in enumerate(prog.phases):
                for c in ph.green:
                    green[c] |= np.uint64(1 << pi)
            phase_dur.extend(durs)
            if controller == FIXED:
                off = prog.offset % prog.cycle() if prog.phases else 0.0
                phase0[k], elapsed0[k] = _advance_fixed(0, 0.0, durs, off)
        junc_phase_off[k + 1] = len(phase_dur)
    return FlatNet(
        n_lanes=n, lane_len=lane_len, lane_cap=lane_cap, lane_kind=lane_kind,
        lane_open=lane_open, lane_left=lane_left, lane_right=lane_right,
        lane_road=lane_road, lane_junction=lane_junc, lane_pred1=lane_pred1,
        lane_succ1=lane_succ1, succ_off=succ_off, succ=succ, pred_off=pred_off,
        pred=pred, road_ids=road_ids, road_lane_off=road_lane_off,
        road_lanes=road_lanes, junction_ids=junction_ids, junc_signal=junc_signal,
        junc_phase_off=junc_phase_off, phase_dur=np.array(phase_dur, dtype=np.float64),
        lane_green_mask=green, junc_phase0=phase0, junc_elapsed0=elapsed0,
        geo_off=geo_off, geo_cum=np.array(cums, dtype=np.float64),
        geo_angle=np.array(angs, dtype=np.float64),
    )


def flatten_trips(flat: FlatNet, trips) -> FlatTrips:
    """Validate like world.py:181-198 and order by id (vix = rank of id)."""
    n = flat.n_lanes
    for t in trips:
        for lid in (t.origin_lane, t.dest_lane):
            if not (0 <= lid < n) or flat.lane_kind[lid] != KIND_ROAD:
                raise InputError(f"trip {t.id}: lane {lid} is not a road lane")
        if not 0.0 <= t.origin_s <= flat.lane_len[t.origin_lane]:
            raise InputError(f"trip {t.id}: origin_s outside its lane")
        if t.departure < 0:
            raise InputError(f"trip {t.id}: negative departure")
    ordered = sorted(trips, key=lambda t: t.id)
    for a, b in zip(ordered, ordered[1:]):
        if a.id == b.id:
            raise InputError("duplicate trip ids")
    return FlatTrips(
        ids=[t.id for t in ordered],
        key=np.array([t.id & MASK64 for t in ordered], dtype=np.uint64),
        origin_lane=np.array([t.origin_lane for t in ordered], dtype=np.int32),
        origin_s=np.array([t.origin_s for t in ordered], dtype=np.float64),
        dest_lane=np.array([t.dest_lane for t in ordered], dtype=np.int32),
        departure=np.array([t.departure for t in ordered], dtype=np.float64),
    )


def record_angles(f: FlatNet, lane: np.ndarray, s: np.ndarray) -> np.ndarray:
    """Heading (deg clockwise from north) per vehicle, as world.py:777-779.

    Angles were precomputed per centerline segment with the reference's own
    float expression (geometry.py:45-52); here only the segment is selected,
    by the same bisect rule (geometry.py:30-33) on s clamped to the lane.
    """
    lane = np.asarray(lane, dtype=np.int64)
    s = np.minimum(np.asarray(s, dtype=np.float64), f.lane_len[lane])
    lo = f.geo_off[lane]
    nseg = f.geo_off[lane + 1] - lo
    out = f.geo_angle[lo].copy() if lane.size else np.zeros(0)
    for k in np.nonzero(nseg > 1)[0]:
        a, b = int(lo[k]), int(lo[k] + nseg[k])
        i = int(np.searchsorted(f.geo_cum[a:b], s[k], side="right")) - 1
        out[k] = f.geo_angle[a + min(max(i, 0), b - a - 1)]
    return out
