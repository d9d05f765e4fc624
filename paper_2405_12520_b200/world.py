"""Drop-in ``World`` for the reference's trafficsim.engine.world.World.

Same constructor, methods, attributes, return types and errors as the
reference class (trafficsim/engine/world.py:111-834), but every step runs on
the B200 through the C-ABI in include/tsb200.h (csrc/): one CUDA graph per
step, the vehicle state resident in HBM, and host round trips only for
queries.  There is no CPU fallback: without the native library or a CUDA
device, construction raises ``EngineError``.

Queries run on the device: ``get_vehicle`` gathers just the requested
vehicle (tsb_get_vehicles), ``record_step`` / ``records_arrays`` receive the
id-sorted records with their headings (tsb_records).  ``prepare`` -- the
whole per-lane index of world.py:227-242 by definition -- downloads the
snapshot layout once per step.
"""

from __future__ import annotations

import ctypes as C
import math
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .cabi import VIEW_DTYPE, TsbReport, pack_network, pack_params, pack_trips
from .errors import InputError
from .flat import KIND_CONNECTOR, FlatNet, FlatTrips, flatten_network, flatten_trips
from .network import CLOSED, OPEN
from .params import EngineConfig
from .records import RoadWindow, VehicleRecord
from .routing import Router

WAITING = "waiting"
DRIVING = "driving"
FINISHED = "finished"
DROPPED = "dropped"
_STATUS = {0: WAITING, 1: DRIVING, 2: FINISHED, 3: DROPPED}
_INT32_MAX = 2**31 - 1
# IDM powers (idm.py:25, idm.py:30): POW_GLIBC evaluates them exactly as
# glibc's pow() -- what CPython's `**` calls -- so trajectories are bit-identical
# to the reference's; POW_CORRECT rounds them correctly.
POW_CORRECT, POW_GLIBC = 0, 1


_new = object.__new__


@dataclass(frozen=True)
class StepReport:
    time: float
    driving: int
    waiting: int
    finished: int
    dropped: int
    injected_now: int
    finished_now: int


# tsb_report (include/tsb200.h): time f64, step_no i64 (skipped), then the
# StepReport counters as i64, in StepReport's field order
_REPORT_FIELDS = ("time", "driving", "waiting", "finished", "dropped", "injected_now", "finished_now")
_REPORT_FMT = struct.Struct("<d8x6q")
assert tuple(StepReport.__dataclass_fields__) == _REPORT_FIELDS
assert [TsbReport.time.offset, TsbReport.driving.offset, TsbReport.finished_now.offset] == [0, 16, 56]


@dataclass
class StatusView:
    id: int
    lane_id: int
    s: float
    v: float
    status: str
    route_index: int
    depart_time: float
    finish_time: float | None


@dataclass
class SimulationOutput:
    steps: int
    dt: float
    finished: list[tuple[int, float, float]]
    driving_at_end: int
    unserved: int
    dropped: int
    total_trips: int
    road_windows: list[RoadWindow] = field(default_factory=list)
    vehicle_updates: int = 0

    def travel_durations(self) -> list[float]:
        return [fin - dep for _, dep, fin in self.finished]


def _route_index(flat: FlatNet, lane: int, rp: int) -> int:
    # route_index == 2 * road_pos + (lane is a connector): invariant of
    # world.py:478-487 under transitions, lane changes and reverts
    return 2 * rp + (1 if flat.lane_kind[lane] == KIND_CONNECTOR else 0)


def _nonempty_f64(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if a.size else np.zeros(1, dtype=np.float64)


class World:
    """B200 engine behind the reference ``World`` interface."""

    def __init__(self, net, trips, config: EngineConfig | None = None, seed: int = 0,
                 device: int = 0, _flat: FlatNet | None = None, _flat_trips: FlatTrips | None = None,
                 pow_mode: int = POW_GLIBC):
        config = config or EngineConfig()
        config.validate()
        self.net = net
        self.config = config
        self.seed = seed
        self._flat = _flat if _flat is not None else flatten_network(net, config.controller)
        self._ft = _flat_trips if _flat_trips is not None else flatten_trips(self._flat, trips)
        self.total_trips = len(self._ft.ids)
        self._h = None
        packed_net = pack_network(self._flat)
        packed_trips = pack_trips(self._ft)
        params = pack_params(config, seed, pow_mode=pow_mode)
        self.pow_mode = pow_mode
        h = C.c_void_p()
        _native.check(_native.lib().tsb_create(C.byref(packed_net.struct), C.byref(packed_trips.struct),
                                               C.byref(params), device, C.byref(h)))
        self._h = h
        f = self._flat
        geo_off = np.ascontiguousarray(f.geo_off, dtype=np.int64)
        geo_cum = _nonempty_f64(f.geo_cum)
        geo_ang = _nonempty_f64(f.geo_angle)
        _native.check(_native.lib().tsb_set_geometry(h, geo_off.ctypes.data, int(geo_off[-1]),
                                                     geo_cum.ctypes.data, geo_ang.ctypes.data))
        self.router = Router(net, flat=self._flat) if net is not None else None
        self._report = TsbReport()
        # step() hot path: the bound entry point, the report's argument and a
        # byte view of it (the StepReport fields in one unpack)
        self._step_fn = _native.lib().tsb_step
        self._report_ref = C.byref(self._report)
        self._report_mv = memoryview(self._report).cast("B")
        self._finished: list[tuple[int, float, float]] = []
        self._fin_seen = 0
        self._mirror = None
        self._acc = None
        self._vix_of = {tid: k for k, tid in enumerate(self._ft.ids)}
        self._road_index = {rid: k for k, rid in enumerate(self._flat.road_ids)}
        self._junc_index = {jid: k for k, jid in enumerate(self._flat.junction_ids)}

    @classmethod
    def from_flat(cls, flat: FlatNet, flat_trips: FlatTrips, config: EngineConfig | None = None,
                  seed: int = 0, device: int = 0, pow_mode: int = None) -> "World":
        """Construct from pre-flattened inputs (large synthetic configs)."""
        return cls(None, None, config, seed, device, _flat=flat, _flat_trips=flat_trips,
                   pow_mode=POW_GLIBC if pow_mode is None else pow_mode)

    # ------------------------------------------------------------ lifecycle

    def close(self) -> None:
        if self._h is not None:
            _native.lib().tsb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _live(self):
        if self._h is None:
            raise InputError("world is closed")
        return self._h

    # ------------------------------------------------------------ counters

    @property
    def time(self) -> float:
        return self._report.time

    @property
    def vehicle_updates(self) -> int:
        return self._report.vehicle_updates

    @property
    def dropped(self) -> int:
        return self._report.dropped

    @property
    def finished(self) -> list[tuple[int, float, float]]:
        total = self._report.finished
        if self._fin_seen < total:
            cap = total - self._fin_seen
            vix = np.zeros(cap, dtype=np.int32)
            t = np.zeros(cap, dtype=np.float64)
            n = C.c_int64()
            _native.check(_native.lib().tsb_finished(self._live(), self._fin_seen, cap, vix.ctypes.data,
                                                     t.ctypes.data, C.byref(n)))
            dep = self._ft.departure
            ids = self._ft.ids
            for k in range(n.value):
                i = int(vix[k])
                self._finished.append((ids[i], float(dep[i]), float(t[k])))
            self._fin_seen += n.value
        return self._finished

    def driving_count(self) -> int:
        return int(self._report.driving)

    def waiting_count(self) -> int:
        return int(self._report.waiting)

    # ------------------------------------------------------------ stepping

    def _advance(self, n: int) -> None:
        while n > 0:
            k = min(n, _INT32_MAX)
            _native.check(_native.lib().tsb_step(self._live(), k, C.byref(self._report)))
            n -= k
        self._mirror = None
        self._acc = None

    def step(self) -> StepReport:
        rc = self._step_fn(self._live(), 1, self._report_ref)
        if rc:
            _native.check(rc)
        self._mirror = None
        self._acc = None
        # StepReport(time, driving, waiting, finished, dropped, injected_now,
        # finished_now) from the tsb_report bytes, filled without the frozen
        # dataclass's per-field __setattr__ (a third of the call's host time)
        rep = _new(StepReport)
        rep.__dict__.update(zip(_REPORT_FIELDS, _REPORT_FMT.unpack_from(self._report_mv)))
        return rep

    def run(self, steps: int, recorder=None) -> SimulationOutput:
        if steps < 0:
            raise InputError("steps must be non-negative")
        start = self.vehicle_updates
        if recorder is None:
            self._advance(steps)
        else:
            for _ in range(steps):
                self.step()
                self.record_step(recorder)
        horizon = steps * self.config.dt
        return SimulationOutput(
            steps=steps, dt=self.config.dt, finished=list(self.finished),
            driving_at_end=self.driving_count(), unserved=self.waiting_count(),
            dropped=self.dropped, total_trips=self.total_trips,
            road_windows=self.road_windows(horizon) if steps else [],
            vehicle_updates=self.vehicle_updates - start,
        )

    # ------------------------------------------------------------ state mirror

    def _state(self):
        if self._mirror is not None:
            return self._mirror
        n = self.total_trips
        cap = max(n, 1)
        nd = C.c_int32()
        ls = np.zeros(self._flat.n_lanes + 1, dtype=np.int32)
        vix = np.zeros(cap, dtype=np.int32)
        lane = np.zeros(cap, dtype=np.int32)
        rp = np.zeros(cap, dtype=np.int32)
        s = np.zeros(cap, dtype=np.float64)
        v = np.zeros(cap, dtype=np.float64)
        h = self._live()
        _native.check(_native.lib().tsb_state(h, C.byref(nd), ls.ctypes.data, vix.ctypes.data,
                                              lane.ctypes.data, rp.ctypes.data, s.ctypes.data, v.ctypes.data))
        st = np.zeros(cap, dtype=np.uint8)
        fin = np.zeros(cap, dtype=np.float64)
        l_lane = np.zeros(cap, dtype=np.int32)
        l_s = np.zeros(cap, dtype=np.float64)
        l_v = np.zeros(cap, dtype=np.float64)
        l_rp = np.zeros(cap, dtype=np.int32)
        _native.check(_native.lib().tsb_status(h, st.ctypes.data, fin.ctypes.data, l_lane.ctypes.data,
                                               l_s.ctypes.data, l_v.ctypes.data, l_rp.ctypes.data))
        m = nd.value
        pos = np.full(cap, -1, dtype=np.int64)
        pos[vix[:m]] = np.arange(m)
        self._mirror = dict(n=m, lane_start=ls, vix=vix[:m], lane=lane[:m], rp=rp[:m], s=s[:m], v=v[:m],
                            status=st[:n], finish=fin[:n], l_lane=l_lane[:n], l_s=l_s[:n], l_v=l_v[:n],
                            l_rp=l_rp[:n], pos=pos)
        return self._mirror

    def prepare(self):
        """(lane id -> vehicle ids front-first, vehicle id -> (lane, s, v)); world.py:211-225."""
        m = self._state()
        ids = self._ft.ids
        index: dict[int, list[int]] = {}
        for k in range(m["n"]):
            index.setdefault(int(m["lane"][k]), []).append(ids[int(m["vix"][k])])
        snapshot = {ids[int(m["vix"][k])]: (int(m["lane"][k]), float(m["s"][k]), float(m["v"][k]))
                    for k in range(m["n"])}
        return index, snapshot

    def _route_index(self, lane: int, rp: int) -> int:
        return _route_index(self._flat, lane, rp)

    def vehicle_views(self, vix) -> np.ndarray:
        """Device-side StatusView data for dense vehicle indices (tsb_get_vehicles):
        a structured array (s, v, finish_time, lane, road_pos, status)."""
        q = np.ascontiguousarray(vix, dtype=np.int32)
        out = np.zeros(len(q), dtype=VIEW_DTYPE)
        _native.check(_native.lib().tsb_get_vehicles(self._live(), q.ctypes.data, len(q), out.ctypes.data))
        return out

    def _status_view(self, vehicle_id: int, k: int, o) -> StatusView:
        status = _STATUS[int(o["status"])]
        lane, rp = int(o["lane"]), int(o["road_pos"])
        return StatusView(id=vehicle_id, lane_id=lane, s=float(o["s"]), v=float(o["v"]), status=status,
                          route_index=self._route_index(lane, rp) if status in (DRIVING, FINISHED) else 0,
                          depart_time=float(self._ft.departure[k]),
                          finish_time=float(o["finish_time"]) if status == FINISHED else None)

    def get_vehicle(self, vehicle_id: int) -> StatusView:
        """world.py:706-714, answered on the device for this one vehicle."""
        k = self._vix_of.get(vehicle_id)
        if k is None:
            raise InputError(f"unknown vehicle {vehicle_id}")
        return self._status_view(vehicle_id, k, self.vehicle_views([k])[0])

    def min_front_gap(self) -> float:
        g = C.c_double()
        _native.check(_native.lib().tsb_min_front_gap(self._live(), C.byref(g)))
        return g.value

    # ------------------------------------------------------------ records

    def records_arrays(self) -> dict:
        """The step's vehicle records as numpy arrays, sorted by id -- the batch
        form of record_step (world.py:771-782), gathered,
        id-ordered and given their headings (geometry.py:45-52) on the device
        (tsb_records): keys ``t`` (float), ``vix`` (dense index), ``id``,
        ``lane``, ``road_pos``, ``s``, ``v``, ``angle_deg``."""
        n = max(self.total_trips, 1)
        vix = np.zeros(n, dtype=np.int32)
        lane = np.zeros(n, dtype=np.int32)
        rp = np.zeros(n, dtype=np.int32)
        s = np.zeros(n, dtype=np.float64)
        v = np.zeros(n, dtype=np.float64)
        ang = np.zeros(n, dtype=np.float64)
        m = C.c_int32()
        _native.check(_native.lib().tsb_records(self._live(), n, vix.ctypes.data, lane.ctypes.data, rp.ctypes.data,
                                                s.ctypes.data, v.ctypes.data, ang.ctypes.data, C.byref(m)))
        k = m.value
        vix = vix[:k]
        ids = self._ft.ids
        dense = len(ids) == 0 or (ids[0] == 0 and ids[-1] == len(ids) - 1)
        id_arr = vix.astype(np.int64) if dense else np.array([ids[i] for i in vix.tolist()], dtype=object)
        return {"t": self.time, "vix": vix, "id": id_arr, "lane": lane[:k], "road_pos": rp[:k], "s": s[:k],
                "v": v[:k], "angle_deg": ang[:k]}

    def record_step(self, recorder) -> None:
        """One VehicleRecord per driving vehicle, sorted by id (world.py:771-782)."""
        r = self.records_arrays()
        t = r["t"]
        ids = self._ft.ids
        for i, l, a, b, g in zip(r["vix"].tolist(), r["lane"].tolist(), r["s"].tolist(), r["v"].tolist(),
                                 r["angle_deg"].tolist()):
            recorder.write(VehicleRecord(t=t, id=ids[i], lane=l, s=a, v=b, angle_deg=g))

    # ------------------------------------------------------------ road aggregate

    def _road_acc(self):
        if self._acc is None:
            nw = int(self.time / self.config.speed_window) + 2
            nr = len(self._flat.road_ids)
            s = np.zeros((max(nr, 1), nw), dtype=np.float64)
            c = np.zeros((max(nr, 1), nw), dtype=np.int64)
            _native.check(_native.lib().tsb_road_acc(self._live(), nw, s.ctypes.data, c.ctypes.data))
            self._acc = (s[:nr], c[:nr])
        return self._acc

    def road_free_flow(self, road_id: str) -> float:
        lids = self.net.roads[road_id] if self.net is not None else \
            self._flat.road_lanes[self._flat.road_lane_off[self._road_index[road_id]]:
                                  self._flat.road_lane_off[self._road_index[road_id] + 1]]
        return sum(float(self._flat.lane_cap[lid]) for lid in lids) / len(lids)

    def get_road_speed(self, road_id: str, window: tuple[float, float]) -> float:
        """Mean recorded speed on a road over [t0, t1); free-flow if empty (world.py:746-761)."""
        if road_id not in self._road_index:
            raise InputError(f"unknown road {road_id}")
        t0, t1 = window
        w = self.config.speed_window
        s, c = self._road_acc()
        r = self._road_index[road_id]
        total, count = 0.0, 0
        for wi in range(int(t0 // w), int(math.ceil(t1 / w))):
            if 0 <= wi < s.shape[1] and c[r, wi] > 0:
                total += float(s[r, wi])
                count += int(c[r, wi])
        if count == 0:
            return self.road_free_flow(road_id)
        return total / count

    def road_windows(self, horizon: float) -> list[RoadWindow]:
        w = self.config.speed_window
        n_windows = max(1, int(math.ceil(horizon / w - 1e-9)))
        s, c = self._road_acc()
        out: list[RoadWindow] = []
        for rid in sorted(self._road_index):
            r = self._road_index[rid]
            for wi in range(n_windows):
                if wi < s.shape[1] and c[r, wi] > 0:
                    speed = float(s[r, wi]) / int(c[r, wi])
                else:
                    speed = self.road_free_flow(rid)
                out.append(RoadWindow(road=rid, window_start=wi * w,
                                      window_end=min((wi + 1) * w, horizon), mean_speed=speed))
        return out

    # ------------------------------------------------------------ control surface

    def set_lane_max_speed(self, lane_id: int, max_speed: float) -> None:
        if self.net is None or lane_id not in self.net.lanes:
            raise InputError(f"unknown lane {lane_id}")
        if max_speed <= 0:
            raise InputError("max_speed must be positive")
        self.net.lanes[lane_id].max_speed = max_speed
        self._flat.lane_cap[lane_id] = max_speed
        _native.check(_native.lib().tsb_set_lane(self._live(), lane_id, max_speed,
                                                 int(self._flat.lane_open[lane_id])))
        self.router.rebuild()

    def set_lane_restriction(self, lane_id: int, restriction: str) -> None:
        if self.net is None or lane_id not in self.net.lanes:
            raise InputError(f"unknown lane {lane_id}")
        if restriction not in (OPEN, CLOSED):
            raise InputError(f"unknown restriction {restriction!r}")
        self.net.lanes[lane_id].restriction = restriction
        self._flat.lane_open[lane_id] = 1 if restriction == OPEN else 0
        _native.check(_native.lib().tsb_set_lane(self._live(), lane_id, float(self._flat.lane_cap[lane_id]),
                                                 int(self._flat.lane_open[lane_id])))
        self.router.rebuild()

    def set_signal_phase(self, junction_id: str, phase_index: int) -> None:
        j = self._junc_index.get(junction_id)
        if j is None:
            raise InputError(f"unknown junction {junction_id}")
        if not self._flat.junc_signal[j]:
            raise InputError(f"junction {junction_id} is unsignalized")
        n_ph = int(self._flat.junc_phase_off[j + 1] - self._flat.junc_phase_off[j])
        if not 0 <= phase_index < n_ph:
            raise InputError(f"phase index {phase_index} out of range (program has {n_ph} phases)")
        _native.check(_native.lib().tsb_set_signal_phase(self._live(), j, phase_index))

    def signal_state(self):
        nj = max(len(self._flat.junction_ids), 1)
        ph = np.zeros(nj, dtype=np.int32)
        el = np.zeros(nj, dtype=np.float64)
        _native.check(_native.lib().tsb_signal_state(self._live(), ph.ctypes.data, el.ctypes.data))
        return ph[: len(self._flat.junction_ids)], el[: len(self._flat.junction_ids)]


def run(world: World, steps: int, recorder=None) -> SimulationOutput:
    return world.run(steps, recorder)
