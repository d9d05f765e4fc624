"""ctypes binding of liboracle.so -- TEST INFRASTRUCTURE ONLY (see oracle.c).

``OracleWorld`` exposes the same query surface the GPU ``World`` uses so
parity tests can compare the two field by field.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2405_12520_b200.cabi import TsbReport, pack_network, pack_params, pack_trips, ptr
from paper_2405_12520_b200.flat import flatten_network, flatten_trips, record_angles
from paper_2405_12520_b200.params import EngineConfig
from paper_2405_12520_b200.records import VehicleRecord

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return os.path.join(_HERE, "liboracle.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        src = os.path.join(_HERE, "oracle.c")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            build()
        L = C.CDLL(path)
        vp = C.c_void_p
        L.orc_create.argtypes = [vp, vp, vp, C.POINTER(vp)]
        L.orc_destroy.argtypes = [vp]
        L.orc_step.argtypes = [vp, C.c_int32, C.POINTER(TsbReport)]
        L.orc_report.argtypes = [vp, C.POINTER(TsbReport)]
        L.orc_state.argtypes = [vp] + [vp] * 7
        L.orc_status.argtypes = [vp, vp, vp, vp]
        L.orc_finished.argtypes = [vp, C.c_int64, C.c_int64, vp, vp, C.POINTER(C.c_int64)]
        L.orc_road_acc.argtypes = [vp, C.c_int32, vp, vp]
        L.orc_min_front_gap.argtypes = [vp, C.POINTER(C.c_double)]
        L.orc_set_lane.argtypes = [vp, C.c_int32, C.c_double, C.c_int32]
        L.orc_set_signal_phase.argtypes = [vp, C.c_int32, C.c_int32]
        L.orc_signal_state.argtypes = [vp, vp, vp]
        L.orc_route_cost.argtypes = [vp, C.c_int32, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int32)]
        L.orc_idm_accel.argtypes = [vp, C.c_double, C.c_double, C.c_double, C.c_double]
        L.orc_idm_accel.restype = C.c_double
        L.orc_keyed_uniform4.argtypes = [C.c_uint64] * 4
        L.orc_keyed_uniform4.restype = C.c_double
        L.orc_set_threads.argtypes = [vp, C.c_int32]
        L.orc_reach.argtypes = [vp, C.c_int32, vp, vp]
        L.orc_pow_cr.argtypes = [C.c_double, C.c_int32]
        L.orc_pow_cr.restype = C.c_double
        _LIB = L
    return _LIB


class OracleRouter:
    """Router.dist_to key sets from the oracle's own reverse Dijkstra
    (routing.py:47-68), for building demand without the product library
    (bench.py's CPU arm).  Same interface as Router.reachable_sets."""

    def __init__(self, net, config: EngineConfig | None = None, flat=None):
        self._w = OracleWorld(net, [], config, flat=flat)
        self._n = self._w.flat.n_lanes

    def reachable_sets(self, dests) -> dict:
        d = np.asarray(dests, dtype=np.int32)
        out = np.zeros((len(d), max(self._n, 1)), dtype=np.uint8)
        lib().orc_reach(self._w._h, len(d), d.ctypes.data, out.ctypes.data)
        return {int(k): out[i].astype(bool) for i, k in enumerate(d)}

    def close(self):
        self._w.close()


class OracleWorld:
    """CPU reference engine on flattened inputs (pow_mode 1 = libm pow)."""

    def __init__(self, net, trips, config: EngineConfig | None = None, seed: int = 0,
                 pow_mode: int = 1, flat=None):
        self.config = config or EngineConfig()
        self.config.validate()
        self.flat = flat if flat is not None else flatten_network(net, self.config.controller)
        self.trips = flatten_trips(self.flat, trips)
        self._net = pack_network(self.flat)
        self._tr = pack_trips(self.trips)
        self._p = pack_params(self.config, seed, pow_mode)
        h = C.c_void_p()
        rc = lib().orc_create(C.byref(self._net.struct), C.byref(self._tr.struct), C.byref(self._p), C.byref(h))
        if rc != 0:
            raise RuntimeError(f"orc_create failed: {rc}")
        self._h = h
        self._fin_seen = 0
        self.finished: list[tuple[int, float, float]] = []

    def set_threads(self, n: int):
        lib().orc_set_threads(self._h, n)

    def close(self):
        if self._h:
            lib().orc_destroy(self._h)
            self._h = None

    __del__ = close

    def step(self, n: int = 1) -> TsbReport:
        r = TsbReport()
        lib().orc_step(self._h, n, C.byref(r))
        return r

    def report(self) -> TsbReport:
        r = TsbReport()
        lib().orc_report(self._h, C.byref(r))
        return r

    def state(self):
        """Lane-sorted snapshot: dict of arrays (vix, lane, road_pos, s, v) + lane_start."""
        n = len(self.trips.ids)
        nd = C.c_int32()
        ls = np.zeros(self.flat.n_lanes + 1, dtype=np.int32)
        out = {k: np.zeros(max(n, 1), dtype=t) for k, t in
               (("vix", np.int32), ("lane", np.int32), ("road_pos", np.int32), ("s", np.float64), ("v", np.float64))}
        lib().orc_state(self._h, C.byref(nd), ptr(ls, np.int32), *(out[k].ctypes.data for k in
                        ("vix", "lane", "road_pos", "s", "v")))
        res = {k: a[: nd.value].copy() for k, a in out.items()}
        res["lane_start"] = ls
        return res

    def status(self):
        n = max(len(self.trips.ids), 1)
        st = np.zeros(n, dtype=np.uint8)
        fin = np.zeros(n, dtype=np.float64)
        ri = np.zeros(n, dtype=np.int32)
        lib().orc_status(self._h, st.ctypes.data, fin.ctypes.data, ri.ctypes.data)
        m = len(self.trips.ids)
        return st[:m], fin[:m], ri[:m]

    def finished_list(self):
        cap = max(len(self.trips.ids), 1)
        vix = np.zeros(cap, dtype=np.int32)
        t = np.zeros(cap, dtype=np.float64)
        n = C.c_int64()
        lib().orc_finished(self._h, self._fin_seen, cap, vix.ctypes.data, t.ctypes.data, C.byref(n))
        for k in range(n.value):
            i = int(vix[k])
            self.finished.append((self.trips.ids[i], float(self.trips.departure[i]), float(t[k])))
        self._fin_seen += n.value
        return self.finished

    def road_acc(self, n_windows: int):
        nr = len(self.flat.road_ids)
        s = np.zeros((max(nr, 1), n_windows), dtype=np.float64)
        c = np.zeros((max(nr, 1), n_windows), dtype=np.int64)
        lib().orc_road_acc(self._h, n_windows, s.ctypes.data, c.ctypes.data)
        return s[:nr], c[:nr]

    def min_front_gap(self) -> float:
        g = C.c_double()
        lib().orc_min_front_gap(self._h, C.byref(g))
        return g.value

    def signal_state(self):
        nj = max(len(self.flat.junction_ids), 1)
        ph = np.zeros(nj, dtype=np.int32)
        el = np.zeros(nj, dtype=np.float64)
        lib().orc_signal_state(self._h, ph.ctypes.data, el.ctypes.data)
        return ph[: len(self.flat.junction_ids)], el[: len(self.flat.junction_ids)]

    def set_lane(self, lane: int, max_speed: float, open_: bool):
        self.flat.lane_cap[lane] = max_speed
        self.flat.lane_open[lane] = 1 if open_ else 0
        return lib().orc_set_lane(self._h, lane, max_speed, 1 if open_ else 0)

    def set_signal_phase(self, junction: int, phase: int):
        return lib().orc_set_signal_phase(self._h, junction, phase)

    def records(self):
        """VehicleRecords of the current state, sorted by id (world.py:771-782)."""
        st = self.state()
        order = np.argsort(st["vix"], kind="stable")
        lane, s, v, vix = st["lane"][order], st["s"][order], st["v"][order], st["vix"][order]
        ang = record_angles(self.flat, lane, s)
        t = self.report().time
        ids = self.trips.ids
        return [VehicleRecord(t=t, id=ids[int(i)], lane=int(l), s=float(a), v=float(b), angle_deg=float(g))
                for i, l, a, b, g in zip(vix, lane, s, v, ang)]
