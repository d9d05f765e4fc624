"""Loaders for the reference-generated fixtures in tests/golden/ and a
scenario runner shared by the oracle tests (CPU) and the GPU tests.

The fixtures were produced by tests/golden/make_golden.py from the reference
package itself; nothing here reads /root/reference, so this module works on
the GPU box.
"""

from __future__ import annotations

import hashlib
import json
import math
import os

import numpy as np

from paper_2405_12520_b200 import Trip
from paper_2405_12520_b200.flat import FlatNet, FlatTrips, flatten_trips
from paper_2405_12520_b200.records import HashingRecorder

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NET_FIELDS = ("lane_len", "lane_cap", "lane_kind", "lane_open", "lane_left", "lane_right", "lane_road",
              "lane_junction", "lane_pred1", "lane_succ1", "succ_off", "succ", "pred_off", "pred",
              "road_lane_off", "road_lanes", "junc_signal", "junc_phase_off", "phase_dur",
              "lane_green_mask", "junc_phase0", "junc_elapsed0", "geo_off", "geo_cum", "geo_angle")

_cache: dict = {}


def _load(name):
    if name not in _cache:
        path = os.path.join(GOLDEN, name)
        if name.endswith(".npz"):
            with np.load(path) as z:
                _cache[name] = {k: z[k] for k in z.files}
        else:
            with open(path) as fh:
                _cache[name] = json.load(fh)
    return _cache[name]


def scenarios() -> dict:
    return _load("scenarios.json")


def kat() -> dict:
    return _load("kat.json")


def golden_flat(net_name: str, controller: str = "fixed") -> FlatNet:
    """The reference's compiled network (network.py:367-560), flattened."""
    arr = _load("nets.npz")
    meta = _load("nets_meta.json")[net_name]
    kw = {f: arr[f"{net_name}/{f}"].copy() for f in NET_FIELDS}
    if controller != "fixed":
        kw["junc_phase0"] = arr[f"{net_name}/mp_junc_phase0"].copy()
        kw["junc_elapsed0"] = arr[f"{net_name}/mp_junc_elapsed0"].copy()
    return FlatNet(n_lanes=meta["n_lanes"], road_ids=list(meta["road_ids"]),
                   junction_ids=list(meta["junction_ids"]), **kw)


def golden_trips(scenario: str) -> list[Trip]:
    """The reference's trips for a scenario (demand.py:260-284 / fixtures), in generation order."""
    arr = _load("nets.npz")
    p = f"trips/{scenario}/"
    return [Trip(int(i), int(o), float(s), int(d), float(t)) for i, o, s, d, t in
            zip(arr[p + "id"], arr[p + "origin_lane"], arr[p + "origin_s"], arr[p + "dest_lane"],
                arr[p + "departure"])]


def closable_lane(flat: FlatNet, trips) -> int:
    """make_golden.closable_lane restated on flat arrays."""
    used = {t.dest_lane for t in trips} | {t.origin_lane for t in trips}
    cands = [lid for lid in range(flat.n_lanes) if flat.lane_kind[lid] == 0 and lid not in used]
    return cands[len(cands) // 2]


def road_lane(flat: FlatNet, road_id: str, k: int) -> int:
    r = flat.road_ids.index(road_id)
    return int(flat.road_lanes[flat.road_lane_off[r] + k])


def sha(obj) -> str:
    return hashlib.sha256(json.dumps(obj, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


class EngineAdapter:
    """What a scenario run needs from an engine (oracle or GPU World)."""

    def step(self): ...
    def report_row(self) -> list: ...
    def records(self) -> list: ...
    def close_lane(self, lane: int, open_: bool): ...
    def set_speed(self, lane: int, v: float): ...
    def set_phase(self, junction: int, phase: int): ...


def run_scenario(sc: dict, flat: FlatNet, eng, hash_records: bool = True, on_step=None):
    """Replays a golden scenario on `eng`; returns the same fields make_golden stores."""
    trips = golden_trips_for(sc)
    ev_at: dict[int, list] = {}
    for ev in sc["events"]:
        ev_at.setdefault(ev[0], []).append(ev)
    h = HashingRecorder()
    reports, digests = [], {}
    for k in range(1, sc["steps"] + 1):
        for ev in ev_at.get(k - 1, []):
            kind = ev[1]
            if kind in ("close", "open"):
                eng.close_lane(closable_lane(flat, trips), kind == "open")
            elif kind == "speed":
                eng.set_speed(road_lane(flat, ev[2], ev[3]), ev[4])
            elif kind == "phase":
                eng.set_phase(flat.junction_ids.index(ev[2]), ev[3])
        eng.step()
        reports.append(eng.report_row())
        if hash_records:
            for r in eng.records():
                h.write(r)
            if k % 50 == 0 or k == sc["steps"]:
                digests[str(k)] = h.hexdigest()
        if on_step is not None:
            on_step(k)
    return {"reports": reports, "digests": digests, "records": h.count}


def golden_trips_for(sc: dict) -> list[Trip]:
    name = sc["_name"]
    return golden_trips(name)


def named(name: str) -> dict:
    sc = dict(scenarios()[name])
    sc["_name"] = name
    return sc


def flat_trips_for(flat: FlatNet, name: str) -> FlatTrips:
    return flatten_trips(flat, golden_trips(name))


def finite(x):
    return x if not (isinstance(x, float) and math.isinf(x)) else "inf"
