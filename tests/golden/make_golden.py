"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run in the development container, where the read-only reference package
lives at /root/reference/pkg/src (it does not exist on the GPU box, so the
outputs are committed):

    python tests/golden/make_golden.py

Everything here is computed by the reference's own code (trafficsim
World / builders / rng / idm); this repo's package is used only to flatten
the reference's RoadNetwork objects into the array form the oracle and the
engine consume (flat.flatten_network duck-types the reference types).

Outputs
  kat.json        keyed-RNG known answers (rng.py:24-41) and IDM tuples
                  (idm.py:17-31, glibc pow as CPython calls it)
  nets.npz        flattened reference networks (network.py:367-560) and
                  the reference random_trips (demand.py:260-284)
  scenarios.json  per scenario: per-step StepReport counters, cumulative
                  sha256 of the canonical record stream (io.py:385-440) at
                  checkpoints, digests of prepare() / finished /
                  road_windows, min_front_gap
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import random
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
sys.path.insert(0, ROOT)
sys.path.insert(0, REF)

from trafficsim import io as tio  # noqa: E402
from trafficsim import rng as trng  # noqa: E402
from trafficsim.demand import Trip as RTrip  # noqa: E402
from trafficsim.demand import random_trips as r_random_trips  # noqa: E402
from trafficsim.engine import EngineConfig as REngineConfig  # noqa: E402
from trafficsim.engine.idm import idm_accel as r_idm_accel  # noqa: E402
from trafficsim.engine.params import IdmParams as RIdmParams  # noqa: E402
from trafficsim.engine.world import World as RWorld  # noqa: E402
from trafficsim.network import BuildOptions, RawJunction, RawRoad, build_network  # noqa: E402
from trafficsim.network import generate_grid as r_generate_grid  # noqa: E402

from paper_2405_12520_b200.flat import flatten_network  # noqa: E402

NET_FIELDS = ("lane_len", "lane_cap", "lane_kind", "lane_open", "lane_left", "lane_right", "lane_road",
              "lane_junction", "lane_pred1", "lane_succ1", "succ_off", "succ", "pred_off", "pred",
              "road_lane_off", "road_lanes", "junc_signal", "junc_phase_off", "phase_dur",
              "lane_green_mask", "junc_phase0", "junc_elapsed0", "geo_off", "geo_cum", "geo_angle")


# ---------------------------------------------------------------- networks (reference builders)

def r_corridor(lengths=(500.0, 500.0), speed=16.67, lane_count=1):
    xs = [0.0]
    for ln in lengths:
        xs.append(xs[-1] + ln)
    roads = [RawRoad(id=f"r{i}", polyline=[(xs[i], 0.0), (xs[i + 1], 0.0)], lane_count=lane_count,
                     max_speed=speed) for i in range(len(lengths))]
    juncs = [RawJunction(id=f"j{i}", position=(xs[i + 1], 0.0), in_roads=[f"r{i}"], out_roads=[f"r{i + 1}"])
             for i in range(len(lengths) - 1)]
    return build_network(roads, juncs, BuildOptions(coordinate_frame="local"))


def r_cross(arm=150.0, speed=13.9, lane_count=1):
    tips = {"n": (0.0, arm), "s": (0.0, -arm), "e": (arm, 0.0), "w": (-arm, 0.0)}
    roads = []
    for name, tip in tips.items():
        roads.append(RawRoad(id=f"{name}_in", polyline=[tip, (0.0, 0.0)], lane_count=lane_count, max_speed=speed))
        roads.append(RawRoad(id=f"{name}_out", polyline=[(0.0, 0.0), tip], lane_count=lane_count, max_speed=speed))
    j = RawJunction(id="center", position=(0.0, 0.0), in_roads=[f"{n}_in" for n in tips],
                    out_roads=[f"{n}_out" for n in tips])
    return build_network(roads, [j], BuildOptions(coordinate_frame="local"))


def r_ring(n, radius, margin=12.0, speed=16.67):
    pts = [(radius * math.cos(2 * math.pi * k / n), radius * math.sin(2 * math.pi * k / n)) for k in range(n)]
    roads, juncs = [], []
    for k in range(n):
        a, b = pts[k], pts[(k + 1) % n]
        d = math.dist(a, b)
        ux, uy = (b[0] - a[0]) / d, (b[1] - a[1]) / d
        roads.append(RawRoad(id=f"r{k:05d}", polyline=[(a[0] + ux * margin, a[1] + uy * margin),
                                                      (b[0] - ux * margin, b[1] - uy * margin)],
                             lane_count=1, max_speed=speed))
    for k in range(n):
        juncs.append(RawJunction(id=f"j{k:05d}", position=pts[k], in_roads=[f"r{(k - 1) % n:05d}"],
                                 out_roads=[f"r{k:05d}"]))
    return build_network(roads, juncs, BuildOptions(snap_radius=margin + 0.5, allow_boundaries=False,
                                                    coordinate_frame="local"))


def ring_trips(net, per_road=6, seed=2024):
    rng = random.Random(seed)
    roads = list(net.roads)
    out = []
    for k, rid in enumerate(roads):
        lane = net.roads[rid][0]
        dest = net.roads[roads[k - 1]][0]
        for j in range(per_road):
            out.append(RTrip(id=len(out), origin_lane=lane, origin_s=22.0 * j + rng.uniform(0, 4),
                             dest_lane=dest, departure=0.0))
    return out


NETS = {
    "corridor": lambda: r_corridor(),
    "corridor2": lambda: r_corridor(lane_count=2),
    "cross1": lambda: r_cross(),
    "cross2": lambda: r_cross(arm=200.0, lane_count=2),
    "grid33": lambda: r_generate_grid(3, 3),
    "grid44": lambda: r_generate_grid(4, 4),
    "grid44x2": lambda: r_generate_grid(4, 4, lanes_per_direction=2),
    "grid55x3": lambda: r_generate_grid(5, 5, lanes_per_direction=3),
    "grid66s": lambda: r_generate_grid(6, 6, block_length=60.0),
    "grid55x2s": lambda: r_generate_grid(5, 5, block_length=80.0, lanes_per_direction=2),
    "ring100": lambda: r_ring(100, 100 * 200.0 / (2 * math.pi)),
    "town": lambda: tio.load_network("/root/reference/pkg/tests/data/golden/net.json"),
}

# (name, net, trips spec, config kwargs, seed, steps, control events)
SCENARIOS = [
    ("corridor_one", "corridor", ("one",), {}, 0, 200, []),
    ("corridor2_lanes", "corridor2", ("random", 80, 9, (0.0, 120.0)), {}, 9, 300, []),
    ("cross_signals", "cross2", ("random", 120, 3, (0.0, 200.0)), {}, 7, 400, []),
    ("grid44_c1", "grid44", ("random", 1000, 42, (0.0, 3600.0)), {}, 42, 600, []),
    ("determinism_c1b", "grid44x2", ("random", 2500, 42, (0.0, 700.0)), {}, 42, 1000, []),
    ("grid55x3_mobil", "grid55x3", ("random", 3000, 17, (0.0, 400.0)), {}, 17, 500, []),
    ("jammed_reverts", "grid44", ("random", 3000, 11, (0.0, 300.0)), {}, 11, 500, []),
    ("max_pressure", "grid44", ("random", 400, 4, (0.0, 200.0)), {"controller": "max_pressure"}, 4, 400, []),
    ("dense_short_blocks", "grid66s", ("random", 6000, 5, (0.0, 200.0)), {}, 5, 300, []),
    ("dense_two_lane", "grid55x2s", ("random", 6000, 5, (0.0, 300.0)), {}, 5, 300, []),
    ("ring_stop_and_go", "ring100", ("ring",), {}, 1, 300, []),
    ("town_pipeline", "town", ("file",), {}, 42, 600, []),
    ("control_surface", "grid55x3", ("random", 250, 21, (0.0, 300.0)), {}, 21, 400,
     [(60, "close", "auto", 0), (60, "speed", "j1_0:j1_1", 0, 8.0), (90, "phase", "j1_1", 2),
      (200, "open", "auto", 0)]),
]


def make_trips(net, spec):
    if spec[0] == "one":
        return [RTrip(id=0, origin_lane=net.roads["r0"][0], origin_s=0.0, dest_lane=net.roads["r1"][0],
                      departure=5.0)]
    if spec[0] == "random":
        _, n, seed, window = spec
        return r_random_trips(net, n, seed, window=window)
    if spec[0] == "ring":
        return ring_trips(net)
    if spec[0] == "file":
        return tio.load_trips("/root/reference/pkg/tests/data/golden/trips.json")
    raise ValueError(spec)


def sha(obj) -> str:
    return hashlib.sha256(json.dumps(obj, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


def closable_lane(net, trips):
    """A road lane that is no trip's origin or destination (the reference
    raises InputError from step() when a pending trip's destination is
    closed, routing.py:52-54), taken from the middle of the id range."""
    used = {t.dest_lane for t in trips} | {t.origin_lane for t in trips}
    cands = [lid for lid in sorted(net.road_lane_ids()) if lid not in used]
    return cands[len(cands) // 2]


def apply_event(w, net, ev, trips):
    kind = ev[1]
    lane = closable_lane(net, trips) if ev[2] == "auto" else None
    if kind == "close":
        w.set_lane_restriction(lane, "closed")
    elif kind == "open":
        w.set_lane_restriction(lane, "open")
    elif kind == "speed":
        w.set_lane_max_speed(net.roads[ev[2]][ev[3]], ev[4])
    elif kind == "phase":
        w.set_signal_phase(ev[2], ev[3])


def run_scenario(name, netname, net, spec, cfg_kw, seed, steps, events):
    trips = make_trips(net, spec)
    w = RWorld(net, trips, REngineConfig(**cfg_kw), seed=seed)
    h = tio.HashingRecorder()
    reports, digests = [], {}
    t0 = time.time()
    ev_at = {}
    for ev in events:
        ev_at.setdefault(ev[0], []).append(ev)
    for k in range(1, steps + 1):
        for ev in ev_at.get(k - 1, []):
            apply_event(w, net, ev, trips)
        r = w.step()
        reports.append([r.time, r.driving, r.waiting, r.finished, r.dropped, r.injected_now, r.finished_now])
        w.record_step(h)
        if k % 50 == 0 or k == steps:
            digests[str(k)] = h.hexdigest()
    index, snap = w.prepare()
    out = {
        "net": netname, "trips": list(spec), "config": cfg_kw, "seed": seed, "steps": steps,
        "events": events, "reports": reports, "digests": digests, "records": h.count,
        "vehicle_updates": w.vehicle_updates,
        "prepare_sha": sha([[lane, index[lane]] for lane in sorted(index)]),
        "snapshot_sha": sha([[vid, list(snap[vid])] for vid in sorted(snap)]),
        "finished": [list(x) for x in w.finished],
        "road_windows": [[rw.road, rw.window_start, rw.window_end, rw.mean_speed]
                         for rw in w.road_windows(steps * w.config.dt)],
        "min_front_gap": w.min_front_gap(),
        "statuses": {str(t.id): [w.get_vehicle(t.id).lane_id, w.get_vehicle(t.id).s, w.get_vehicle(t.id).v,
                                 w.get_vehicle(t.id).status, w.get_vehicle(t.id).route_index,
                                 w.get_vehicle(t.id).finish_time]
                     for t in sorted(trips, key=lambda t: t.id)[:40]},
        "ref_seconds": round(time.time() - t0, 2),
    }
    w.close()
    return out, trips


def kat():
    keys = [(0, 1, 0, 0), (42, 1, 0, 0), (42, 1, 7, 3), (42, 1, 123456, 3599), (7, 1, 9999999, 100), (-5, 3),
            (2 ** 63 + 5, 1, 1, 1), (2 ** 64 - 1, 1, 2 ** 64 - 1, 2 ** 32), (-1, -1, -1, -1)]
    rnd = random.Random(77)
    for _ in range(60):
        keys.append((rnd.getrandbits(64), 1, rnd.getrandbits(40), rnd.randrange(100000)))
    rng_rows = [[list(k), format(trng.keyed_u64(*k), "#018x"), trng.keyed_uniform(*k)] for k in keys]
    p = RIdmParams()
    rows = []
    for _ in range(4000):
        v = rnd.uniform(0.0, 20.0)
        dv = rnd.uniform(-15.0, 15.0)
        gap = math.inf if rnd.random() < 0.1 else rnd.uniform(1e-6, 120.0)
        cap = rnd.choice([16.67, 13.9, 8.0, 30.0])
        rows.append([v, dv, gap if math.isfinite(gap) else "inf", cap, r_idm_accel(v, dv, gap, p, cap)])
    return {"rng": rng_rows, "idm": rows,
            "idm_params": {"v0": p.v0, "T": p.T, "a_max": p.a_max, "b": p.b, "delta": p.delta, "s0": p.s0}}


def main():
    arrays = {}
    meta = {}
    nets = {}
    for name, fn in NETS.items():
        net = fn()
        nets[name] = net
        f = flatten_network(net)
        for fld in NET_FIELDS:
            arrays[f"{name}/{fld}"] = getattr(f, fld)
        meta[name] = {"n_lanes": f.n_lanes, "road_ids": f.road_ids, "junction_ids": f.junction_ids}
        # max-pressure flattening has no fixed-time pre-advance
        fmp = flatten_network(net, "max_pressure")
        arrays[f"{name}/mp_junc_phase0"] = fmp.junc_phase0
        arrays[f"{name}/mp_junc_elapsed0"] = fmp.junc_elapsed0
    scen = {}
    for (name, netname, spec, cfg_kw, seed, steps, events) in SCENARIOS:
        out, trips = run_scenario(name, netname, nets[netname], spec, cfg_kw, seed, steps, events)
        scen[name] = out
        arrays[f"trips/{name}/id"] = np.array([t.id for t in trips], dtype=np.int64)
        arrays[f"trips/{name}/origin_lane"] = np.array([t.origin_lane for t in trips], dtype=np.int32)
        arrays[f"trips/{name}/origin_s"] = np.array([t.origin_s for t in trips], dtype=np.float64)
        arrays[f"trips/{name}/dest_lane"] = np.array([t.dest_lane for t in trips], dtype=np.int32)
        arrays[f"trips/{name}/departure"] = np.array([t.departure for t in trips], dtype=np.float64)
        print(f"{name}: {out['records']} records, {out['vehicle_updates']} updates, {out['ref_seconds']} s",
              flush=True)
    np.savez_compressed(os.path.join(HERE, "nets.npz"), **arrays)
    with open(os.path.join(HERE, "nets_meta.json"), "w") as fh:
        json.dump(meta, fh, sort_keys=True)
    with open(os.path.join(HERE, "scenarios.json"), "w") as fh:
        json.dump(scen, fh, sort_keys=True)
    with open(os.path.join(HERE, "kat.json"), "w") as fh:
        json.dump(kat(), fh, sort_keys=True)


if __name__ == "__main__":
    main()
