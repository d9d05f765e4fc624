"""Device-side queries (SURVEY 8(b) tsb_get_vehicles / tsb_records, 8(f) rank 2):
World.get_vehicle (world.py:706-714) and World.record_step (world.py:771-782)
answered on the device, against the CPU oracle (pinned to the reference,
test_oracle.py) and, at the bench size, against the full-state download."""

import time

import numpy as np
import pytest

from oracle.bind import OracleWorld
from paper_2405_12520_b200 import EngineConfig, World, generate_grid, random_trips
from paper_2405_12520_b200.flat import record_angles
from paper_2405_12520_b200.records import CollectingRecorder

pytestmark = pytest.mark.gpu

_ST = {0: "waiting", 1: "driving", 2: "finished", 3: "dropped"}


def test_queries_match_oracle_c1b():
    """The published determinism scenario (C1b): every 50 steps, every
    vehicle's StatusView and the id-sorted record stream equal the oracle's."""
    net = generate_grid(4, 4, lanes_per_direction=2)
    trips = random_trips(net, 2500, seed=42, window=(0.0, 700.0))
    g = World(net, trips, EngineConfig(), seed=42)
    r = OracleWorld(net, trips, EngineConfig(), seed=42, pow_mode=1)
    try:
        ids = [t.id for t in sorted(trips, key=lambda t: t.id)]
        for k in range(1, 401):
            g.step()
            r.step(1)
            if k % 50:
                continue
            rec = CollectingRecorder()
            g.record_step(rec)
            assert rec.records == r.records(), f"step {k}: record stream differs"
            st, fin, ri = r.status()
            ost = r.state()
            pos = {int(x): j for j, x in enumerate(ost["vix"])}
            for i, vid in enumerate(ids):
                sv = g.get_vehicle(vid)
                assert sv.status == _ST[int(st[i])], f"step {k}: vehicle {vid} status"
                if sv.status == "driving":
                    j = pos[i]
                    assert (sv.lane_id, sv.s, sv.v) == (int(ost["lane"][j]), float(ost["s"][j]), float(ost["v"][j]))
                    assert sv.route_index == int(ri[i])
                elif sv.status == "finished":
                    assert sv.finish_time == float(fin[i]) and sv.route_index == int(ri[i])
                else:
                    assert sv.finish_time is None
    finally:
        g.close()
        r.close()


def test_m1_queries_at_bench_size():
    """M1 (1M vehicles, the bench workload) after 26 steps: tsb_records equals
    the full-state download re-sorted by id with host-computed headings;
    get_vehicle answers one vehicle on the device in well under a millisecond."""
    from tests.test_gpu_configs import m1_inputs

    net, trips = m1_inputs()
    g = World(net, trips, EngineConfig(), seed=42, pow_mode=0)
    try:
        g.run(26)
        r = g.records_arrays()
        st = g._state()
        order = np.argsort(st["vix"], kind="stable")
        assert np.array_equal(r["vix"], st["vix"][order])
        assert np.all(np.diff(r["vix"]) > 0)
        for k, key in (("lane", "lane"), ("road_pos", "rp"), ("s", "s"), ("v", "v")):
            assert np.array_equal(r[k], st[key][order]), k
        assert np.array_equal(r["angle_deg"], record_angles(g._flat, r["lane"], r["s"]))
        rng = np.random.default_rng(7)
        sample = rng.choice(len(g._ft.ids), 200, replace=False)
        pos = st["pos"]
        for i in sample.tolist():
            sv = g.get_vehicle(g._ft.ids[i])
            p = int(pos[i])
            if p >= 0:
                assert sv.status == "driving"
                assert (sv.lane_id, sv.s, sv.v) == (int(st["lane"][p]), float(st["s"][p]), float(st["v"][p]))
            else:
                assert sv.status != "driving"
        g.get_vehicle(g._ft.ids[0])
        times = []
        for i in sample[:50].tolist():
            t0 = time.perf_counter()
            g.get_vehicle(g._ft.ids[i])
            times.append(time.perf_counter() - t0)
        med = float(np.median(times))
        print(f"M1 get_vehicle: median {med * 1e3:.3f} ms")
        assert med < 1e-3
        t0 = time.perf_counter()
        g.records_arrays()
        print(f"M1 records_arrays ({len(r['vix'])} records): {1e3 * (time.perf_counter() - t0):.1f} ms")
    finally:
        g.close()


def test_query_edge_cases():
    """No trips at all; an unknown id (InputError, world.py:706-709); waiting
    and dropped vehicles report their origin (world.py:196-198)."""
    from paper_2405_12520_b200 import InputError, Trip

    net = generate_grid(3, 3)
    w = World(net, [], EngineConfig(), seed=1)
    try:
        w.run(3)
        assert w.records_arrays()["vix"].size == 0 and w.driving_count() == 0
        with pytest.raises(InputError):
            w.get_vehicle(0)
    finally:
        w.close()
    lanes = sorted(net.road_lane_ids())
    # trip 1 departs later (waiting), trip 2 drives, trip 3's destination lane
    # is closed before it departs (unroutable: dropped)
    trips = [Trip(1, lanes[0], 0.0, lanes[-1], 500.0), Trip(2, lanes[1], 3.0, lanes[-1], 0.0),
             Trip(3, lanes[2], 7.0, lanes[-3], 2.0)]
    w = World(net, trips, EngineConfig(), seed=1)
    r = OracleWorld(net, trips, EngineConfig(), seed=1, pow_mode=1)
    try:
        w.set_lane_restriction(lanes[-3], "closed")
        r.set_lane(lanes[-3], float(net.lanes[lanes[-3]].max_speed), False)
        for _ in range(5):
            w.step()
            r.step(1)
        sv = w.get_vehicle(1)
        assert sv.status == "waiting" and sv.lane_id == lanes[0] and sv.s == 0.0 and sv.v == 0.0
        assert sv.route_index == 0 and sv.finish_time is None
        d = w.get_vehicle(3)
        assert d.status == "dropped" and d.lane_id == lanes[2] and d.s == 7.0 and d.finish_time is None
        assert w.get_vehicle(2).status == "driving" and w.dropped == 1
        st, _, _ = r.status()
        assert [w.get_vehicle(t.id).status for t in trips] == [_ST[int(x)] for x in st]
        rec = CollectingRecorder()
        w.record_step(rec)
        assert rec.records == r.records()
    finally:
        w.close()
        r.close()
