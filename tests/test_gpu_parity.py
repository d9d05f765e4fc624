"""GPU engine vs CPU oracle, step by step (bit-exact, correctly-rounded powers).

The oracle (oracle/oracle.c) is pinned to the reference by test_oracle.py;
here every step's full lane-sorted state (membership, order, road_pos, s, v),
report counters, signal states, arrivals and statuses must be identical.
"""

import numpy as np
import pytest

from paper_2405_12520_b200 import (EngineConfig, MAX_PRESSURE, Trip, generate_grid, make_corridor,
                                   make_cross, make_ring, random_trips)
from tests.parity import run_pair

pytestmark = pytest.mark.gpu


def _close(*ws):
    for w in ws:
        w.close()


def test_corridor_single_trip():
    net = make_corridor()
    o, d = net.roads["r0"][0], net.roads["r1"][0]
    g, r, _ = run_pair(net, [Trip(0, o, 0.0, d, 5.0)], EngineConfig(), 0, 200)
    assert len(g.finished) == 1
    _close(g, r)


def test_cross_signals_and_queues():
    net = make_cross(arm=200.0, lane_count=2)
    trips = random_trips(net, 120, seed=3, window=(0.0, 200.0))
    g, r, _ = run_pair(net, trips, EngineConfig(), 7, 400)
    _close(g, r)


def test_grid44_single_lane():
    net = generate_grid(4, 4)
    trips = random_trips(net, 1000, seed=42, window=(0.0, 3600.0))
    g, r, _ = run_pair(net, trips, EngineConfig(), 42, 600, every=5)
    _close(g, r)


@pytest.mark.parametrize("pow_mode", [1, 0])
def test_grid44_two_lanes_mobil(pow_mode):
    net = generate_grid(4, 4, lanes_per_direction=2)
    trips = random_trips(net, 2500, seed=42, window=(0.0, 700.0))
    g, r, reverts = run_pair(net, trips, EngineConfig(), 42, 1000, every=10, pow_mode=pow_mode)
    _close(g, r)


@pytest.mark.parametrize("pow_mode", [1, 0])
def test_jammed_grid_reverts(pow_mode):
    net = generate_grid(4, 4)
    trips = random_trips(net, 3000, seed=11, window=(0.0, 300.0))
    g, r, reverts = run_pair(net, trips, EngineConfig(), 11, 500, every=5, pow_mode=pow_mode)
    _close(g, r)


def test_max_pressure():
    net = generate_grid(4, 4)
    trips = random_trips(net, 400, seed=4, window=(0.0, 200.0))
    g, r, _ = run_pair(net, trips, EngineConfig(controller=MAX_PRESSURE), 4, 400, every=5)
    _close(g, r)


def test_ring_stop_and_go():
    net = make_ring(100, radius=100 * 200.0 / (2 * np.pi))
    import random
    rng = random.Random(2024)
    trips = []
    roads = list(net.roads)
    for k, rid in enumerate(roads):
        lane = net.roads[rid][0]
        dest = net.roads[roads[k - 1]][0]
        for j in range(6):
            trips.append(Trip(len(trips), lane, 22.0 * j + rng.uniform(0, 4), dest, 0.0))
    g, r, _ = run_pair(net, trips, EngineConfig(), 1, 300, every=3)
    _close(g, r)


@pytest.mark.parametrize("debug", [0, 1, 2, 3, 4, 6])
def test_dense_short_blocks_revert_chains(debug):
    """Up to 35 reverts per step: per-event fast path, forced sequential
    replay (bit 0), forced full regroup (bit 1) and forced closure/component
    resolver (bit 2) must all match the oracle."""
    net = generate_grid(6, 6, block_length=60.0)
    trips = random_trips(net, 6000, seed=5, window=(0.0, 200.0))
    g, r, reverts = run_pair(net, trips, EngineConfig(), 5, 400, every=2, debug=debug)
    assert reverts > 200
    print("reverts", reverts, "sequential-resolve steps", g._report.resolve_sequential)
    _close(g, r)


@pytest.mark.parametrize("debug", [64, 64 | 2 | 8])
def test_snapshot_isolation_poisoned_scratch(debug):
    """Debug bit 6 fills every write-before-read buffer of the step (post-update
    records, sort scratch, the layout the step builds) with 0xff bytes before
    the update: results identical to the oracle means every kernel reads only
    the snapshot and what the step itself wrote (world.py:231-236, 416-419).
    With the full regroup (bit 1) and the gated graph (bit 3) as well."""
    net = generate_grid(5, 5, block_length=80.0, lanes_per_direction=2)
    trips = random_trips(net, 6000, seed=5, window=(0.0, 300.0))
    g, r, reverts = run_pair(net, trips, EngineConfig(), 5, 300, every=3, debug=debug)
    assert reverts > 50
    _close(g, r)


def test_dense_two_lane_reverts():
    net = generate_grid(5, 5, block_length=80.0, lanes_per_direction=2)
    trips = random_trips(net, 6000, seed=5, window=(0.0, 300.0))
    g, r, reverts = run_pair(net, trips, EngineConfig(), 5, 400, every=2)
    assert reverts > 50
    print("reverts", reverts, "sequential-resolve steps", g._report.resolve_sequential)
    _close(g, r)


@pytest.mark.parametrize("pow_mode", [1, 0])
def test_long_queues_oversized_lanes(pow_mode):
    """1.2 km single-lane blocks under heavy demand: lanes with ~160 vehicles
    exercise the off-chip paths of k_lanefix (> 64 members) and k_patch_dirty
    (> 128)."""
    net = generate_grid(3, 3, block_length=1200.0)
    trips = random_trips(net, 6000, seed=8, window=(0.0, 150.0))
    g, r, _ = run_pair(net, trips, EngineConfig(), 8, 500, every=5, pow_mode=pow_mode)
    assert int(np.diff(g._state()["lane_start"]).max()) > 128
    _close(g, r)


def test_long_multilane_queues():
    net = generate_grid(3, 3, block_length=1000.0, lanes_per_direction=2)
    trips = random_trips(net, 8000, seed=8, window=(0.0, 200.0))
    g, r, _ = run_pair(net, trips, EngineConfig(), 8, 500, every=5)
    _close(g, r)


def _star(arms=6, arm=400.0):
    import math
    from paper_2405_12520_b200 import BuildOptions, RawJunction, RawRoad, build_network
    roads = []
    for k in range(arms):
        ang = 2 * math.pi * k / arms
        tip = (arm * math.cos(ang), arm * math.sin(ang))
        roads.append(RawRoad(f"a{k}_in", [tip, (0.0, 0.0)], 1, 13.9))
        roads.append(RawRoad(f"a{k}_out", [(0.0, 0.0), tip], 1, 13.9))
    j = RawJunction("c", [f"a{k}_in" for k in range(arms)], [f"a{k}_out" for k in range(arms)], (0.0, 0.0))
    return build_network(roads, [j], BuildOptions(coordinate_frame="local", allow_uturns=True))


def test_star_junction_many_successors():
    """A 6-arm junction with U-turns: lanes with 6 successor connectors use the
    CSR tail of the 4-wide successor table (conn_from_id)."""
    net = _star()
    assert max(len(l.successors) for l in net.lanes.values()) > 4
    trips = random_trips(net, 600, seed=2, window=(0.0, 300.0))
    g, r, _ = run_pair(net, trips, EngineConfig(), 2, 500, every=5)
    assert len(g.finished) > 50
    _close(g, r)
