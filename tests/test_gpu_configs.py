"""The BASELINE.json configurations as parity cases: the GPU engine against the
CPU oracle (pinned to the reference, test_oracle.py) in the reference's own
arithmetic (glibc pow), bit for bit -- every StepReport counter at every step
and the full lane-sorted state (membership, order, road_pos, s, v) at the
checkpoints.

C1  4x4 grid, 1k vehicles, 3600 steps (BASELINE configs[0])
C2  single-lane ring, 1,250 junctions, 10k vehicles, IDM only, 3600 steps (configs[1]);
    the jittered start settles into IDM's homogeneous equilibrium flow
C3  50x50x2 grid, 200k pre-placed vehicles, first 40 steps (configs[2])
M1  100x100x3 grid, 1M pre-placed vehicles -- the bench workload -- first 3 steps
"""

import math
import random

import numpy as np
import pytest

from paper_2405_12520_b200 import EngineConfig, Router, Trip, generate_grid, make_ring, preplaced_trips, random_trips
from tests.parity import run_pair

pytestmark = pytest.mark.gpu


def _close(*ws):
    for w in ws:
        w.close()


def test_c1_grid44_full_hour():
    net = generate_grid(4, 4)
    trips = random_trips(net, 1000, seed=42, window=(0.0, 3600.0))
    g, r, _ = run_pair(net, trips, EngineConfig(), 42, 3600, every=25)
    assert len(g.finished) > 500
    _close(g, r)


def ring_c2(per_road=8, n_junctions=1250, seed=2024):
    net = make_ring(n_junctions, radius=n_junctions * 200.0 / (2 * math.pi))
    rng = random.Random(seed)
    roads = list(net.roads)
    trips = []
    for k, rid in enumerate(roads):
        lane = net.roads[rid][0]
        dest = net.roads[roads[k - 1]][0]
        for j in range(per_road):
            trips.append(Trip(len(trips), lane, 22.0 * j + rng.uniform(0, 4), dest, 0.0))
    return net, trips


def test_c2_ring_10k_equilibrium():
    net, trips = ring_c2()
    g, r, _ = run_pair(net, trips, EngineConfig(), 42, 3600, every=50)
    st = g._state()
    assert len(st["vix"]) == 10000  # nobody arrives on the ring within the hour
    # the jittered start relaxes to IDM's homogeneous flow: every vehicle at the
    # speed whose equilibrium gap (idm.py:34-37) equals the mean gap (200 m of
    # ring per 8 vehicles, minus the 5 m vehicle length)
    p = EngineConfig().idm
    v = float(st["v"].mean())
    eq_gap = (p.s0 + v * p.T) / math.sqrt(1.0 - (v / p.v0) ** p.delta)
    assert abs(eq_gap - (200.0 / 8 - 5.0)) < 0.2
    assert float(st["v"].max() - st["v"].min()) < 0.01
    _close(g, r)


def test_c3_grid50_200k():
    net = generate_grid(50, 50, lanes_per_direction=2)
    router = Router(net)
    trips = preplaced_trips(net, router, 200_000, 16.0)
    router.close()
    g, r, _ = run_pair(net, trips, EngineConfig(), 42, 40, every=5)
    assert g.driving_count() > 190_000
    _close(g, r)


def test_m1_bench_workload_first_steps():
    net = generate_grid(100, 100, block_length=400.0, lanes_per_direction=3)
    router = Router(net)
    trips = preplaced_trips(net, router, 1_000_000, 29.0)
    router.close()
    g, r, _ = run_pair(net, trips, EngineConfig(), 42, 3, every=1)
    assert g.driving_count() == 1_000_000
    _close(g, r)


def test_m1_into_the_revert_regime():
    """The bench workload at full size (1M vehicles) through step 20, where
    revert chains have started (~20 per step): every StepReport counter each
    step and the whole lane-sorted state at the end, bit for bit against the
    CPU oracle in the reference's arithmetic (glibc pow)."""
    net = generate_grid(100, 100, block_length=400.0, lanes_per_direction=3)
    router = Router(net)
    trips = preplaced_trips(net, router, 1_000_000, 29.0)
    router.close()
    g, r, reverts = run_pair(net, trips, EngineConfig(), 42, 20, every=10)
    assert reverts > 50
    print("reverts in 20 steps:", reverts)
    _close(g, r)
