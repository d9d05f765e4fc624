"""The BASELINE.json configurations as parity cases: the GPU engine against the
CPU oracle (pinned to the reference, test_oracle.py) in the reference's own
arithmetic (glibc pow), bit for bit -- every StepReport counter at every step
and the full lane-sorted state (membership, order, road_pos, s, v) at the
checkpoints.

C1  4x4 grid, 1k vehicles, 3600 steps (BASELINE configs[0])
C2  single-lane ring, 1,250 junctions, 10k vehicles, IDM only, 3600 steps (configs[1]);
    the jittered start settles into IDM's homogeneous equilibrium flow
C3  50x50x2 grid, 200k pre-placed vehicles, first 100 steps (configs[2])
M1  100x100x3 grid, 1M pre-placed vehicles -- the bench workload -- 20 steps in
    the reference arithmetic; 26 steps (the bench window) in the headline's
    correctly-rounded arithmetic, also against the reference arithmetic
C4  100x100x3 grid, 2M pre-placed slots, first 5 steps (configs[3])
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
    """C3 through 100 steps (lane changes, road transitions, reverts)."""
    net = generate_grid(50, 50, lanes_per_direction=2)
    router = Router(net)
    trips = preplaced_trips(net, router, 200_000, 16.0)
    router.close()
    g, r, reverts = run_pair(net, trips, EngineConfig(), 42, 100, every=10)
    assert g.driving_count() > 150_000
    print("C3 reverts in 100 steps:", reverts)
    _close(g, r)


def m1_inputs(n=1_000_000, spacing=29.0):
    net = generate_grid(100, 100, block_length=400.0, lanes_per_direction=3)
    router = Router(net)
    trips = preplaced_trips(net, router, n, spacing)
    router.close()
    return net, trips


def test_c4_2m_first_steps():
    """C4 (100x100x3 grid, 2M pre-placed slots every 22 m; 1.42M routable):
    5 steps bit for bit against the oracle in the reference's arithmetic."""
    net, trips = m1_inputs(2_000_000, 22.0)
    g, r, _ = run_pair(net, trips, EngineConfig(), 42, 5, every=1)
    assert g.driving_count() > 1_400_000
    _close(g, r)


def test_m1_headline_arithmetic():
    """bench.py's headline run at its own config and arithmetic: M1 (1M
    vehicles) in the correctly-rounded power mode (pow_mode=0) through the
    bench window (bulk injection + 5 warm-up + 20 timed steps = 26 steps):
    (1) bit for bit against the oracle in the same arithmetic, every
    StepReport counter each step and the whole lane-sorted state every 5;
    (2) against the oracle in the reference's own arithmetic (glibc pow,
    what trafficsim computes): identical lane membership, order, road_pos,
    statuses and counters, s and v within the north-star tolerance (1e-4
    relative), measured at step 26."""

    from oracle.bind import OracleWorld
    from tests.parity import compare_reports, compare_state

    net, trips = m1_inputs()
    g, r, reverts = run_pair(net, trips, EngineConfig(), 42, 26, every=5, pow_mode=0)
    assert reverts > 50
    r.close()
    ref = OracleWorld(net, trips, EngineConfig(), seed=42, pow_mode=1)
    try:
        ref.step(26)
        compare_reports(g, ref, 26)
        compare_state(g, ref, 26, exact=False, tol=1e-4)
        a, b = g._state(), ref.state()
        ds = float(np.max(np.abs(a["s"] - b["s"])))
        dv = float(np.max(np.abs(a["v"] - b["v"])))
        print(f"M1 pow_mode=0 vs reference arithmetic after 26 steps: max |ds| {ds:.3e} m, max |dv| {dv:.3e} m/s")
        assert np.array_equal(g._state()["status"], ref.status()[0])
    finally:
        ref.close()
        g.close()


def test_m1_bench_workload_first_steps():
    net = generate_grid(100, 100, block_length=400.0, lanes_per_direction=3)
    router = Router(net)
    trips = preplaced_trips(net, router, 1_000_000, 29.0)
    router.close()
    g, r, _ = run_pair(net, trips, EngineConfig(), 42, 3, every=1)
    assert g.driving_count() == 1_000_000
    _close(g, r)


def test_m1_into_the_revert_regime():
    """The bench workload at full size (1M vehicles) through step 100, deep in
    the revert regime (~25 reverts per step): every StepReport counter each
    step and the whole lane-sorted state every 25 steps, bit for bit against
    the CPU oracle in the reference's arithmetic (glibc pow).  (A one-off
    200-step run plus 3 steps at C5 scale: profiles/round2/long_parity_*.log.)"""
    net = generate_grid(100, 100, block_length=400.0, lanes_per_direction=3)
    router = Router(net)
    trips = preplaced_trips(net, router, 1_000_000, 29.0)
    router.close()
    g, r, reverts = run_pair(net, trips, EngineConfig(), 42, 100, every=25)
    assert reverts > 1000
    print("reverts in 100 steps:", reverts)
    _close(g, r)
