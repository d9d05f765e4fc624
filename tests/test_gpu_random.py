"""Randomised parity sweep: small grids of random size, lane count, block
length and demand (seeded, so every run checks the same cases), each run on
the GPU and on the CPU oracle in both power arithmetics, compared bit for bit
every step (StepReport counters) and every 10 steps (the whole lane-sorted
state, signal states), plus arrivals and statuses at the end."""

import random

import pytest

from paper_2405_12520_b200 import MAX_PRESSURE, EngineConfig, generate_grid, random_trips
from tests.parity import run_pair

pytestmark = pytest.mark.gpu


def _cases(n=12, seed=20261017):
    rng = random.Random(seed)
    out = []
    for k in range(n):
        rows, cols = rng.randint(2, 6), rng.randint(2, 6)
        lanes = rng.randint(1, 3)
        block = rng.choice([40.0, 60.0, 90.0, 150.0, 250.0, 400.0])
        trips = rng.randint(200, 4000)
        window = rng.choice([60.0, 200.0, 600.0])
        controller = MAX_PRESSURE if rng.random() < 0.3 else "fixed"
        out.append((k, rows, cols, lanes, block, trips, window, controller, rng.randint(0, 10**6)))
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"case{c[0]}")
@pytest.mark.parametrize("pow_mode", [1, 0])
def test_random_grid_parity(case, pow_mode):
    k, rows, cols, lanes, block, n, window, controller, seed = case
    net = generate_grid(rows, cols, block_length=block, lanes_per_direction=lanes)
    trips = random_trips(net, n, seed=seed, window=(0.0, window))
    g, r, reverts = run_pair(net, trips, EngineConfig(controller=controller), seed % 1000, 250, every=10,
                             pow_mode=pow_mode)
    print(f"case {k}: {rows}x{cols}x{lanes} block {block} m, {n} trips, {controller}: reverts {reverts}")
    g.close()
    r.close()
