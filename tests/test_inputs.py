"""The input builders in paper_2405_12520_b200 (network compiler, grid and
ring generators, random_trips) against the reference's own outputs
(tests/golden/nets.npz, made by tests/golden/make_golden.py).  Lane-id order
and successor order are load-bearing for parity, so the flattened arrays
must be identical, not merely equivalent."""

from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2405_12520_b200 import generate_grid, make_corridor, make_cross, make_ring, random_trips
from paper_2405_12520_b200.flat import flatten_network, flatten_trips
from tests import goldens as G

BUILDERS = {
    "corridor": lambda: make_corridor(),
    "corridor2": lambda: make_corridor(lane_count=2),
    "cross1": lambda: make_cross(),
    "cross2": lambda: make_cross(arm=200.0, lane_count=2),
    "grid33": lambda: generate_grid(3, 3),
    "grid44": lambda: generate_grid(4, 4),
    "grid44x2": lambda: generate_grid(4, 4, lanes_per_direction=2),
    "grid55x3": lambda: generate_grid(5, 5, lanes_per_direction=3),
    "grid66s": lambda: generate_grid(6, 6, block_length=60.0),
    "grid55x2s": lambda: generate_grid(5, 5, block_length=80.0, lanes_per_direction=2),
    "ring100": lambda: make_ring(100, 100 * 200.0 / (2 * math.pi)),
}


@pytest.mark.parametrize("name", sorted(BUILDERS))
@pytest.mark.parametrize("controller", ["fixed", "max_pressure"])
def test_builder_matches_reference_network(name, controller):
    ours = flatten_network(BUILDERS[name](), controller)
    ref = G.golden_flat(name, controller)
    assert ours.n_lanes == ref.n_lanes
    assert ours.road_ids == ref.road_ids
    assert ours.junction_ids == ref.junction_ids
    for f in G.NET_FIELDS:
        a, b = getattr(ours, f), getattr(ref, f)
        assert a.dtype == b.dtype and np.array_equal(a, b), f


@pytest.mark.parametrize("name", [n for n, sc in G.scenarios().items() if sc["trips"][0] == "random"])
def test_random_trips_match_reference(name):
    sc = G.scenarios()[name]
    _, n, seed, window = sc["trips"]
    ours = random_trips(BUILDERS[sc["net"]](), n, seed, window=tuple(window))
    assert ours == G.golden_trips(name)


def test_flatten_trips_orders_by_id_and_validates():
    from paper_2405_12520_b200 import InputError, Trip
    flat = G.golden_flat("corridor")
    o = int(flat.road_lanes[0])
    ft = flatten_trips(flat, [Trip(7, o, 1.0, o, 0.0), Trip(-3, o, 2.0, o, 1.0), Trip(2 ** 70, o, 0.0, o, 0.0)])
    assert ft.ids == [-3, 7, 2 ** 70]
    assert ft.key.tolist() == [(-3) & (2 ** 64 - 1), 7, 2 ** 70 & (2 ** 64 - 1)]
    with pytest.raises(InputError):
        flatten_trips(flat, [Trip(1, o, 1.0, o, 0.0), Trip(1, o, 1.0, o, 0.0)])
    with pytest.raises(InputError):
        flatten_trips(flat, [Trip(1, o, -1.0, o, 0.0)])
    with pytest.raises(InputError):
        flatten_trips(flat, [Trip(1, o, 1.0, o, -0.5)])
    conn = int(np.nonzero(flat.lane_kind == 1)[0][0])
    with pytest.raises(InputError):
        flatten_trips(flat, [Trip(1, conn, 0.0, o, 0.0)])
