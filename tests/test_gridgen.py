"""Native grid builder (csrc/gridgen.cpp, gridgen.grid_flat) against the
Python builder (pinned to the reference by test_inputs.py) array for array,
and against the reference itself by sha256 at the bench scales (M1/C4:
100x100x3, C5: 200x200x3; tests/golden/scale_sha.json, made from the
reference by tests/golden/make_scale_sha.py)."""

import json
import math
import os
import random
import time

import numpy as np
import pytest

from paper_2405_12520_b200 import Router, generate_grid, preplaced_trips
from paper_2405_12520_b200 import _native
from paper_2405_12520_b200.flat import flatten_network
from paper_2405_12520_b200.gridgen import grid_flat
from tests.goldens import NET_FIELDS

HERE = os.path.dirname(os.path.abspath(__file__))


def test_vector_norm_matches_cpython_math_dist():
    """math.dist / math.hypot are CPython's vector_norm, restated in C++."""
    rng = random.Random(11)
    L = _native.lib()
    for _ in range(100_000):
        p = [rng.uniform(-1e4, 1e4) for _ in range(4)]
        if rng.random() < 0.3:  # grid-like coordinates: quarter-metre offsets
            p = [round(x * 4) / 4 for x in p]
        assert L.tsb_py_dist(*p) == math.dist(p[:2], p[2:])


@pytest.mark.parametrize("args", [(2, 2, 200.0, 1), (4, 4, 200.0, 2), (5, 5, 200.0, 3), (6, 6, 60.0, 1),
                                  (5, 5, 80.0, 2), (3, 7, 137.3, 2), (12, 9, 400.0, 3), (4, 4, 30.0, 4)])
@pytest.mark.parametrize("controller", ["fixed", "max_pressure"])
def test_grid_flat_equals_python_builder(args, controller):
    f, jpos = grid_flat(*args, controller=controller)
    net = generate_grid(*args)
    g = flatten_network(net, controller)
    assert f.n_lanes == g.n_lanes and f.road_ids == g.road_ids and f.junction_ids == g.junction_ids
    for k in NET_FIELDS:
        a, b = getattr(f, k), getattr(g, k)
        assert a.dtype == b.dtype and np.array_equal(a, b), k
    assert np.array_equal(jpos, np.array([net.junctions[j].position for j in g.junction_ids]))


def _sha(f):
    import hashlib

    h = hashlib.sha256()
    h.update(str(f.n_lanes).encode())
    h.update("\n".join(f.road_ids).encode())
    h.update("\n".join(f.junction_ids).encode())
    for k in NET_FIELDS:
        a = getattr(f, k)
        h.update(k.encode())
        h.update(a.dtype.str.encode())
        h.update(a.tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("rows,cols", [(100, 100), (200, 200)])
def test_grid_flat_matches_reference_at_scale(rows, cols):
    """M1/C4 (100x100x3) and C5 (200x200x3) grids: sha256 of every flattened
    array equals the reference's (its own generate_grid, flattened), built
    in seconds."""
    ref = json.load(open(os.path.join(HERE, "golden", "scale_sha.json")))
    for ctl in ("fixed", "max_pressure"):
        t0 = time.time()
        f, _ = grid_flat(rows, cols, 400.0, 3, controller=ctl)
        dt = time.time() - t0
        exp = ref[f"grid{rows}x{cols}_400_3_{ctl}"]
        assert f.n_lanes == exp["n_lanes"]
        assert _sha(f) == exp["sha256"], (rows, cols, ctl)
        assert dt < 10.0


def test_preplaced_trips_from_flat_equal_from_network():
    net = generate_grid(6, 6, block_length=200.0, lanes_per_direction=2)
    f, _ = grid_flat(6, 6, 200.0, 2)
    r1, r2 = Router(net), Router(None, flat=f)
    try:
        assert preplaced_trips(net, r1, 1500, 16.0) == preplaced_trips(f, r2, 1500, 16.0)
    finally:
        r1.close()
        r2.close()
