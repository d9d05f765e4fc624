"""INTEGRATION.md's claim that the drop-in World accepts the reference's own
input objects (RoadNetwork, Trip, EngineConfig), checked in the development
container where the reference package is importable (skipped elsewhere).
The flattening of the reference objects must equal the flattening of this
package's rebuilt inputs, and on a CPU-only host construction must stop at
the device with EngineError (no CPU fallback)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF)
    try:
        import trafficsim.demand as d
        import trafficsim.engine as e
        import trafficsim.network as n
        yield n, d, e
    finally:
        sys.path.remove(REF)


def test_reference_objects_flatten_like_ours(ref):
    n, d, e = ref
    from paper_2405_12520_b200 import EngineConfig, generate_grid, random_trips
    from paper_2405_12520_b200.cabi import pack_params
    from paper_2405_12520_b200.flat import flatten_network, flatten_trips
    rnet = n.generate_grid(3, 3, lanes_per_direction=2)
    rtrips = d.random_trips(rnet, 50, 7, window=(0.0, 100.0))
    a, b = flatten_network(rnet), flatten_network(generate_grid(3, 3, lanes_per_direction=2))
    for f in ("lane_len", "succ", "succ_off", "lane_green_mask", "junc_elapsed0", "geo_angle"):
        assert np.array_equal(getattr(a, f), getattr(b, f))
    ta = flatten_trips(a, rtrips)
    tb = flatten_trips(b, random_trips(generate_grid(3, 3, lanes_per_direction=2), 50, 7, window=(0.0, 100.0)))
    assert ta.ids == tb.ids and np.array_equal(ta.origin_s, tb.origin_s)
    pr, po = pack_params(e.EngineConfig(), 42), pack_params(EngineConfig(), 42)
    assert bytes(pr) == bytes(po)


def test_world_with_reference_inputs_needs_the_device(ref):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    n, d, e = ref
    from paper_2405_12520_b200 import EngineError, World
    rnet = n.generate_grid(2, 2)
    with pytest.raises(EngineError):
        World(rnet, d.random_trips(rnet, 5, 1, window=(0.0, 10.0)), e.EngineConfig(), seed=1)
