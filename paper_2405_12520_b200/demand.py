"""Trip type and synthetic demand generators (input side of the hot path).

``Trip`` mirrors trafficsim/demand.py:47-53.  ``random_trips`` restates the
reference's uniform generator (demand.py:260-284) bit-for-bit: the same numpy
Philox stream keyed by (seed, 0) (rng.py:44-47) and the same draw order, so
BASELINE configs C1/C1b produce identical trips here and on the GPU box.
``preplaced_trips`` is the routable pre-placed demand of SURVEY appendix C
used for the large configs (C3, M1, C4, C5).
"""

from __future__ import annotations

import random
from dataclasses import dataclass

import numpy as np

from .errors import InputError

_MASK64 = (1 << 64) - 1


@dataclass(frozen=True)
class Trip:
    id: int
    origin_lane: int
    origin_s: float
    dest_lane: int
    departure: float


def philox_stream(seed: int, index: int) -> np.random.Generator:
    key = np.array([seed & _MASK64, index & _MASK64], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


def random_trips(net, count: int, seed: int, window=(0.0, 3600.0)) -> list[Trip]:
    if count < 0:
        raise InputError("count must be non-negative")
    t0, t1 = window
    if not t0 < t1:
        raise InputError("window must satisfy t_start < t_end")
    pool = sorted(net.road_lane_ids())
    if not pool:
        raise InputError("network has no road lanes")
    g = philox_stream(seed, 0)
    out = []
    for k in range(count):
        o = pool[int(g.integers(len(pool)))]
        os_ = g.random() * 0.5 * net.lanes[o].length
        d = pool[int(g.integers(len(pool)))]
        dep = t0 + g.random() * (t1 - t0)
        out.append(Trip(k, o, os_, d, dep))
    out.sort(key=lambda t: (t.departure, t.id))
    return out


def preplaced_trips(net, router, n_vehicles: int, spacing: float, seed: int = 1234,
                    pool_size: int = 256, draws: int = 32) -> list[Trip]:
    """Pre-placed, routable demand.

    Road lanes in id order get slots at ``spacing * k`` (k = 0, 1, ... while
    the slot fits the lane); each slot's destination is the first of
    ``draws`` candidates from a fixed pool of ``pool_size`` road lanes from
    which the origin is routable.  Departure 0; ids sorted by
    (destination, lane, s) so injection hits the router's LRU.  Slots with
    no routable candidate are skipped.  The first ``n_vehicles`` are kept.
    """
    rng = random.Random(seed)
    if hasattr(net, "lane_kind"):  # a FlatNet (gridgen.grid_flat): same lanes, same lengths
        lanes = [int(x) for x in np.nonzero(net.lane_kind == 0)[0]]
        lane_len = net.lane_len.tolist()
    else:
        lanes = sorted(net.road_lane_ids())
        lane_len = {lid: net.lanes[lid].length for lid in lanes}
    pool = sorted(rng.sample(lanes, min(pool_size, len(lanes))))
    reach = router.reachable_sets(pool)     # dest -> set-like of origins
    slots = []
    for lid in lanes:
        length = lane_len[lid]
        k = 0
        while spacing * k <= length:
            slots.append((lid, spacing * k))
            k += 1
    picked = []
    for lid, s in slots:
        if len(picked) >= n_vehicles:
            break
        dest = None
        for _ in range(draws):
            cand = pool[rng.randrange(len(pool))]
            if cand != lid and reach[cand][lid]:
                dest = cand
                break
        if dest is not None:
            picked.append((dest, lid, s))
    picked.sort()
    return [Trip(i, lid, s, dest, 0.0) for i, (dest, lid, s) in enumerate(picked)]
