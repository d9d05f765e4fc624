"""Router with the reference interface (trafficsim/engine/routing.py:19-117),
backed by the native host router in csrc/router.cpp.

Free-flow-time shortest lane routes: reverse Dijkstra over open lanes weighted
length / max_speed, tight-edge extraction with the smallest successor id.
Routing stays on the host (it runs at first injection attempts and
reroutes, not per step); batch routing at engine creation is multithreaded.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native
from .cabi import pack_network
from .errors import InputError, NoRouteError
from .flat import KIND_ROAD, flatten_network
from .network import OPEN, ROAD


class Router:
    def __init__(self, net, cache_size: int = 256, flat=None):
        self.net = net
        self.cache_size = cache_size  # API parity; results do not depend on caching
        self._flat = flat
        self._h = None
        self.rebuild()

    def rebuild(self) -> None:
        """Refresh weights after speed or restriction changes (routing.py:29-45)."""
        self.close()
        self._flat = flatten_network(self.net) if self._flat is None else self._refresh(self._flat)
        self._packed = pack_network(self._flat)
        h = C.c_void_p()
        _native.check(_native.lib().tsb_router_create(C.byref(self._packed.struct), C.byref(h)))
        self._h = h

    def _refresh(self, flat):
        if self.net is None:  # built from a FlatNet alone (gridgen.grid_flat): flat is authoritative
            return flat
        for lid, lane in self.net.lanes.items():
            flat.lane_cap[lid] = lane.max_speed
            flat.lane_open[lid] = 1 if lane.restriction == OPEN else 0
        return flat

    def close(self):
        if getattr(self, "_h", None):
            _native.lib().tsb_router_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def weight(self, lane_id: int) -> float:
        lane = self.net.lanes[lane_id]
        if lane.restriction != OPEN:
            raise KeyError(lane_id)
        return lane.length / lane.max_speed

    def route(self, origin_lane: int, dest_lane: int) -> list[int]:
        for lid in (origin_lane, dest_lane):
            if lid not in self.net.lanes:
                raise InputError(f"unknown lane {lid}")
            if self.net.lanes[lid].kind != ROAD:
                raise InputError(f"lane {lid} is not a road lane")
        if self.net.lanes[dest_lane].restriction != OPEN:
            raise InputError(f"destination lane {dest_lane} is closed or unknown")
        cap = max(self._flat.n_lanes, 1)
        buf = np.zeros(cap, dtype=np.int32)
        n = C.c_int32()
        cost = C.c_double()
        _native.check(_native.lib().tsb_router_route(self._h, origin_lane, dest_lane, cap,
                                                     buf.ctypes.data, C.byref(n), C.byref(cost)))
        if n.value == 0:
            raise NoRouteError(f"no route from lane {origin_lane} to lane {dest_lane}")
        return [int(x) for x in buf[: n.value]]

    def route_cost(self, path: list[int]) -> float:
        cost = 0.0
        for lid in reversed(path):
            cost = self.weight(lid) + cost
        return cost

    def reachable_sets(self, dests: list[int]) -> dict:
        """dest -> boolean array over lanes: origin can reach dest (dist_to keys)."""
        n = self._flat.n_lanes
        d = np.asarray(dests, dtype=np.int32)
        out = np.zeros((len(dests), max(n, 1)), dtype=np.uint8)
        _native.check(_native.lib().tsb_router_reach(self._h, len(dests), d.ctypes.data, out.ctypes.data))
        return {int(k): out[i].astype(bool) for i, k in enumerate(dests)}


def roads_of_route(net, path: list[int]) -> list[str]:
    """Ordered road ids visited by a lane route (routing.py:110-117)."""
    roads: list[str] = []
    for lid in path:
        lane = net.lanes[lid]
        if lane.kind == ROAD and (not roads or roads[-1] != lane.parent):
            roads.append(lane.parent)
    return roads
