"""Native grid builder (csrc/gridgen.cpp): ``generate_grid`` + ``flatten_network``
in one C++ pass, for the large synthetic configs (M1, C4, C5: SURVEY 8(f)
rank 4).

``grid_flat(rows, cols, ...)`` returns the same ``FlatNet`` as
``flatten_network(generate_grid(rows, cols, ...), controller)`` -- the
reference's lane numbering, geometry and signal programs (network.py:367-560)
-- plus the junction positions (for the sharded partition), without building
a Python ``RoadNetwork``.  Pinned array for array against the Python builder
and by sha256 against the reference at the bench scales
(tests/test_gridgen.py).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native
from .errors import InputError
from .flat import FlatNet
from .params import FIXED, MAX_PRESSURE

# tsb_grid_export order: (FlatNet field or extra, dtype, size index in tsb_grid_sizes)
_ARRAYS = (
    ("lane_len", np.float64, 0), ("lane_cap", np.float64, 0), ("lane_kind", np.int8, 0),
    ("lane_open", np.uint8, 0), ("lane_left", np.int32, 0), ("lane_right", np.int32, 0),
    ("lane_road", np.int32, 0), ("lane_junction", np.int32, 0), ("lane_pred1", np.int32, 0),
    ("lane_succ1", np.int32, 0), ("succ_off", np.int32, "n+1"), ("succ", np.int32, 1),
    ("pred_off", np.int32, "n+1"), ("pred", np.int32, 2), ("road_lane_off", np.int32, "r+1"),
    ("road_lanes", np.int32, 4), ("junc_signal", np.uint8, 5), ("junc_phase_off", np.int32, "j+1"),
    ("phase_dur", np.float64, 6), ("lane_green_mask", np.uint64, 0), ("junc_phase0", np.int32, 5),
    ("junc_elapsed0", np.float64, 5), ("geo_off", np.int64, "n+1"), ("geo_cum", np.float64, 7),
    ("geo_angle", np.float64, 7), ("junc_pos", np.float64, "2j"), ("road_ids", np.uint8, 8),
    ("junction_ids", np.uint8, 9),
)


def grid_flat(rows: int, cols: int, block_length: float = 200.0, lanes_per_direction: int = 1,
              max_speed: float = 16.67, controller: str = FIXED):
    """(FlatNet, junction positions [n_junctions, 2] in junction_ids order)."""
    if controller not in (FIXED, MAX_PRESSURE):
        raise InputError(f"unknown controller {controller!r}")
    L = _native.lib()
    h = C.c_void_p()
    rc = L.tsb_grid_build(rows, cols, float(block_length), lanes_per_direction, float(max_speed),
                          0 if controller == FIXED else 1, C.byref(h))
    if rc != 0:
        raise InputError("invalid grid parameters")
    try:
        sz = np.zeros(10, dtype=np.int64)
        _native.check(L.tsb_grid_sizes(h, sz.ctypes.data))
        n, nr, nj = int(sz[0]), int(sz[3]), int(sz[5])
        count = {"n+1": n + 1, "r+1": nr + 1, "j+1": nj + 1, "2j": 2 * nj}
        arrs = {}
        for name, dt, k in _ARRAYS:
            m = count[k] if isinstance(k, str) else int(sz[k])
            arrs[name] = np.zeros(m, dtype=dt)
        ptrs = (C.c_void_p * len(_ARRAYS))(*[arrs[name].ctypes.data for name, _, _ in _ARRAYS])
        _native.check(L.tsb_grid_export(h, ptrs))
    finally:
        L.tsb_grid_destroy(h)
    road_ids = arrs.pop("road_ids").tobytes().decode().split("\n")
    junction_ids = arrs.pop("junction_ids").tobytes().decode().split("\n")
    jpos = arrs.pop("junc_pos").reshape(-1, 2)
    flat = FlatNet(n_lanes=n, road_ids=road_ids, junction_ids=junction_ids, **arrs)
    return flat, jpos
