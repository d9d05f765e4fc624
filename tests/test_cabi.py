"""The C-ABI boundary without a GPU: libtsb200.so loads, exports every entry
point include/tsb200.h declares, its host-only router agrees with the
oracle's, and engine creation fails loudly (EngineError, never a CPU
fallback) when no CUDA device is present."""

from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2405_12520_b200 import _native
from paper_2405_12520_b200.cabi import pack_network
from tests import goldens as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "tsb200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tsb_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_surface():
    syms = declared_symbols()
    for s in ("tsb_create", "tsb_step", "tsb_state", "tsb_destroy", "tsb_last_error", "tsb_road_acc",
              "tsb_min_front_gap", "tsb_set_lane", "tsb_set_signal_phase", "tsb_finished", "tsb_status",
              "tsb_get_vehicles", "tsb_records", "tsb_set_geometry", "tsb_grid_build", "tsb_grid_export"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    L = _native.lib()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing


def test_python_signatures_cover_the_header():
    assert set(declared_symbols()) <= set(_native.SIGNATURES)


def test_exports_are_c_linkage():
    out = os.popen(f"nm -D --defined-only {_native.LIB_PATH}").read()
    for s in declared_symbols():
        assert re.search(rf"\bT {s}$", out, flags=re.M), s


def _router(net_name):
    L = _native.lib()
    flat = G.golden_flat(net_name)
    pk = pack_network(flat)
    h = C.c_void_p()
    _native.check(L.tsb_router_create(C.byref(pk.struct), C.byref(h)))
    return L, flat, pk, h


def test_host_router_matches_oracle_route_costs():
    """routing.py:70-107: the engine's native router (used at injection and
    on reroute) against the oracle's restatement on the same network."""
    from oracle.bind import OracleWorld, lib as olib
    from paper_2405_12520_b200 import EngineConfig
    L, flat, pk, h = _router("grid44x2")
    o = OracleWorld(None, [], EngineConfig(), 0, pow_mode=1, flat=flat)
    try:
        roads = np.nonzero(flat.lane_kind == 0)[0]
        rng = np.random.default_rng(3)
        buf = np.zeros(4096, dtype=np.int32)
        checked = 0
        for _ in range(300):
            a, b = (int(x) for x in rng.choice(roads, 2))
            n = C.c_int32()
            cost = C.c_double()
            _native.check(L.tsb_router_route(h, a, b, 4096, buf.ctypes.data, C.byref(n), C.byref(cost)))
            oc = C.c_double()
            onr = C.c_int32()
            olib().orc_route_cost(o._h, a, b, C.byref(oc), C.byref(onr))
            if n.value == 0:
                assert oc.value < 0
            else:
                checked += 1
                assert cost.value == oc.value
                assert buf[0] == a and buf[n.value - 1] == b
        assert checked > 50
    finally:
        o.close()
        L.tsb_router_destroy(h)


def test_router_reach_sets():
    L, flat, pk, h = _router("grid44")
    try:
        roads = np.nonzero(flat.lane_kind == 0)[0].astype(np.int32)
        dests = roads[:5].copy()
        reach = np.zeros(5 * flat.n_lanes, dtype=np.uint8)
        _native.check(L.tsb_router_reach(h, 5, dests.ctypes.data, reach.ctypes.data))
        reach = reach.reshape(5, flat.n_lanes)
        for k, d in enumerate(dests):
            assert reach[k, d] == 1
            for o in roads[:10]:
                n = C.c_int32()
                buf = np.zeros(4096, dtype=np.int32)
                _native.check(L.tsb_router_route(h, int(o), int(d), 4096, buf.ctypes.data, C.byref(n), None))
                assert (n.value > 0) == bool(reach[k, o])
    finally:
        L.tsb_router_destroy(h)


def test_engine_creation_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2405_12520_b200 import EngineError, World, generate_grid
    with pytest.raises(EngineError):
        World(generate_grid(2, 2), [])
