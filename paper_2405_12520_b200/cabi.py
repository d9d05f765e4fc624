"""ctypes mirrors of the plain-data structs in include/tsb200.h.

Used to pass a ``FlatNet`` / ``FlatTrips`` / ``EngineConfig`` across the
C-ABI.  ``pack_*`` keep the numpy arrays alive on the returned holder so the
pointers stay valid for the duration of the call.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from .flat import FlatNet, FlatTrips
from .params import FIXED

_p = C.POINTER


class TsbNetwork(C.Structure):
    _fields_ = [
        ("n_lanes", C.c_int32),
        ("lane_len", _p(C.c_double)), ("lane_cap", _p(C.c_double)),
        ("lane_kind", _p(C.c_int8)), ("lane_open", _p(C.c_uint8)),
        ("lane_left", _p(C.c_int32)), ("lane_right", _p(C.c_int32)),
        ("lane_road", _p(C.c_int32)), ("lane_junction", _p(C.c_int32)),
        ("lane_pred1", _p(C.c_int32)), ("lane_succ1", _p(C.c_int32)),
        ("succ_off", _p(C.c_int32)), ("succ", _p(C.c_int32)),
        ("pred_off", _p(C.c_int32)), ("pred", _p(C.c_int32)),
        ("n_roads", C.c_int32),
        ("road_lane_off", _p(C.c_int32)), ("road_lanes", _p(C.c_int32)),
        ("n_junctions", C.c_int32),
        ("junc_signal", _p(C.c_uint8)), ("junc_phase_off", _p(C.c_int32)),
        ("phase_dur", _p(C.c_double)), ("lane_green_mask", _p(C.c_uint64)),
        ("junc_phase0", _p(C.c_int32)), ("junc_elapsed0", _p(C.c_double)),
    ]


class TsbTrips(C.Structure):
    _fields_ = [
        ("n", C.c_int32),
        ("key", _p(C.c_uint64)),
        ("origin_lane", _p(C.c_int32)),
        ("origin_s", _p(C.c_double)),
        ("dest_lane", _p(C.c_int32)),
        ("departure", _p(C.c_double)),
    ]


class TsbParams(C.Structure):
    _fields_ = [(k, C.c_double) for k in (
        "dt", "lookahead", "idm_v0", "idm_T", "idm_a_max", "idm_b", "idm_delta", "idm_s0",
        "mobil_politeness", "mobil_threshold", "mobil_b_safe", "mobil_eval_prob",
        "vehicle_length", "speed_window", "amber", "s0_floor", "mp_interval", "mp_min_green")] + [
        ("controller", C.c_int32), ("pow_mode", C.c_int32), ("seed", C.c_uint64)]


class TsbReport(C.Structure):
    _fields_ = [("time", C.c_double), ("step_no", C.c_int64)] + [
        (k, C.c_int64) for k in ("driving", "waiting", "finished", "dropped", "injected_now",
                                 "finished_now", "vehicle_updates", "reverts_last",
                                 "resolve_sequential", "reverts_total")]


class TsbVehicleView(C.Structure):
    _fields_ = [("s", C.c_double), ("v", C.c_double), ("finish_time", C.c_double),
                ("lane", C.c_int32), ("road_pos", C.c_int32), ("status", C.c_int32), ("pad", C.c_int32)]


# numpy view of an array of tsb_vehicle_view
VIEW_DTYPE = np.dtype([("s", "<f8"), ("v", "<f8"), ("finish_time", "<f8"), ("lane", "<i4"),
                       ("road_pos", "<i4"), ("status", "<i4"), ("pad", "<i4")])


class TsbShard(C.Structure):
    _fields_ = [
        ("rank", C.c_int32), ("nranks", C.c_int32),
        ("zone", _p(C.c_uint8)),
        ("export_off", _p(C.c_int32)), ("export_lanes", _p(C.c_int32)),
        ("import_off", _p(C.c_int32)), ("import_lanes", _p(C.c_int32)),
        ("export_kind", _p(C.c_uint8)), ("import_kind", _p(C.c_uint8)),
    ]


_CT = {np.float64: C.c_double, np.int8: C.c_int8, np.uint8: C.c_uint8,
       np.int32: C.c_int32, np.uint64: C.c_uint64, np.int64: C.c_int64}


def ptr(arr: np.ndarray, dtype):
    """Pointer to a contiguous array of exactly ``dtype`` (no silent casts)."""
    if arr.dtype != np.dtype(dtype) or not arr.flags["C_CONTIGUOUS"]:
        raise TypeError(f"expected contiguous {np.dtype(dtype)}, got {arr.dtype}")
    return arr.ctypes.data_as(_p(_CT[np.dtype(dtype).type]))


class Packed:
    """Holder keeping arrays alive next to the struct that points at them."""

    def __init__(self, struct, keep):
        self.struct = struct
        self.keep = keep


def _nonempty(a: np.ndarray, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a if a.size else np.zeros(1, dtype=dtype)


def pack_network(f: FlatNet) -> Packed:
    fields = {
        "lane_len": np.float64, "lane_cap": np.float64, "lane_kind": np.int8,
        "lane_open": np.uint8, "lane_left": np.int32, "lane_right": np.int32,
        "lane_road": np.int32, "lane_junction": np.int32, "lane_pred1": np.int32,
        "lane_succ1": np.int32, "succ_off": np.int32, "succ": np.int32,
        "pred_off": np.int32, "pred": np.int32, "road_lane_off": np.int32,
        "road_lanes": np.int32, "junc_signal": np.uint8, "junc_phase_off": np.int32,
        "phase_dur": np.float64, "lane_green_mask": np.uint64, "junc_phase0": np.int32,
        "junc_elapsed0": np.float64,
    }
    keep = {k: _nonempty(getattr(f, k), t) for k, t in fields.items()}
    s = TsbNetwork(n_lanes=f.n_lanes, n_roads=len(f.road_ids), n_junctions=len(f.junction_ids),
                   **{k: ptr(a, fields[k]) for k, a in keep.items()})
    return Packed(s, keep)


def pack_trips(t: FlatTrips) -> Packed:
    fields = {"key": np.uint64, "origin_lane": np.int32, "origin_s": np.float64,
              "dest_lane": np.int32, "departure": np.float64}
    keep = {k: _nonempty(getattr(t, k), tp) for k, tp in fields.items()}
    s = TsbTrips(n=len(t.ids), **{k: ptr(a, fields[k]) for k, a in keep.items()})
    return Packed(s, keep)


def pack_shard(plan) -> Packed:
    """tsb_shard from a shard.ShardPlan."""
    def csr(lists):
        off = np.zeros(len(lists) + 1, dtype=np.int32)
        off[1:] = np.cumsum([len(x) for x in lists])
        flat = np.concatenate([np.asarray(x, dtype=np.int32) for x in lists]) if lists else np.zeros(0, np.int32)
        return off, _nonempty(flat, np.int32)
    eo, el = csr(plan.export_lanes)
    io, il = csr(plan.import_lanes)
    ek = _nonempty(np.concatenate([np.asarray(x, dtype=np.uint8) for x in plan.export_kind])
                   if plan.export_kind else np.zeros(0, np.uint8), np.uint8)
    ik = _nonempty(np.concatenate([np.asarray(x, dtype=np.uint8) for x in plan.import_kind])
                   if plan.import_kind else np.zeros(0, np.uint8), np.uint8)
    zone = _nonempty(plan.zone, np.uint8)
    keep = dict(zone=zone, eo=eo, el=el, io=io, il=il, ek=ek, ik=ik)
    s = TsbShard(rank=plan.rank, nranks=plan.nranks, zone=ptr(zone, np.uint8),
                 export_off=ptr(eo, np.int32), export_lanes=ptr(el, np.int32),
                 import_off=ptr(io, np.int32), import_lanes=ptr(il, np.int32),
                 export_kind=ptr(ek, np.uint8), import_kind=ptr(ik, np.uint8))
    return Packed(s, keep)


def pack_params(cfg, seed: int, pow_mode: int = 1) -> TsbParams:
    return TsbParams(
        dt=cfg.dt, lookahead=cfg.lookahead,
        idm_v0=cfg.idm.v0, idm_T=cfg.idm.T, idm_a_max=cfg.idm.a_max, idm_b=cfg.idm.b,
        idm_delta=cfg.idm.delta, idm_s0=cfg.idm.s0,
        mobil_politeness=cfg.mobil.politeness, mobil_threshold=cfg.mobil.threshold,
        mobil_b_safe=cfg.mobil.b_safe, mobil_eval_prob=cfg.mobil.eval_prob,
        vehicle_length=cfg.vehicle_length, speed_window=cfg.speed_window, amber=cfg.amber,
        s0_floor=cfg.s0_floor, mp_interval=cfg.mp_interval, mp_min_green=cfg.mp_min_green,
        controller=0 if cfg.controller == FIXED else 1, pow_mode=pow_mode,
        seed=seed & ((1 << 64) - 1),
    )
