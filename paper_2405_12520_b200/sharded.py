"""Multi-GPU engine: one process per GPU, lanes partitioned into spatial bands.

SURVEY.md 8(e).  Every rank builds the same network, trips and routes (the
inputs are replicated; they are small next to the vehicle state), owns the
lanes of its band (shard.py) and simulates them plus a halo of ghost lanes.
One step on rank r is

1. the single-GPU step graph over own + ghost vehicles (csrc/kernels.cu): the
   update of ghosts reproduces exactly what their owner computes for every
   vehicle that can affect an own lane this step (transitions into own lanes,
   revert partners); chains that would leave the exactly-computed zone make
   the engine fail loudly (TSB_ECAP), never silently diverge;
2. one exchange: each rank packs the vehicles of its own lanes that lie in a
   peer's halo and the peers' packets become its ghosts for the next step.
   Two transports:
   * p2p=True (device-driven): the pack kernel writes each message straight
     into the peer's receive slot (peer memory mapped with CUDA IPC; NVLink
     P2P between GPUs), releases the peer's arrival flag, waits for its own
     flags and imports -- all enqueued on the engine stream, no host
     synchronisation and no collective per step (tsb_shard_p2p_*);
   * otherwise tsb_shard_export / tsb_shard_import around
     `torch.distributed.all_to_all_single` on device tensors (NCCL), or gloo
     with host staging;
3. step counters (driving, waiting, finished, ...) are summed over ranks.

Vehicles migrate implicitly: a vehicle that crosses into a peer's band was a
ghost there, so the peer already holds its exact new state.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native, shard
from .cabi import VIEW_DTYPE, TsbReport, pack_network, pack_params, pack_shard, pack_trips
from .errors import InputError
from .flat import FlatNet, FlatTrips, flatten_network, flatten_trips
from .params import EngineConfig

RECORD_BYTES = 32


def alltoall_packets(send, out_bytes: np.ndarray, recv, group=None, host_staging: bool = False):
    """Variable-size all-to-all of byte packets: send[:sum(out_bytes)] holds
    the packets for ranks 0..N-1 back to back; returns (received bytes, the
    per-source sizes).  Device tensors go through NCCL; with host_staging the
    bytes travel through host memory (gloo, tests)."""
    import torch
    import torch.distributed as dist

    dev = send.device
    sizes_out = torch.tensor(out_bytes, dtype=torch.int64)
    sizes_in = torch.zeros(len(out_bytes), dtype=torch.int64)
    if not host_staging and dev.type == "cuda":
        sizes_out, sizes_in = sizes_out.to(dev), sizes_in.to(dev)
    dist.all_to_all_single(sizes_in, sizes_out, group=group)
    in_b = sizes_in.cpu().numpy().astype(np.int64)
    n_out, n_in = int(out_bytes.sum()), int(in_b.sum())
    if n_in > recv.numel():
        raise InputError("receive buffer too small")
    s, r = send[:n_out], recv[:n_in]
    if host_staging and dev.type == "cuda":
        r_h = torch.zeros(n_in, dtype=torch.uint8)
        dist.all_to_all_single(r_h, s.cpu(), in_b.tolist(), out_bytes.tolist(), group=group)
        r.copy_(r_h)
    else:
        dist.all_to_all_single(r, s, in_b.tolist(), out_bytes.tolist(), group=group)
    return r, in_b


class ShardedWorld:
    """One rank of the sharded engine (call collectively on every rank)."""

    def __init__(self, flat: FlatNet, ft: FlatTrips, junc_pos: np.ndarray, config: EngineConfig | None,
                 seed: int, rank: int, nranks: int, device: int = 0, group=None, host_staging: bool = False,
                 pow_mode: int = 1, p2p: bool = False, local_lanes: bool = True):
        import torch
        import torch.distributed as dist

        self.config = config or EngineConfig()
        self.config.validate()
        self.rank, self.nranks = rank, nranks
        self.group = group
        self.dist = dist
        self.torch = torch
        self.host_staging = host_staging
        self.flat, self.ft = flat, ft
        self.plan = shard.plan_all(flat, junc_pos, nranks, self.config)[rank]
        pn, pt = pack_network(flat), pack_trips(ft)
        params = pack_params(self.config, seed, pow_mode=pow_mode)
        h = C.c_void_p()
        self.local_lanes = local_lanes
        if local_lanes:
            # the rank's zone renumbered into a compact local lane space: every
            # lane-proportional buffer and kernel of the rank shrinks to it
            lflat, self.l2g, lplan = shard.local_network(flat, self.plan)
            pl, ps = pack_network(lflat), pack_shard(lplan)
            l2g = np.ascontiguousarray(self.l2g, dtype=np.int32)
            _native.check(_native.lib().tsb_create_sharded_local(
                C.byref(pn.struct), C.byref(pl.struct), l2g.ctypes.data, C.byref(pt.struct), C.byref(params),
                device, C.byref(ps.struct), C.byref(h)))
            self._eng_zone, gflat = lplan.zone, lflat
        else:
            ps = pack_shard(self.plan)
            _native.check(_native.lib().tsb_create_sharded(C.byref(pn.struct), C.byref(pt.struct), C.byref(params),
                                                           device, C.byref(ps.struct), C.byref(h)))
            self.l2g = np.arange(flat.n_lanes, dtype=np.int32)
            self._eng_zone, gflat = self.plan.zone, flat
        self._h = h
        geo_off = np.ascontiguousarray(gflat.geo_off, dtype=np.int64)
        geo_cum = np.ascontiguousarray(gflat.geo_cum if len(gflat.geo_cum) else np.zeros(1), dtype=np.float64)
        geo_ang = np.ascontiguousarray(gflat.geo_angle if len(gflat.geo_angle) else np.zeros(1), dtype=np.float64)
        _native.check(_native.lib().tsb_set_geometry(h, geo_off.ctypes.data, int(geo_off[-1]),
                                                     geo_cum.ctypes.data, geo_ang.ctypes.data))
        self._report = TsbReport()
        self.net = None
        self._flat = flat
        self._ft = ft
        self._road_index = {rid: k for k, rid in enumerate(flat.road_ids)}
        self._vix_of = {tid: k for k, tid in enumerate(ft.ids)}
        self._finished: list = []
        self._fin_seen = 0
        self.device = torch.device("cuda", device)
        # a packet holds at most every vehicle (32 B) plus one int32 count per lane entry
        n_exp = sum(len(x) for x in self.plan.export_lanes)
        n_imp = sum(len(x) for x in self.plan.import_lanes)
        self._send = torch.zeros(len(ft.ids) * RECORD_BYTES + 4 * n_exp + 32 * nranks + 64, dtype=torch.uint8,
                                 device=self.device)
        self._recv = torch.zeros(len(ft.ids) * RECORD_BYTES + 4 * n_imp + 32 * nranks + 64, dtype=torch.uint8,
                                 device=self.device)
        self.exchanged_bytes = 0
        self.p2p = p2p
        self.p2p_error = None
        self._ipc_mapped = []  # peer buffers opened through CUDA IPC (closed in close())
        if p2p:
            # every rank maps every peer's memory, or all keep the collective
            # transport together (e.g. no peer access between the devices)
            self.p2p = self._setup_p2p()
        self._exchange()  # initial ghosts (empty network: zero vehicles)

    def _setup_p2p(self) -> bool:
        """Receive slots and arrival flags of every rank mapped into every
        other rank (CUDA IPC handles exchanged once through the process
        group).  Every rank runs the same collectives whatever fails locally;
        the engines switch to the device exchange only if every rank mapped
        every peer (else all keep the collective transport)."""
        import os

        L = _native.lib()
        recv, flags, slot = C.c_void_p(), C.c_void_p(), C.c_int64()
        hr, hf = (C.c_uint8 * 64)(), (C.c_uint8 * 64)()
        ok = True
        try:
            if os.environ.get("TSB_P2P_FAIL_RANK") == str(self.rank):  # test hook: this rank cannot map
                raise RuntimeError("P2P mapping disabled by TSB_P2P_FAIL_RANK")
            _native.check(L.tsb_shard_p2p_alloc(self._h, C.byref(recv), C.byref(flags), C.byref(slot)))
            _native.check(L.tsb_ipc_handle(recv, hr))
            _native.check(L.tsb_ipc_handle(flags, hf))
        except Exception as exc:  # noqa: BLE001 -- reported, then the fallback
            ok, self.p2p_error = False, repr(exc)
        got = [None] * self.nranks
        self.dist.all_gather_object(got, (ok, bytes(hr), bytes(hf), self.p2p_error), group=self.group)
        if not all(g[0] for g in got):
            self.p2p_error = "; ".join(f"rank {q}: {g[3]}" for q, g in enumerate(got) if not g[0])
            return False
        pr, pf = (C.c_void_p * self.nranks)(), (C.c_void_p * self.nranks)()
        try:
            for q, (_, br, bf, _) in enumerate(got):
                if q == self.rank:
                    pr[q], pf[q] = recv, flags
                    continue
                a, b = C.c_void_p(), C.c_void_p()
                _native.check(L.tsb_ipc_open((C.c_uint8 * 64).from_buffer_copy(br), C.byref(a)))
                self._ipc_mapped.append(a)
                _native.check(L.tsb_ipc_open((C.c_uint8 * 64).from_buffer_copy(bf), C.byref(b)))
                self._ipc_mapped.append(b)
                pr[q], pf[q] = a, b
        except Exception as exc:  # noqa: BLE001
            ok, self.p2p_error = False, repr(exc)
        errs = [None] * self.nranks  # (also orders every mapping before the first exchange)
        self.dist.all_gather_object(errs, (ok, self.p2p_error), group=self.group)
        if not all(g[0] for g in errs):
            self.p2p_error = "; ".join(f"rank {q}: {g[1]}" for q, g in enumerate(errs) if not g[0])
            return False
        _native.check(L.tsb_shard_p2p_set_peers(self._h, pr, pf))
        return True

    @classmethod
    def from_network(cls, net, trips, config=None, seed=0, rank=0, nranks=1, device=0, group=None,
                     host_staging=False, p2p=False, local_lanes=True):
        config = config or EngineConfig()
        flat = flatten_network(net, config.controller)
        ft = flatten_trips(flat, trips)
        jp = np.array([net.junctions[j].position for j in flat.junction_ids], dtype=np.float64).reshape(-1, 2)
        return cls(flat, ft, jp, config, seed, rank, nranks, device, group, host_staging, p2p=p2p,
                   local_lanes=local_lanes)

    def close(self):
        if self._h is not None:
            L = _native.lib()
            L.tsb_destroy(self._h)  # (synchronises the device: no kernel still uses the mappings)
            self._h = None
            for ptr in getattr(self, "_ipc_mapped", []):
                L.tsb_ipc_close(ptr)
            self._ipc_mapped = []

    __del__ = close

    # ------------------------------------------------------------ exchange

    def _exchange(self):
        if self.p2p:
            _native.check(_native.lib().tsb_shard_p2p_exchange(self._h))
            return
        torch = self.torch
        out_b = np.zeros(self.nranks, dtype=np.int64)
        _native.check(_native.lib().tsb_shard_export(self._h, C.c_void_p(self._send.data_ptr()),
                                                     self._send.numel(), out_b.ctypes.data))
        _, in_b = alltoall_packets(self._send, out_b, self._recv, self.group, self.host_staging)
        torch.cuda.current_stream(self.device).synchronize()
        self.exchanged_bytes += int(out_b.sum())
        _native.check(_native.lib().tsb_shard_import(self._h, C.c_void_p(self._recv.data_ptr()), in_b.ctypes.data))

    # ------------------------------------------------------------ stepping

    def step_local(self, n: int = 1):
        """n steps, exchanging ghosts after each (no global reductions)."""
        if self.p2p:
            # the step graph ends with the exchange: n graph replays, no host
            # synchronisation until the report
            _native.check(_native.lib().tsb_step_async(self._h, n))
            _native.check(_native.lib().tsb_report_get(self._h, C.byref(self._report)))
            return
        for _ in range(n):
            _native.check(_native.lib().tsb_step(self._h, 1, C.byref(self._report)))
            self._exchange()

    def exchange_bytes(self) -> int:
        """Bytes this rank sent to its peers so far (either transport)."""
        if self.p2p:
            out = C.c_int64()
            _native.check(_native.lib().tsb_exchange_bytes(self._h, C.byref(out)))
            return int(out.value)
        return self.exchanged_bytes

    def set_p2p_timeout(self, seconds: float) -> None:
        """Bound of the device-side wait for a peer's step (TSB_ECUDA on expiry)."""
        _native.check(_native.lib().tsb_set_p2p_timeout(self._h, float(seconds)))

    def report(self) -> dict:
        """StepReport counters summed over ranks (time and step are shared)."""
        torch, dist = self.torch, self.dist
        r = self._report
        keys = ("driving", "waiting", "finished", "dropped", "injected_now", "finished_now", "vehicle_updates")
        t = torch.tensor([getattr(r, k) for k in keys], dtype=torch.int64)
        if not self.host_staging:
            t = t.to(self.device)
        dist.all_reduce(t, group=self.group)
        out = dict(zip(keys, (int(x) for x in t.cpu().tolist())))
        out["time"] = r.time
        return out

    def own_state(self):
        """This rank's own vehicles, lane-sorted: dict of arrays (vix, lane, road_pos, s, v)."""
        n = max(len(self.ft.ids), 1)
        nd = C.c_int32()
        ls = np.zeros(len(self.l2g) + 1, dtype=np.int32)
        out = {k: np.zeros(2 * n, dtype=t) for k, t in (("vix", np.int32), ("lane", np.int32),
                                                         ("road_pos", np.int32), ("s", np.float64),
                                                         ("v", np.float64))}
        _native.check(_native.lib().tsb_state(self._h, C.byref(nd), ls.ctypes.data, out["vix"].ctypes.data,
                                              out["lane"].ctypes.data, out["road_pos"].ctypes.data,
                                              out["s"].ctypes.data, out["v"].ctypes.data))
        m = nd.value
        own = (self._eng_zone[out["lane"][:m]] & shard.ZONE_OWN) > 0
        res = {k: a[:m][own] for k, a in out.items()}
        res["lane"] = self.l2g[res["lane"]]  # global lane ids (ascending map: the lane-major order holds)
        return res

    # ------------------------------------------------------------ queries (collective: every rank calls)
    #
    # The reference's query surface (world.py:706-714, 746-804, 771-782, 447-493)
    # over the whole sharded network: each rank answers for its own lanes on the
    # device (tsb_get_vehicles / tsb_records / tsb_finished / tsb_road_acc) and
    # the answers are merged across ranks.

    @property
    def time(self) -> float:
        return self._report.time

    def _gather(self, obj) -> list:
        out = [None] * self.nranks
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def get_vehicle(self, vehicle_id: int):
        """StatusView of one vehicle: the rank driving it on its own lanes (or
        where it finished / was dropped) answers; nobody -> still waiting."""
        from .world import _STATUS, StatusView, _route_index

        k = self._vix_of.get(vehicle_id)
        if k is None:
            raise InputError(f"unknown vehicle {vehicle_id}")
        q = np.array([k], dtype=np.int32)
        o = np.zeros(1, dtype=VIEW_DTYPE)
        _native.check(_native.lib().tsb_get_vehicles(self._h, q.ctypes.data, 1, o.ctypes.data))
        mine = list(o[0].tolist())
        if mine[5] in (1, 2):
            mine[3] = int(self.l2g[mine[3]])  # this rank's local lane id -> global
        views = self._gather(tuple(mine))
        pick = next((v for v in views if v[5] in (1, 2, 3)), views[0])  # driving, finished, dropped
        s, v, fin, lane, rp, st, _ = pick
        status = _STATUS[st] if st >= 0 else _STATUS[0]
        dep = float(self.ft.departure[k])
        if status in ("driving", "finished"):
            return StatusView(id=vehicle_id, lane_id=lane, s=s, v=v, status=status,
                              route_index=_route_index(self.flat, lane, rp), depart_time=dep,
                              finish_time=fin if status == "finished" else None)
        return StatusView(id=vehicle_id, lane_id=int(self.ft.origin_lane[k]), s=float(self.ft.origin_s[k]),
                          v=0.0, status=status, route_index=0, depart_time=dep, finish_time=None)

    def records_arrays(self) -> dict:
        """record_step's records over all ranks, sorted by id (each rank's own
        lanes gathered and headed on its device, merged by vix)."""
        n = max(len(self.ft.ids), 1)
        bufs = {k: np.zeros(n, dtype=t) for k, t in (("vix", np.int32), ("lane", np.int32), ("road_pos", np.int32),
                                                     ("s", np.float64), ("v", np.float64),
                                                     ("angle_deg", np.float64))}
        m = C.c_int32()
        _native.check(_native.lib().tsb_records(self._h, n, *(bufs[k].ctypes.data for k in
                                                            ("vix", "lane", "road_pos", "s", "v", "angle_deg")),
                                                C.byref(m)))
        mine = {k: a[:m.value] for k, a in bufs.items()}
        mine["lane"] = self.l2g[mine["lane"]].astype(np.int32)  # global lane ids
        parts = self._gather(mine)
        out = {k: np.concatenate([p[k] for p in parts]) for k in bufs}
        order = np.argsort(out["vix"], kind="stable")
        out = {k: a[order] for k, a in out.items()}
        ids = self.ft.ids
        dense = len(ids) == 0 or (ids[0] == 0 and ids[-1] == len(ids) - 1)
        out["id"] = out["vix"].astype(np.int64) if dense else np.array([ids[i] for i in out["vix"].tolist()],
                                                                       dtype=object)
        out["t"] = self.time
        return out

    def record_step(self, recorder) -> None:
        from .records import VehicleRecord

        r = self.records_arrays()
        ids = self.ft.ids
        for i, l, a, b, g in zip(r["vix"].tolist(), r["lane"].tolist(), r["s"].tolist(), r["v"].tolist(),
                                 r["angle_deg"].tolist()):
            recorder.write(VehicleRecord(t=r["t"], id=ids[i], lane=l, s=a, v=b, angle_deg=g))

    @property
    def finished(self) -> list:
        """Arrivals of every rank merged in the reference's order (step, then
        id: world.py:447-493 commits in id order; finish time = step end)."""
        cap = max(len(self.ft.ids), 1)
        vix = np.zeros(cap, dtype=np.int32)
        t = np.zeros(cap, dtype=np.float64)
        n = C.c_int64()
        _native.check(_native.lib().tsb_finished(self._h, self._fin_seen, cap, vix.ctypes.data, t.ctypes.data,
                                                 C.byref(n)))
        self._fin_seen += n.value
        parts = self._gather((vix[:n.value], t[:n.value]))
        new = sorted((float(tt), int(x)) for pv, pt in parts for x, tt in zip(pv.tolist(), pt.tolist()))
        dep, ids = self.ft.departure, self.ft.ids
        self._finished.extend((ids[x], float(dep[x]), tt) for tt, x in new)
        return self._finished

    def _road_acc(self):
        """Road aggregate over ranks (each road accumulated by its owner only)."""
        torch = self.torch
        nw = int(self.time / self.config.speed_window) + 2
        nr = len(self.flat.road_ids)
        s = np.zeros((max(nr, 1), nw), dtype=np.float64)
        c = np.zeros((max(nr, 1), nw), dtype=np.int64)
        _native.check(_native.lib().tsb_road_acc(self._h, nw, s.ctypes.data, c.ctypes.data))
        ts, tc = torch.from_numpy(s), torch.from_numpy(c)
        if not self.host_staging:
            ts, tc = ts.to(self.device), tc.to(self.device)
        self.dist.all_reduce(ts, group=self.group)
        self.dist.all_reduce(tc, group=self.group)
        return ts.cpu().numpy()[:nr], tc.cpu().numpy()[:nr]

    def road_free_flow(self, road_id: str) -> float:
        from .world import World

        return World.road_free_flow(self, road_id)

    def get_road_speed(self, road_id: str, window: tuple[float, float]) -> float:
        from .world import World

        return World.get_road_speed(self, road_id, window)

    def road_windows(self, horizon: float) -> list:
        from .world import World

        return World.road_windows(self, horizon)
