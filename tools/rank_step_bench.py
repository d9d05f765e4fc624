"""Rank-local step time of the sharded engine (no exchange, one GPU): rank r of
N lane bands of M1 (bench.py's workload), created with the compact local
lane space (tsb_create_sharded_local) and with the whole network's lane
numbering (tsb_create_sharded); own vehicles only (no peers, so no ghosts).
Prints one JSON line per (rank, numbering)."""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2405_12520_b200 import EngineConfig, _native, shard  # noqa: E402
from paper_2405_12520_b200.cabi import TsbReport, pack_network, pack_params, pack_shard, pack_trips  # noqa: E402


def main():
    nranks = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    ranks = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [nranks // 2]
    steps = 50
    _, flat, _, ft, jp = bench.build_workload(1_000_000, 29.0)
    cfg = EngineConfig()
    plans = shard.plan_all(flat, jp, nranks, cfg)
    L = _native.lib()
    pn, pt, params = pack_network(flat), pack_trips(ft), pack_params(cfg, 42, pow_mode=0)
    for r in ranks:
        for local in (True, False):
            h = C.c_void_p()
            if local:
                lflat, l2g, lplan = shard.local_network(flat, plans[r])
                pl, ps = pack_network(lflat), pack_shard(lplan)
                l2g = np.ascontiguousarray(l2g, dtype=np.int32)
                _native.check(L.tsb_create_sharded_local(C.byref(pn.struct), C.byref(pl.struct), l2g.ctypes.data,
                                                         C.byref(pt.struct), C.byref(params), 0, C.byref(ps.struct),
                                                         C.byref(h)))
                nl = lflat.n_lanes
            else:
                ps = pack_shard(plans[r])
                _native.check(L.tsb_create_sharded(C.byref(pn.struct), C.byref(pt.struct), C.byref(params), 0,
                                                   C.byref(ps.struct), C.byref(h)))
                nl = flat.n_lanes
            rep = TsbReport()
            _native.check(L.tsb_step(h, 1, C.byref(rep)))   # injection of the rank's own vehicles
            _native.check(L.tsb_step(h, 10, C.byref(rep)))
            ms = C.c_double()
            _native.check(L.tsb_time_steps(h, steps, C.byref(ms)))
            _native.check(L.tsb_report_get(h, C.byref(rep)))
            print(json.dumps({"nranks": nranks, "rank": r, "numbering": "local" if local else "global",
                              "lanes": nl, "driving": rep.driving, "ms_per_step": ms.value / steps}), flush=True)
            L.tsb_destroy(h)


if __name__ == "__main__":
    main()
