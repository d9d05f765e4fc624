"""Host-side logic of the sharded engine (CPU): the lane partition and the
halo zones (paper_2405_12520_b200/shard.py) and the packet transport over a
real 2-rank gloo process group."""

from __future__ import annotations

import math
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2405_12520_b200 import EngineConfig, generate_grid, make_ring
from paper_2405_12520_b200 import shard
from paper_2405_12520_b200.flat import KIND_CONNECTOR, KIND_ROAD, flatten_network

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _plans(net, n):
    flat = flatten_network(net)
    jp = np.array([net.junctions[j].position for j in flat.junction_ids], dtype=np.float64)
    return flat, shard.plan_all(flat, jp, n, EngineConfig())


@pytest.mark.parametrize("n", [2, 3, 4])
def test_partition_covers_lanes_and_keeps_roads_whole(n):
    flat, plans = _plans(generate_grid(6, 6, lanes_per_direction=2), n)
    owner = plans[0].lane_owner
    valid = flat.lane_kind >= 0
    assert np.all(owner[valid] >= 0) and np.all(owner[valid] < n)
    for r in range(len(flat.road_ids)):
        lanes = flat.road_lanes[flat.road_lane_off[r]:flat.road_lane_off[r + 1]]
        assert len(set(owner[lanes].tolist())) == 1
    counts = np.bincount(owner[valid], minlength=n)
    assert counts.min() > 0.5 * counts.mean()  # balanced bands
    for p in plans:
        own = (p.zone & shard.ZONE_OWN) > 0
        assert np.array_equal(own, owner == p.rank)
        assert np.all(p.zone[own] & shard.ZONE_EXACT)  # own lanes are computed exactly


def test_halo_holds_lookahead_and_feeders():
    net = generate_grid(6, 6, lanes_per_direction=2)
    flat, plans = _plans(net, 2)
    cfg = EngineConfig()
    travel = shard.max_step_travel(flat, cfg)
    for p in plans:
        own = set(np.nonzero(p.lane_owner == p.rank)[0].tolist())
        zone = p.zone > 0
        reads = shard._reach(flat, own, cfg.lookahead + travel, downstream=True)
        feeders = shard._reach(flat, own, travel, downstream=False)
        assert all(zone[x] for x in reads | feeders)


def test_export_import_lists_are_mutual():
    flat, plans = _plans(generate_grid(8, 8, lanes_per_direction=3), 4)
    for p in plans:
        for q in range(4):
            assert np.array_equal(p.export_lanes[q], plans[q].import_lanes[p.rank])
            if q != p.rank:
                imp = plans[q].import_lanes[p.rank]
                assert np.all(p.lane_owner[imp] == p.rank)
                assert np.all(plans[q].zone[imp] & shard.ZONE_HALO)


@pytest.mark.parametrize("n", [2, 3])
def test_max_pressure_lanes_are_counted_or_imported(n):
    """Max-pressure sharded: for every junction with a connector in a rank's
    zone, each connector's predecessor and successor lane is own (counted
    locally) or imported from its owner as a count-only entry (kind 1); the
    owner's export list mirrors it, and fixed-time plans carry no such entries."""
    net = generate_grid(6, 6, lanes_per_direction=2)
    flat = flatten_network(net, "max_pressure")
    jp = np.array([net.junctions[j].position for j in flat.junction_ids], dtype=np.float64)
    plans = shard.plan_all(flat, jp, n, EngineConfig(controller="max_pressure"))
    fixed = shard.plan_all(flat, jp, n, EngineConfig())
    for p, pf in zip(plans, fixed):
        assert all(not np.any(k) for k in pf.import_kind)
        conn = np.nonzero((flat.lane_kind == KIND_CONNECTOR) & (p.zone > 0))[0]
        juncs = set(flat.lane_junction[conn].tolist())
        need = set()
        for c in np.nonzero(flat.lane_kind == KIND_CONNECTOR)[0]:
            if flat.lane_junction[c] in juncs:
                need |= {int(flat.lane_pred1[c]), int(flat.lane_succ1[c])}
        got = set()
        for q in range(n):
            lanes, kinds = p.import_lanes[q], p.import_kind[q]
            assert np.all(np.diff(kinds.astype(int)) >= 0)  # kind-1 entries follow the halo lanes
            mp = lanes[kinds == 1]
            assert np.all(p.lane_owner[mp] == q)
            got |= set(mp.tolist())
            assert np.array_equal(plans[q].export_lanes[p.rank], lanes)
            assert np.array_equal(plans[q].export_kind[p.rank], kinds)
        own = {x for x in need if p.lane_owner[x] == p.rank}
        assert need == own | got and not (own & got)


@pytest.mark.parametrize("controller", ["fixed", "max_pressure"])
def test_local_lane_space(controller):
    """shard.local_network: the rank's lanes in ascending global order; own and
    halo lanes, exchange lanes and whole roads present; every own lane keeps
    all of its successors and predecessors (only the zone edge loses any);
    lane references and exchange lists map back to the global ids."""
    net = generate_grid(8, 8, lanes_per_direction=3)
    flat = flatten_network(net, controller)
    jp = np.array([net.junctions[j].position for j in flat.junction_ids], dtype=np.float64)
    for p in shard.plan_all(flat, jp, 3, EngineConfig(controller=controller)):
        lf, l2g, lp = shard.local_network(flat, p)
        assert np.all(np.diff(l2g) > 0) and lf.n_lanes == len(l2g) < flat.n_lanes
        assert set(np.nonzero(p.zone > 0)[0].tolist()) <= set(l2g.tolist())
        assert np.array_equal(lp.zone, p.zone[l2g])
        for q in range(p.nranks):
            assert np.array_equal(l2g[lp.import_lanes[q]], p.import_lanes[q])
            assert np.array_equal(l2g[lp.export_lanes[q]], p.export_lanes[q])
        for r in range(len(lf.road_ids)):
            mine = lf.road_lanes[lf.road_lane_off[r]:lf.road_lane_off[r + 1]]
            full = flat.road_lanes[flat.road_lane_off[r]:flat.road_lane_off[r + 1]]
            assert len(mine) in (0, len(full)) and np.array_equal(l2g[mine], full[:len(mine)])
        for l in np.nonzero(lp.zone & shard.ZONE_OWN)[0]:
            g = l2g[l]
            for off, idx, loff, lidx in ((flat.succ_off, flat.succ, lf.succ_off, lf.succ),
                                         (flat.pred_off, flat.pred, lf.pred_off, lf.pred)):
                assert np.array_equal(l2g[lidx[loff[l]:loff[l + 1]]], idx[off[g]:off[g + 1]])
        for k in ("lane_left", "lane_right", "lane_pred1", "lane_succ1"):
            a, b = getattr(lf, k), getattr(flat, k)[l2g]
            ok = a >= 0
            assert np.array_equal(l2g[a[ok]], b[ok])
        assert np.array_equal(lf.lane_len, flat.lane_len[l2g])


def test_ring_two_ranks():
    net = make_ring(40, radius=40 * 200.0 / (2 * math.pi))
    flat, plans = _plans(net, 2)
    assert all(len(p.import_lanes[1 - p.rank]) > 0 for p in plans)


def test_packet_transport_two_ranks_gloo():
    """alltoall_packets (the engine's exchange) on a 2-process gloo group."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29631",
           os.path.join(ROOT, "tests", "dist", "transport_worker.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert "TRANSPORT_OK 2" in out.stdout, out.stdout[-2000:] + out.stderr[-2000:]
