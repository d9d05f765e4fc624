"""Lane partitioning and halo zones for the sharded (multi-GPU) engine.

SURVEY.md 8(e): the road graph is split into spatial bands of junctions; a
connector belongs to its junction's rank and a road (all its lanes) to the
rank of its upstream junction.  Each rank then simulates its own lanes plus a
halo of foreign lanes (an overlapping decomposition), so that everything
that can influence its own lanes within ONE step is computed locally from
exact inputs:

* reads of the update (world.py:261-397): the lane, its road siblings (MOBIL)
  and the lanes within `lookahead` downstream (_sense);
* vehicles that can enter an own lane in one step (transitions, lane
  changes) -- lanes within one step's travel upstream;
* revert partners (world.py:501-559): lanes own vehicles can enter, whose
  sweep may send them back.

After every step each rank sends the vehicles of its own lanes that lie in a
neighbour's halo to that neighbour (one all-to-all of boundary lanes); the
neighbour uses them as read-only ghosts for the next step.  Lanes marked
EXACT are those whose post-step content is computed exactly; the engine
checks at run time that every revert chain touching an own lane stays inside
EXACT lanes and fails loudly otherwise (never silently wrong).
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass

import numpy as np

from .flat import KIND_CONNECTOR, KIND_ROAD, FlatNet

ZONE_OWN, ZONE_HALO, ZONE_EXACT = 1, 2, 4


@dataclass
class ShardPlan:
    rank: int
    nranks: int
    lane_owner: np.ndarray   # int32 per lane (-1 for id holes)
    zone: np.ndarray         # uint8 per lane: OWN | HALO, EXACT
    export_lanes: list       # per destination rank: own lanes in its halo (ascending), then pressure lanes
    import_lanes: list       # per source rank: its lanes in my halo (ascending), then pressure lanes
    export_kind: list = None  # per destination rank: 0 halo lane, 1 max-pressure count only
    import_kind: list = None


def lane_owners(flat: FlatNet, junc_pos: np.ndarray, nranks: int) -> np.ndarray:
    """Bands of junctions sorted by (y, x), balanced by lane count."""
    nj = len(flat.junction_ids)
    n = flat.n_lanes
    # a road's upstream junction: the junction of its predecessor connectors
    # (else its successors'); all lanes of a road share it
    road_junc = np.full(len(flat.road_ids), -1, dtype=np.int64)
    for r in range(len(flat.road_ids)):
        for lane in flat.road_lanes[flat.road_lane_off[r]:flat.road_lane_off[r + 1]]:
            preds = flat.pred[flat.pred_off[lane]:flat.pred_off[lane + 1]]
            conns = [int(p) for p in preds if flat.lane_kind[p] == KIND_CONNECTOR]
            if conns:
                road_junc[r] = flat.lane_junction[conns[0]]
                break
        if road_junc[r] < 0:
            for lane in flat.road_lanes[flat.road_lane_off[r]:flat.road_lane_off[r + 1]]:
                succ = flat.succ[flat.succ_off[lane]:flat.succ_off[lane + 1]]
                conns = [int(s) for s in succ if flat.lane_kind[s] == KIND_CONNECTOR]
                if conns:
                    road_junc[r] = flat.lane_junction[conns[0]]
                    break
        if road_junc[r] < 0:
            road_junc[r] = 0
    lane_junc = np.full(n, -1, dtype=np.int64)
    is_conn = flat.lane_kind == KIND_CONNECTOR
    lane_junc[is_conn] = flat.lane_junction[is_conn]
    is_road = flat.lane_kind == KIND_ROAD
    lane_junc[is_road] = road_junc[flat.lane_road[is_road]]
    weight = np.bincount(lane_junc[lane_junc >= 0], minlength=nj).astype(np.float64)
    order = np.lexsort((junc_pos[:, 0], junc_pos[:, 1]))  # by y, then x
    cum = np.cumsum(weight[order])
    total = cum[-1] if len(cum) else 0.0
    band = np.minimum((cum - weight[order] * 0.5) * nranks // max(total, 1.0), nranks - 1).astype(np.int32)
    junc_rank = np.empty(nj, dtype=np.int32)
    junc_rank[order] = band
    owner = np.full(n, -1, dtype=np.int32)
    ok = lane_junc >= 0
    owner[ok] = junc_rank[lane_junc[ok]]
    return owner


def _csr_lists(off, idx, n):
    return [idx[off[i]:off[i + 1]] for i in range(n)]


def _reach(flat: FlatNet, seeds, dist: float, downstream: bool) -> set:
    """Lanes whose near end lies within `dist` of a seed's boundary, walking
    successors from the seeds' ends (downstream) or predecessors from their
    starts (upstream).  The distance to a lane is the length of the lanes
    strictly between it and the seed."""
    off, idx = (flat.succ_off, flat.succ) if downstream else (flat.pred_off, flat.pred)
    best: dict[int, float] = {}
    dq = deque((int(s), -1.0) for s in seeds)
    while dq:
        lane, d = dq.popleft()
        base = 0.0 if d < 0 else d + float(flat.lane_len[lane])
        if base >= dist:
            continue
        for nb in idx[off[lane]:off[lane + 1]]:
            nb = int(nb)
            if flat.lane_kind[nb] < 0:
                continue
            if nb not in best or best[nb] > base:
                best[nb] = base
                dq.append((nb, base))
    return set(best)


def _siblings(flat: FlatNet, lanes: set) -> set:
    out = set(lanes)
    for lane in lanes:
        if flat.lane_kind[lane] == KIND_ROAD:
            r = flat.lane_road[lane]
            out.update(int(x) for x in flat.road_lanes[flat.road_lane_off[r]:flat.road_lane_off[r + 1]])
    return out


def max_step_travel(flat: FlatNet, config) -> float:
    """Upper bound of one vehicle's displacement in one step (m)."""
    vmax = max(float(config.idm.v0), float(flat.lane_cap[flat.lane_kind >= 0].max(initial=0.0)))
    return vmax * config.dt + 0.5 * config.idm.a_max * config.dt * config.dt + 1.0


def plan_shard(flat: FlatNet, owner: np.ndarray, rank: int, nranks: int, config) -> ShardPlan:
    n = flat.n_lanes
    travel = max_step_travel(flat, config)
    own = set(int(x) for x in np.nonzero(owner == rank)[0])

    def down(seeds, dist):
        return _reach(flat, seeds, dist, downstream=True)

    def up(seeds, dist):
        return _reach(flat, seeds, dist, downstream=False)

    # lanes own vehicles may enter (revert partners) and lanes that may feed them
    near = _siblings(flat, own | down(own, 2 * travel))
    feed = _siblings(flat, near | up(near, 2 * travel))
    # everything those vehicles read: downstream lookahead from anywhere on the lane
    zone_set = _siblings(flat, feed | down(feed, config.lookahead + travel))
    zone = np.zeros(n, dtype=np.uint8)
    for lane in zone_set:
        zone[lane] = ZONE_OWN if owner[lane] == rank else ZONE_HALO
    for lane in own:
        zone[lane] = ZONE_OWN
    # exact_update(L): L's siblings and its downstream reads are in the zone
    in_zone = zone > 0
    exact_update = np.zeros(n, dtype=bool)
    for lane in zone_set | own:
        sib = _siblings(flat, {lane})
        reads = down({lane}, config.lookahead + travel)
        exact_update[lane] = all(in_zone[x] for x in sib | reads)
    # exact_lane(H): every lane whose vehicles can end in H this step is exact_update
    for lane in zone_set | own:
        src = _siblings(flat, {lane}) | up({lane}, travel)
        if all(exact_update[x] for x in src if flat.lane_kind[x] >= 0):
            zone[lane] |= ZONE_EXACT
    pressure = pressure_lanes(flat, zone) if getattr(config, "controller", "fixed") == "max_pressure" else set()
    export_lanes, import_lanes, import_kind = [], [], []
    for q in range(nranks):
        if q == rank:
            export_lanes.append(np.zeros(0, dtype=np.int32))
            import_lanes.append(np.zeros(0, dtype=np.int32))
            import_kind.append(np.zeros(0, dtype=np.uint8))
            continue
        export_lanes.append(None)
        halo = sorted(x for x in zone_set if owner[x] == q and zone[x] & ZONE_HALO)
        mp = sorted(x for x in pressure if owner[x] == q)
        import_lanes.append(np.array(halo + mp, dtype=np.int32))
        import_kind.append(np.array([0] * len(halo) + [1] * len(mp), dtype=np.uint8))
    return ShardPlan(rank, nranks, owner, zone, export_lanes, import_lanes, None, import_kind)


def pressure_lanes(flat: FlatNet, zone: np.ndarray) -> set:
    """Max-pressure sharded (signals.py:64-86, world.py:627-647): the lanes
    whose post-sweep counts decide the phase of every junction with a
    connector in this rank's zone (the junctions its vehicles may read): each
    connector's predecessor and successor road lane.  Own lanes are counted
    locally; the owners send the others' counts with every exchange, and each
    rank advances those junctions itself at the start of the next step."""
    conn = np.nonzero((flat.lane_kind == KIND_CONNECTOR) & (zone > 0))[0]
    juncs = set(int(flat.lane_junction[c]) for c in conn)
    out = set()
    for c in np.nonzero(flat.lane_kind == KIND_CONNECTOR)[0]:
        if int(flat.lane_junction[c]) in juncs:
            out.add(int(flat.lane_pred1[c]))
            out.add(int(flat.lane_succ1[c]))
    return out


def plan_all(flat: FlatNet, junc_pos: np.ndarray, nranks: int, config) -> list[ShardPlan]:
    """Plans for every rank (export lists are the peers' import lists)."""
    owner = lane_owners(flat, junc_pos, nranks)
    plans = [plan_shard(flat, owner, r, nranks, config) for r in range(nranks)]
    for r, p in enumerate(plans):
        p.export_lanes = [plans[q].import_lanes[r] if q != r else np.zeros(0, dtype=np.int32)
                          for q in range(nranks)]
        p.export_kind = [plans[q].import_kind[r] if q != r else np.zeros(0, dtype=np.uint8)
                         for q in range(nranks)]
    return plans


def local_network(flat: FlatNet, plan: ShardPlan):
    """The rank's zone as a compact local lane space (tsb_create_sharded_local).

    Local lanes are the rank's own and halo lanes, the max-pressure lanes it
    counts or imports, and their roads' sibling lanes, in ascending global id
    (l2g is increasing, so every lane-id comparison -- MOBIL ties, the sweep
    order, revert chains -- is unchanged).  Lane references that leave the
    local set (a halo lane's successors at the zone edge) become -1; roads and
    junctions keep their global indices (routes are sequences of global road
    ids).  Returns (local FlatNet, l2g, local ShardPlan)."""
    from dataclasses import replace

    n = flat.n_lanes
    keep = set(np.nonzero(plan.zone > 0)[0].tolist())
    for lists in (plan.import_lanes, plan.export_lanes):
        for x in lists:
            keep.update(int(v) for v in x)
    keep = _siblings(flat, keep)
    l2g = np.array(sorted(keep), dtype=np.int32)
    g2l = np.full(n, -1, dtype=np.int32)
    g2l[l2g] = np.arange(len(l2g), dtype=np.int32)

    def remap(a):
        a = np.asarray(a)
        out = np.full(a.shape, -1, dtype=np.int32)
        ok = a >= 0
        out[ok] = g2l[a[ok]]
        return out

    def csr(off, idx):
        lists = [remap(idx[off[g]:off[g + 1]]) for g in l2g]
        lists = [x[x >= 0] for x in lists]
        o = np.zeros(len(l2g) + 1, dtype=np.int32)
        o[1:] = np.cumsum([len(x) for x in lists]) if len(lists) else []
        v = np.concatenate(lists).astype(np.int32) if lists else np.zeros(0, np.int32)
        return o, v

    succ_off, succ = csr(flat.succ_off, flat.succ)
    pred_off, pred = csr(flat.pred_off, flat.pred)
    nr = len(flat.road_ids)
    rl = [remap(flat.road_lanes[flat.road_lane_off[r]:flat.road_lane_off[r + 1]]) for r in range(nr)]
    rl = [x[x >= 0] for x in rl]
    road_lane_off = np.zeros(nr + 1, dtype=np.int32)
    road_lane_off[1:] = np.cumsum([len(x) for x in rl])
    road_lanes = np.concatenate(rl).astype(np.int32) if rl else np.zeros(0, np.int32)
    nseg = (flat.geo_off[l2g + 1] - flat.geo_off[l2g]).astype(np.int64)
    geo_off = np.zeros(len(l2g) + 1, dtype=np.int64)
    geo_off[1:] = np.cumsum(nseg)
    seg_idx = np.concatenate([np.arange(flat.geo_off[g], flat.geo_off[g + 1]) for g in l2g]) if len(l2g) \
        else np.zeros(0, np.int64)
    lflat = replace(
        flat, n_lanes=len(l2g),
        lane_len=flat.lane_len[l2g].copy(), lane_cap=flat.lane_cap[l2g].copy(),
        lane_kind=flat.lane_kind[l2g].copy(), lane_open=flat.lane_open[l2g].copy(),
        lane_left=remap(flat.lane_left[l2g]), lane_right=remap(flat.lane_right[l2g]),
        lane_road=flat.lane_road[l2g].copy(), lane_junction=flat.lane_junction[l2g].copy(),
        lane_pred1=remap(flat.lane_pred1[l2g]), lane_succ1=remap(flat.lane_succ1[l2g]),
        succ_off=succ_off, succ=succ, pred_off=pred_off, pred=pred,
        road_lane_off=road_lane_off, road_lanes=road_lanes,
        lane_green_mask=flat.lane_green_mask[l2g].copy(),
        geo_off=geo_off, geo_cum=flat.geo_cum[seg_idx].copy(), geo_angle=flat.geo_angle[seg_idx].copy(),
    )
    lplan = ShardPlan(plan.rank, plan.nranks, plan.lane_owner[l2g].copy(), plan.zone[l2g].copy(),
                      [remap(x) for x in plan.export_lanes], [remap(x) for x in plan.import_lanes],
                      plan.export_kind, plan.import_kind)
    for x in lplan.export_lanes + lplan.import_lanes:
        assert np.all(x >= 0), "an exchange lane is outside the local lane set"
    return lflat, l2g, lplan
