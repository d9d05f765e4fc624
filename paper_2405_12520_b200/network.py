"""Lane-level road network types and the input builders used by tests/bench.

The engine consumes a ``RoadNetwork`` exactly as the reference defines it
(trafficsim/network.py:57-113): lanes keyed by integer id, roads as lists of
lane ids (leftmost first), junctions with connector lists and an optional
fixed-time signal program.  ``World`` duck-types the object, so the reference's
own ``RoadNetwork`` is accepted as well.

The builders below (``build_network``, ``generate_grid``) are *input
generators*: the GPU box has no copy of the reference package, so synthetic
networks must be compiled here with the same lane numbering, geometry and
signal programs as the reference compiler (network.py:367-560).  Lane-id
order is load-bearing for parity (ties, feasibility sets, revert chains), so
every numbering rule is restated verbatim and pinned by
``tests/test_inputs.py`` against fixtures produced by the reference.
"""

from __future__ import annotations

import math
from bisect import bisect_right
from dataclasses import dataclass, field

from .errors import BuildError, InputError, SchemaError

Point = tuple[float, float]

ROAD = "road"
CONNECTOR = "connector"
OPEN = "open"
CLOSED = "closed"

STRAIGHT = "straight"
LEFT = "left"
RIGHT = "right"
UTURN = "uturn"

EARTH_RADIUS_M = 6371008.8


# --------------------------------------------------------------------------
# types (field-compatible with trafficsim.network)


@dataclass
class RawRoad:
    id: str
    polyline: list[Point]
    lane_count: int
    max_speed: float


@dataclass
class RawJunction:
    id: str
    in_roads: list[str]
    out_roads: list[str]
    position: Point


@dataclass
class Lane:
    id: int
    parent: str
    kind: str
    centerline: list[Point]
    length: float
    max_speed: float
    predecessors: list[int] = field(default_factory=list)
    successors: list[int] = field(default_factory=list)
    restriction: str = OPEN
    turn: str | None = None
    left: int | None = None
    right: int | None = None


@dataclass
class SignalPhase:
    duration: float
    green: tuple[int, ...]


@dataclass
class SignalProgram:
    phases: list[SignalPhase]
    offset: float = 0.0

    def cycle(self) -> float:
        return sum(p.duration for p in self.phases)


@dataclass
class Junction:
    id: str
    position: Point
    connectors: list[int] = field(default_factory=list)
    signal: SignalProgram | None = None


@dataclass
class RoadNetwork:
    lanes: dict[int, Lane]
    roads: dict[str, list[int]]
    junctions: dict[str, Junction]
    zone_hint: dict[int, int] | None = None

    def lane(self, lane_id: int) -> Lane:
        return self.lanes[lane_id]

    def road_lane_ids(self) -> list[int]:
        return [lid for ids in self.roads.values() for lid in ids]

    def road_of(self, lane_id: int) -> str:
        ln = self.lanes[lane_id]
        if ln.kind != ROAD:
            raise InputError(f"lane {lane_id} is not a road lane")
        return ln.parent


@dataclass
class BuildOptions:
    lane_width: float = 3.5
    snap_radius: float = 5.0
    allow_boundaries: bool = True
    allow_uturns: bool = False
    coordinate_frame: str = "auto"
    green_duration: float = 30.0
    clearance_duration: float = 3.0
    signal_min_approaches: int = 3


# --------------------------------------------------------------------------
# planar geometry (same float operations as trafficsim/geometry.py:18-89)


def arc_length(pts: list[Point]) -> float:
    # builtin sum(): CPython >= 3.12 compensates, exactly as the reference does
    return sum(math.dist(pts[k], pts[k + 1]) for k in range(len(pts) - 1))


def vertex_arclengths(pts: list[Point]) -> list[float]:
    out = [0.0]
    for k in range(len(pts) - 1):
        out.append(out[-1] + math.dist(pts[k], pts[k + 1]))
    return out


def segment_index(cum: list[float], s: float) -> int:
    k = bisect_right(cum, s) - 1
    return min(max(k, 0), len(cum) - 2)


def heading_at(pts: list[Point], cum: list[float], s: float) -> float:
    """Degrees clockwise from +y of the segment holding arc position ``s``."""
    k = segment_index(cum, s)
    dx = pts[k + 1][0] - pts[k][0]
    dy = pts[k + 1][1] - pts[k][1]
    if dx == 0.0 and dy == 0.0:
        return 0.0
    return math.degrees(math.atan2(dx, dy)) % 360.0


def _unit_right_normals(pts: list[Point]) -> list[Point]:
    out = []
    for (x0, y0), (x1, y1) in zip(pts, pts[1:]):
        dx, dy = x1 - x0, y1 - y0
        h = math.hypot(dx, dy)
        out.append((dy / h, -dx / h))
    return out


def shift_polyline(pts: list[Point], d: float) -> list[Point]:
    """Offset to the right of travel by ``d`` with capped miter joins."""
    if d == 0.0:
        return [tuple(p) for p in pts]
    nrm = _unit_right_normals(pts)
    last = len(pts) - 1
    res: list[Point] = []
    for k, (px, py) in enumerate(pts):
        if k == 0:
            nx, ny = nrm[0]
        elif k == last:
            nx, ny = nrm[-1]
        else:
            (ax, ay), (bx, by) = nrm[k - 1], nrm[k]
            mx, my = ax + bx, ay + by
            ml = math.hypot(mx, my)
            if ml < 1e-9:
                nx, ny = ax, ay
            else:
                mx, my = mx / ml, my / ml
                sc = max(mx * bx + my * by, 0.25)
                nx, ny = mx / sc, my / sc
        res.append((px + d * nx, py + d * ny))
    return res


def _looks_lonlat(pts) -> bool:
    return all(-180.0 <= x <= 180.0 and -90.0 <= y <= 90.0 for x, y in pts)


def _azimuthal(pts, center):
    lon0, lat0 = math.radians(center[0]), math.radians(center[1])
    s0, c0 = math.sin(lat0), math.cos(lat0)
    res = []
    for lon_d, lat_d in pts:
        lon, lat = math.radians(lon_d), math.radians(lat_d)
        sl, cl = math.sin(lat), math.cos(lat)
        dl = lon - lon0
        cc = min(max(s0 * sl + c0 * cl * math.cos(dl), -1.0), 1.0)
        c = math.acos(cc)
        if c < 1e-12:
            res.append((0.0, 0.0))
            continue
        k = EARTH_RADIUS_M * c / math.sin(c)
        res.append((k * cl * math.sin(dl), k * (c0 * sl - s0 * cl * math.cos(dl))))
    return res


def _to_local(roads, junctions, frame):
    if frame == "local":
        return roads, junctions
    groups = [r.polyline for r in roads] + [[j.position] for j in junctions]
    if frame == "auto" and (not groups or not all(_looks_lonlat(g) for g in groups)):
        return roads, junctions
    xs = [x for g in groups for x, _ in g]
    ys = [y for g in groups for _, y in g]
    center = ((min(xs) + max(xs)) / 2.0, (min(ys) + max(ys)) / 2.0)
    return (
        [RawRoad(r.id, _azimuthal(r.polyline, center), r.lane_count, r.max_speed) for r in roads],
        [RawJunction(j.id, list(j.in_roads), list(j.out_roads), _azimuthal([j.position], center)[0])
         for j in junctions],
    )


# --------------------------------------------------------------------------
# junction rules (network.py:264-364)


def classify_turn(h_in: float, h_out: float) -> str:
    theta = (h_out - h_in + 180.0) % 360.0 - 180.0
    if abs(theta) < 30.0:
        return STRAIGHT
    if 30.0 <= theta < 150.0:
        return RIGHT
    if -150.0 < theta <= -30.0:
        return LEFT
    return UTURN


def lane_pairs(n_in: int, n_out: int, turn: str) -> list[tuple[int, int]]:
    """(in lane index, out lane index) pairs; index 0 is leftmost."""
    if turn == STRAIGHT:
        return [(k, min(k, n_out - 1)) for k in range(n_in)]
    if turn == RIGHT:
        return [(n_in - 1, n_out - 1)]
    if turn in (LEFT, UTURN):
        return [(0, 0)]
    raise ValueError(turn)


def _approach_groups(in_roads: list[str], heading: dict[str, float]) -> list[list[str]]:
    todo = sorted(in_roads)
    groups: list[list[str]] = []
    while todo:
        a = todo.pop(0)
        mate = next(
            (b for b in todo if abs((heading[b] - heading[a] + 180.0) % 360.0 - 180.0) >= 135.0),
            None,
        )
        if mate is None:
            groups.append([a])
        else:
            todo.remove(mate)
            groups.append([a, mate])
    return groups


def _fixed_program(conns: list[Lane], in_roads, heading, source_road, opts) -> SignalProgram:
    dur = opts.green_duration + opts.clearance_duration
    phases: list[SignalPhase] = []
    for grp in _approach_groups(in_roads, heading):
        members = set(grp)
        mine = [c for c in conns if source_road[c.id] in members]
        through = sorted(c.id for c in mine if c.turn in (STRAIGHT, RIGHT))
        turning = sorted(c.id for c in mine if c.turn in (LEFT, UTURN))
        for ids in (through, turning):
            if ids:
                phases.append(SignalPhase(dur, tuple(ids)))
    if not phases:
        phases.append(SignalPhase(dur, tuple(sorted(c.id for c in conns))))
    return SignalProgram(phases=phases, offset=0.0)


# --------------------------------------------------------------------------
# compiler


def build_network(roads: list[RawRoad], junctions: list[RawJunction],
                  options: BuildOptions | None = None) -> RoadNetwork:
    """Compile raw roads/junctions into lanes, connectors and signal programs.

    Numbering follows the reference exactly: road lanes first, roads in
    sorted-id order, leftmost lane first; then connectors junction by
    junction (sorted ids), in-road x out-road pairs in sorted order.
    """
    opts = options or BuildOptions()
    for r in roads:
        if r.lane_count < 1 or r.max_speed <= 0 or len(r.polyline) < 2:
            raise BuildError(f"road {r.id!r}: invalid raw fields")
    roads, junctions = _to_local(roads, junctions, opts.coordinate_frame)
    by_id = {r.id: r for r in roads}

    ends: dict[str, str] = {}
    starts: dict[str, str] = {}
    for j in junctions:
        if not j.in_roads or not j.out_roads:
            raise BuildError(f"junction {j.id!r}: needs both incoming and outgoing roads")
        for table, rids, tip, word in ((ends, j.in_roads, -1, "end"), (starts, j.out_roads, 0, "start")):
            for rid in rids:
                if math.dist(by_id[rid].polyline[tip], j.position) > opts.snap_radius:
                    raise BuildError(
                        f"road {rid!r}: {word} point does not snap to junction {j.id!r} "
                        f"within {opts.snap_radius} m")
                if table.get(rid, j.id) != j.id:
                    kind = "incoming" if tip == -1 else "outgoing"
                    raise SchemaError(f"road {rid!r}: claimed as {kind} by two junctions")
                table[rid] = j.id
    if not opts.allow_boundaries:
        for r in roads:
            if r.id not in ends or r.id not in starts:
                raise BuildError(f"road {r.id!r}: endpoint not attached to any junction")

    lanes: dict[int, Lane] = {}
    road_lanes: dict[str, list[int]] = {}
    nid = 0
    for rid in sorted(by_id):
        r = by_id[rid]
        ids = list(range(nid, nid + r.lane_count))
        for k, lid in enumerate(ids):
            line = shift_polyline(r.polyline, (k + 0.5 - r.lane_count / 2.0) * opts.lane_width)
            lanes[lid] = Lane(id=lid, parent=rid, kind=ROAD, centerline=line,
                              length=arc_length(line), max_speed=r.max_speed)
        for a, b in zip(ids, ids[1:]):
            lanes[a].right = b
            lanes[b].left = a
        road_lanes[rid] = ids
        nid += r.lane_count

    h_in: dict[str, float] = {}
    h_out: dict[str, float] = {}
    for rid, r in by_id.items():
        cum = vertex_arclengths(r.polyline)
        h_in[rid] = heading_at(r.polyline, cum, cum[-1])
        h_out[rid] = heading_at(r.polyline, cum, 0.0)

    juncs: dict[str, Junction] = {}
    for j in sorted(junctions, key=lambda q: q.id):
        made: list[Lane] = []
        source_road: dict[int, str] = {}
        for rin in sorted(j.in_roads):
            for rout in sorted(j.out_roads):
                turn = classify_turn(h_in[rin], h_out[rout])
                if turn == UTURN and not opts.allow_uturns:
                    continue
                a_ids, b_ids = road_lanes[rin], road_lanes[rout]
                for i, k in lane_pairs(len(a_ids), len(b_ids), turn):
                    src, dst = lanes[a_ids[i]], lanes[b_ids[k]]
                    line = [src.centerline[-1], dst.centerline[0]]
                    c = Lane(id=nid, parent=j.id, kind=CONNECTOR, centerline=line,
                             length=arc_length(line),
                             max_speed=min(src.max_speed, dst.max_speed),
                             predecessors=[src.id], successors=[dst.id], turn=turn)
                    lanes[nid] = c
                    src.successors.append(nid)
                    dst.predecessors.append(nid)
                    made.append(c)
                    source_road[nid] = rin
                    nid += 1
        if not made:
            raise BuildError(f"junction {j.id!r}: no feasible connector")
        prog = None
        if len(j.in_roads) >= opts.signal_min_approaches:
            prog = _fixed_program(made, j.in_roads, h_in, source_road, opts)
        juncs[j.id] = Junction(id=j.id, position=j.position,
                               connectors=sorted(c.id for c in made), signal=prog)

    for ln in lanes.values():
        ln.predecessors.sort()
        ln.successors.sort()
    return RoadNetwork(lanes=lanes, roads=road_lanes, junctions=juncs)


def generate_grid(rows: int, cols: int, block_length: float = 200.0,
                  lanes_per_direction: int = 1, max_speed: float = 16.67) -> RoadNetwork:
    """Manhattan grid compiled through ``build_network`` (network.py:507-560)."""
    if rows < 2 or cols < 2:
        raise InputError("grid needs rows >= 2 and cols >= 2")
    if block_length <= 0 or lanes_per_direction < 1 or max_speed <= 0:
        raise InputError("invalid grid parameters")
    margin = min(block_length / 4.0, 12.0)
    pos = {f"j{r}_{c}": (c * block_length, r * block_length)
           for r in range(rows) for c in range(cols)}
    incoming: dict[str, list[str]] = {j: [] for j in pos}
    outgoing: dict[str, list[str]] = {j: [] for j in pos}
    raw: list[RawRoad] = []

    def link(a: str, b: str) -> None:
        (ax, ay), (bx, by) = pos[a], pos[b]
        d = math.dist((ax, ay), (bx, by))
        ux, uy = (bx - ax) / d, (by - ay) / d
        rid = f"{a}:{b}"
        raw.append(RawRoad(rid, [(ax + ux * margin, ay + uy * margin),
                                 (bx - ux * margin, by - uy * margin)],
                           lanes_per_direction, max_speed))
        outgoing[a].append(rid)
        incoming[b].append(rid)

    for r in range(rows):
        for c in range(cols):
            here = f"j{r}_{c}"
            for there in ((f"j{r}_{c + 1}" if c + 1 < cols else None),
                          (f"j{r + 1}_{c}" if r + 1 < rows else None)):
                if there is not None:
                    link(here, there)
                    link(there, here)
    rj = [RawJunction(j, incoming[j], outgoing[j], pos[j]) for j in sorted(pos)]
    opts = BuildOptions(snap_radius=margin + 0.5, allow_boundaries=False, coordinate_frame="local")
    return build_network(raw, rj, opts)


def make_ring(n_junctions: int, radius: float, margin: float = 12.0,
              max_speed: float = 16.67, lane_count: int = 1) -> RoadNetwork:
    """Single-lane unsignalized ring (BASELINE config C2).

    N junctions on a circle, one road from each junction to the next with
    ``margin`` trimmed at both ends, compiled through ``build_network``.
    """
    pts = [(radius * math.cos(2 * math.pi * k / n_junctions),
            radius * math.sin(2 * math.pi * k / n_junctions)) for k in range(n_junctions)]
    roads, juncs = [], []
    for k in range(n_junctions):
        a, b = pts[k], pts[(k + 1) % n_junctions]
        d = math.dist(a, b)
        ux, uy = (b[0] - a[0]) / d, (b[1] - a[1]) / d
        roads.append(RawRoad(f"r{k:05d}", [(a[0] + ux * margin, a[1] + uy * margin),
                                           (b[0] - ux * margin, b[1] - uy * margin)],
                             lane_count, max_speed))
    for k in range(n_junctions):
        juncs.append(RawJunction(f"j{k:05d}", [f"r{(k - 1) % n_junctions:05d}"], [f"r{k:05d}"], pts[k]))
    return build_network(roads, juncs, BuildOptions(snap_radius=margin + 0.5,
                                                    allow_boundaries=False,
                                                    coordinate_frame="local"))


def make_corridor(lengths=(500.0, 500.0), speed=16.67, lane_count=1) -> RoadNetwork:
    """Straight unsignalized chain (reference tests/conftest.py:17-43)."""
    xs = [0.0]
    for ln in lengths:
        xs.append(xs[-1] + ln)
    roads = [RawRoad(f"r{i}", [(xs[i], 0.0), (xs[i + 1], 0.0)], lane_count, speed)
             for i in range(len(lengths))]
    juncs = [RawJunction(f"j{i}", [f"r{i}"], [f"r{i + 1}"], (xs[i + 1], 0.0))
             for i in range(len(lengths) - 1)]
    return build_network(roads, juncs, BuildOptions(coordinate_frame="local"))


def make_cross(arm=150.0, speed=13.9, lane_count=1, allow_uturns=False) -> RoadNetwork:
    """Four-arm signalized cross (reference tests/conftest.py:46-64)."""
    tips = {"n": (0.0, arm), "s": (0.0, -arm), "e": (arm, 0.0), "w": (-arm, 0.0)}
    roads = []
    for name, tip in tips.items():
        roads.append(RawRoad(f"{name}_in", [tip, (0.0, 0.0)], lane_count, speed))
        roads.append(RawRoad(f"{name}_out", [(0.0, 0.0), tip], lane_count, speed))
    j = RawJunction("center", [f"{n}_in" for n in tips], [f"{n}_out" for n in tips], (0.0, 0.0))
    return build_network(roads, [j], BuildOptions(coordinate_frame="local", allow_uturns=allow_uturns))
