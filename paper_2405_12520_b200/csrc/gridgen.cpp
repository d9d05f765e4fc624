// gridgen.cpp -- native builder of the synthetic Manhattan grids (SURVEY 8(f)
// rank 4): the reference's generate_grid (trafficsim/network.py:507-560)
// compiled through its build_network (network.py:367-505) and flattened the
// way paper_2405_12520_b200/flat.py flattens a RoadNetwork, straight into the
// struct-of-arrays the engine uploads -- no per-lane Python objects.  A
// 200x200x3 grid (1.27M lanes) takes seconds instead of minutes.
//
// Every number is produced by the same IEEE operations as the reference's
// CPython code: math.dist / math.hypot are CPython 3.12's vector_norm
// (Modules/mathmodule.c: frexp scaling, exact double-length squares,
// one differential correction), math.degrees multiplies by 180/pi, Python's
// float % takes the sign of the divisor, atan2 is libm's.  Lane ids, road and
// junction order follow the reference's sorted-string rules.  Pinned array
// for array against the Python builder (itself pinned to the reference) and
// by sha256 against the reference at 100x100x3 and 200x200x3
// (tests/test_gridgen.py, tests/golden/scale_sha.json).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/tsb200.h"

namespace {

struct DL {
  double hi, lo;
};
inline DL dl_mul(double x, double y) {
  const double h = x * y;
  return DL{h, std::fma(x, y, -h)};
}
inline DL dl_fast_sum(double a, double b) {
  const double h = a + b;
  return DL{h, (a - h) + b};
}

// CPython 3.12 vector_norm for finite, non-negative entries (math.hypot,
// math.dist).
double vector_norm(int n, double* vec, double max) {
  if (std::isinf(max)) return max;
  if (max == 0.0 || n <= 1) return max;
  int max_e;
  std::frexp(max, &max_e);
  if (max_e < -1023) {
    for (int i = 0; i < n; i++) vec[i] /= 2.2250738585072014e-308;  // DBL_MIN
    return 2.2250738585072014e-308 * vector_norm(n, vec, max / 2.2250738585072014e-308);
  }
  const double scale = std::ldexp(1.0, -max_e);
  double csum = 1.0, frac1 = 0.0, frac2 = 0.0;
  for (int i = 0; i < n; i++) {
    const double x = vec[i] * scale;
    const DL pr = dl_mul(x, x);
    const DL sm = dl_fast_sum(csum, pr.hi);
    csum = sm.hi;
    frac1 += pr.lo;
    frac2 += sm.lo;
  }
  double h = std::sqrt(csum - 1.0 + (frac1 + frac2));
  const DL pr = dl_mul(-h, h);
  const DL sm = dl_fast_sum(csum, pr.hi);
  csum = sm.hi;
  frac1 += pr.lo;
  frac2 += sm.lo;
  const double x = csum - 1.0 + (frac1 + frac2);
  h += x / (2.0 * h);
  return h / scale;
}

double py_hypot(double a, double b) {
  double v[2] = {std::fabs(a), std::fabs(b)};
  double mx = v[0];
  if (v[1] > mx) mx = v[1];
  return vector_norm(2, v, mx);
}

struct P2 {
  double x, y;
};
double py_dist(P2 p, P2 q) {
  double v[2] = {std::fabs(p.x - q.x), std::fabs(p.y - q.y)};
  double mx = v[0];
  if (v[1] > mx) mx = v[1];
  return vector_norm(2, v, mx);
}

// Python float % (result has the sign of the divisor)
double py_mod(double a, double w) {
  double m = std::fmod(a, w);
  if (m != 0.0) {
    if ((w < 0) != (m < 0)) m += w;
  } else {
    m = std::copysign(0.0, w);
  }
  return m;
}
double py_degrees(double x) {
  static const double radToDeg = 180.0 / 3.14159265358979323846;
  return radToDeg * x;
}
// geometry.heading_deg_at on a segment (geometry.py:45-52)
double heading(P2 a, P2 b) {
  const double dx = b.x - a.x, dy = b.y - a.y;
  if (dx == 0.0 && dy == 0.0) return 0.0;
  return py_mod(py_degrees(std::atan2(dx, dy)), 360.0);
}

enum Turn { STRAIGHT, RIGHT, LEFT, UTURN };
Turn classify_turn(double h_in, double h_out) {  // network.py classify_turn
  const double theta = py_mod(h_out - h_in + 180.0, 360.0) - 180.0;
  if (std::fabs(theta) < 30.0) return STRAIGHT;
  if (30.0 <= theta && theta < 150.0) return RIGHT;
  if (-150.0 < theta && theta <= -30.0) return LEFT;
  return UTURN;
}

struct Road {
  std::string id;
  P2 p0, p1;
  int a, b;  // junction indices (source, target) in generation order
};

}  // namespace

struct tsb_grid {
  int32_t n_lanes = 0;
  std::vector<double> lane_len, lane_cap;
  std::vector<int8_t> lane_kind;
  std::vector<uint8_t> lane_open;
  std::vector<int32_t> lane_left, lane_right, lane_road, lane_junc, lane_pred1, lane_succ1;
  std::vector<int32_t> succ_off, succ, pred_off, pred;
  std::vector<int32_t> road_lane_off, road_lanes;
  std::vector<uint8_t> junc_signal;
  std::vector<int32_t> junc_phase_off;
  std::vector<double> phase_dur;
  std::vector<uint64_t> green;
  std::vector<int32_t> phase0;
  std::vector<double> elapsed0;
  std::vector<int64_t> geo_off;
  std::vector<double> geo_cum, geo_angle;
  std::vector<double> junc_pos;  // x, y per junction (sorted-id order)
  std::string road_ids, junction_ids;  // '\n'-joined, in flat order
};

extern "C" {

double tsb_py_dist(double ax, double ay, double bx, double by) { return py_dist(P2{ax, ay}, P2{bx, by}); }

int tsb_grid_build(int32_t rows, int32_t cols, double block_length, int32_t lanes_per_direction, double max_speed,
                   int32_t controller, tsb_grid** out) {
  *out = nullptr;
  if (rows < 2 || cols < 2 || !(block_length > 0) || lanes_per_direction < 1 || !(max_speed > 0))
    return TSB_EINVAL;
  auto* g = new tsb_grid();
  const double lane_width = 3.5;
  const double margin = std::min(block_length / 4.0, 12.0);
  // junctions in generation order r, c; their ids sorted as strings
  const int nj = rows * cols;
  std::vector<std::string> jname(nj);
  std::vector<P2> jpos(nj);
  for (int r = 0; r < rows; r++)
    for (int c = 0; c < cols; c++) {
      jname[r * cols + c] = "j" + std::to_string(r) + "_" + std::to_string(c);
      jpos[r * cols + c] = P2{(double)c * block_length, (double)r * block_length};
    }
  // roads in link() order (network.py:530-552), per junction in/out lists
  std::vector<Road> roads;
  roads.reserve((size_t)4 * nj);
  std::vector<std::vector<int>> incoming(nj), outgoing(nj);
  auto link = [&](int a, int b) {
    const P2 A = jpos[a], B = jpos[b];
    const double d = py_dist(A, B);
    const double ux = (B.x - A.x) / d, uy = (B.y - A.y) / d;
    Road rd;
    rd.id = jname[a] + ":" + jname[b];
    rd.p0 = P2{A.x + ux * margin, A.y + uy * margin};
    rd.p1 = P2{B.x - ux * margin, B.y - uy * margin};
    rd.a = a;
    rd.b = b;
    outgoing[a].push_back((int)roads.size());
    incoming[b].push_back((int)roads.size());
    roads.push_back(rd);
  };
  for (int r = 0; r < rows; r++)
    for (int c = 0; c < cols; c++) {
      const int here = r * cols + c;
      if (c + 1 < cols) {
        link(here, here + 1);
        link(here + 1, here);
      }
      if (r + 1 < rows) {
        link(here, here + cols);
        link(here + cols, here);
      }
    }
  const int nr = (int)roads.size();
  // road lanes: roads in sorted-id order, leftmost lane first
  std::vector<int> rorder(nr);
  for (int k = 0; k < nr; k++) rorder[k] = k;
  std::sort(rorder.begin(), rorder.end(), [&](int x, int y) { return roads[x].id < roads[y].id; });
  std::vector<int> rindex(nr);  // road -> flat road index
  for (int k = 0; k < nr; k++) rindex[rorder[k]] = k;
  const int L = lanes_per_direction;
  struct LaneTmp {
    P2 c0, c1;  // centerline
    std::vector<int32_t> succ, pred;
  };
  const int64_t n_road_lanes = (int64_t)nr * L;
  std::vector<LaneTmp> lanes;
  lanes.reserve((size_t)n_road_lanes + (size_t)nj * 16 * L);
  std::vector<double> len, cap;
  std::vector<int8_t> kind;
  std::vector<int32_t> left, right, lroad, ljunc, pred1, succ1;
  for (int k = 0; k < nr; k++) {
    const Road& rd = roads[rorder[k]];
    // shift_polyline (geometry.py offset_polyline): a two-point polyline
    // moves by d along its unit right normal
    const double dx = rd.p1.x - rd.p0.x, dy = rd.p1.y - rd.p0.y;
    const double h = py_hypot(dx, dy);
    const double nx = dy / h, ny = -dx / h;
    for (int q = 0; q < L; q++) {
      const int32_t lid = (int32_t)lanes.size();
      const double off = ((double)q + 0.5 - (double)L / 2.0) * lane_width;
      LaneTmp t;
      if (off == 0.0) {
        t.c0 = rd.p0;
        t.c1 = rd.p1;
      } else {
        t.c0 = P2{rd.p0.x + off * nx, rd.p0.y + off * ny};
        t.c1 = P2{rd.p1.x + off * nx, rd.p1.y + off * ny};
      }
      lanes.push_back(t);
      len.push_back(py_dist(t.c0, t.c1));
      cap.push_back(max_speed);
      kind.push_back(TSB_KIND_ROAD);
      left.push_back(q > 0 ? lid - 1 : -1);
      right.push_back(q + 1 < L ? lid + 1 : -1);
      lroad.push_back(k);
      ljunc.push_back(-1);
      pred1.push_back(-1);
      succ1.push_back(-1);
    }
  }
  auto first_lane = [&](int road) { return rindex[road] * L; };
  std::vector<double> h_in(nr), h_out(nr);
  for (int k = 0; k < nr; k++) {
    h_in[k] = heading(roads[k].p0, roads[k].p1);
    h_out[k] = h_in[k];
  }
  // junctions in sorted-id order: connectors and the fixed-time program
  std::vector<int> jorder(nj);
  for (int k = 0; k < nj; k++) jorder[k] = k;
  std::sort(jorder.begin(), jorder.end(), [&](int x, int y) { return jname[x] < jname[y]; });
  g->junc_signal.assign(nj, 0);
  g->junc_phase_off.assign(nj + 1, 0);
  g->phase0.assign(nj, 0);
  g->elapsed0.assign(nj, 0.0);
  std::vector<std::pair<int32_t, uint64_t>> greens;
  auto by_name = [&](std::vector<int> v) {
    std::sort(v.begin(), v.end(), [&](int x, int y) { return roads[x].id < roads[y].id; });
    return v;
  };
  for (int ji = 0; ji < nj; ji++) {
    const int j = jorder[ji];
    struct Conn {
      int32_t id;
      int src_road;
      Turn turn;
    };
    std::vector<Conn> made;
    const std::vector<int> ins = by_name(incoming[j]), outs = by_name(outgoing[j]);
    for (int rin : ins)
      for (int rout : outs) {
        const Turn turn = classify_turn(h_in[rin], h_out[rout]);
        if (turn == UTURN) continue;  // allow_uturns = False
        std::vector<std::pair<int, int>> pairs;
        if (turn == STRAIGHT) {
          for (int k = 0; k < L; k++) pairs.push_back({k, std::min(k, L - 1)});
        } else if (turn == RIGHT) {
          pairs.push_back({L - 1, L - 1});
        } else {
          pairs.push_back({0, 0});
        }
        for (auto [a, b] : pairs) {
          const int32_t src = first_lane(rin) + a, dst = first_lane(rout) + b;
          const int32_t nid = (int32_t)lanes.size();
          LaneTmp t;
          t.c0 = lanes[src].c1;
          t.c1 = lanes[dst].c0;
          t.pred.push_back(src);
          t.succ.push_back(dst);
          lanes.push_back(t);
          lanes[src].succ.push_back(nid);
          lanes[dst].pred.push_back(nid);
          len.push_back(py_dist(t.c0, t.c1));
          cap.push_back(std::min(cap[src], cap[dst]));
          kind.push_back(TSB_KIND_CONNECTOR);
          left.push_back(-1);
          right.push_back(-1);
          lroad.push_back(-1);
          ljunc.push_back(ji);
          pred1.push_back(src);
          succ1.push_back(dst);
          made.push_back(Conn{nid, rin, turn});
        }
      }
    if (made.empty()) {
      delete g;
      return TSB_EINVAL;
    }
    if ((int)incoming[j].size() >= 3) {  // signal_min_approaches
      // _fixed_program: approach groups of opposite in-roads (sorted ids)
      const double dur = 30.0 + 3.0;
      std::vector<int> todo = ins;
      std::vector<std::vector<int>> groups;
      while (!todo.empty()) {
        const int a = todo.front();
        todo.erase(todo.begin());
        int mate = -1;
        for (size_t k = 0; k < todo.size(); k++) {
          const int b = todo[k];
          if (std::fabs(py_mod(h_in[b] - h_in[a] + 180.0, 360.0) - 180.0) >= 135.0) {
            mate = (int)k;
            break;
          }
        }
        if (mate < 0) {
          groups.push_back({a});
        } else {
          groups.push_back({a, todo[mate]});
          todo.erase(todo.begin() + mate);
        }
      }
      int nph = 0;
      auto add_phase = [&](const std::vector<int32_t>& ids) {
        for (int32_t cid : ids) greens.push_back({cid, 1ull << nph});
        g->phase_dur.push_back(dur);
        nph++;
      };
      for (const auto& grp : groups) {
        std::vector<int32_t> through, turning;
        for (const Conn& cn : made) {
          if (std::find(grp.begin(), grp.end(), cn.src_road) == grp.end()) continue;
          (cn.turn == STRAIGHT || cn.turn == RIGHT ? through : turning).push_back(cn.id);
        }
        std::sort(through.begin(), through.end());
        std::sort(turning.begin(), turning.end());
        if (!through.empty()) add_phase(through);
        if (!turning.empty()) add_phase(turning);
      }
      if (nph == 0) {
        std::vector<int32_t> all;
        for (const Conn& cn : made) all.push_back(cn.id);
        std::sort(all.begin(), all.end());
        add_phase(all);
      }
      if (nph > 64) {
        delete g;
        return TSB_EINVAL;
      }
      g->junc_signal[ji] = 1;
    }
    g->junc_phase_off[ji + 1] = (int32_t)g->phase_dur.size();
  }
  (void)controller;  // offset 0: the fixed-time pre-advance leaves (phase 0, elapsed 0) either way
  const int32_t n = (int32_t)lanes.size();
  g->n_lanes = n;
  g->lane_len = std::move(len);
  g->lane_cap = std::move(cap);
  g->lane_kind = std::move(kind);
  g->lane_open.assign(n, 1);
  g->lane_left = std::move(left);
  g->lane_right = std::move(right);
  g->lane_road = std::move(lroad);
  g->lane_junc = std::move(ljunc);
  g->lane_pred1 = std::move(pred1);
  g->lane_succ1 = std::move(succ1);
  g->succ_off.assign(n + 1, 0);
  g->pred_off.assign(n + 1, 0);
  for (int32_t l = 0; l < n; l++) {
    auto& t = lanes[l];
    std::sort(t.succ.begin(), t.succ.end());
    std::sort(t.pred.begin(), t.pred.end());
    g->succ_off[l + 1] = g->succ_off[l] + (int32_t)t.succ.size();
    g->pred_off[l + 1] = g->pred_off[l] + (int32_t)t.pred.size();
  }
  g->succ.reserve(g->succ_off[n]);
  g->pred.reserve(g->pred_off[n]);
  for (int32_t l = 0; l < n; l++) {
    g->succ.insert(g->succ.end(), lanes[l].succ.begin(), lanes[l].succ.end());
    g->pred.insert(g->pred.end(), lanes[l].pred.begin(), lanes[l].pred.end());
  }
  g->road_lane_off.resize(nr + 1);
  g->road_lanes.resize((size_t)nr * L);
  for (int k = 0; k <= nr; k++) g->road_lane_off[k] = k * L;
  for (int64_t k = 0; k < (int64_t)nr * L; k++) g->road_lanes[k] = (int32_t)k;
  g->green.assign(n, 0);
  for (auto [cid, bit] : greens) g->green[cid] |= bit;
  // centerline geometry: one segment per lane (cum = [0], its heading)
  g->geo_off.resize(n + 1);
  g->geo_cum.assign(n, 0.0);
  g->geo_angle.resize(n);
  for (int32_t l = 0; l <= n; l++) g->geo_off[l] = l;
  for (int32_t l = 0; l < n; l++) g->geo_angle[l] = heading(lanes[l].c0, lanes[l].c1);
  g->junc_pos.resize(2 * (size_t)nj);
  for (int ji = 0; ji < nj; ji++) {
    g->junc_pos[2 * ji] = jpos[jorder[ji]].x;
    g->junc_pos[2 * ji + 1] = jpos[jorder[ji]].y;
    g->junction_ids += (ji ? "\n" : "") + jname[jorder[ji]];
  }
  for (int k = 0; k < nr; k++) g->road_ids += (k ? "\n" : "") + roads[rorder[k]].id;
  *out = g;
  return TSB_OK;
}

int tsb_grid_sizes(const tsb_grid* g, int64_t* sizes) {
  sizes[0] = g->n_lanes;
  sizes[1] = (int64_t)g->succ.size();
  sizes[2] = (int64_t)g->pred.size();
  sizes[3] = (int64_t)g->road_lane_off.size() - 1;
  sizes[4] = (int64_t)g->road_lanes.size();
  sizes[5] = (int64_t)g->junc_signal.size();
  sizes[6] = (int64_t)g->phase_dur.size();
  sizes[7] = (int64_t)g->geo_cum.size();
  sizes[8] = (int64_t)g->road_ids.size();
  sizes[9] = (int64_t)g->junction_ids.size();
  return TSB_OK;
}

int tsb_grid_export(const tsb_grid* g, void* const* dst) {
  int k = 0;
  auto put = [&](const auto& v) {
    if (dst[k] && !v.empty()) std::memcpy(dst[k], v.data(), v.size() * sizeof(v[0]));
    k++;
  };
  put(g->lane_len);
  put(g->lane_cap);
  put(g->lane_kind);
  put(g->lane_open);
  put(g->lane_left);
  put(g->lane_right);
  put(g->lane_road);
  put(g->lane_junc);
  put(g->lane_pred1);
  put(g->lane_succ1);
  put(g->succ_off);
  put(g->succ);
  put(g->pred_off);
  put(g->pred);
  put(g->road_lane_off);
  put(g->road_lanes);
  put(g->junc_signal);
  put(g->junc_phase_off);
  put(g->phase_dur);
  put(g->green);
  put(g->phase0);
  put(g->elapsed0);
  put(g->geo_off);
  put(g->geo_cum);
  put(g->geo_angle);
  put(g->junc_pos);
  put(g->road_ids);
  put(g->junction_ids);
  return TSB_OK;
}

void tsb_grid_destroy(tsb_grid* g) { delete g; }

}  // extern "C"
