// router.cpp -- host restatement of trafficsim/engine/routing.py.
//
// Reverse Dijkstra over open lanes weighted length/max_speed (routing.py:29-45,
// 47-68); route extraction follows tight edges w(u) + dist(v) == dist(u),
// smallest successor id first (routing.py:70-101).  Because fp addition is
// monotone, the settled distances are the unique solution of the Bellman
// equation dist(u) = min_v fl(w(u) + dist(v)), so they are bitwise equal to
// the reference's heapq values regardless of heap tie order.  The LRU of the
// reference only affects speed and is replaced by batch routing grouped by
// destination, multithreaded over destinations.
#include "router.h"

#include <algorithm>
#include <queue>
#include <thread>
#include <vector>

namespace tsb {

Router::Router(int32_t n_lanes, const int8_t* kind, const double* len, const double* cap, const uint8_t* open,
               const int32_t* succ_off, const int32_t* succ, const int32_t* pred_off, const int32_t* pred,
               const int32_t* lane_road)
    : n_(n_lanes),
      kind_(kind, kind + n_lanes),
      len_(len, len + n_lanes),
      cap_(cap, cap + n_lanes),
      open_(open, open + n_lanes),
      succ_off_(succ_off, succ_off + n_lanes + 1),
      succ_(succ, succ + succ_off[n_lanes]),
      pred_off_(pred_off, pred_off + n_lanes + 1),
      pred_(pred, pred + pred_off[n_lanes]),
      road_(lane_road, lane_road + n_lanes) {
  rebuild();
}

void Router::set_lane(int32_t lane, double max_speed, bool open) {
  cap_[lane] = max_speed;
  open_[lane] = open ? 1 : 0;
  rebuild();
}

void Router::rebuild() {
  w_.assign(n_, -1.0);
  for (int32_t l = 0; l < n_; l++)
    if (kind_[l] >= 0 && open_[l]) w_[l] = len_[l] / cap_[l];
}

void Router::dist_to(int32_t dest, std::vector<double>& dist) const {
  dist.assign(n_, -1.0);
  if (dest < 0 || dest >= n_ || w_[dest] < 0) return;
  using Item = std::pair<double, int32_t>;
  std::priority_queue<Item, std::vector<Item>, std::greater<Item>> heap;
  heap.push({w_[dest], dest});
  while (!heap.empty()) {
    auto [d, u] = heap.top();
    heap.pop();
    if (dist[u] >= 0) continue;
    dist[u] = d;
    for (int32_t k = pred_off_[u]; k < pred_off_[u + 1]; k++) {
      int32_t p = pred_[k];
      if (w_[p] < 0 || dist[p] >= 0) continue;
      heap.push({w_[p] + d, p});
    }
  }
}

bool Router::extract(int32_t origin, int32_t dest, const std::vector<double>& dist, std::vector<int32_t>* lanes,
                     std::vector<int32_t>* roads) const {
  if (dist[origin] < 0) return false;
  int32_t u = origin;
  for (;;) {
    if (lanes) lanes->push_back(u);
    if (roads && kind_[u] == 0 && (roads->empty() || roads->back() != road_[u])) roads->push_back(road_[u]);
    if (u == dest) return true;
    int32_t nxt = -1;
    for (int32_t k = succ_off_[u]; k < succ_off_[u + 1]; k++) {
      int32_t v = succ_[k];
      if (w_[v] < 0 || dist[v] < 0) continue;
      if (w_[u] + dist[v] == dist[u]) {
        nxt = v;
        break;
      }
    }
    if (nxt < 0) return false;  // extraction stalled (routing.py:96-99)
    u = nxt;
  }
}

bool Router::route(int32_t origin, int32_t dest, std::vector<int32_t>* lanes, std::vector<int32_t>* roads,
                   double* cost) const {
  std::vector<double> dist;
  dist_to(dest, dist);
  if (origin < 0 || origin >= n_ || dist[origin] < 0) return false;
  if (cost) *cost = dist[origin];
  return extract(origin, dest, dist, lanes, roads);
}

void Router::route_batch(const std::vector<int32_t>& origins, const std::vector<int32_t>& dests,
                         std::vector<std::vector<int32_t>>& roads_out, std::vector<uint8_t>& ok) const {
  const size_t n = origins.size();
  roads_out.assign(n, {});
  ok.assign(n, 0);
  std::vector<size_t> order(n);
  for (size_t i = 0; i < n; i++) order[i] = i;
  std::sort(order.begin(), order.end(), [&](size_t a, size_t b) { return dests[a] < dests[b]; });
  std::vector<std::pair<size_t, size_t>> groups;  // [begin, end) in order
  for (size_t i = 0; i < n;) {
    size_t j = i;
    while (j < n && dests[order[j]] == dests[order[i]]) j++;
    groups.push_back({i, j});
    i = j;
  }
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  unsigned nt = std::min<unsigned>(hw, (unsigned)std::max<size_t>(1, groups.size()));
  std::vector<std::thread> pool;
  std::atomic<size_t> next{0};
  for (unsigned t = 0; t < nt; t++)
    pool.emplace_back([&]() {
      std::vector<double> dist;
      for (;;) {
        size_t g = next.fetch_add(1);
        if (g >= groups.size()) break;
        dist_to(dests[order[groups[g].first]], dist);
        for (size_t q = groups[g].first; q < groups[g].second; q++) {
          size_t i = order[q];
          std::vector<int32_t> r;
          if (extract(origins[i], dests[i], dist, nullptr, &r)) {
            roads_out[i] = std::move(r);
            ok[i] = 1;
          }
        }
      }
    });
  for (auto& th : pool) th.join();
}

void Router::reach(const std::vector<int32_t>& dests, uint8_t* out) const {
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  std::atomic<size_t> next{0};
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < std::min<unsigned>(hw, (unsigned)std::max<size_t>(1, dests.size())); t++)
    pool.emplace_back([&]() {
      std::vector<double> dist;
      for (;;) {
        size_t k = next.fetch_add(1);
        if (k >= dests.size()) break;
        dist_to(dests[k], dist);
        for (int32_t l = 0; l < n_; l++) out[k * (size_t)n_ + l] = dist[l] >= 0 ? 1 : 0;
      }
    });
  for (auto& th : pool) th.join();
}

}  // namespace tsb
