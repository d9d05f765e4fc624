// router.h -- host router (restates trafficsim/engine/routing.py).
#pragma once
#include <atomic>
#include <cstdint>
#include <vector>

namespace tsb {

class Router {
 public:
  Router(int32_t n_lanes, const int8_t* kind, const double* len, const double* cap, const uint8_t* open,
         const int32_t* succ_off, const int32_t* succ, const int32_t* pred_off, const int32_t* pred,
         const int32_t* lane_road);
  void set_lane(int32_t lane, double max_speed, bool open);
  // dist[l] = cost from l to dest inclusive of both endpoints, -1 if unreachable.
  void dist_to(int32_t dest, std::vector<double>& dist) const;
  bool route(int32_t origin, int32_t dest, std::vector<int32_t>* lanes, std::vector<int32_t>* roads,
             double* cost) const;
  // roads_of_route for many (origin, dest) pairs, one Dijkstra per distinct dest.
  void route_batch(const std::vector<int32_t>& origins, const std::vector<int32_t>& dests,
                   std::vector<std::vector<int32_t>>& roads_out, std::vector<uint8_t>& ok) const;
  void reach(const std::vector<int32_t>& dests, uint8_t* out) const;
  int32_t n_lanes() const { return n_; }

 private:
  void rebuild();
  bool extract(int32_t origin, int32_t dest, const std::vector<double>& dist, std::vector<int32_t>* lanes,
               std::vector<int32_t>* roads) const;
  int32_t n_;
  std::vector<int8_t> kind_;
  std::vector<double> len_, cap_;
  std::vector<uint8_t> open_;
  std::vector<int32_t> succ_off_, succ_, pred_off_, pred_, road_;
  std::vector<double> w_;
};

}  // namespace tsb
