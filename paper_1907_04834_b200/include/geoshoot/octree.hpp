// geoshoot/octree.hpp -- the reference's Octree value type (reference
// octree.hpp:17-87), backed by the device octree of include/geoshoot_b200.h.
//
// build() runs the sm_100a Morton-replay build; the host keeps a mirror of the
// node records (same fields as the reference's Node) for inspection. Node
// order is the device's depth-first pre-order (root = 0) rather than the
// reference's creation order; children[], counts, boxes and (up to summation
// order) sums are the reference's. Leaf chains list bucket members newest
// first, as the reference's insertion does.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "geoshoot/core.hpp"

extern "C" {
struct gs_tree;
}

namespace geoshoot {

class Octree {
 public:
  static constexpr int max_depth = 32;
  static constexpr std::int32_t no_child = -1;

  struct Node {
    Vec3 cell_min, cell_max;
    Vec3 actual_min, actual_max;
    Vec3 position_sum;
    Vec3 momentum_sum;
    Vec3 alpha_sum;
    Vec3 beta_sum;
    std::uint32_t count = 0;
    std::int32_t children[8] = {no_child, no_child, no_child, no_child,
                                no_child, no_child, no_child, no_child};
    std::int32_t first_point = -1;
    bool leaf = true;
    Vec3 centroid() const { return position_sum * (1.0 / count); }
  };

  /// Empty tree over an explicit root cell; points arrive through insert().
  Octree(const Vec3& cell_min, const Vec3& cell_max);
  /// Root cell = bounding box padded by 1e-9 * extent (reference octree.cpp:25-40).
  static Octree build(const PointSet& q, const MomentumSet& p);

  /// Adds point `index` (must equal point_count()); throws OutOfBounds outside
  /// the root cell. Inserts are O(1): the device tree over the explicit root
  /// cell is (re)built once, on the first use after a run of inserts, so an
  /// insert loop costs one O(N) build in total (reference octree.cpp:74-117
  /// inserts in O(depth) each; the resulting tree is the same).
  void insert(std::uint32_t index, const Vec3& position, const Vec3& momentum);
  void accumulate_adjoints(const std::vector<Vec3>& alpha, const std::vector<Vec3>& beta);
  static double min_distance(const Node& node, const Vec3& x);

  std::size_t point_count() const { return points_.size(); }
  std::size_t node_count() const { sync(); return nodes_.size(); }
  const Node& node(std::size_t i) const { sync(); return nodes_[i]; }
  const Node& root() const { sync(); return nodes_.front(); }
  const std::vector<Vec3>& points() const { return points_; }
  const std::vector<Vec3>& momenta() const { return momenta_; }
  const std::vector<std::int32_t>& next_point() const { sync(); return next_point_; }
  static int octant_of(const Node& node, const Vec3& x);

  /// The device tree (built on first use); nullptr for an empty tree.
  gs_tree* device() const;
  /// Per-point adjoint arrays whose values the device tree holds (the last
  /// accumulate_adjoints, or the last bh_point_hessian_products upload): a
  /// per-point query passing the same arrays re-uses the device copy.
  const Vec3* device_alpha() const { return dev_alpha_; }
  const Vec3* device_beta() const { return dev_beta_; }
  void note_device_adjoints(const Vec3* a, const Vec3* b) const { dev_alpha_ = a; dev_beta_ = b; }

  Octree(Octree&&) noexcept;
  Octree& operator=(Octree&&) noexcept;
  Octree(const Octree&) = delete;
  Octree& operator=(const Octree&) = delete;
  ~Octree();

 private:
  Octree() = default;
  void rebuild(bool explicit_root) const;
  void mirror() const;
  void sync() const {
    if (dirty_) rebuild(true);
  }

  mutable std::vector<Node> nodes_;
  std::vector<Vec3> points_;
  std::vector<Vec3> momenta_;
  mutable std::vector<std::int32_t> next_point_;
  Vec3 root_min_, root_max_;
  bool explicit_root_ = false;
  mutable bool dirty_ = false;  // inserts since the last device build
  mutable gs_tree* dev_ = nullptr;
  mutable const Vec3* dev_alpha_ = nullptr;
  mutable const Vec3* dev_beta_ = nullptr;
};

}  // namespace geoshoot
