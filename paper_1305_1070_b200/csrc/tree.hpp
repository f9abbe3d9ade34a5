// Separator tree and nested dissection, host side, built once per device.
//
// Bit-exact restatement of the reference partitioner so that the cluster
// ids, dof lists, levels and fold order are identical to what the CPU solver
// would use:
//   SeparatorTree::build   proj/src/partition.cpp:19-91
//   dissect                proj/src/partition.cpp:159-230
//   bfs_coordinates        proj/src/partition.cpp:234-267
//   nested_dissection      proj/src/partition.cpp:271-326
//   validate_partition     proj/src/partition.cpp:340-363
#pragma once

#include <array>
#include <utility>
#include <vector>

#include "common.hpp"

namespace negfb {

struct Cluster {
  int id = -1;
  int level = 0;     // 1 = leaf, levels() = root
  int parent = -1;   // -1 for the root
  std::vector<int> dofs;       // ascending
  std::vector<int> children;   // in id order
  std::vector<int> anc;        // ancestors, nearest first
  int size() const { return static_cast<int>(dofs.size()); }
};

class Tree {
 public:
  // `clusters` carry parent links and dof lists (ids = positions).
  static Tree build(std::vector<Cluster> clusters, int n_dofs);

  int num_clusters() const { return static_cast<int>(c_.size()); }
  int num_dofs() const { return n_; }
  int levels() const { return levels_; }
  int root() const { return root_; }
  const Cluster& cluster(int i) const { return c_[static_cast<std::size_t>(i)]; }
  int dof_cluster(int d) const { return dof_cluster_[static_cast<std::size_t>(d)]; }
  int local_index(int d) const { return local_[static_cast<std::size_t>(d)]; }
  bool is_ancestor(int anc, int node) const;
  const std::vector<int>& fold_order() const { return fold_order_; }

 private:
  std::vector<Cluster> c_;
  std::vector<int> dof_cluster_, local_, fold_order_;
  int n_ = 0, levels_ = 0, root_ = -1;
};

struct Graph {
  int n = 0;
  std::vector<std::array<int, 2>> edges;  // u < v, deduplicated
  std::vector<std::vector<int>> adjacency() const;
};

// Off-diagonal pattern of (rows, cols) as an undirected simple graph
// (proj/src/sparse.cpp:61-72).
Graph graph_of_pattern(int n, const std::vector<std::pair<int, int>>& entries);

Tree nested_dissection(const Graph& g, const std::vector<std::vector<int>>& atomic_groups,
                       int max_leaf, const std::vector<std::array<double, 2>>& coords);

// Edges joining clusters that are not ancestor-related: {u, v, cu, cv}.
std::vector<std::array<int, 4>> partition_violations(const Tree& t, const Graph& g);

}  // namespace negfb
