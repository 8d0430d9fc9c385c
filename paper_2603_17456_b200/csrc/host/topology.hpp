// Fabric model: directed capacitated links, star and folded-Clos fat-tree
// builders (topology.cpp:98-165), shortest-path routes with the reference's
// lowest-link-id tie break (topology.cpp:32-81).
//
// The reference materialises a dense n x n route table (1.6 GB at 4096 hosts).
// Here routes are produced on demand from one reverse BFS per destination and
// only for the (src, dst) pairs the simulation can use; the device receives
// them as a CSR table (route id -> link list).
#pragma once
#include <string>
#include <unordered_map>
#include <vector>

#include "config.hpp"

namespace mfh {

enum class NodeRole : unsigned char { Prefill, Decode, Switch };

struct Link {
  int from = -1;
  int to = -1;
  double capacity = 0.0;
};

class Fabric {
 public:
  int add_node(NodeRole role);
  int add_link(int from, int to, double capacity);
  void add_duplex(int a, int b, double capacity);

  // Link ids of the route src -> dst (empty when src == dst). Throws SimError
  // for unreachable pairs, like Topology::route (topology.cpp:83-89).
  std::vector<int> route(int src, int dst) const;

  int nodes() const { return static_cast<int>(roles_.size()); }
  int hosts() const { return hosts_; }
  const std::vector<Link>& links() const { return links_; }

  static Fabric star(int hosts, double capacity);
  // oversub >= 1 divides the capacity of every switch-to-switch link (edge-agg
  // and agg-core); 1 is the reference's uniform fabric (topology.cpp:108-145).
  // Oversubscription is an oracle extension: the reference has no such key.
  static Fabric fat_tree(int hosts, double capacity, double oversub = 1.0);
  static Fabric from(const Config& cfg);

 private:
  const std::vector<int>& dist_to(int dst) const;
  std::vector<NodeRole> roles_;
  std::vector<Link> links_;
  std::vector<std::vector<int>> out_;  // link ids per node, ascending
  std::vector<std::vector<int>> in_;
  int hosts_ = 0;
  mutable std::unordered_map<int, std::vector<int>> dist_cache_;
};

// CSR route table for the device
struct RouteTable {
  std::vector<int> off{0};
  std::vector<int> links;
  int rmax = 0;
  std::unordered_map<long long, int> index;  // (src<<32|dst) -> route id

  int add(const Fabric& f, int src, int dst);
  int count() const { return static_cast<int>(off.size()) - 1; }
};

}  // namespace mfh
