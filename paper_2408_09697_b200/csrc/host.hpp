// Host-side model of the heterogeneous graph and the planning objects that
// stay on the CPU (the meta-partitioner is O(|A|log|A|+|R|), BASELINE.json
// north_star). Everything here reproduces the reference's host algorithms
// bit-for-bit (same libstdc++ RNG engines and distributions), so that the GPU
// path consumes identical graphs, plans, initial weights and batches.
//
// Reference counterparts (under /root/reference/proj):
//   Graph / Csr / Relation           include/hetsim/hetgraph.hpp:29-74
//   gen_synthetic                    src/harness.cpp:74-186
//   build_hetgraph / add_reverse     src/hetgraph.cpp:96-156
//   Metatree / meta_partition        include/hetsim/metapartition.hpp:17-111
//   init_model / init_learnable      src/hgnn.cpp:39-81
//   hop_relation_sets / rels_by_dst  src/hgnn.cpp:16-37
//   make_batches                     src/harness.cpp:327-340
//   profile_miss_penalty / allocate  src/cache.cpp:11-33, 65-85
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace hetgpu {

using NodeId = std::uint32_t;

// splitmix64 finaliser over a + phi*(b+1) (sampling.cpp:9-15); shared by host
// and device (the device copy lives in kernels.cuh).
inline std::uint64_t mix_seed(std::uint64_t a, std::uint64_t b) {
  std::uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// std::mt19937_64(seed) engines whose next outputs are outputs starts[c] (ascending) of
// that stream, by polynomial jump-ahead (mt_jump.cpp): a long stream generated in
// concurrent chunks, bit-identical to the serial one.
std::vector<std::mt19937_64> mt64_jump_engines(std::uint64_t seed, const std::vector<std::uint64_t>& starts);

enum class Storage : int { Absent = 0, Dense = 1, Learnable = 2 };

// Destination-major adjacency of one relation: indptr over dst nodes, source
// ids in insertion order within each destination.
struct Adjacency {
  std::vector<std::uint64_t> offsets;  // n_dst + 1
  std::vector<NodeId> sources;
  std::uint64_t degree(NodeId d) const { return offsets[d + 1] - offsets[d]; }
};

struct RelationInfo {
  int src_type = -1;
  int edge_type = -1;
  int dst_type = -1;
  bool reverse = false;
  Adjacency adj;
};

struct NodeTypeInfo {
  std::string name;
  std::uint64_t count = 0;
  int dim = 0;
  Storage storage = Storage::Absent;
  int elem_bytes = 4;
  std::vector<float> dense;  // [count x dim] row-major, Storage::Dense only
};

struct Graph {
  std::vector<NodeTypeInfo> types;
  std::vector<std::string> edge_type_names;
  std::vector<RelationInfo> rels;
  int target = 0;
  int num_classes = 0;
  std::vector<std::int32_t> labels;

  int num_types() const { return static_cast<int>(types.size()); }
  int num_rels() const { return static_cast<int>(rels.size()); }
  std::uint64_t total_edges() const;
  void validate() const;
};

// ---- synthetic generation (harness.hpp:22-50) --------------------------------
struct SpecNodeType {
  std::string name;
  std::uint64_t count = 0;
  int dim = 0;
  Storage storage = Storage::Dense;
};
struct SpecRelation {
  std::string src, edge, dst;
  std::uint64_t edges = 0;
  bool powerlaw = false;
  double alpha = 2.0;
};
struct Spec {
  std::string name;
  std::string target;
  int num_classes = 2;
  double label_noise = 0.0;
  std::vector<SpecNodeType> node_types;
  std::vector<SpecRelation> relations;
  bool add_reverse = true;
  std::vector<std::string> self_paired;
};

Graph generate(const Spec& spec, std::uint64_t seed);

// ---- HGC1 container (container.hpp:8-19; container.cpp:47-154) -----------------
std::string container_header(const Graph& g);  // the reference's exact JSON header
void save_container(const Graph& g, const std::string& path);
Graph load_container(const std::string& path);
// The header of a container as a Graph skeleton (types, relations, labels; no
// adjacency or features) plus the file offset of every relation's dst-major (src, dst)
// u32 pairs and of every dense type's f32 rows: the device loader streams those.
struct ContainerLayout {
  Graph meta;
  std::vector<std::uint64_t> rel_edges, rel_offset, dense_offset;
};
ContainerLayout container_layout(const std::string& path);

// Builds the dst-major adjacency of every relation from (src, dst) pairs in
// insertion order (hetgraph.cpp:126-156). Features start Absent.
Graph assemble(std::vector<std::string> type_names, std::vector<std::uint64_t> counts,
               std::vector<std::string> edge_names, const std::vector<int>& rel_src,
               const std::vector<int>& rel_dst,
               const std::vector<std::vector<std::pair<NodeId, NodeId>>>& pairs, int target,
               int num_classes);

// Appends the transposed relation for every forward relation except those in
// `self_paired` (hetgraph.cpp:96-124).
void append_reverse(Graph& g, const std::vector<int>& self_paired);

// ---- metatree and meta-partitioning ----------------------------------------
struct TreePos {
  int type = -1;
  int depth = 0;
  int parent = -1;
  int rel = -1;
  std::vector<int> children;
};

struct Tree {
  std::vector<TreePos> pos;
  int k = 0;
  int root_type = -1;
  int root_child_ancestor(int p) const;
};

struct SubTree {
  int id = -1;
  int child_pos = -1;
  std::vector<int> positions;
  std::vector<int> rel_multiset;
  std::vector<int> rel_unique;
  std::vector<int> types_unique;
  std::uint64_t weight = 0;
};

struct Part {
  std::vector<int> sub_ids;
  std::vector<int> relations;
  std::vector<int> node_types;
  std::uint64_t weight = 0;
  bool replica = false;
  int replica_index = 0;
  int replica_count = 1;
};

struct Plan {
  int p = 0;
  Tree tree;
  std::vector<SubTree> subs;
  std::vector<Part> parts;
  bool deduplicated = false;
  std::vector<int> owners_of_sub(int sub_id) const;
};

// Schema-level view: vertex weight = node count, link weight = edge count.
struct Schema {
  std::vector<std::uint64_t> vertex_weight;
  struct Link {
    int rel = -1;
    int src = -1, dst = -1;
    std::uint64_t weight = 0;
  };
  std::vector<Link> links;
};

Schema schema_of(const Graph& g);
Tree bfs_tree(const Schema& s, int root, int k);
Tree metapath_tree(const Schema& s, int root, const std::vector<std::vector<int>>& paths);
std::vector<int> lpt(const std::vector<std::uint64_t>& weights, int p);
Plan meta_partition(const Schema& s, int root, int k, int p);
// work-aware alternative (not the reference policy): groups of workers replicate sets of
// sub-metatrees, minimising the busiest worker's share of `work` (one value per sub)
Plan work_aware_partition(const Schema& s, int root, int k, int p, const std::vector<double>& work,
                          const std::vector<double>& learn_rows = {}, double merge_cost = 6.0,
                          const std::vector<bool>& learnable_types = {});
std::vector<int> cacheable_types(const Plan& plan, int part);

// hop_relation_sets (hgnn.cpp:28-37): allowed relations per hop, ascending.
std::vector<std::vector<int>> hop_relations(const Tree& t, int k);
// rels_by_dst_at_depth (hgnn.cpp:16-26)
std::map<int, std::vector<int>> relations_into_at_depth(const Tree& t, int depth);

// ---- model parameters --------------------------------------------------------
struct SlotId {
  int rel = -1;
  int layer = 0;
  bool operator<(const SlotId& o) const { return rel != o.rel ? rel < o.rel : layer < o.layer; }
};

struct WeightInit {
  int in_dim = 0, out_dim = 0;
  std::vector<double> values;  // row-major [in_dim x out_dim]
};

struct ModelInit {
  int k = 1, hidden = 16, num_classes = 2;
  std::vector<int> input_dims;
  std::map<SlotId, WeightInit> weights;
  int out_dim(int layer) const { return layer == k ? num_classes : hidden; }
};

ModelInit init_model(const Graph& g, const Tree& t, int hidden, std::uint64_t seed);
// Learnable tables: uniform in [-1/sqrt(d), 1/sqrt(d)] per type (hgnn.cpp:64-81).
std::map<int, std::vector<double>> init_learnable(const Graph& g, std::uint64_t seed);

// ---- batch-invariant RAF bookkeeping ---------------------
// run_raf_batch recomputes these every batch although they depend only on the
// plan: structural_boundaries (raf.cpp:306-340), boundary_cut_edges
// (raf.cpp:521-528) and the contributor sets behind the slot part of
// sync_bytes (raf.cpp:217, 414, 496-503). Meta view: a depth-1 position is the
// only crossing kind; a slot's contributors are the owners of the root children
// whose subtrees hold a position with that (relation, layer).
struct RafAccounting {
  std::vector<std::uint64_t> boundary_counts;          // per worker
  std::uint64_t boundary_cut_edges = 0;
  std::map<SlotId, std::vector<int>> slot_contributors;  // ascending worker ids
  std::map<int, std::vector<int>> leaf_owners;           // learnable leaf type -> possible contributors
};
// top_owners[ci]: owning workers of root child ci (tree.pos[0].children order)
RafAccounting raf_accounting(const Graph& g, const Tree& t, const std::vector<std::vector<int>>& top_owners, int p);
// the same for a meta plan's view (raf_view_from_plan, raf.cpp:43-57)
RafAccounting plan_accounting(const Graph& g, const Plan& plan);

// make_batches (harness.cpp:327-340): shuffled target ids in batch_size chunks.
std::vector<std::vector<NodeId>> make_batches(const Graph& g, int batch_size, int max_batches,
                                              std::uint64_t seed);

// ---- cache planning (cache.hpp) ---------------------------------------------
struct CostModel {
  double read_ns_per_byte = 1.0;
  double write_ns_per_byte = 1.0;
  double fixed_overhead_ns = 1000.0;
  int elem_bytes = 4;
};
struct TypePenalty {
  bool learnable = false;
  std::uint64_t record_bytes = 0;
  double transfer_ns = 0.0;
  double ratio = 0.0;
};
std::vector<TypePenalty> miss_penalty(const Graph& g, const CostModel& cm);
struct CacheAlloc {
  std::uint64_t budget = 0;
  std::vector<std::uint64_t> bytes, capacity;
};
CacheAlloc allocate_cache(std::uint64_t budget, const std::vector<std::vector<std::uint64_t>>& counts,
                          const std::vector<TypePenalty>& prof);

}  // namespace hetgpu
