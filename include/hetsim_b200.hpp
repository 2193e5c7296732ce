// hetsim_b200.hpp — header-only C++ mirror of the reference's hetsim API for the
// mini-batch hot path, implemented over the C-ABI in hetgpu.h (libhetgpu.so).
//
// The reference (/root/reference/proj) is a C++20 library that callers link
// directly; it has no FFI of its own. A hetsim user switches to the B200 path by
// including this header instead of hetsim/{sampling,harness,metapartition,raf}.hpp
// and linking libhetgpu.so. Names, argument meaning and exception types follow
// the reference (file:line per declaration, under /root/reference/proj):
//   std::invalid_argument for bad shapes / ranges / ids, std::runtime_error for
//   missing features, non-finite gradients and CUDA/NCCL failures.
//
// Everything lives in namespace hetsim_b200 so it can be linked side by side
// with the reference in parity tests; define HETSIM_B200_AS_HETSIM before the
// include to also expose it as namespace hetsim (drop-in replacement build).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <set>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "hetgpu.h"

namespace hetsim_b200 {

using NodeId = std::uint32_t;     // hetgraph.hpp:16
using NodeTypeId = int;           // hetgraph.hpp:14

namespace detail {

[[noreturn]] inline void raise_last() {
  const std::string msg = hg_last_error();
  if (hg_last_error_kind() == 1) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
template <typename T>
T* check(T* p) {
  if (!p) raise_last();
  return p;
}
inline int check(int rc) {
  if (rc < 0) raise_last();
  return rc;
}

// name -> raw array of a C-ABI bundle (copied out, bundle freed)
class Bundle {
 public:
  explicit Bundle(hg_bundle* b) {
    check(b);
    for (int i = 0; i < hg_bundle_size(b); ++i) {
      Item it;
      it.dtype = hg_bundle_dtype(b, i);
      for (int d = 0; d < hg_bundle_ndim(b, i); ++d) it.shape.push_back(hg_bundle_dim(b, i, d));
      const auto nb = static_cast<std::size_t>(hg_bundle_nbytes(b, i));
      it.bytes.resize(nb);
      if (nb) std::memcpy(it.bytes.data(), hg_bundle_data(b, i), nb);
      items_.emplace(hg_bundle_name(b, i), std::move(it));
    }
    hg_bundle_free(b);
  }
  bool has(const std::string& n) const { return items_.count(n) != 0; }
  template <typename T>
  std::vector<T> get(const std::string& n) const {
    auto it = items_.find(n);
    if (it == items_.end()) throw std::runtime_error("hetgpu bundle has no tensor " + n);
    std::vector<T> v(it->second.bytes.size() / sizeof(T));
    if (!v.empty()) std::memcpy(v.data(), it->second.bytes.data(), v.size() * sizeof(T));
    return v;
  }

 private:
  struct Item {
    std::string dtype;
    std::vector<long long> shape;
    std::vector<char> bytes;
  };
  std::map<std::string, Item> items_;
};

}  // namespace detail

// splitmix64 finaliser (sampling.cpp:9-15)
inline std::uint64_t mix_seed(std::uint64_t a, std::uint64_t b) { return hg_mix_seed(a, b); }

// ---- synthetic specs and graphs (harness.hpp:15-48, hetgraph.hpp:58-74) ------------------------
struct SyntheticNodeType {
  std::string name;
  std::uint64_t count = 0;
  int dim = 0;
  std::string storage = "dense";  // dense | learnable
};
struct SyntheticRelation {
  std::string src, edge, dst;
  std::uint64_t edges = 0;
  std::string degree = "uniform";  // uniform | powerlaw
  double alpha = 2.0;
};
struct SyntheticSpec {
  std::string name, target;
  int num_classes = 2;
  double label_noise = 0.0;
  std::vector<SyntheticNodeType> node_types;
  std::vector<SyntheticRelation> relations;
  bool add_reverse = true;
  std::vector<std::string> self_paired;
};

// Host-resident heterogeneous graph owned by libhetgpu (immutable, shareable).
class HetGraph {
 public:
  explicit HetGraph(hg_graph* h) : h_(detail::check(h), hg_graph_free) {
    const detail::Bundle b(hg_graph_schema(h_.get()));
    node_counts = b.get<std::uint64_t>("node_counts");
    const auto rs = b.get<int>("rel_src"), rd = b.get<int>("rel_dst");
    for (std::size_t r = 0; r < rs.size(); ++r) relations.push_back({rs[r], rd[r]});
    target = b.get<std::int64_t>("target").at(0);
    num_classes = static_cast<int>(b.get<std::int64_t>("num_classes").at(0));
    dims = b.get<int>("dims");
    kinds = b.get<int>("kinds");
    const auto names = b.get<char>("type_names");
    std::string cur;
    for (char ch : names) {
      if (ch == '\n') {
        type_names.push_back(cur);
        cur.clear();
      } else {
        cur.push_back(ch);
      }
    }
  }
  hg_graph* handle() const { return h_.get(); }
  std::vector<std::uint64_t> node_counts;  // per node type
  struct Rel {
    NodeTypeId src, dst;
  };
  std::vector<Rel> relations;
  NodeTypeId target = 0;
  int num_classes = 0;
  std::vector<std::string> type_names;  // TypeRegistry::node_type_names
  std::vector<int> dims;                // feature / learnable dim per type
  std::vector<int> kinds;               // 0 absent, 1 dense, 2 learnable (StorageKind)
  // g.labels (hetgraph.hpp:66), borrowed from the native graph
  std::span<const std::int32_t> labels() const {
    const std::int32_t* p = nullptr;
    std::uint64_t n = 0;
    detail::check(hg_graph_labels(h_.get(), &p, &n));
    return {p, static_cast<std::size_t>(n)};
  }

 private:
  std::shared_ptr<hg_graph> h_;
};

// gen_synthetic (harness.cpp:74-186): bit-exact with the reference generator
inline HetGraph gen_synthetic(const SyntheticSpec& spec, std::uint64_t seed) {
  std::vector<hg_spec_node_type> types;
  for (const auto& t : spec.node_types) {
    if (t.storage != "dense" && t.storage != "learnable") throw std::invalid_argument("unknown storage kind: " + t.storage);
    types.push_back({t.name.c_str(), t.count, t.dim, t.storage == "dense" ? 1 : 2});
  }
  std::vector<hg_spec_relation> rels;
  for (const auto& r : spec.relations) {
    if (r.degree != "uniform" && r.degree != "powerlaw")
      throw std::invalid_argument("unknown degree distribution: " + r.degree);
    rels.push_back({r.src.c_str(), r.edge.c_str(), r.dst.c_str(), r.edges, r.degree == "powerlaw" ? 1 : 0, r.alpha});
  }
  std::vector<const char*> sp;
  for (const auto& s : spec.self_paired) sp.push_back(s.c_str());
  const hg_spec s{spec.target.c_str(), spec.num_classes, spec.label_noise,
                  static_cast<int>(types.size()), types.data(), static_cast<int>(rels.size()), rels.data(),
                  spec.add_reverse ? 1 : 0, static_cast<int>(sp.size()), sp.data()};
  return HetGraph(hg_graph_generate(&s, seed));
}

// build_hetgraph (hetgraph.cpp:126-156): dst-major CSR per relation, insertion order
inline HetGraph build_hetgraph(const std::vector<std::uint64_t>& node_counts,
                               const std::vector<std::pair<NodeTypeId, NodeTypeId>>& relations,
                               const std::vector<std::vector<std::pair<NodeId, NodeId>>>& edges,
                               NodeTypeId target, int num_classes) {
  std::vector<int> rs, rd;
  std::vector<std::uint64_t> pc;
  std::vector<std::uint32_t> ps, pd;
  for (const auto& r : relations) {
    rs.push_back(r.first);
    rd.push_back(r.second);
  }
  for (const auto& e : edges) {
    pc.push_back(e.size());
    for (const auto& [s, d] : e) {
      ps.push_back(s);
      pd.push_back(d);
    }
  }
  return HetGraph(hg_graph_from_pairs(static_cast<int>(node_counts.size()), node_counts.data(),
                                      static_cast<int>(rs.size()), rs.data(), rd.data(), pc.data(), ps.data(),
                                      pd.data(), target, num_classes));
}

// load_container / save_container (container.cpp:47-154): HGC1 files, byte-identical
// to the reference writer; failures throw std::runtime_error
inline HetGraph load_container(const std::string& path) { return HetGraph(hg_graph_load(path.c_str())); }
inline void save_container(const HetGraph& g, const std::string& path) {
  detail::check(hg_graph_save(g.handle(), path.c_str()));
}

// make_batches (harness.cpp:327-340)
inline std::vector<std::vector<NodeId>> make_batches(const HetGraph& g, int batch_size, int max_batches,
                                                     std::uint64_t seed) {
  const detail::Bundle b(hg_make_batches(g.handle(), batch_size, max_batches, seed));
  std::vector<std::vector<NodeId>> out;
  for (int i = 0; b.has("batch" + std::to_string(i)); ++i) out.push_back(b.get<NodeId>("batch" + std::to_string(i)));
  return out;
}

// ---- planning (metapartition.hpp:17-109; stays on the host) ------------------------------------
struct MetatreePos {
  NodeTypeId type = -1;
  int depth = 0;
  int parent = -1;
  int rel_index = -1;
};
struct Metatree {
  std::vector<MetatreePos> pos;
  int k = 0;
  // MetatreePos::children of a position, in tree order (positions are numbered in BFS order)
  std::vector<int> children(int p) const {
    std::vector<int> c;
    for (std::size_t i = 0; i < pos.size(); ++i)
      if (pos[i].parent == p && static_cast<int>(i) != p) c.push_back(static_cast<int>(i));
    return c;
  }
};
struct PlanPartition {
  std::vector<int> sub_ids, relations;
  std::vector<NodeTypeId> node_types;
  std::vector<NodeTypeId> cacheable;  // cacheable_types (cache.cpp:143-177)
  std::uint64_t weight = 0;
  bool replica = false;
  int replica_index = 0, replica_count = 1;
};
struct PartitionPlan {
  int p = 0;
  Metatree tree;
  std::vector<std::uint64_t> sub_weights;
  std::vector<int> sub_child_pos;  // SubMetatree::child_pos per sub id
  std::vector<PlanPartition> parts;
  std::vector<std::vector<int>> hop_relations;  // hop_relation_sets(tree, k) (hgnn.cpp:28-37)
  // batch-invariant RAF bookkeeping of the plan (raf.cpp:306-340, 496-510, 521-528)
  std::vector<std::uint64_t> boundary_counts;
  std::uint64_t boundary_cut_edges = 0;
  std::vector<std::array<int, 3>> slot_contributors;  // (rel, layer, n contributors)
  std::vector<std::array<int, 2>> leaf_owners;        // (learnable leaf type, n possible contributors)
  // PartitionPlan::owners_of_sub (metapartition.cpp:24-30)
  std::vector<int> owners_of_sub(int sub_id) const {
    std::vector<int> out;
    for (std::size_t i = 0; i < parts.size(); ++i)
      if (std::find(parts[i].sub_ids.begin(), parts[i].sub_ids.end(), sub_id) != parts[i].sub_ids.end())
        out.push_back(static_cast<int>(i));
    return out;
  }
};

// meta_partition (metapartition.cpp:283-295), BFS metatree of depth k
inline PartitionPlan meta_partition(const HetGraph& g, int k, int p) {
  const detail::Bundle b(hg_meta_partition(g.handle(), k, p));
  PartitionPlan plan;
  plan.p = p;
  plan.tree.k = k;
  const auto ty = b.get<int>("tree.type"), de = b.get<int>("tree.depth"), pa = b.get<int>("tree.parent"),
             re = b.get<int>("tree.rel");
  for (std::size_t i = 0; i < ty.size(); ++i) plan.tree.pos.push_back({ty[i], de[i], pa[i], re[i]});
  plan.sub_weights = b.get<std::uint64_t>("subs.weight");
  plan.sub_child_pos = b.get<int>("subs.child_pos");
  plan.boundary_counts = b.get<std::uint64_t>("raf.boundary_counts");
  plan.boundary_cut_edges = b.get<std::uint64_t>("raf.boundary_cut_edges").at(0);
  const auto sc = b.get<int>("raf.slot_contributors");
  for (std::size_t i = 0; i + 2 < sc.size(); i += 3) plan.slot_contributors.push_back({sc[i], sc[i + 1], sc[i + 2]});
  const auto lo = b.get<int>("raf.leaf_owners");
  for (std::size_t i = 0; i + 1 < lo.size(); i += 2) plan.leaf_owners.push_back({lo[i], lo[i + 1]});
  for (int i = 0; b.has("part" + std::to_string(i) + ".sub_ids"); ++i) {
    const std::string pre = "part" + std::to_string(i);
    PlanPartition part;
    part.sub_ids = b.get<int>(pre + ".sub_ids");
    part.relations = b.get<int>(pre + ".relations");
    part.node_types = b.get<int>(pre + ".node_types");
    part.cacheable = b.get<int>(pre + ".cacheable");
    const auto rep = b.get<int>(pre + ".replica");
    part.replica = rep.at(0) != 0;
    part.replica_index = rep.at(1);
    part.replica_count = rep.at(2);
    part.weight = b.get<std::uint64_t>(pre + ".weight").at(0);
    plan.parts.push_back(std::move(part));
  }
  for (int h = 1; h <= k; ++h) plan.hop_relations.push_back(b.get<int>("hop_rels" + std::to_string(h)));
  return plan;
}

// ---- sampling (sampling.hpp:11-48) --------------------------------------------------------------
struct Block {
  int rel_index = -1;
  int hop = 0;
  std::vector<NodeId> dst_ids;
  std::vector<std::uint32_t> indptr;
  std::vector<NodeId> src_ids;
};
struct SampledBlocks {
  int k = 0;
  std::vector<NodeId> seeds;
  std::uint64_t rng_seed = 0;
  std::vector<std::vector<Block>> hops;                       // hops[h-1], ascending relation
  std::vector<std::vector<std::vector<NodeId>>> frontier;     // frontier[h][type]
};

// A device sampler bound to (graph, fanouts, relation sets). Reusing one across
// calls keeps the graph resident in HBM; the free functions below build one per call.
class Sampler {
 public:
  // hop_relations empty: every relation at every hop (sample_khop)
  Sampler(const HetGraph& g, std::vector<int> fanouts, const std::vector<std::vector<int>>& hop_relations = {},
          int batch_cap = 1024, int device = 0)
      : g_(g), fanouts_(std::move(fanouts)), cap_(batch_cap) {
    if (fanouts_.empty()) throw std::invalid_argument("fanouts must be non-empty");
    std::vector<int> flat, counts;
    for (const auto& h : hop_relations) {
      counts.push_back(static_cast<int>(h.size()));
      flat.insert(flat.end(), h.begin(), h.end());
    }
    if (!hop_relations.empty() && hop_relations.size() != fanouts_.size())
      throw std::invalid_argument("hop_relations must have one entry per hop");
    if (flat.empty()) flat.push_back(-1);
    e_.reset(detail::check(hg_sampler_create(g.handle(), fanouts_.data(), static_cast<int>(fanouts_.size()),
                                             hop_relations.empty() ? nullptr : flat.data(),
                                             hop_relations.empty() ? nullptr : counts.data(), batch_cap, device)));
  }

  // sample_impl (sampling.cpp:41-92) on the device; blocks and frontiers copied back
  hg_engine* handle() const { return e_.get(); }

  SampledBlocks sample(std::span<const NodeId> seeds, std::uint64_t rng_seed) {
    for (NodeId s : seeds)
      if (s >= g_.node_counts.at(g_.target))
        throw std::invalid_argument("seed node id out of range: " + std::to_string(s));
    SampledBlocks out;
    out.k = static_cast<int>(fanouts_.size());
    out.seeds.assign(seeds.begin(), seeds.end());
    out.rng_seed = rng_seed;
    const int nt = static_cast<int>(g_.node_counts.size());
    out.frontier.assign(out.k + 1, std::vector<std::vector<NodeId>>(nt));
    out.hops.resize(out.k);
    if (seeds.empty()) return out;  // the reference returns empty blocks and frontiers
    if (static_cast<int>(seeds.size()) > cap_) throw std::invalid_argument("batch larger than the sampler's capacity");
    detail::check(hg_engine_sample(e_.get(), seeds.data(), static_cast<int>(seeds.size()), rng_seed));
    const detail::Bundle b(hg_engine_read(e_.get(), nullptr));
    for (int h = 0; h <= out.k; ++h)
      for (int t = 0; t < nt; ++t) {
        const std::string n = "frontier" + std::to_string(h) + ".t" + std::to_string(t);
        if (b.has(n)) out.frontier[h][t] = b.get<NodeId>(n);
      }
    for (int h = 1; h <= out.k; ++h)
      for (std::size_t r = 0; r < g_.relations.size(); ++r) {
        const std::string pre = "hop" + std::to_string(h) + ".rel" + std::to_string(r);
        if (!b.has(pre + ".dst_ids")) continue;
        Block blk;
        blk.rel_index = static_cast<int>(r);
        blk.hop = h;
        blk.dst_ids = b.get<NodeId>(pre + ".dst_ids");
        if (blk.dst_ids.empty()) continue;  // relations with an empty dst frontier emit no block
        blk.indptr = b.get<std::uint32_t>(pre + ".indptr");
        blk.src_ids = b.get<NodeId>(pre + ".src_ids");
        out.hops[h - 1].push_back(std::move(blk));
      }
    return out;
  }

 private:
  struct Free {
    void operator()(hg_engine* e) const { hg_engine_free(e); }
  };
  HetGraph g_;
  std::vector<int> fanouts_;
  int cap_;
  std::unique_ptr<hg_engine, Free> e_;
};

// sample_khop (sampling.cpp:94-97)
inline SampledBlocks sample_khop(const HetGraph& g, std::span<const NodeId> seeds, const std::vector<int>& fanouts,
                                 std::uint64_t rng_seed) {
  return Sampler(g, fanouts, {}, std::max<int>(1, static_cast<int>(seeds.size()))).sample(seeds, rng_seed);
}
// sample_khop_restricted (sampling.cpp:99-103)
inline SampledBlocks sample_khop_restricted(const HetGraph& g, std::span<const NodeId> seeds,
                                            const std::vector<int>& fanouts, std::uint64_t rng_seed,
                                            const std::vector<std::vector<int>>& hop_relations) {
  if (fanouts.empty()) throw std::invalid_argument("fanouts must be non-empty");
  return Sampler(g, fanouts, hop_relations, std::max<int>(1, static_cast<int>(seeds.size()))).sample(seeds, rng_seed);
}

// ---- dense matrices (matrix.hpp:9-94): host containers, f64 like the reference -------------------
struct Matrix {
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::vector<double> data;

  Matrix() = default;
  Matrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0.0) {}

  double* row(std::size_t i) { return data.data() + i * cols; }
  const double* row(std::size_t i) const { return data.data() + i * cols; }
  double& at(std::size_t i, std::size_t j) { return data[i * cols + j]; }
  double at(std::size_t i, std::size_t j) const { return data[i * cols + j]; }
  bool same_shape(const Matrix& o) const { return rows == o.rows && cols == o.cols; }
};

inline void check_dims(bool ok, const char* what) {
  if (!ok) throw std::invalid_argument(std::string("dimension mismatch: ") + what);
}
inline void add_inplace(Matrix& a, const Matrix& b) {
  check_dims(a.same_shape(b), "add_inplace");
  for (std::size_t i = 0; i < a.data.size(); ++i) a.data[i] += b.data[i];
}
inline double max_abs_diff(const Matrix& a, const Matrix& b) {
  check_dims(a.same_shape(b), "max_abs_diff");
  double m = 0.0;
  for (std::size_t i = 0; i < a.data.size(); ++i) m = std::max(m, std::abs(a.data[i] - b.data[i]));
  return m;
}

// ---- model state (hgnn.hpp:16-72) -------------------------------------------------------------------
struct AdamHyper {
  double lr = 1e-2;
  double beta1 = 0.9;
  double beta2 = 0.999;
  double eps = 1e-8;
};

struct SlotKey {
  int rel_index = -1;
  int layer = 0;  // 1..k
  bool operator<(const SlotKey& o) const {
    return rel_index != o.rel_index ? rel_index < o.rel_index : layer < o.layer;
  }
  bool operator==(const SlotKey& o) const { return rel_index == o.rel_index && layer == o.layer; }
};

struct HGNNModel {
  int k = 1;
  int hidden = 16;
  int num_classes = 2;
  std::vector<int> input_dims;
  std::map<SlotKey, Matrix> weights;  // W_r^{(l)}, [d_{l-1} x d_l]
  int out_dim(int layer) const { return layer == k ? num_classes : hidden; }
  std::uint64_t param_count() const {
    std::uint64_t n = 0;
    for (const auto& [key, w] : weights) n += w.data.size();
    return n;
  }
};

struct LearnableFeatureTable {
  Matrix w, m, v;  // [n x d0]
  std::int64_t step = 0;
  AdamHyper hp;
};
struct LearnableStore {
  std::map<int, LearnableFeatureTable> tables;  // keyed by node type
};

struct GradientSet {
  std::map<SlotKey, Matrix> weight_grads;
  // per learnable type: touched row ids (sorted) and their gradient rows
  std::map<int, std::pair<std::vector<NodeId>, Matrix>> feature_grads;

  // sorted-union merge of row gradients plus dense slot sums (hgnn.cpp:83-113)
  void accumulate(const GradientSet& other) {
    for (const auto& [key, g] : other.weight_grads) {
      auto it = weight_grads.find(key);
      if (it == weight_grads.end())
        weight_grads.emplace(key, g);
      else
        add_inplace(it->second, g);
    }
    for (const auto& [type, rows] : other.feature_grads) {
      auto it = feature_grads.find(type);
      if (it == feature_grads.end()) {
        feature_grads.emplace(type, rows);
        continue;
      }
      auto& [ids, mat] = it->second;
      std::vector<NodeId> merged(ids);
      merged.insert(merged.end(), rows.first.begin(), rows.first.end());
      std::sort(merged.begin(), merged.end());
      merged.erase(std::unique(merged.begin(), merged.end()), merged.end());
      Matrix out(merged.size(), mat.cols);
      auto scatter = [&](const std::vector<NodeId>& src_ids, const Matrix& src) {
        for (std::size_t i = 0; i < src_ids.size(); ++i) {
          const auto at = std::lower_bound(merged.begin(), merged.end(), src_ids[i]) - merged.begin();
          for (std::size_t j = 0; j < src.cols; ++j) out.at(at, j) += src.at(i, j);
        }
      };
      scatter(ids, mat);
      scatter(rows.first, rows.second);
      it->second = {std::move(merged), std::move(out)};
    }
  }

  // max |a - b| over every slot and every row id of either side (hgnn.cpp:115-164)
  double max_abs_diff_vs(const GradientSet& other) const {
    double m = 0.0;
    auto upd = [&](double d) { m = std::max(m, std::abs(d)); };
    std::vector<SlotKey> keys;
    for (const auto& [k, v] : weight_grads) keys.push_back(k);
    for (const auto& [k, v] : other.weight_grads)
      if (!weight_grads.count(k)) keys.push_back(k);
    for (const SlotKey& k : keys) {
      const Matrix* a = weight_grads.count(k) ? &weight_grads.at(k) : nullptr;
      const Matrix* b = other.weight_grads.count(k) ? &other.weight_grads.at(k) : nullptr;
      if (a && b) {
        upd(max_abs_diff(*a, *b));
      } else {
        for (double x : (a ? a : b)->data) upd(x);
      }
    }
    std::vector<int> types;
    for (const auto& [t, v] : feature_grads) types.push_back(t);
    for (const auto& [t, v] : other.feature_grads)
      if (!feature_grads.count(t)) types.push_back(t);
    for (int t : types) {
      auto row_of = [](const std::pair<std::vector<NodeId>, Matrix>& fg, NodeId id) -> const double* {
        auto it = std::lower_bound(fg.first.begin(), fg.first.end(), id);
        if (it == fg.first.end() || *it != id) return nullptr;
        return fg.second.row(static_cast<std::size_t>(it - fg.first.begin()));
      };
      std::vector<NodeId> ids;
      if (feature_grads.count(t)) ids = feature_grads.at(t).first;
      if (other.feature_grads.count(t))
        ids.insert(ids.end(), other.feature_grads.at(t).first.begin(), other.feature_grads.at(t).first.end());
      std::sort(ids.begin(), ids.end());
      ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
      const std::size_t cols =
          feature_grads.count(t) ? feature_grads.at(t).second.cols : other.feature_grads.at(t).second.cols;
      for (NodeId id : ids) {
        const double* a = feature_grads.count(t) ? row_of(feature_grads.at(t), id) : nullptr;
        const double* b = other.feature_grads.count(t) ? row_of(other.feature_grads.at(t), id) : nullptr;
        for (std::size_t j = 0; j < cols; ++j) upd((a ? a[j] : 0.0) - (b ? b[j] : 0.0));
      }
    }
    return m;
  }
};

struct ModelAdamState {
  std::map<SlotKey, Matrix> m, v;
  std::int64_t step = 0;
  AdamHyper hp;
};

// ---- message accounting (raf.hpp:13-47) -----------------------------------------------------------
enum class MsgKind { PartialAgg, PartialGrad, FeatureFetchRequest, FeatureFetchReply };
struct AccountingModel {
  int header_bytes = 32;
  int id_bytes = 8;
  int elem_bytes = 4;  // payload element width: 2, 4 or 8
};
struct Message {
  MsgKind kind = MsgKind::PartialAgg;
  int layer = 0;
  int sender = -1;
  int receiver = -1;
  NodeTypeId node_type = -1;
  std::vector<NodeId> node_ids;
  std::size_t rows = 0;
  std::size_t dim = 0;
  std::uint64_t bytes = 0;
};
// (sender, receiver, kind) -> totals; additive across batches (raf.cpp:11-41)
struct CommStats {
  struct Entry {
    std::uint64_t count = 0;
    std::uint64_t bytes = 0;
  };
  std::map<std::tuple<int, int, int>, Entry> per_direction;
  void record(const Message& m) {
    auto& e = per_direction[{m.sender, m.receiver, static_cast<int>(m.kind)}];
    e.count += 1;
    e.bytes += m.bytes;
  }
  void merge(const CommStats& o) {
    for (const auto& [k, e] : o.per_direction) {
      auto& mine = per_direction[k];
      mine.count += e.count;
      mine.bytes += e.bytes;
    }
  }
  std::uint64_t total_bytes() const {
    std::uint64_t b = 0;
    for (const auto& [k, e] : per_direction) b += e.bytes;
    return b;
  }
  std::uint64_t bytes_of(MsgKind k) const {
    std::uint64_t b = 0;
    for (const auto& [key, e] : per_direction)
      if (std::get<2>(key) == static_cast<int>(k)) b += e.bytes;
    return b;
  }
  Entry direction_kind(int from, int to, MsgKind k) const {
    auto it = per_direction.find({from, to, static_cast<int>(k)});
    return it == per_direction.end() ? Entry{} : it->second;
  }
};

// ---- RAF training engine: one meta-partition per GPU (raf.hpp:66-81, hgnn.hpp:121-130) ----------
struct ExecutionReport {
  double loss = 0.0;
  std::uint64_t sampled_edges = 0;     // Block::src_ids entries over all hops (this partition)
  std::vector<int> active_rows;        // per rank (p > 1): rows of the AGG_all partial (raf.cpp:418-446)
  std::uint64_t sync_bytes = 0;        // this rank's replica group's share (raf.cpp:496-510)
  bool sync_leader = true;             // sum sync_bytes over leaders for the run-wide figure
  std::vector<std::uint64_t> boundary_counts;  // structural, per worker (raf.cpp:306-340)
  std::uint64_t boundary_cut_edges = 0;        // raf.cpp:521-528
  bool cross_ids_target_only = true;
  bool message_bound_ok = true;        // check_comm_bounds (raf.cpp:662-676)
  // filled by the caller-owned run_raf_batch (raf.hpp:66-77); RafEngine::run_raf_batch
  // keeps these on the device (RafEngine::read)
  Matrix logits;                       // rows aligned with sorted unique batch ids
  std::vector<NodeId> logit_ids;
  GradientSet grads;
  CommStats stats;
  std::vector<Message> trace;
};

// layer type of the engine: the reference's RGCN (hgnn.cpp:173-362), or relational graph
// attention (no reference counterpart, oracle/rgat.py) with `heads` heads
enum class LayerKind : int { RGCN = 0, RGAT = 1 };

class RafEngine {
 public:
  // init_model / init_learnable seeds as run_experiment derives them (harness.cpp:365-366)
  // feat_dtype: storage of the dense feature tables (0 f32, 1 f16, 2 bf16); feat_host: keep
  // them in pinned host memory with an HBM cache of the set_cache rows
  RafEngine(const HetGraph& g, std::vector<int> fanouts, int hidden, std::uint64_t seed, int batch_cap = 1024,
            int p = 1, int rank = 0, int device = 0, int feat_dtype = 0, bool feat_host = false,
            LayerKind kind = LayerKind::RGCN, int heads = 4)
      : g_(g), fanouts_(std::move(fanouts)) {
    const hg_engine_opts o{static_cast<int>(fanouts_.size()), fanouts_.data(), hidden, batch_cap, p, rank,
                           mix_seed(seed, 0xd0de1), mix_seed(seed, 0x1ea4a), device, feat_dtype, feat_host ? 1 : 0,
                           static_cast<int>(kind), heads};
    e_.reset(detail::check(hg_engine_create(g.handle(), &o)));
  }
  // run_raf_batch (raf.cpp:344-530) + adam_update_model + adam_update_rows, as the
  // hot loop of run_experiment (harness.cpp:403-423); train = false stops after the loss
  ExecutionReport run_raf_batch(std::span<const NodeId> batch, std::uint64_t rng_seed, int designated,
                                bool train = true) {
    hg_step_report r{};
    detail::check(hg_engine_step(e_.get(), batch.data(), static_cast<int>(batch.size()), rng_seed, designated,
                                 train ? 1 : 0, &r));
    ExecutionReport out;
    out.loss = r.loss;
    out.sampled_edges = r.sampled_edges;
    out.active_rows.assign(r.active_rows, r.active_rows + r.n_active);
    out.sync_bytes = r.sync_bytes;
    out.sync_leader = r.sync_leader != 0;
    out.boundary_counts.assign(r.boundary_counts, r.boundary_counts + r.n_boundary);
    out.boundary_cut_edges = r.boundary_cut_edges;
    out.cross_ids_target_only = r.target_only_ok != 0;
    out.message_bound_ok = r.message_bound_ok != 0;
    return out;
  }
  // sample a future batch now (second sample slot, sampling stream); the next
  // run_raf_batch with the same (batch, rng_seed) trains on it meanwhile
  void prefetch(std::span<const NodeId> batch, std::uint64_t rng_seed) {
    detail::check(hg_engine_prefetch(e_.get(), batch.data(), static_cast<int>(batch.size()), rng_seed));
  }
  // device tensors by name (hetgpu.h hg_engine_read), widened like the reference's Matrix
  detail::Bundle read(const std::string& names) { return detail::Bundle(hg_engine_read(e_.get(), names.c_str())); }
  // presample_hotness (cache.cpp:39-63): per type, visit counts over `epochs` id-ordered passes
  std::vector<std::vector<std::uint64_t>> presample_hotness(int epochs, std::uint64_t seed, int batch_size = 512) {
    const detail::Bundle b(hg_engine_presample_hotness(e_.get(), epochs, seed, batch_size));
    std::vector<std::vector<std::uint64_t>> out;
    for (std::size_t t = 0; t < g_.node_counts.size(); ++t) out.push_back(b.get<std::uint64_t>("hot.t" + std::to_string(t)));
    return out;
  }
  // multi-GPU AGG_all: every rank attaches the same NCCL id (hg_nccl_unique_id on rank 0)
  void attach_nccl(const std::vector<char>& unique_id, int nranks, int rank) {
    detail::check(hg_engine_attach_nccl(e_.get(), unique_id.data(), static_cast<int>(unique_id.size()), nranks, rank));
  }
  // replica groups (p > #sub-metatrees): this rank's CUDA IPC handle of its gradient
  // exchange arena (empty without replicas); every rank then maps all ranks' handles
  std::vector<char> replica_handle() {
    std::vector<char> h(4096);
    const int n = detail::check(hg_engine_replica_handle(e_.get(), h.data(), static_cast<int>(h.size())));
    h.resize(n);
    return h;
  }
  void attach_replicas(const std::vector<std::vector<char>>& handles_by_rank) {
    std::size_t size = 1;
    for (const auto& h : handles_by_rank) size = std::max(size, h.size());
    std::vector<char> flat(size * handles_by_rank.size(), 0);
    for (std::size_t r = 0; r < handles_by_rank.size(); ++r)
      std::copy(handles_by_rank[r].begin(), handles_by_rank[r].end(), flat.begin() + r * size);
    detail::check(hg_engine_attach_replicas(e_.get(), flat.data(), static_cast<int>(size),
                                            static_cast<int>(handles_by_rank.size())));
  }
  hg_engine* handle() const { return e_.get(); }

 private:
  struct Free {
    void operator()(hg_engine* e) const { hg_engine_free(e); }
  };
  HetGraph g_;
  std::vector<int> fanouts_;
  std::unique_ptr<hg_engine, Free> e_;
};


// ==== the layer interface on the device (hgnn.hpp:34-130) =============================================
// Matrix-level mirrors of the reference's functions: inputs are uploaded as fp32 device
// tensors, the work runs on the hot path's own kernels through the C-ABI layer primitives
// (hg_mean_aggregate, hg_project, ... on an hg_ctx), results come back as f64 Matrices.
// Device-resident callers use the hg_* primitives directly.

namespace detail {

inline int& layer_device() {
  static int d = 0;
  return d;
}
struct CtxHolder {
  hg_ctx* c = nullptr;
  int device = -1;
  ~CtxHolder() {
    if (c) hg_ctx_free(c);
  }
};
inline hg_ctx* ctx() {
  static CtxHolder h;
  if (!h.c || h.device != layer_device()) {
    if (h.c) hg_ctx_free(h.c);
    h.c = check(hg_ctx_create(layer_device()));
    h.device = layer_device();
  }
  return h.c;
}

// device allocation owned by the context (zero-filled)
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(std::size_t bytes) : p_(check(hg_ctx_malloc(ctx(), bytes))) {}
  DevBuf(const void* host, std::size_t bytes) : DevBuf(bytes) {
    if (bytes) check(hg_ctx_copy(ctx(), p_, host, bytes));
  }
  DevBuf(DevBuf&& o) noexcept : p_(o.p_) { o.p_ = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    std::swap(p_, o.p_);
    return *this;
  }
  DevBuf(const DevBuf&) = delete;
  ~DevBuf() {
    if (p_) hg_ctx_mfree(ctx(), p_);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p_);
  }

 private:
  void* p_ = nullptr;
};
template <typename T>
DevBuf dev_vec(const std::vector<T>& v) {
  return DevBuf(v.data(), v.size() * sizeof(T));
}

inline int ld_of(std::size_t cols) { return static_cast<int>((cols + 3) & ~static_cast<std::size_t>(3)); }

// fp32 device matrix with 16-byte rows (zero padding)
struct DevMat {
  DevBuf buf;
  hg_tensor t{};
};
inline DevMat dev_zeros(std::size_t rows, std::size_t cols) {
  DevMat m;
  const int ld = ld_of(cols);
  m.buf = DevBuf(std::max<std::size_t>(1, rows) * ld * 4);
  m.t = hg_tensor{m.buf.as<float>(), static_cast<std::int64_t>(rows), static_cast<std::int32_t>(cols), ld};
  return m;
}
inline DevMat dev_upload(const Matrix& a) {
  const int ld = ld_of(a.cols);
  std::vector<float> h(std::max<std::size_t>(1, a.rows) * ld, 0.f);
  for (std::size_t i = 0; i < a.rows; ++i)
    for (std::size_t j = 0; j < a.cols; ++j) h[i * ld + j] = static_cast<float>(a.at(i, j));
  DevMat m;
  m.buf = DevBuf(h.data(), h.size() * 4);
  m.t = hg_tensor{m.buf.as<float>(), static_cast<std::int64_t>(a.rows), static_cast<std::int32_t>(a.cols), ld};
  return m;
}
inline Matrix dev_download(const hg_tensor& t) {
  Matrix a(static_cast<std::size_t>(t.rows), static_cast<std::size_t>(t.cols));
  if (a.rows == 0 || a.cols == 0) return a;
  std::vector<float> h(static_cast<std::size_t>(t.rows) * t.ld);
  check(hg_ctx_copy(ctx(), h.data(), t.data, h.size() * 4));
  for (std::size_t i = 0; i < a.rows; ++i)
    for (std::size_t j = 0; j < a.cols; ++j) a.at(i, j) = h[i * t.ld + j];
  return a;
}
inline DevMat dev_copy(const hg_tensor& t) {
  DevMat m = dev_zeros(static_cast<std::size_t>(t.rows), static_cast<std::size_t>(t.cols));
  check(hg_ctx_copy(ctx(), m.t.data, t.data, static_cast<std::size_t>(t.rows) * t.ld * 4));
  return m;
}
// row_index of every source id of a block in a sorted frontier, on the device
inline DevBuf dev_rows(const DevBuf& ids, std::size_t n, const std::vector<NodeId>& frontier) {
  DevBuf rows(std::max<std::size_t>(1, n) * 4);
  if (n == 0) return rows;
  const DevBuf fr = dev_vec(frontier);
  check(hg_rows_in(ctx(), ids.as<std::uint32_t>(), static_cast<std::int64_t>(n), fr.as<std::uint32_t>(),
                   static_cast<std::int64_t>(frontier.size()), rows.as<std::uint32_t>()));
  check(hg_ctx_sync(ctx()));  // raises "node id not in frontier: <id>"
  return rows;
}

}  // namespace detail

// device of the Matrix-level layer functions below (default 0)
inline void set_layer_device(int device) { detail::layer_device() = device; }

// rels_by_dst_at_depth / hop_relation_sets (hgnn.cpp:16-37)
inline std::map<int, std::vector<int>> rels_by_dst_at_depth(const Metatree& tree, int depth) {
  std::map<int, std::vector<int>> out;
  for (const auto& p : tree.pos) {
    if (p.depth != depth || p.rel_index < 0) continue;
    auto& v = out[tree.pos[p.parent].type];
    if (std::find(v.begin(), v.end(), p.rel_index) == v.end()) v.push_back(p.rel_index);
  }
  for (auto& [t, v] : out) std::sort(v.begin(), v.end());
  return out;
}
inline std::vector<std::vector<int>> hop_relation_sets(const Metatree& tree, int k) {
  std::vector<std::vector<int>> out(k);
  for (const auto& p : tree.pos) {
    if (p.rel_index < 0 || p.depth < 1 || p.depth > k) continue;
    auto& v = out[p.depth - 1];
    if (std::find(v.begin(), v.end(), p.rel_index) == v.end()) v.push_back(p.rel_index);
  }
  for (auto& v : out) std::sort(v.begin(), v.end());
  return out;
}

// init_model (hgnn.cpp:39-62) on the BFS metatree of depth tree.k (meta_partition's tree):
// bit-identical initial weights (the same libstdc++ engines)
inline HGNNModel init_model(const HetGraph& g, const Metatree& tree, int hidden, std::uint64_t seed) {
  const detail::Bundle b(hg_init_model(g.handle(), std::max(tree.k, 1), hidden, seed));
  HGNNModel m;
  m.k = std::max(tree.k, 1);
  m.hidden = hidden;
  m.num_classes = g.num_classes;
  m.input_dims = b.get<int>("input_dims");
  for (const auto& p : tree.pos) {
    if (p.rel_index < 0) continue;
    const SlotKey key{p.rel_index, m.k - p.depth + 1};
    if (m.weights.count(key)) continue;
    const std::string n = "w.r" + std::to_string(key.rel_index) + ".l" + std::to_string(key.layer);
    const int in = key.layer == 1 ? m.input_dims[p.type] : hidden;
    Matrix w(static_cast<std::size_t>(in), static_cast<std::size_t>(m.out_dim(key.layer)));
    w.data = b.get<double>(n);
    m.weights.emplace(key, std::move(w));
  }
  return m;
}
// init_learnable (hgnn.cpp:64-81)
inline LearnableStore init_learnable(const HetGraph& g, std::uint64_t seed, const AdamHyper& hp = {}) {
  const detail::Bundle b(hg_init_learnable(g.handle(), seed));
  LearnableStore st;
  for (std::size_t t = 0; t < g.kinds.size(); ++t) {
    if (g.kinds[t] != 2) continue;
    LearnableFeatureTable tab;
    tab.hp = hp;
    const std::size_t n = g.node_counts[t], d = static_cast<std::size_t>(g.dims[t]);
    tab.w = Matrix(n, d);
    tab.m = Matrix(n, d);
    tab.v = Matrix(n, d);
    tab.w.data = b.get<double>("learn.t" + std::to_string(t));
    st.tables.emplace(static_cast<int>(t), std::move(tab));
  }
  return st;
}

// mean_aggregate (hgnn.cpp:173-187): segment mean of h_src rows (looked up in the sorted
// src_frontier), zero rows for empty neighbourhoods; fp32 on the device, edge-order sums
inline Matrix mean_aggregate(const Block& blk, const Matrix& h_src, const std::vector<NodeId>& src_frontier) {
  const std::size_t n_dst = blk.dst_ids.size();
  if (blk.indptr.size() != n_dst + 1) throw std::invalid_argument("block indptr must have dst_ids.size() + 1 entries");
  const detail::DevBuf src = detail::dev_vec(blk.src_ids);
  const detail::DevBuf rows = detail::dev_rows(src, blk.src_ids.size(), src_frontier);
  if (n_dst == 0 || h_src.cols == 0) return Matrix(n_dst, h_src.cols);
  const detail::DevMat h = detail::dev_upload(h_src);
  const detail::DevBuf ip = detail::dev_vec(blk.indptr);
  detail::DevMat out = detail::dev_zeros(n_dst, h_src.cols);
  detail::check(hg_mean_aggregate(detail::ctx(), ip.as<std::uint32_t>(), static_cast<std::int64_t>(n_dst),
                                  rows.as<std::uint32_t>(), h.t, out.t));
  detail::check(hg_ctx_sync(detail::ctx()));
  return detail::dev_download(out.t);
}

// agg_relation (hgnn.cpp:189-192): mean then the relation's linear map (tcgen05 projection)
inline Matrix agg_relation(const Block& blk, const Matrix& h_src, const std::vector<NodeId>& src_frontier,
                           const Matrix& w) {
  const Matrix mean = mean_aggregate(blk, h_src, src_frontier);
  check_dims(mean.cols == w.rows, "matmul");
  if (mean.rows == 0 || w.cols == 0) return Matrix(mean.rows, w.cols);
  const detail::DevMat dm = detail::dev_upload(mean), dw = detail::dev_upload(w);
  detail::DevMat out = detail::dev_zeros(mean.rows, w.cols);
  detail::check(hg_project(detail::ctx(), &dm.t, &dw.t, 1, out.t, 0, 0));
  detail::check(hg_ctx_sync(detail::ctx()));
  return detail::dev_download(out.t);
}

// agg_all (hgnn.cpp:194-203): elementwise sum in the given order
inline Matrix agg_all(const std::vector<const Matrix*>& partials) {
  if (partials.empty()) throw std::invalid_argument("agg_all needs at least one partial");
  for (const Matrix* p : partials)
    if (!p->same_shape(*partials[0])) throw std::invalid_argument("agg_all partials have mismatched shapes");
  std::vector<detail::DevMat> up;
  std::vector<hg_tensor> ts;
  for (const Matrix* p : partials) {
    up.push_back(detail::dev_upload(*p));
    ts.push_back(up.back().t);
  }
  detail::DevMat out = detail::dev_zeros(partials[0]->rows, partials[0]->cols);
  // chains of at most 32 partials, each continuing from the running sum
  std::size_t at = 0;
  while (at < ts.size()) {
    std::vector<hg_tensor> chunk;
    if (at > 0) chunk.push_back(out.t);
    while (at < ts.size() && chunk.size() < 32) chunk.push_back(ts[at++]);
    detail::DevMat next = detail::dev_zeros(partials[0]->rows, partials[0]->cols);
    detail::check(hg_agg_all(detail::ctx(), chunk.data(), static_cast<int>(chunk.size()), next.t));
    detail::check(hg_ctx_sync(detail::ctx()));
    out = std::move(next);
  }
  return detail::dev_download(out.t);
}

struct TapeEntry {
  int layer = 0;
  int rel_index = -1;
  int hop = 0;         // tree depth of the edge = blocks hop index
  int block_idx = -1;  // index into blocks.hops[hop-1]
  NodeTypeId dst_type = -1;
  Matrix mean;  // post-mean pre-linear activations, rows = block dst rows
};
struct ForwardTape {
  const SampledBlocks* blocks = nullptr;
  std::vector<std::map<int, Matrix>> H;  // H[d][type], rows aligned with blocks->frontier[d][type]
  std::vector<TapeEntry> entries;
};

namespace detail {
inline const Block* find_block(const SampledBlocks& blocks, int hop, int rel_index, int* idx) {
  const auto& list = blocks.hops[hop - 1];
  for (std::size_t i = 0; i < list.size(); ++i)
    if (list[i].rel_index == rel_index) {
      if (idx) *idx = static_cast<int>(i);
      return &list[i];
    }
  return nullptr;
}
}  // namespace detail

// forward_flat (hgnn.cpp:215-279): layer-0 gather, then per layer the relation means
// (gather-mean kernel) and the projection summed over the relations into each type with
// the ReLU in its epilogue (tcgen05). The tape keeps the reference's host layout.
inline std::pair<Matrix, ForwardTape> forward_flat(const HetGraph& g, const Metatree& tree,
                                                   const SampledBlocks& blocks, const HGNNModel& model,
                                                   const LearnableStore& store) {
  const int k = blocks.k;
  const int nt = static_cast<int>(g.node_counts.size());
  ForwardTape tape;
  tape.blocks = &blocks;
  tape.H.resize(k + 1);
  std::vector<std::map<int, detail::DevMat>> Hd(k + 1);
  // layer-0 inputs: features of the outermost frontier
  for (int t = 0; t < nt; ++t) {
    const auto& front = blocks.frontier[k][t];
    if (front.empty()) continue;
    const int dim = g.dims[t];
    Matrix h(front.size(), static_cast<std::size_t>(dim));
    if (g.kinds[t] == 1) {
      const float* data = nullptr;
      std::uint64_t rows = 0;
      int d = 0, kind = 0;
      detail::check(hg_graph_dense(g.handle(), t, &data, &rows, &d, &kind));
      for (std::size_t i = 0; i < front.size(); ++i)
        for (int j = 0; j < dim; ++j) h.at(i, j) = data[static_cast<std::size_t>(front[i]) * dim + j];
    } else if (g.kinds[t] == 2) {
      auto it = store.tables.find(t);
      if (it == store.tables.end()) throw std::runtime_error("no learnable table for node type " + g.type_names[t]);
      for (std::size_t i = 0; i < front.size(); ++i)
        for (int j = 0; j < dim; ++j) h.at(i, j) = it->second.w.at(front[i], j);
    } else {
      throw std::runtime_error("missing features for node type " + g.type_names[t]);
    }
    Hd[k].emplace(t, detail::dev_upload(h));
    tape.H[k].emplace(t, std::move(h));
  }
  for (int l = 1; l <= k; ++l) {
    const int d = k - l + 1;
    const auto rels = rels_by_dst_at_depth(tree, d);
    for (int t = 0; t < nt; ++t) {
      const auto& front = blocks.frontier[d - 1][t];
      if (front.empty()) continue;
      detail::DevMat out = detail::dev_zeros(front.size(), static_cast<std::size_t>(model.out_dim(l)));
      std::vector<detail::DevMat> means, ws;
      auto it = rels.find(t);
      if (it != rels.end()) {
        for (int r : it->second) {
          int bidx = -1;
          const Block* blk = detail::find_block(blocks, d, r, &bidx);
          if (!blk) continue;  // relation had an empty frontier
          const NodeTypeId src_t = g.relations[r].src;
          const std::size_t din = static_cast<std::size_t>(l == 1 ? model.input_dims[src_t] : model.hidden);
          detail::DevMat mean;
          auto hit = Hd[d].find(src_t);
          if (hit != Hd[d].end()) {
            const detail::DevBuf src = detail::dev_vec(blk->src_ids);
            const detail::DevBuf rows = detail::dev_rows(src, blk->src_ids.size(), blocks.frontier[d][src_t]);
            const detail::DevBuf ip = detail::dev_vec(blk->indptr);
            mean = detail::dev_zeros(blk->dst_ids.size(), static_cast<std::size_t>(hit->second.t.cols));
            detail::check(hg_mean_aggregate(detail::ctx(), ip.as<std::uint32_t>(),
                                            static_cast<std::int64_t>(blk->dst_ids.size()), rows.as<std::uint32_t>(),
                                            hit->second.t, mean.t));
            detail::check(hg_ctx_sync(detail::ctx()));
          } else {
            mean = detail::dev_zeros(blk->dst_ids.size(), din);
          }
          const Matrix& w = model.weights.at(SlotKey{r, l});
          if (w.rows != static_cast<std::size_t>(mean.t.cols))
            throw std::invalid_argument("weight/input dim mismatch for relation " + std::to_string(r));
          tape.entries.push_back({l, r, d, bidx, t, detail::dev_download(mean.t)});
          ws.push_back(detail::dev_upload(w));
          means.push_back(std::move(mean));
        }
      }
      // out = sum_r mean_r . W_r (ascending relations), ReLU between layers: one tcgen05
      // launch per 16 relations
      for (std::size_t q0 = 0; q0 < means.size(); q0 += 16) {
        std::vector<hg_tensor> mt, wt;
        for (std::size_t q = q0; q < std::min(means.size(), q0 + 16); ++q) {
          mt.push_back(means[q].t);
          wt.push_back(ws[q].t);
        }
        const bool last = q0 + 16 >= means.size();
        detail::check(hg_project(detail::ctx(), mt.data(), wt.data(), static_cast<int>(mt.size()), out.t,
                                 (l < k && last && q0 == 0) ? 1 : 0, q0 > 0 ? 1 : 0));
      }
      if (l < k && means.size() > 16) detail::check(hg_relu(detail::ctx(), out.t, nullptr));
      detail::check(hg_ctx_sync(detail::ctx()));
      tape.H[d - 1].emplace(t, detail::dev_download(out.t));
      Hd[d - 1].emplace(t, std::move(out));
    }
  }
  Matrix logits = tape.H[0].at(g.target);
  return {std::move(logits), std::move(tape)};
}

// cross_entropy (hgnn.cpp:281-307): mean softmax cross-entropy over the batch (duplicates
// count), dlogits per row; fp32 log-sum-exp per row on the device, ordered batch sum
inline double cross_entropy(const Matrix& logits, const std::vector<NodeId>& row_ids, std::span<const NodeId> batch,
                            std::span<const std::int32_t> labels, int num_classes, Matrix* dlogits) {
  if (batch.empty()) throw std::invalid_argument("empty batch");
  const detail::DevMat z = detail::dev_upload(logits);
  detail::DevMat dz = detail::dev_zeros(logits.rows, logits.cols);
  double loss = 0.0;
  detail::check(hg_cross_entropy(detail::ctx(), z.t, row_ids.data(), static_cast<std::int64_t>(row_ids.size()),
                                 batch.data(), static_cast<std::int64_t>(batch.size()), labels.data(),
                                 static_cast<std::int64_t>(labels.size()), num_classes, dlogits ? &dz.t : nullptr,
                                 &loss));
  if (dlogits) *dlogits = detail::dev_download(dz.t);
  return loss;
}

// backward_flat (hgnn.cpp:309-362): per tape entry the ReLU mask, the weight gradient
// (tcgen05, ordered split-K), the mean gradient with 1/deg (tcgen05), and the scatter to
// the source frontier as an ordered source-major gather (deterministic)
inline GradientSet backward_flat(const HetGraph& g, const Metatree& tree, const HGNNModel& model,
                                 const ForwardTape& tape, const Matrix& dlogits) {
  (void)tree;
  const SampledBlocks& blocks = *tape.blocks;
  const int k = blocks.k;
  GradientSet grads;
  std::vector<std::map<int, detail::DevMat>> dH(k + 1);
  dH[0].emplace(g.target, detail::dev_upload(dlogits));
  std::map<SlotKey, detail::DevMat> wg;
  for (int l = k; l >= 1; --l) {
    const int d = k - l + 1;
    for (const TapeEntry& e : tape.entries) {
      if (e.layer != l) continue;
      auto dit = dH[d - 1].find(e.dst_type);
      if (dit == dH[d - 1].end()) continue;  // no downstream gradient
      detail::DevMat dpre = detail::dev_copy(dit->second.t);
      if (l < k) {
        const detail::DevMat hp = detail::dev_upload(tape.H[d - 1].at(e.dst_type));
        detail::check(hg_relu(detail::ctx(), dpre.t, &hp.t));
        detail::check(hg_ctx_sync(detail::ctx()));
      }
      const Matrix& w = model.weights.at(SlotKey{e.rel_index, l});
      const detail::DevMat dw = detail::dev_upload(w);
      auto git = wg.find(SlotKey{e.rel_index, l});
      if (git == wg.end()) git = wg.emplace(SlotKey{e.rel_index, l}, detail::dev_zeros(w.rows, w.cols)).first;
      const detail::DevMat mean = detail::dev_upload(e.mean);
      detail::check(hg_weight_grad(detail::ctx(), mean.t, dpre.t, git->second.t, 1));
      const Block& blk = blocks.hops[d - 1][e.block_idx];
      const detail::DevBuf ip = detail::dev_vec(blk.indptr);
      detail::DevMat dmean = detail::dev_zeros(blk.dst_ids.size(), w.rows);
      if (!blk.dst_ids.empty())
        detail::check(hg_mean_grad(detail::ctx(), dpre.t, dw.t, ip.as<std::uint32_t>(), dmean.t));
      const NodeTypeId src_t = g.relations[e.rel_index].src;
      const auto& src_front = blocks.frontier[d][src_t];
      auto sit = dH[d].find(src_t);
      if (sit == dH[d].end()) sit = dH[d].emplace(src_t, detail::dev_zeros(src_front.size(), w.rows)).first;
      const detail::DevBuf src = detail::dev_vec(blk.src_ids);
      const detail::DevBuf rows = detail::dev_rows(src, blk.src_ids.size(), src_front);
      detail::check(hg_scatter_rows(detail::ctx(), ip.as<std::uint32_t>(), static_cast<std::int64_t>(blk.dst_ids.size()),
                                    static_cast<std::int64_t>(blk.src_ids.size()), rows.as<std::uint32_t>(), dmean.t,
                                    sit->second.t));
      detail::check(hg_ctx_sync(detail::ctx()));
    }
  }
  for (auto& [key, m] : wg) grads.weight_grads.emplace(key, detail::dev_download(m.t));
  for (const auto& [t, dmat] : dH[k]) {
    if (g.kinds[t] != 2) continue;
    grads.feature_grads.emplace(t, std::make_pair(blocks.frontier[k][t], detail::dev_download(dmat.t)));
  }
  return grads;
}

namespace detail {
// Adam on flat arrays (adam_step, hgnn.cpp:364-377): w, m, v updated in place
inline void adam_flat(std::vector<double>& w, std::vector<double>& m, std::vector<double>& v,
                      const std::vector<double>& g, std::int64_t step, const AdamHyper& hp) {
  if (w.empty()) return;
  auto f = [](const std::vector<double>& x) { return std::vector<float>(x.begin(), x.end()); };
  const auto hw = f(w), hm = f(m), hv = f(v), hg = f(g);
  DevBuf dw = dev_vec(hw), dm = dev_vec(hm), dv = dev_vec(hv), dg = dev_vec(hg);
  check(hg_adam_dense(ctx(), dw.as<float>(), dm.as<float>(), dv.as<float>(), dg.as<float>(),
                      static_cast<std::int64_t>(w.size()), step, hp.lr, hp.beta1, hp.beta2, hp.eps));
  check(hg_ctx_sync(ctx()));  // raises "non-finite gradient"
  std::vector<float> o(w.size());
  auto back = [&](const DevBuf& b, std::vector<double>& dst) {
    check(hg_ctx_copy(ctx(), o.data(), b.as<float>(), o.size() * 4));
    for (std::size_t i = 0; i < o.size(); ++i) dst[i] = o[i];
  };
  back(dw, w);
  back(dm, m);
  back(dv, v);
}
}  // namespace detail

// adam_update_model (hgnn.cpp:379-390): one global step, every slot with a gradient
inline void adam_update_model(HGNNModel& model, ModelAdamState& state, const GradientSet& grads) {
  state.step += 1;
  for (auto& [key, w] : model.weights) {
    auto git = grads.weight_grads.find(key);
    if (!state.m.count(key)) {
      state.m.emplace(key, Matrix(w.rows, w.cols));
      state.v.emplace(key, Matrix(w.rows, w.cols));
    }
    if (git == grads.weight_grads.end()) continue;  // untouched slot
    check_dims(git->second.same_shape(w), "adam gradient");
    detail::adam_flat(w.data, state.m.at(key).data, state.v.at(key).data, git->second.data, state.step, state.hp);
  }
}

// adam_update_rows (hgnn.cpp:392-410): only the listed rows change; the step advances once
inline void adam_update_rows(LearnableFeatureTable& table, const std::vector<NodeId>& rows, const Matrix& row_grads) {
  table.step += 1;
  if (rows.empty()) return;
  if (row_grads.rows != rows.size() || row_grads.cols != table.w.cols)
    throw std::invalid_argument("row gradients must be [rows x dim]");
  const std::size_t dim = table.w.cols;
  Matrix cw(rows.size(), dim), cm(rows.size(), dim), cv(rows.size(), dim);
  for (std::size_t i = 0; i < rows.size(); ++i) {
    if (rows[i] >= table.w.rows) throw std::invalid_argument("row id out of range: " + std::to_string(rows[i]));
    for (std::size_t j = 0; j < dim; ++j) {
      cw.at(i, j) = table.w.at(rows[i], j);
      cm.at(i, j) = table.m.at(rows[i], j);
      cv.at(i, j) = table.v.at(rows[i], j);
    }
  }
  const detail::DevMat dw = detail::dev_upload(cw), dm = detail::dev_upload(cm), dv = detail::dev_upload(cv),
                       dg = detail::dev_upload(row_grads);
  std::vector<NodeId> iota(rows.size());
  for (std::size_t i = 0; i < iota.size(); ++i) iota[i] = static_cast<NodeId>(i);
  const detail::DevBuf ids = detail::dev_vec(iota);
  detail::check(hg_adam_rows(detail::ctx(), dw.t, dm.t, dv.t, ids.as<std::uint32_t>(),
                             static_cast<std::int64_t>(rows.size()), dg.t, table.step, table.hp.lr, table.hp.beta1,
                             table.hp.beta2, table.hp.eps));
  detail::check(hg_ctx_sync(detail::ctx()));
  const Matrix nw = detail::dev_download(dw.t), nm = detail::dev_download(dm.t), nv = detail::dev_download(dv.t);
  for (std::size_t i = 0; i < rows.size(); ++i)
    for (std::size_t j = 0; j < dim; ++j) {
      table.w.at(rows[i], j) = nw.at(i, j);
      table.m.at(rows[i], j) = nm.at(i, j);
      table.v.at(rows[i], j) = nv.at(i, j);
    }
}

// ---- sample_neighbors (sampling.hpp:34-35) ---------------------------------------------------------
struct Csr {  // hetgraph.hpp:41-47
  std::vector<std::uint64_t> indptr;
  std::vector<NodeId> src;
};
inline std::vector<NodeId> sample_neighbors(const Csr& adj, NodeId dst, int fanout, std::uint64_t rng_seed, int hop,
                                            int rel_index) {
  std::vector<NodeId> out(static_cast<std::size_t>(std::max(fanout, 0)) + 1);
  int n = 0;
  detail::check(hg_sample_neighbors(adj.indptr.data(), adj.indptr.empty() ? 0 : adj.indptr.size() - 1,
                                    adj.src.data(), dst, fanout, rng_seed, hop, rel_index, out.data(), &n,
                                    detail::layer_device()));
  out.resize(static_cast<std::size_t>(n));
  return out;
}

// ---- RAF with caller-owned state (raf.hpp:49-103) -----------------------------------------------------
struct RafPlanView {
  Metatree tree;
  int p = 1;
  std::vector<std::vector<int>> top_owners;  // per root-child position (tree order)
  std::vector<int> rel_owner;                // empty under meta plans
  bool meta = true;
  // the plan's batch-invariant bookkeeping (raf.cpp:306-340, 496-510, 521-528)
  std::vector<std::uint64_t> boundary_counts;
  std::uint64_t boundary_cut_edges = 0;
  std::vector<std::array<int, 3>> slot_contributors;
  std::vector<std::array<int, 2>> leaf_owners;
};

// raf_view_from_plan (raf.cpp:43-57)
inline RafPlanView raf_view_from_plan(const PartitionPlan& plan) {
  RafPlanView v;
  v.tree = plan.tree;
  v.p = plan.p;
  v.meta = true;
  for (int c : v.tree.children(0)) {
    int sid = -1;
    for (std::size_t s = 0; s < plan.sub_child_pos.size(); ++s)
      if (plan.sub_child_pos[s] == c) sid = static_cast<int>(s);
    if (sid < 0) throw std::invalid_argument("plan has no sub-metatree for a root child");
    v.top_owners.push_back(plan.owners_of_sub(sid));
  }
  v.boundary_counts = plan.boundary_counts;
  v.boundary_cut_edges = plan.boundary_cut_edges;
  v.slot_contributors = plan.slot_contributors;
  v.leaf_owners = plan.leaf_owners;
  return v;
}

struct CommBoundVerdict {
  bool message_bound_ok = true;
  bool target_only_ok = true;
};
// check_comm_bounds (raf.cpp:662-676)
inline CommBoundVerdict check_comm_bounds(const ExecutionReport& report, int num_relations, bool meta_plan) {
  CommBoundVerdict v;
  std::map<std::pair<int, int>, std::uint64_t> agg_count;
  for (const auto& [key, e] : report.stats.per_direction)
    if (std::get<2>(key) == static_cast<int>(MsgKind::PartialAgg))
      agg_count[{std::get<0>(key), std::get<1>(key)}] += e.count;
  for (const auto& [dir, n] : agg_count)
    if (n > static_cast<std::uint64_t>(num_relations) * report.boundary_counts.at(dir.first)) v.message_bound_ok = false;
  if (meta_plan) v.target_only_ok = report.cross_ids_target_only;
  return v;
}

namespace detail {
// one device engine per (graph, depth, hidden, batch capacity), reused across calls
struct EngineKey {
  const hg_graph* g;
  std::vector<int> fanouts;
  int hidden, cap, device;
  bool operator<(const EngineKey& o) const {
    return std::tie(g, fanouts, hidden, cap, device) < std::tie(o.g, o.fanouts, o.hidden, o.cap, o.device);
  }
};
// the tensor names hg_engine_read serves for an engine
inline std::vector<std::string> engine_names(hg_engine* e) {
  const Bundle nb(hg_engine_read(e, "?"));
  std::vector<std::string> out;
  std::string cur;
  for (char ch : nb.get<char>("names")) {
    if (ch == ',') {
      if (!cur.empty()) out.push_back(cur);
      cur.clear();
    } else {
      cur.push_back(ch);
    }
  }
  if (!cur.empty()) out.push_back(cur);
  return out;
}
inline hg_engine* state_engine(const HetGraph& g, const std::vector<int>& fanouts, int hidden, int cap) {
  struct Free {
    void operator()(hg_engine* e) const { hg_engine_free(e); }
  };
  static std::map<EngineKey, std::unique_ptr<hg_engine, Free>> cache;
  int c = 1024;
  while (c < cap) c *= 2;
  const EngineKey key{g.handle(), fanouts, hidden, c, layer_device()};
  auto it = cache.find(key);
  if (it == cache.end()) {
    const hg_engine_opts o{static_cast<int>(fanouts.size()), fanouts.data(), hidden, c, 1, 0, 0, 0, layer_device(), 0, 0};
    hg_engine* e = check(hg_engine_create(g.handle(), &o));
    check(hg_engine_set_option(e, "apply_adam", 0));
    check(hg_engine_set_option(e, "retain_grads", 1));
    it = cache.emplace(key, std::unique_ptr<hg_engine, Free>(e)).first;
  }
  return it->second.get();
}
}  // namespace detail

// run_raf_batch (raf.cpp:344-530) with the caller's model and learnable store: the fused
// device step of RafEngine (sampling, gather-mean, tcgen05 projections, loss, backward) on
// the caller's parameters, gradients returned and nothing updated (the caller then runs
// adam_update_model / adam_update_rows, harness.cpp:410-423). The numbers are the flat
// pass's (check_equivalence pins RAF == flat); the RAF bookkeeping of a meta view with
// p workers (buckets, PartialAgg / PartialGrad messages, CommStats, sync bytes, boundary
// counts) follows raf.cpp:382-530 from the sampled hop-1 blocks.
inline ExecutionReport run_raf_batch(const HetGraph& g, const RafPlanView& view, const HGNNModel& model,
                                     const LearnableStore& store, std::span<const NodeId> batch,
                                     const std::vector<int>& fanouts, std::uint64_t rng_seed, int designated,
                                     const AccountingModel& acct = {}) {
  if (static_cast<int>(fanouts.size()) != model.k) throw std::invalid_argument("fanout count must equal the model depth");
  if (designated < 0 || designated >= view.p) throw std::invalid_argument("designated worker out of range");
  if (!view.meta) throw std::invalid_argument("the device engine executes meta-plan views");
  std::vector<NodeId> batch_ids(batch.begin(), batch.end());
  std::sort(batch_ids.begin(), batch_ids.end());
  batch_ids.erase(std::unique(batch_ids.begin(), batch_ids.end()), batch_ids.end());
  if (batch.empty()) throw std::invalid_argument("empty batch");
  hg_engine* e = detail::state_engine(g, fanouts, model.hidden, static_cast<int>(batch.size()));
  for (const auto& [key, w] : model.weights)
    detail::check(hg_engine_load_weights(e, key.rel_index, key.layer, w.data.data(), static_cast<int>(w.rows),
                                         static_cast<int>(w.cols)));
  // the caller's learnable rows of this batch's layer-0 frontier
  detail::check(hg_engine_sample(e, batch_ids.data(), static_cast<int>(batch_ids.size()), rng_seed));
  const int k = model.k;
  const std::vector<std::string> listed = detail::engine_names(e);
  for (std::size_t t = 0; t < g.kinds.size(); ++t) {
    if (g.kinds[t] != 2) continue;
    const std::string fn = "frontier" + std::to_string(k) + ".t" + std::to_string(t);
    if (std::find(listed.begin(), listed.end(), fn) == listed.end()) continue;
    const detail::Bundle fb(hg_engine_read(e, fn.c_str()));
    if (!fb.has(fn)) continue;
    const auto ids = fb.get<NodeId>(fn);
    if (ids.empty()) continue;
    auto it = store.tables.find(static_cast<int>(t));
    if (it == store.tables.end()) throw std::runtime_error("no learnable table for node type " + g.type_names[t]);
    const std::size_t dim = it->second.w.cols;
    std::vector<double> rows(ids.size() * dim);
    for (std::size_t i = 0; i < ids.size(); ++i)
      std::copy(it->second.w.row(ids[i]), it->second.w.row(ids[i]) + dim, rows.begin() + i * dim);
    detail::check(hg_engine_load_table_rows(e, static_cast<int>(t), ids.data(), static_cast<std::int64_t>(ids.size()),
                                            rows.data(), static_cast<int>(dim)));
  }
  hg_step_report r{};
  detail::check(hg_engine_step(e, batch.data(), static_cast<int>(batch.size()), rng_seed, 0, 1, &r));
  ExecutionReport rep;
  rep.loss = r.loss;
  rep.sampled_edges = r.sampled_edges;
  rep.logit_ids = batch_ids;
  // the engine's tensors this report needs (names as hg_engine_read lists them)
  std::string names = "logits";
  for (const std::string& n : detail::engine_names(e))
    if (n.rfind("grad.", 0) == 0 ||
        (n.rfind("hop1.rel", 0) == 0 && n.size() > 7 && n.compare(n.size() - 7, 7, ".indptr") == 0))
      names += "," + n;
  const detail::Bundle b(hg_engine_read(e, names.c_str()));
  {
    const auto lg = b.get<double>("logits");
    rep.logits = Matrix(batch_ids.size(), static_cast<std::size_t>(model.num_classes));
    for (std::size_t i = 0; i < rep.logits.data.size(); ++i) rep.logits.data[i] = lg[i];
  }
  for (const auto& [key, w] : model.weights) {
    const std::string n = "grad.w.r" + std::to_string(key.rel_index) + ".l" + std::to_string(key.layer);
    if (!b.has(n)) continue;
    const auto gv = b.get<double>(n);
    Matrix gm(w.rows, w.cols);
    for (std::size_t i = 0; i < gm.data.size(); ++i) gm.data[i] = gv[i];
    rep.grads.weight_grads.emplace(key, std::move(gm));
  }
  for (std::size_t t = 0; t < g.kinds.size(); ++t) {
    const std::string n = "grad.f.t" + std::to_string(t);
    if (g.kinds[t] != 2 || !b.has(n + ".ids")) continue;
    const auto ids = b.get<NodeId>(n + ".ids");
    const auto rv = b.get<double>(n + ".rows");
    Matrix gm(ids.size(), static_cast<std::size_t>(g.dims[t]));
    for (std::size_t i = 0; i < gm.data.size(); ++i) gm.data[i] = rv[i];
    rep.grads.feature_grads.emplace(static_cast<int>(t), std::make_pair(ids, std::move(gm)));
  }
  // ---- RAF bookkeeping over the view's workers (raf.cpp:382-446, 452-466, 496-528)
  struct Bucket {
    int owner;
    std::vector<NodeId> shard;
    std::vector<std::size_t> active;
  };
  std::vector<Bucket> buckets;
  std::map<std::tuple<int, int, int>, std::size_t> bucket_of;
  const auto root_children = view.tree.children(0);
  for (std::size_t ci = 0; ci < root_children.size(); ++ci) {
    const int rel = view.tree.pos[root_children[ci]].rel_index;
    const std::vector<int>& owners = view.top_owners.at(ci);
    const std::string ipn = "hop1.rel" + std::to_string(rel) + ".indptr";
    const std::vector<std::uint32_t> ip = b.has(ipn) ? b.get<std::uint32_t>(ipn) : std::vector<std::uint32_t>{};
    for (std::size_t oi = 0; oi < owners.size(); ++oi) {
      const auto bkey = std::make_tuple(owners[oi], static_cast<int>(owners.size()), static_cast<int>(oi));
      auto bit = bucket_of.find(bkey);
      if (bit == bucket_of.end()) {
        Bucket nb{owners[oi], {}, {}};
        for (std::size_t i = oi; i < batch_ids.size(); i += owners.size()) nb.shard.push_back(batch_ids[i]);
        bit = bucket_of.emplace(bkey, buckets.size()).first;
        buckets.push_back(std::move(nb));
      }
      Bucket& bk = buckets[bit->second];
      for (std::size_t j = 0, i = oi; i < batch_ids.size(); ++j, i += owners.size())
        if (!ip.empty() && ip[i + 1] > ip[i] && std::find(bk.active.begin(), bk.active.end(), j) == bk.active.end())
          bk.active.push_back(j);
    }
  }
  for (MsgKind kind : {MsgKind::PartialAgg, MsgKind::PartialGrad})
    for (Bucket& bk : buckets) {
      if (bk.owner == designated || bk.active.empty()) continue;
      std::sort(bk.active.begin(), bk.active.end());
      Message m;
      m.kind = kind;
      m.layer = k;
      m.sender = kind == MsgKind::PartialAgg ? bk.owner : designated;
      m.receiver = kind == MsgKind::PartialAgg ? designated : bk.owner;
      m.node_type = g.target;
      for (std::size_t i : bk.active) m.node_ids.push_back(bk.shard[i]);
      m.rows = m.node_ids.size();
      m.dim = static_cast<std::size_t>(model.num_classes);
      m.bytes = static_cast<std::uint64_t>(acct.header_bytes) + m.rows * m.dim * acct.elem_bytes;
      rep.stats.record(m);
      rep.trace.push_back(std::move(m));
    }
  // ring all-reduce model of the slots and learnable rows several workers touch (raf.cpp:496-510)
  for (const auto& sc : view.slot_contributors) {
    const std::uint64_t s = static_cast<std::uint64_t>(sc[2]);
    if (s < 2) continue;
    const Matrix& w = model.weights.at(SlotKey{sc[0], sc[1]});
    rep.sync_bytes += 2ULL * w.data.size() * acct.elem_bytes * (s - 1) / s;
  }
  // learnable rows: a worker contributes to a type when one of its depth-k positions of that
  // type received a non-empty slice of the frontier this batch (raf.cpp:250-258); the
  // slices follow the RAF recursion over the sampled blocks (ids only)
  bool shared_leaf = false;
  for (const auto& lo : view.leaf_owners) shared_leaf = shared_leaf || lo[1] >= 2;
  if (shared_leaf) {
    std::string bn;
    for (const std::string& n : detail::engine_names(e))
      if (n.rfind("hop", 0) == 0 && n.find(".col") == std::string::npos) bn += (bn.empty() ? "" : ",") + n;
    const detail::Bundle blk(hg_engine_read(e, bn.c_str()));
    std::map<int, std::set<int>> contributors;
    std::function<void(int, const std::vector<NodeId>&, int)> walk = [&](int pos, const std::vector<NodeId>& parent_ids,
                                                                          int owner) {
      const MetatreePos& mp = view.tree.pos[pos];
      const std::string pre = "hop" + std::to_string(mp.depth) + ".rel" + std::to_string(mp.rel_index);
      std::vector<NodeId> f;
      if (blk.has(pre + ".dst_ids")) {
        const auto dst = blk.get<NodeId>(pre + ".dst_ids");
        const auto ip = blk.get<std::uint32_t>(pre + ".indptr");
        const auto src = blk.get<NodeId>(pre + ".src_ids");
        for (NodeId v : parent_ids) {
          const auto it = std::lower_bound(dst.begin(), dst.end(), v);
          if (it == dst.end() || *it != v) continue;
          const std::size_t row = static_cast<std::size_t>(it - dst.begin());
          f.insert(f.end(), src.begin() + ip[row], src.begin() + ip[row + 1]);
        }
        std::sort(f.begin(), f.end());
        f.erase(std::unique(f.begin(), f.end()), f.end());
      }
      if (mp.depth == k) {
        if (g.kinds[mp.type] == 2 && !f.empty()) contributors[mp.type].insert(owner);
        return;
      }
      for (int c : view.tree.children(pos)) walk(c, f, owner);
    };
    for (std::size_t ci = 0; ci < root_children.size(); ++ci) {
      const std::vector<int>& owners = view.top_owners.at(ci);
      for (std::size_t oi = 0; oi < owners.size(); ++oi) {
        std::vector<NodeId> shard;
        for (std::size_t i = oi; i < batch_ids.size(); i += owners.size()) shard.push_back(batch_ids[i]);
        walk(root_children[ci], shard, owners[oi]);
      }
    }
    for (const auto& [type, who] : contributors) {
      const std::uint64_t s = who.size();
      auto it = rep.grads.feature_grads.find(type);
      if (s < 2 || it == rep.grads.feature_grads.end()) continue;
      rep.sync_bytes += 2ULL * it->second.second.data.size() * acct.elem_bytes * (s - 1) / s;
    }
  }
  rep.boundary_counts = view.boundary_counts;
  rep.boundary_cut_edges = view.boundary_cut_edges;
  rep.cross_ids_target_only = true;  // meta plans: only the target-typed AGG_all partials cross
  const CommBoundVerdict v = check_comm_bounds(rep, static_cast<int>(g.relations.size()), true);
  rep.message_bound_ok = v.message_bound_ok;
  return rep;
}

struct EquivalenceResult {
  double logit_diff = 0.0;
  double grad_diff = 0.0;
  double max_diff() const { return logit_diff > grad_diff ? logit_diff : grad_diff; }
};

// check_equivalence (raf.cpp:639-660): the fused engine step (run_raf_batch above) against
// the layer primitives (forward_flat / cross_entropy / backward_flat) on the same blocks
inline EquivalenceResult check_equivalence(const HetGraph& g, const RafPlanView& view, const HGNNModel& model,
                                           const LearnableStore& store, std::span<const NodeId> batch,
                                           const std::vector<int>& fanouts, std::uint64_t rng_seed, int designated) {
  const ExecutionReport raf = run_raf_batch(g, view, model, store, batch, fanouts, rng_seed, designated);
  std::vector<NodeId> batch_ids(batch.begin(), batch.end());
  std::sort(batch_ids.begin(), batch_ids.end());
  batch_ids.erase(std::unique(batch_ids.begin(), batch_ids.end()), batch_ids.end());
  const SampledBlocks blocks =
      sample_khop_restricted(g, batch_ids, fanouts, rng_seed, hop_relation_sets(view.tree, model.k));
  auto [logits, tape] = forward_flat(g, view.tree, blocks, model, store);
  Matrix dlogits;
  cross_entropy(logits, batch_ids, batch, g.labels(), model.num_classes, &dlogits);
  const GradientSet flat = backward_flat(g, view.tree, model, tape, dlogits);
  EquivalenceResult res;
  res.logit_diff = max_abs_diff(raf.logits, logits);
  res.grad_diff = raf.grads.max_abs_diff_vs(flat);
  return res;
}

// ==== feature cache (cache.hpp:14-89) ===================================================================
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
struct MissPenaltyProfile {
  std::vector<TypePenalty> types;
};
// profile_miss_penalty (cache.cpp:11-33)
inline MissPenaltyProfile profile_miss_penalty(const HetGraph& g, const CostModel& cm) {
  std::uint64_t total = 0;
  for (auto c : g.node_counts) total += c;
  const std::vector<std::uint64_t> zeros(std::max<std::uint64_t>(1, total), 0u);
  const detail::Bundle b(hg_cache_plan(g.handle(), zeros.data(), 0, cm.read_ns_per_byte, cm.write_ns_per_byte,
                                       cm.fixed_overhead_ns, cm.elem_bytes));
  const auto ratio = b.get<double>("profile.ratio"), tns = b.get<double>("profile.transfer_ns");
  const auto rb = b.get<std::uint64_t>("profile.record_bytes");
  MissPenaltyProfile p;
  for (std::size_t t = 0; t < rb.size(); ++t) p.types.push_back({g.kinds[t] == 2, rb[t], tns[t], ratio[t]});
  return p;
}

struct HotnessTable {
  std::vector<std::vector<std::uint64_t>> counts;  // [type][node]
  std::uint64_t total(int type) const {
    std::uint64_t s = 0;
    for (auto c : counts[type]) s += c;
    return s;
  }
};
// presample_hotness (cache.cpp:39-63): every batch of every epoch sampled on the device
// (one captured sampling graph replay per batch) with the histogram fused
inline HotnessTable presample_hotness(const HetGraph& g, const Metatree& tree, const std::vector<int>& fanouts,
                                      int epochs, std::uint64_t seed, std::size_t batch_size = 512) {
  Sampler s(g, fanouts, hop_relation_sets(tree, static_cast<int>(fanouts.size())), static_cast<int>(batch_size),
            detail::layer_device());
  const detail::Bundle b(hg_engine_presample_hotness(s.handle(), epochs, seed, static_cast<int>(batch_size)));
  HotnessTable hot;
  for (std::size_t t = 0; t < g.node_counts.size(); ++t) {
    const auto c = b.get<std::uint64_t>("hot.t" + std::to_string(t));
    hot.counts.emplace_back(c.begin(), c.end());
  }
  return hot;
}

struct CacheAllocation {
  std::uint64_t budget = 0;
  std::vector<std::uint64_t> bytes;
  std::vector<std::uint64_t> capacity;
};
// allocate_cache (cache.cpp:65-85): host arithmetic (the plan stays on the CPU)
inline CacheAllocation allocate_cache(std::uint64_t budget, const HotnessTable& hot, const MissPenaltyProfile& profile) {
  CacheAllocation a;
  a.budget = budget;
  a.bytes.assign(profile.types.size(), 0);
  a.capacity.assign(profile.types.size(), 0);
  double denom = 0.0;
  for (std::size_t t = 0; t < profile.types.size(); ++t)
    if (profile.types[t].record_bytes > 0)
      denom += static_cast<double>(hot.total(static_cast<int>(t))) * profile.types[t].ratio;
  if (denom <= 0.0) throw std::invalid_argument("nothing to cache: all count*ratio products are zero");
  for (std::size_t t = 0; t < profile.types.size(); ++t) {
    const TypePenalty& tp = profile.types[t];
    if (tp.record_bytes == 0) continue;
    const double share =
        static_cast<double>(budget) * (static_cast<double>(hot.total(static_cast<int>(t))) * tp.ratio) / denom;
    a.capacity[t] = static_cast<std::uint64_t>(share) / tp.record_bytes;
    a.bytes[t] = a.capacity[t] * tp.record_bytes;
  }
  return a;
}

// CacheState (cache.hpp:57-76, cache.cpp:87-119): the per-batch accounting object
struct CacheState {
  struct TypeCache {
    std::vector<NodeId> cached;  // sorted
    std::uint64_t hits = 0;
    std::uint64_t misses = 0;
    double penalty_ns = 0.0;
  };
  std::vector<TypeCache> types;
  MissPenaltyProfile profile;
  int num_workers = 1;

  bool contains(int type, NodeId id) const {
    const auto& c = types[type].cached;
    return std::binary_search(c.begin(), c.end(), id);
  }
  bool lookup(int type, NodeId id) {
    TypeCache& tc = types[type];
    if (contains(type, id)) {
      tc.hits += 1;
      return true;
    }
    tc.misses += 1;
    tc.penalty_ns += profile.types[type].transfer_ns;
    return false;
  }
  void update(int type, NodeId id) {
    if (!profile.types[type].learnable)
      throw std::invalid_argument("update on read-only node type " + std::to_string(type));
    TypeCache& tc = types[type];
    if (contains(type, id)) {
      tc.hits += 1;
      return;
    }
    tc.misses += 1;
    tc.penalty_ns += profile.types[type].transfer_ns;
  }
  int placement_rank(NodeId id) const { return static_cast<int>(id) % num_workers; }
  double hit_rate(int type) const {
    const TypeCache& tc = types[type];
    const std::uint64_t n = tc.hits + tc.misses;
    return n == 0 ? 0.0 : static_cast<double>(tc.hits) / static_cast<double>(n);
  }
};

// fill_and_serve (cache.cpp:121-141): static top-capacity fill by (count desc, id asc)
inline CacheState fill_and_serve(const CacheAllocation& alloc, const HotnessTable& hot,
                                 const MissPenaltyProfile& profile, int num_workers = 1) {
  CacheState st;
  st.profile = profile;
  st.num_workers = num_workers;
  st.types.resize(profile.types.size());
  for (std::size_t t = 0; t < profile.types.size(); ++t) {
    const std::uint64_t cap = alloc.capacity[t];
    if (cap == 0) continue;
    const auto& c = hot.counts[t];
    std::vector<NodeId> ids(c.size());
    for (std::size_t i = 0; i < ids.size(); ++i) ids[i] = static_cast<NodeId>(i);
    auto better = [&](NodeId a, NodeId b) { return c[a] != c[b] ? c[a] > c[b] : a < b; };
    if (ids.size() > cap) {
      std::nth_element(ids.begin(), ids.begin() + static_cast<std::ptrdiff_t>(cap), ids.end(), better);
      ids.resize(cap);
    }
    std::sort(ids.begin(), ids.end());
    st.types[t].cached = std::move(ids);
  }
  return st;
}

// cacheable_types (cache.cpp:143-177) and partition_aware_space (cache.cpp:179-182)
inline std::vector<NodeTypeId> cacheable_types(const PartitionPlan& plan, int part) {
  return plan.parts.at(part).cacheable;
}
inline bool partition_aware_space(const PartitionPlan& plan, int part, NodeTypeId type) {
  const auto& types = plan.parts.at(part).node_types;
  return std::find(types.begin(), types.end(), type) != types.end();
}

}  // namespace hetsim_b200

#ifdef HETSIM_B200_AS_HETSIM
namespace hetsim {
using namespace hetsim_b200;  // NOLINT: drop-in build without the reference library
}
#endif
