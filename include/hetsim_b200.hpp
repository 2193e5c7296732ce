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
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
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
  }
  hg_graph* handle() const { return h_.get(); }
  std::vector<std::uint64_t> node_counts;  // per node type
  struct Rel {
    NodeTypeId src, dst;
  };
  std::vector<Rel> relations;
  NodeTypeId target = 0;
  int num_classes = 0;

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
  std::vector<PlanPartition> parts;
  std::vector<std::vector<int>> hop_relations;  // hop_relation_sets(tree, k) (hgnn.cpp:28-37)
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
};

class RafEngine {
 public:
  // init_model / init_learnable seeds as run_experiment derives them (harness.cpp:365-366)
  RafEngine(const HetGraph& g, std::vector<int> fanouts, int hidden, std::uint64_t seed, int batch_cap = 1024,
            int p = 1, int rank = 0, int device = 0)
      : g_(g), fanouts_(std::move(fanouts)) {
    const hg_engine_opts o{static_cast<int>(fanouts_.size()), fanouts_.data(), hidden, batch_cap, p, rank,
                           mix_seed(seed, 0xd0de1), mix_seed(seed, 0x1ea4a), device};
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
  std::vector<std::vector<std::uint32_t>> presample_hotness(int epochs, std::uint64_t seed, int batch_size = 512) {
    const detail::Bundle b(hg_engine_presample_hotness(e_.get(), epochs, seed, batch_size));
    std::vector<std::vector<std::uint32_t>> out;
    for (std::size_t t = 0; t < g_.node_counts.size(); ++t) out.push_back(b.get<std::uint32_t>("hot.t" + std::to_string(t)));
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

}  // namespace hetsim_b200

#ifdef HETSIM_B200_AS_HETSIM
namespace hetsim {
using namespace hetsim_b200;  // NOLINT: drop-in build without the reference library
}
#endif
