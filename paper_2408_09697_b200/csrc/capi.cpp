// extern "C" boundary (include/hetgpu.h): converts C arguments into the host
// layer / engine calls and C++ exceptions into return codes + last error.
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <map>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/hetgpu.h"
#include "engine.hpp"
#include "gemm.cuh"
#include "host.hpp"
#include "layers.hpp"

#ifdef HG_WITH_NCCL
#include <nccl.h>
#endif

using namespace hetgpu;

struct hg_graph {
  Graph g;
};
struct hg_engine {
  std::unique_ptr<Engine> e;
#ifdef HG_WITH_NCCL
  ncclComm_t comm = nullptr;
  ncclComm_t rcomm = nullptr;  // replica group (ncclCommSplit of comm)
#endif
};
struct hg_ctx {
  std::unique_ptr<LayerCtx> c;
};
struct hg_bundle {
  struct Item {
    std::string name, dtype;
    std::vector<long long> shape;
    std::vector<char> data;
  };
  std::vector<Item> items;

  template <typename T>
  void add(const std::string& n, const char* dt, const std::vector<T>& v, std::vector<long long> shape = {}) {
    Item it;
    it.name = n;
    it.dtype = dt;
    it.shape = shape.empty() ? std::vector<long long>{static_cast<long long>(v.size())} : shape;
    it.data.resize(v.size() * sizeof(T));
    if (!v.empty()) std::memcpy(it.data.data(), v.data(), it.data.size());
    items.push_back(std::move(it));
  }
};

namespace {

thread_local std::string g_err;
thread_local int g_err_kind = 0;

template <typename R, typename F>
R guard(R fail, F&& f) {
  try {
    g_err.clear();
    g_err_kind = 0;
    return f();
  } catch (const std::invalid_argument& ex) {
    g_err = ex.what();
    g_err_kind = 1;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    g_err_kind = 2;
  }
  return fail;
}

std::vector<int> ivec(const int* p, int n) { return p ? std::vector<int>(p, p + n) : std::vector<int>{}; }

// work: n_subs sampled-work values, optionally followed by n_subs learnable-row counts
Plan work_aware_plan(const Graph& g, int k, int p, const double* work, int n_work) {
  const Schema sch = schema_of(g);
  const int n_subs = static_cast<int>(meta_partition(sch, g.target, k, 1).subs.size());
  std::vector<double> w(work, work + std::min(n_work, n_subs)), l;
  if (n_work == 2 * n_subs) l.assign(work + n_subs, work + n_work);
  std::vector<bool> learnable(g.num_types());
  for (int t = 0; t < g.num_types(); ++t) learnable[t] = g.types[t].storage == Storage::Learnable;
  return work_aware_partition(sch, g.target, k, p, w, l, 6.0, learnable);
}

EngineOptions engine_options(const hg_engine_opts& o) {
  EngineOptions eo;
  eo.k = o.k;
  eo.fanouts = ivec(o.fanouts, o.k);
  eo.hidden = o.hidden;
  eo.batch_cap = o.batch_cap;
  eo.p = o.p;
  eo.rank = o.rank;
  eo.model_seed = o.model_seed;
  eo.learn_seed = o.learn_seed;
  eo.device = o.device;
  eo.feat_dtype = o.feat_dtype;
  eo.feat_host = o.feat_host;
  if (o.model != 0 && o.model != 1) throw std::invalid_argument("model must be 0 (RGCN) or 1 (RGAT)");
  eo.model = o.model;
  eo.heads = o.heads > 0 ? o.heads : 4;
  return eo;
}

}  // namespace

extern "C" {

const char* hg_last_error(void) { return g_err.c_str(); }
int hg_last_error_kind(void) { return g_err_kind; }
const char* hg_version(void) { return "hetgpu 0.1 (sm_100a)"; }

int hg_bundle_size(const hg_bundle* b) { return static_cast<int>(b->items.size()); }
const char* hg_bundle_name(const hg_bundle* b, int i) { return b->items[i].name.c_str(); }
const char* hg_bundle_dtype(const hg_bundle* b, int i) { return b->items[i].dtype.c_str(); }
int hg_bundle_ndim(const hg_bundle* b, int i) { return static_cast<int>(b->items[i].shape.size()); }
long long hg_bundle_dim(const hg_bundle* b, int i, int d) { return b->items[i].shape[d]; }
long long hg_bundle_nbytes(const hg_bundle* b, int i) { return static_cast<long long>(b->items[i].data.size()); }
const void* hg_bundle_data(const hg_bundle* b, int i) { return b->items[i].data.data(); }
void hg_bundle_free(hg_bundle* b) { delete b; }

uint64_t hg_mix_seed(uint64_t a, uint64_t b) { return mix_seed(a, b); }

int hg_mt64_outputs(uint64_t seed, uint64_t start, uint64_t n, uint64_t* out) {
  return guard<int>(-1, [&] {
    std::mt19937_64 e = mt64_jump_engines(seed, {start})[0];
    for (uint64_t i = 0; i < n; ++i) out[i] = e();
    return 0;
  });
}

// ---- graphs ----------------------------------------------------------------------------
hg_graph* hg_graph_generate(const hg_spec* spec, uint64_t seed) {
  return guard<hg_graph*>(nullptr, [&] {
    Spec s;
    s.target = spec->target;
    s.num_classes = spec->num_classes;
    s.label_noise = spec->label_noise;
    s.add_reverse = spec->add_reverse != 0;
    for (int i = 0; i < spec->n_types; ++i) {
      const hg_spec_node_type& t = spec->types[i];
      if (t.storage != 1 && t.storage != 2) throw std::invalid_argument("unknown storage kind");
      s.node_types.push_back({t.name, t.count, t.dim, t.storage == 1 ? Storage::Dense : Storage::Learnable});
    }
    for (int i = 0; i < spec->n_rels; ++i) {
      const hg_spec_relation& r = spec->rels[i];
      s.relations.push_back({r.src, r.edge, r.dst, r.edges, r.powerlaw != 0, r.alpha});
    }
    for (int i = 0; i < spec->n_self_paired; ++i) s.self_paired.push_back(spec->self_paired[i]);
    auto* h = new hg_graph;
    h->g = generate(s, seed);
    return h;
  });
}

hg_graph* hg_graph_from_csr(int n_types, const uint64_t* counts, int n_rels, const int* rel_src, const int* rel_dst,
                            const int* rel_reverse, const uint64_t* indptr, const uint32_t* src, const int* kinds,
                            const int* dims, const float* dense, int target, int num_classes, const int32_t* labels) {
  return guard<hg_graph*>(nullptr, [&] {
    auto* h = new hg_graph;
    Graph& g = h->g;
    std::size_t dense_off = 0;
    for (int t = 0; t < n_types; ++t) {
      NodeTypeInfo nt;
      nt.name = "t" + std::to_string(t);
      nt.count = counts[t];
      nt.dim = dims[t];
      nt.storage = static_cast<Storage>(kinds[t]);
      if (nt.storage == Storage::Dense) {
        const std::size_t n = nt.count * static_cast<std::size_t>(nt.dim);
        nt.dense.assign(dense + dense_off, dense + dense_off + n);
        dense_off += n;
      }
      g.types.push_back(std::move(nt));
    }
    std::size_t ip = 0, sp = 0;
    for (int r = 0; r < n_rels; ++r) {
      RelationInfo rel;
      rel.src_type = rel_src[r];
      rel.dst_type = rel_dst[r];
      rel.edge_type = r;
      rel.reverse = rel_reverse && rel_reverse[r];
      const std::size_t nd = counts[rel.dst_type];
      rel.adj.offsets.assign(indptr + ip, indptr + ip + nd + 1);
      ip += nd + 1;
      const std::size_t ne = rel.adj.offsets.back();
      rel.adj.sources.assign(src + sp, src + sp + ne);
      sp += ne;
      g.edge_type_names.push_back("e" + std::to_string(r));
      g.rels.push_back(std::move(rel));
    }
    g.target = target;
    g.num_classes = num_classes;
    g.labels.assign(labels, labels + counts[target]);
    g.validate();
    return h;
  });
}

hg_graph* hg_graph_from_pairs(int n_types, const uint64_t* counts, int n_rels, const int* rel_src, const int* rel_dst,
                              const uint64_t* pair_counts, const uint32_t* pair_src, const uint32_t* pair_dst,
                              int target, int num_classes) {
  return guard<hg_graph*>(nullptr, [&] {
    std::vector<std::string> names, enames;
    for (int t = 0; t < n_types; ++t) names.push_back("t" + std::to_string(t));
    std::vector<std::vector<std::pair<NodeId, NodeId>>> pairs(n_rels);
    std::size_t off = 0;
    for (int r = 0; r < n_rels; ++r) {
      enames.push_back("e" + std::to_string(r));
      for (std::uint64_t e = 0; e < pair_counts[r]; ++e, ++off) pairs[r].emplace_back(pair_src[off], pair_dst[off]);
    }
    auto* h = new hg_graph;
    h->g = assemble(names, std::vector<std::uint64_t>(counts, counts + n_types), enames, ivec(rel_src, n_rels),
                    ivec(rel_dst, n_rels), pairs, target, num_classes);
    return h;
  });
}

hg_graph* hg_graph_load(const char* path) {
  return guard<hg_graph*>(nullptr, [&] {
    auto* h = new hg_graph;
    h->g = load_container(path ? path : "");
    return h;
  });
}

int hg_graph_save(const hg_graph* g, const char* path) {
  return guard<int>(-1, [&] {
    save_container(g->g, path ? path : "");
    return 0;
  });
}

void hg_graph_free(hg_graph* g) { delete g; }

hg_bundle* hg_graph_schema(const hg_graph* h) {
  return guard<hg_bundle*>(nullptr, [&] {
    const Graph& g = h->g;
    auto* b = new hg_bundle;
    std::vector<std::uint64_t> counts;
    std::vector<int> kinds, dims, rs, rd;
    for (const auto& t : g.types) {
      counts.push_back(t.count);
      kinds.push_back(static_cast<int>(t.storage));
      dims.push_back(t.dim);
    }
    for (int r = 0; r < g.num_rels(); ++r) {
      rs.push_back(g.rels[r].src_type);
      rd.push_back(g.rels[r].dst_type);
    }
    b->add("node_counts", "<u8", counts);
    b->add("kinds", "<i4", kinds);
    b->add("dims", "<i4", dims);
    b->add("target", "<i8", std::vector<long long>{g.target});
    b->add("num_classes", "<i8", std::vector<long long>{g.num_classes});
    b->add("rel_src", "<i4", rs);
    b->add("rel_dst", "<i4", rd);
    std::string names;  // node type names, '\n'-separated (hetgraph.hpp TypeRegistry)
    for (const auto& t : g.types) names += t.name + "\n";
    b->add("type_names", "|u1", std::vector<char>(names.begin(), names.end()));
    return b;
  });
}

hg_bundle* hg_graph_export(const hg_graph* h) {
  return guard<hg_bundle*>(nullptr, [&] {
    const Graph& g = h->g;
    auto* b = new hg_bundle;
    std::vector<std::uint64_t> counts;
    std::vector<int> kinds, dims, rs, rd, rr;
    for (const auto& t : g.types) {
      counts.push_back(t.count);
      kinds.push_back(static_cast<int>(t.storage));
      dims.push_back(t.dim);
    }
    b->add("node_counts", "<u8", counts);
    b->add("kinds", "<i4", kinds);
    b->add("dims", "<i4", dims);
    b->add("labels", "<i4", g.labels);
    b->add("target", "<i8", std::vector<long long>{g.target});
    b->add("num_classes", "<i8", std::vector<long long>{g.num_classes});
    for (int r = 0; r < g.num_rels(); ++r) {
      rs.push_back(g.rels[r].src_type);
      rd.push_back(g.rels[r].dst_type);
      rr.push_back(g.rels[r].reverse ? 1 : 0);
      b->add("rel" + std::to_string(r) + ".indptr", "<u8", g.rels[r].adj.offsets);
      b->add("rel" + std::to_string(r) + ".src", "<u4", g.rels[r].adj.sources);
    }
    b->add("rel_src", "<i4", rs);
    b->add("rel_dst", "<i4", rd);
    b->add("rel_reverse", "<i4", rr);
    for (int t = 0; t < g.num_types(); ++t)
      if (g.types[t].storage == Storage::Dense)
        b->add("feat.t" + std::to_string(t), "<f4", g.types[t].dense,
               {static_cast<long long>(g.types[t].count), g.types[t].dim});
    return b;
  });
}

// ---- planning ------------------------------------------------------------------------------
namespace {
hg_bundle* plan_bundle(const Graph& g, const Plan& plan, int k) {
  {
    auto* b = new hg_bundle;
    std::vector<int> ty, de, pa, re;
    for (const auto& ps : plan.tree.pos) {
      ty.push_back(ps.type);
      de.push_back(ps.depth);
      pa.push_back(ps.parent);
      re.push_back(ps.rel);
    }
    b->add("tree.type", "<i4", ty);
    b->add("tree.depth", "<i4", de);
    b->add("tree.parent", "<i4", pa);
    b->add("tree.rel", "<i4", re);
    std::vector<int> sc;
    std::vector<std::uint64_t> sw;
    for (const auto& s : plan.subs) {
      sc.push_back(s.child_pos);
      sw.push_back(s.weight);
    }
    b->add("subs.child_pos", "<i4", sc);
    b->add("subs.weight", "<u8", sw);
    for (std::size_t i = 0; i < plan.parts.size(); ++i) {
      const Part& part = plan.parts[i];
      const std::string pre = "part" + std::to_string(i);
      b->add(pre + ".sub_ids", "<i4", part.sub_ids);
      b->add(pre + ".relations", "<i4", part.relations);
      b->add(pre + ".node_types", "<i4", part.node_types);
      b->add(pre + ".cacheable", "<i4", cacheable_types(plan, static_cast<int>(i)));
      b->add(pre + ".replica", "<i4", std::vector<int>{part.replica ? 1 : 0, part.replica_index, part.replica_count});
      b->add(pre + ".weight", "<u8", std::vector<std::uint64_t>{part.weight});
    }
    const auto hr = hop_relations(plan.tree, k);
    for (int i = 0; i < k; ++i) b->add("hop_rels" + std::to_string(i + 1), "<i4", hr[i]);
    // batch-invariant RAF bookkeeping of this plan (raf.cpp:306-340, 496-503, 521-528)
    const RafAccounting a = plan_accounting(g, plan);
    b->add("raf.boundary_counts", "<u8", a.boundary_counts);
    b->add("raf.boundary_cut_edges", "<u8", std::vector<std::uint64_t>{a.boundary_cut_edges});
    std::vector<int> slot_rows;  // (rel, layer, n_contributors) per slot
    for (const auto& [id, who] : a.slot_contributors) {
      slot_rows.push_back(id.rel);
      slot_rows.push_back(id.layer);
      slot_rows.push_back(static_cast<int>(who.size()));
    }
    b->add("raf.slot_contributors", "<i4", slot_rows);
    std::vector<int> leaf_rows;  // (learnable leaf type, n_possible_contributors)
    for (const auto& [t, who] : a.leaf_owners) {
      leaf_rows.push_back(t);
      leaf_rows.push_back(static_cast<int>(who.size()));
    }
    b->add("raf.leaf_owners", "<i4", leaf_rows);
    return b;
  }
}
}  // namespace

hg_bundle* hg_meta_partition(const hg_graph* h, int k, int p) {
  return guard<hg_bundle*>(nullptr, [&] {
    const Graph& g = h->g;
    return plan_bundle(g, meta_partition(schema_of(g), g.target, k, p), k);
  });
}

hg_bundle* hg_meta_partition_work_aware(const hg_graph* h, int k, int p, const double* work, int n_work) {
  return guard<hg_bundle*>(nullptr, [&] {
    const Graph& g = h->g;
    return plan_bundle(g, work_aware_plan(g, k, p, work, n_work), k);
  });
}

// sampled work of every sub-metatree: mean sampled edges per batch of a sampler restricted
// to the sub's relations at each hop, over n_batches make_batches batches
hg_bundle* hg_sub_work(const hg_graph* h, const int* fanouts, int k, int n_batches, int batch_size, uint64_t seed,
                       int device) {
  return guard<hg_bundle*>(nullptr, [&] {
    const Graph& g = h->g;
    if (k < 1 || !fanouts) throw std::invalid_argument("fanouts must be non-empty");
    const Plan plan = meta_partition(schema_of(g), g.target, k, 1);
    const auto batches = make_batches(g, batch_size, n_batches, seed);
    std::vector<double> work, learn;
    for (const SubTree& st : plan.subs) {
      EngineOptions eo;
      eo.k = k;
      eo.fanouts = ivec(fanouts, k);
      eo.batch_cap = batch_size;
      eo.device = device;
      eo.sample_only = true;
      eo.hop_relations.assign(k, {});
      for (int pos : st.positions) {
        const TreePos& tp = plan.tree.pos[pos];
        if (tp.rel >= 0 && tp.depth >= 1 && tp.depth <= k) eo.hop_relations[tp.depth - 1].push_back(tp.rel);
      }
      Engine e(g, eo);
      double edges = 0, rows = 0;
      for (std::size_t i = 0; i < batches.size(); ++i) {
        e.sample_only(batches[i].data(), static_cast<int>(batches[i].size()), mix_seed(seed, 0xb000 + i));
        edges += static_cast<double>(e.sampled_edges());
        rows += static_cast<double>(e.learnable_leaf_rows());
      }
      const double nb = std::max<double>(1.0, static_cast<double>(batches.size()));
      work.push_back(edges / nb);
      learn.push_back(rows / nb);
    }
    auto* b = new hg_bundle;
    b->add("work", "<f8", work);
    b->add("learn_rows", "<f8", learn);
    return b;
  });
}

hg_engine* hg_engine_create_work_aware(const hg_graph* g, const hg_engine_opts* o, const double* work, int n_work) {
  return guard<hg_engine*>(nullptr, [&] {
    EngineOptions eo = engine_options(*o);
    eo.sub_work.assign(work, work + n_work);
    auto* h = new hg_engine;
    h->e = std::make_unique<Engine>(g->g, eo);
    return h;
  });
}

hg_bundle* hg_make_batches(const hg_graph* h, int batch_size, int max_batches, uint64_t seed) {
  return guard<hg_bundle*>(nullptr, [&] {
    auto* b = new hg_bundle;
    const auto batches = make_batches(h->g, batch_size, max_batches, seed);
    for (std::size_t i = 0; i < batches.size(); ++i) b->add("batch" + std::to_string(i), "<u4", batches[i]);
    return b;
  });
}

// ---- engine --------------------------------------------------------------------------------
hg_engine* hg_engine_create_from_container(const char* path, const hg_engine_opts* o) {
  return guard<hg_engine*>(nullptr, [&] {
    const EngineOptions eo = engine_options(*o);
    auto* h = new hg_engine;
    h->e = std::make_unique<Engine>(std::string(path), eo);
    return h;
  });
}

hg_engine* hg_engine_create(const hg_graph* g, const hg_engine_opts* o) {
  return guard<hg_engine*>(nullptr, [&] {
    const EngineOptions eo = engine_options(*o);
    auto* h = new hg_engine;
    h->e = std::make_unique<Engine>(g->g, eo);
    return h;
  });
}

hg_engine* hg_sampler_create(const hg_graph* g, const int* fanouts, int k, const int* hop_rel_flat,
                             const int* hop_rel_counts, int batch_cap, int device) {
  return guard<hg_engine*>(nullptr, [&] {
    if (k < 1 || !fanouts) throw std::invalid_argument("fanouts must be non-empty");
    EngineOptions eo;
    eo.k = k;
    eo.fanouts = ivec(fanouts, k);
    eo.batch_cap = batch_cap;
    eo.device = device;
    eo.sample_only = true;
    if (!hop_rel_flat || !hop_rel_counts) {
      eo.all_relations = true;
    } else {
      int at = 0;
      for (int h = 0; h < k; ++h) {
        eo.hop_relations.emplace_back(hop_rel_flat + at, hop_rel_flat + at + hop_rel_counts[h]);
        at += hop_rel_counts[h];
      }
    }
    auto* h = new hg_engine;
    h->e = std::make_unique<Engine>(g->g, eo);
    return h;
  });
}

void hg_engine_free(hg_engine* e) {
  if (!e) return;
  // the engine first: its captured step graphs hold NCCL work on the communicator
  e->e.reset();
#ifdef HG_WITH_NCCL
  if (e->rcomm) ncclCommDestroy(e->rcomm);
  if (e->comm) ncclCommDestroy(e->comm);
#endif
  delete e;
}

int hg_engine_step(hg_engine* e, const uint32_t* batch, int n, uint64_t rng_seed, int designated, int train,
                   hg_step_report* out) {
  return guard<int>(-1, [&] {
    if (n <= 0) throw std::invalid_argument("empty batch");
    const StepReport r = e->e->step(batch, n, rng_seed, designated, train != 0);
    if (out) {
      out->loss = r.loss;
      out->sampled_edges = r.sampled_edges;
      out->n_active = static_cast<int>(std::min<std::size_t>(64, r.active_rows.size()));
      for (int i = 0; i < out->n_active; ++i) out->active_rows[i] = r.active_rows[i];
      out->sync_bytes = r.sync_bytes;
      out->sync_leader = r.sync_leader ? 1 : 0;
      out->message_bound_ok = r.message_bound_ok ? 1 : 0;
      out->target_only_ok = r.target_only_ok ? 1 : 0;
      out->boundary_cut_edges = r.boundary_cut_edges;
      out->n_boundary = static_cast<int>(std::min<std::size_t>(64, r.boundary_counts.size()));
      for (int i = 0; i < out->n_boundary; ++i) out->boundary_counts[i] = r.boundary_counts[i];
    }
    return 0;
  });
}

int hg_engine_prefetch(hg_engine* e, const uint32_t* batch, int n, uint64_t rng_seed) {
  return guard<int>(-1, [&] {
    e->e->prefetch(batch, n, rng_seed);
    return 0;
  });
}

int hg_engine_sample(hg_engine* e, const uint32_t* batch, int n, uint64_t rng_seed) {
  return guard<int>(-1, [&] {
    e->e->sample_only(batch, n, rng_seed);
    return 0;
  });
}

hg_bundle* hg_engine_read(hg_engine* e, const char* names) {
  return guard<hg_bundle*>(nullptr, [&] {
    std::vector<std::string> want;
    if (names && std::string(names) == "?") {
      std::string all;
      for (const auto& n : e->e->tensor_names()) all += (all.empty() ? "" : ",") + n;
      auto* b = new hg_bundle;
      b->add("names", "|u1", std::vector<char>(all.begin(), all.end()));
      return b;
    }
    if (names && *names) {
      std::string s(names);
      std::size_t at = 0;
      while (at <= s.size()) {
        const std::size_t c = s.find(',', at);
        const std::string n = s.substr(at, c == std::string::npos ? std::string::npos : c - at);
        if (!n.empty()) want.push_back(n);
        if (c == std::string::npos) break;
        at = c + 1;
      }
    } else {
      want = e->e->tensor_names();
    }
    auto* b = new hg_bundle;
    for (const auto& n : want) {
      hg_bundle::Item it;
      it.name = n;
      if (!e->e->read_tensor(n, it.dtype, it.shape, it.data)) {
        delete b;
        throw std::invalid_argument("unknown tensor: " + n);
      }
      b->items.push_back(std::move(it));
    }
    return b;
  });
}

int hg_engine_bench(hg_engine* e, const uint32_t* batches, const int* lens, const uint64_t* seeds, int n_steps,
                    int train, double* out_ms, uint64_t* out_edges, double* out_loss) {
  return guard<int>(-1, [&] {
    Engine& en = *e->e;
    std::size_t total = 0;
    for (int i = 0; i < n_steps; ++i) {
      if (lens[i] <= 0) throw std::invalid_argument("empty batch");
      if (lens[i] > en.batch_cap()) throw std::invalid_argument("batch larger than the engine's batch capacity");
      en.validate_batch(batches + total, lens[i]);
      total += lens[i];
    }
    // inputs resident in HBM before the timed region: batch ids and per-step scalars
    std::vector<StepScalars> sc(n_steps);
    for (int i = 0; i < n_steps; ++i) sc[i] = en.next_scalars(seeds[i], lens[i], 0, train != 0);
    std::uint32_t* d_all = nullptr;
    StepScalars* d_sc = nullptr;
    HG_CUDA(cudaMalloc(&d_all, std::max<std::size_t>(4, total * 4)));
    HG_CUDA(cudaMalloc(&d_sc, sizeof(StepScalars) * std::max(1, n_steps)));
    // on the engine's (non-blocking) stream and complete before the timed region: a
    // pageable legacy-stream copy may return before its DMA has landed
    HG_CUDA(cudaMemcpyAsync(d_all, batches, total * 4, cudaMemcpyHostToDevice, en.stream()));
    HG_CUDA(cudaMemcpyAsync(d_sc, sc.data(), sizeof(StepScalars) * n_steps, cudaMemcpyHostToDevice, en.stream()));
    HG_CUDA(cudaStreamSynchronize(en.stream()));
    cudaEvent_t a, b;
    HG_CUDA(cudaEventCreate(&a));
    HG_CUDA(cudaEventCreate(&b));
    en.quiesce();
    HG_CUDA(cudaEventRecord(a, en.stream()));
    HG_CUDA(cudaStreamWaitEvent(en.sample_stream(), a, 0));  // sampling is inside the timed region
    std::vector<std::size_t> off(n_steps + 1, 0);
    for (int i = 0; i < n_steps; ++i) off[i + 1] = off[i] + lens[i];
    std::uint64_t edges = 0;
    double loss = 0.0;
    // HG_BENCH_PHASE (diagnostics only): "sample" times the sampling graphs alone,
    // "serial" runs sampling and training back to back without overlap
    const char* phase_env = std::getenv("HG_BENCH_PHASE");
    const std::string phase = phase_env ? phase_env : "";
    if (phase == "sample") {
      for (int i = 0; i < n_steps; ++i) {
        en.prefetch_device(d_all + off[i], lens[i], d_sc + i);
        en.drop_pending();
      }
      HG_CUDA(cudaEventRecord(b, en.sample_stream()));
    } else if (phase == "serial") {
      for (int i = 0; i < n_steps; ++i) {
        en.prefetch_device(d_all + off[i], lens[i], d_sc + i);
        en.train_device(d_sc + i, train != 0);
        HG_CUDA(cudaEventRecord(b, en.stream()));
        HG_CUDA(cudaStreamWaitEvent(en.sample_stream(), b, 0));
      }
      HG_CUDA(cudaEventRecord(b, en.stream()));
    } else {
      // batch i+1 is sampled (sampling stream) while batch i trains
      if (n_steps > 0) en.prefetch_device(d_all + off[0], lens[0], d_sc + 0);
      for (int i = 0; i < n_steps; ++i) {
        if (i + 1 < n_steps) en.prefetch_device(d_all + off[i + 1], lens[i + 1], d_sc + i + 1);
        en.train_device(d_sc + i, train != 0);
      }
      HG_CUDA(cudaEventRecord(b, en.stream()));
    }
    HG_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    HG_CUDA(cudaEventElapsedTime(&ms, a, b));
    const StepReport last = en.finish_step();
    loss = last.loss;
    edges = last.sampled_edges;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(d_all);
    cudaFree(d_sc);
    *out_ms = ms;
    if (out_edges) *out_edges = edges;
    if (out_loss) *out_loss = loss;
    return 0;
  });
}

void hg_engine_profile(hg_engine* e, int on) {
  e->e->set_profiling(on != 0);
  e->e->reset_profile();
}

hg_bundle* hg_engine_profile_read(hg_engine* e) {
  return guard<hg_bundle*>(nullptr, [&] {
    auto* b = new hg_bundle;
    const auto ms = e->e->kernel_ms();
    const auto bytes = e->e->kernel_bytes();
    const auto launches = e->e->kernel_launches();
    for (const auto& [k, v] : ms) {
      b->add("kernel." + k + ".ms", "<f8", std::vector<double>{v});
      b->add("kernel." + k + ".launches", "<i8", std::vector<long long>{launches.at(k)});
    }
    (void)bytes;
    b->add("alg_bytes", "<f8", e->e->algorithmic_bytes());
    return b;
  });
}

int hg_engine_info(hg_engine* e, uint64_t* param_count, uint64_t* device_bytes, int* model_step) {
  return guard<int>(-1, [&] {
    if (param_count) *param_count = e->e->param_count();
    if (device_bytes) *device_bytes = e->e->device_bytes();
    if (model_step) *model_step = e->e->model_step();
    return 0;
  });
}

int hg_engine_set_option(hg_engine* e, const char* name, int value) {
  return guard<int>(-1, [&] {
    const std::string n(name ? name : "");
    if (n == "retain_grads")
      e->e->set_retain_grads(value != 0);
    else if (n == "graphs")
      e->e->set_graphs(value != 0);
    else if (n == "umma")
      e->e->set_umma(value != 0);
    else if (n == "elem_bytes")
      e->e->set_elem_bytes(value);
    else if (n == "trace_sampler")
      e->e->set_trace_sampler(value != 0);
    else if (n == "shard_merge")
      e->e->set_shard_merge(value != 0);
    else if (n == "apply_adam")
      e->e->set_apply_adam(value != 0);
    else
      throw std::invalid_argument("unknown engine option: " + n);
    return 0;
  });
}

hg_bundle* hg_selftest_contractions(const int* cases, int n_cases, int device) {
  return guard<hg_bundle*>(nullptr, [&] {
    HG_CUDA(cudaSetDevice(device));
    std::vector<std::vector<int>> cs;
    for (int i = 0; i < n_cases; ++i) cs.push_back({cases[4 * i], cases[4 * i + 1], cases[4 * i + 2], cases[4 * i + 3]});
    const auto errs = selftest_contractions(cs);
    std::vector<double> flat;
    for (const auto& e : errs) flat.insert(flat.end(), e.begin(), e.end());
    auto* b = new hg_bundle;
    b->add("err", "<f8", flat, {static_cast<long long>(errs.size()), 3});
    return b;
  });
}

int hg_engine_count_launches(hg_engine* e, int n, int train) {
  return guard<int>(-1, [&] { return e->e->count_launches(n, train != 0); });
}

// ---- cache -----------------------------------------------------------------------------------
hg_bundle* hg_engine_presample_hotness(hg_engine* e, int epochs, uint64_t seed, int batch_size) {
  return guard<hg_bundle*>(nullptr, [&] {
    const auto counts = e->e->presample_hotness(epochs, seed, batch_size);
    auto* b = new hg_bundle;
    for (std::size_t t = 0; t < counts.size(); ++t) b->add("hot.t" + std::to_string(t), "<u8", counts[t]);
    return b;
  });
}

hg_bundle* hg_cache_plan(const hg_graph* h, const uint64_t* counts, uint64_t budget, double read_ns, double write_ns,
                         double overhead_ns, int elem_bytes) {
  return guard<hg_bundle*>(nullptr, [&] {
    const Graph& g = h->g;
    CostModel cm;
    cm.read_ns_per_byte = read_ns;
    cm.write_ns_per_byte = write_ns;
    cm.fixed_overhead_ns = overhead_ns;
    cm.elem_bytes = elem_bytes;
    const auto prof = miss_penalty(g, cm);
    std::vector<std::vector<std::uint64_t>> hot(g.num_types());
    std::size_t off = 0;
    for (int t = 0; t < g.num_types(); ++t) {
      hot[t].assign(counts + off, counts + off + g.types[t].count);
      off += g.types[t].count;
    }
    auto* b = new hg_bundle;
    std::vector<double> ratio, tns;
    std::vector<std::uint64_t> rb;
    for (const auto& tp : prof) {
      ratio.push_back(tp.ratio);
      tns.push_back(tp.transfer_ns);
      rb.push_back(tp.record_bytes);
    }
    b->add("profile.ratio", "<f8", ratio);
    b->add("profile.transfer_ns", "<f8", tns);
    b->add("profile.record_bytes", "<u8", rb);
    if (budget == 0) return b;
    const CacheAlloc a = allocate_cache(budget, hot, prof);
    b->add("alloc.bytes", "<u8", a.bytes);
    b->add("alloc.capacity", "<u8", a.capacity);
    // static top-capacity fill by (count desc, id asc), ids re-sorted (cache.cpp:121-141)
    for (int t = 0; t < g.num_types(); ++t) {
      std::vector<NodeId> keep;
      const std::uint64_t cap = a.capacity[t];
      if (cap > 0) {
        std::vector<NodeId> ids(hot[t].size());
        std::iota(ids.begin(), ids.end(), 0u);
        const auto& c = hot[t];
        auto better = [&](NodeId x, NodeId y) { return c[x] != c[y] ? c[x] > c[y] : x < y; };
        if (ids.size() > cap) {
          std::nth_element(ids.begin(), ids.begin() + cap, ids.end(), better);
          ids.resize(cap);
        }
        std::sort(ids.begin(), ids.end());
        keep = std::move(ids);
      }
      b->add("cached.t" + std::to_string(t), "<u4", keep);
    }
    return b;
  });
}

int hg_engine_set_cache(hg_engine* e, const uint32_t* ids, const uint64_t* lens, int n_types) {
  return guard<int>(-1, [&] {
    std::vector<std::vector<NodeId>> sets(n_types);
    std::size_t off = 0;
    for (int t = 0; t < n_types; ++t) {
      sets[t].assign(ids + off, ids + off + lens[t]);
      off += lens[t];
    }
    e->e->set_cache(sets);
    return 0;
  });
}

hg_bundle* hg_engine_cache_counters(hg_engine* e) {
  return guard<hg_bundle*>(nullptr, [&] {
    auto* b = new hg_bundle;
    const auto c = e->e->cache_counters();
    for (std::size_t t = 0; t < c.size(); ++t)
      b->add("cache.t" + std::to_string(t), "<u8", std::vector<std::uint64_t>{c[t].first, c[t].second});
    return b;
  });
}

// ---- NCCL --------------------------------------------------------------------------------------
int hg_nccl_unique_id(void* out, int cap) {
  return guard<int>(-1, [&] {
#ifdef HG_WITH_NCCL
    ncclUniqueId id;
    if (cap < static_cast<int>(sizeof(id))) throw std::invalid_argument("unique id buffer too small");
    if (ncclGetUniqueId(&id) != ncclSuccess) throw std::runtime_error("ncclGetUniqueId failed");
    std::memcpy(out, &id, sizeof(id));
    return static_cast<int>(sizeof(id));
#else
    (void)out;
    (void)cap;
    throw std::runtime_error("built without NCCL");
    return -1;
#endif
  });
}

int hg_engine_replica_handle(hg_engine* e, void* out, int cap) {
  return guard<int>(-1, [&] {
    const std::vector<char> h = e->e->replica_handle();
    if (static_cast<int>(h.size()) > cap) throw std::invalid_argument("handle buffer too small");
    if (!h.empty()) std::memcpy(out, h.data(), h.size());
    return static_cast<int>(h.size());
  });
}

int hg_engine_attach_replicas(hg_engine* e, const void* handles, int handle_bytes, int nranks) {
  return guard<int>(-1, [&] {
    std::vector<std::vector<char>> hs(nranks);
    const char* p = static_cast<const char*>(handles);
    for (int r = 0; r < nranks; ++r) hs[r].assign(p + static_cast<std::size_t>(r) * handle_bytes,
                                                 p + static_cast<std::size_t>(r + 1) * handle_bytes);
    e->e->attach_replicas(hs);
    return 0;
  });
}

int hg_engine_attach_nccl(hg_engine* e, const void* unique_id, int id_bytes, int nranks, int rank) {
  return guard<int>(-1, [&] {
#ifdef HG_WITH_NCCL
    ncclUniqueId id;
    if (id_bytes != static_cast<int>(sizeof(id))) throw std::invalid_argument("bad unique id size");
    std::memcpy(&id, unique_id, sizeof(id));
    if (ncclCommInitRank(&e->comm, nranks, id, rank) != ncclSuccess) throw std::runtime_error("ncclCommInitRank failed");
    // every rank joins the split (collective); replicas of one sub-metatree set
    // share a colour, the others opt out
    const int color = e->e->replica_color();
    if (ncclCommSplit(e->comm, color >= 0 ? color : NCCL_SPLIT_NOCOLOR, e->e->replica_pos(), &e->rcomm, nullptr) !=
        ncclSuccess)
      throw std::runtime_error("ncclCommSplit failed");
    e->e->attach_comm(e->comm, e->rcomm);
    return 0;
#else
    (void)e;
    (void)unique_id;
    (void)id_bytes;
    (void)nranks;
    (void)rank;
    throw std::runtime_error("built without NCCL");
    return -1;
#endif
  });
}


// ---- model state (init_model / init_learnable, hgnn.cpp:39-81) -------------------------
hg_bundle* hg_init_model(const hg_graph* h, int k, int hidden, uint64_t seed) {
  return guard<hg_bundle*>(nullptr, [&] {
    const Graph& g = h->g;
    const Tree tree = bfs_tree(schema_of(g), g.target, k);
    const ModelInit mi = init_model(g, tree, hidden, seed);
    auto* b = new hg_bundle;
    b->add("input_dims", "<i4", mi.input_dims);
    b->add("k", "<i4", std::vector<int>{mi.k});
    for (const auto& [id, w] : mi.weights)
      b->add("w.r" + std::to_string(id.rel) + ".l" + std::to_string(id.layer), "<f8", w.values,
             {static_cast<long long>(w.in_dim), static_cast<long long>(w.out_dim)});
    return b;
  });
}

hg_bundle* hg_init_learnable(const hg_graph* h, uint64_t seed) {
  return guard<hg_bundle*>(nullptr, [&] {
    const Graph& g = h->g;
    auto* b = new hg_bundle;
    for (auto& [t, v] : init_learnable(g, seed))
      b->add("learn.t" + std::to_string(t), "<f8", v,
             {static_cast<long long>(g.types[t].count), static_cast<long long>(g.types[t].dim)});
    return b;
  });
}

int hg_graph_dense(const hg_graph* h, int type, const float** data, uint64_t* rows, int* dim, int* kind) {
  return guard<int>(-1, [&] {
    const Graph& g = h->g;
    if (type < 0 || type >= g.num_types()) throw std::invalid_argument("unknown node type " + std::to_string(type));
    const NodeTypeInfo& t = g.types[type];
    if (data) *data = t.storage == Storage::Dense ? t.dense.data() : nullptr;
    if (rows) *rows = t.count;
    if (dim) *dim = t.dim;
    if (kind) *kind = static_cast<int>(t.storage);
    return 0;
  });
}

int hg_graph_labels(const hg_graph* h, const int32_t** labels, uint64_t* n) {
  return guard<int>(-1, [&] {
    if (labels) *labels = h->g.labels.data();
    if (n) *n = h->g.labels.size();
    return 0;
  });
}

int hg_engine_load_weights(hg_engine* e, int rel, int layer, const double* w, int din, int dout) {
  return guard<int>(-1, [&] {
    e->e->load_weights(rel, layer, w, din, dout);
    return 0;
  });
}

int hg_engine_load_table_rows(hg_engine* e, int type, const uint32_t* ids, int64_t n, const double* rows, int dim) {
  return guard<int>(-1, [&] {
    e->e->load_table_rows(type, ids, n, rows, dim);
    return 0;
  });
}

// ---- layer interface (hgnn.hpp:76-130) on device tensors ------------------------------------
namespace {
DevTensor dt(const hg_tensor& t) { return DevTensor{t.data, t.rows, t.cols, t.ld}; }
std::vector<DevTensor> dts(const hg_tensor* t, int n) {
  std::vector<DevTensor> v;
  for (int i = 0; i < n; ++i) v.push_back(dt(t[i]));
  return v;
}
AdamHyper hyper(double lr, double b1, double b2, double eps) {
  AdamHyper hp;
  hp.lr = lr;
  hp.beta1 = b1;
  hp.beta2 = b2;
  hp.eps = eps;
  return hp;
}
}  // namespace

hg_ctx* hg_ctx_create(int device) {
  return guard<hg_ctx*>(nullptr, [&] {
    auto* c = new hg_ctx;
    c->c = std::make_unique<LayerCtx>(device);
    return c;
  });
}
void hg_ctx_free(hg_ctx* c) { delete c; }
int hg_ctx_sync(hg_ctx* c) {
  return guard<int>(-1, [&] {
    c->c->sync();
    return 0;
  });
}
void* hg_ctx_malloc(hg_ctx* c, size_t bytes) {
  return guard<void*>(nullptr, [&] {
    HG_CUDA(cudaSetDevice(c->c->device()));
    void* p = nullptr;
    HG_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
    // zero-fill on the context's (non-blocking) stream: ordered before every later
    // primitive and copy on it (a legacy-stream memset would race with them)
    HG_CUDA(cudaMemsetAsync(p, 0, std::max<size_t>(bytes, 16), c->c->stream()));
    return p;
  });
}
int hg_ctx_mfree(hg_ctx* c, void* p) {
  return guard<int>(-1, [&] {
    HG_CUDA(cudaStreamSynchronize(c->c->stream()));
    HG_CUDA(cudaFree(p));
    return 0;
  });
}
int hg_ctx_copy(hg_ctx* c, void* dst, const void* src, size_t bytes) {
  return guard<int>(-1, [&] {
    HG_CUDA(cudaSetDevice(c->c->device()));
    HG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->c->stream()));
    HG_CUDA(cudaStreamSynchronize(c->c->stream()));
    return 0;
  });
}
int hg_rows_in(hg_ctx* c, const uint32_t* ids, int64_t n, const uint32_t* sorted, int64_t n_sorted, uint32_t* rows) {
  return guard<int>(-1, [&] {
    c->c->rows_in(ids, n, sorted, n_sorted, rows);
    return 0;
  });
}
int hg_mean_aggregate(hg_ctx* c, const uint32_t* indptr, int64_t n_dst, const uint32_t* src_rows, hg_tensor h_src,
                      hg_tensor out) {
  return guard<int>(-1, [&] {
    c->c->mean_aggregate(indptr, n_dst, src_rows, dt(h_src), dt(out));
    return 0;
  });
}
int hg_project(hg_ctx* c, const hg_tensor* means, const hg_tensor* ws, int nrel, hg_tensor out, int relu,
               int accumulate) {
  return guard<int>(-1, [&] {
    const auto m = dts(means, nrel), w = dts(ws, nrel);
    c->c->project(m.data(), w.data(), nrel, dt(out), relu != 0, accumulate != 0);
    return 0;
  });
}
int hg_agg_all(hg_ctx* c, const hg_tensor* partials, int n, hg_tensor out) {
  return guard<int>(-1, [&] {
    const auto p = dts(partials, n);
    c->c->agg_all(p.data(), n, dt(out));
    return 0;
  });
}
int hg_relu(hg_ctx* c, hg_tensor x, const hg_tensor* mask) {
  return guard<int>(-1, [&] {
    const DevTensor mk = mask ? dt(*mask) : DevTensor{};
    c->c->relu(dt(x), mask ? &mk : nullptr);
    return 0;
  });
}
int hg_gather_rows(hg_ctx* c, hg_tensor table, const uint32_t* ids, int64_t n, hg_tensor out) {
  return guard<int>(-1, [&] {
    c->c->gather_rows(dt(table), ids, n, dt(out));
    return 0;
  });
}
int hg_cross_entropy(hg_ctx* c, hg_tensor logits, const uint32_t* row_ids, int64_t n_rows, const uint32_t* batch,
                     int64_t n_batch, const int32_t* labels, int64_t n_labels, int num_classes,
                     const hg_tensor* dlogits, double* loss) {
  return guard<int>(-1, [&] {
    const DevTensor dz = dlogits ? dt(*dlogits) : DevTensor{};
    const double l = c->c->cross_entropy(dt(logits), row_ids, n_rows, batch, n_batch, labels, n_labels, num_classes,
                                         dlogits ? &dz : nullptr);
    if (loss) *loss = l;
    return 0;
  });
}
int hg_weight_grad(hg_ctx* c, hg_tensor mean, hg_tensor dpre, hg_tensor dw, int accumulate) {
  return guard<int>(-1, [&] {
    c->c->weight_grad(dt(mean), dt(dpre), dt(dw), accumulate != 0);
    return 0;
  });
}
int hg_mean_grad(hg_ctx* c, hg_tensor dpre, hg_tensor w, const uint32_t* indptr, hg_tensor dmean) {
  return guard<int>(-1, [&] {
    c->c->mean_grad(dt(dpre), dt(w), indptr, dt(dmean));
    return 0;
  });
}
int hg_scatter_rows(hg_ctx* c, const uint32_t* indptr, int64_t n_dst, int64_t n_edges, const uint32_t* src_rows,
                    hg_tensor dmean, hg_tensor dh_src) {
  return guard<int>(-1, [&] {
    c->c->scatter_rows(indptr, n_dst, n_edges, src_rows, dt(dmean), dt(dh_src));
    return 0;
  });
}
int hg_adam_dense(hg_ctx* c, float* w, float* m, float* v, const float* g, int64_t n, int64_t step, double lr,
                  double beta1, double beta2, double eps) {
  return guard<int>(-1, [&] {
    c->c->adam_dense(w, m, v, g, n, step, hyper(lr, beta1, beta2, eps));
    return 0;
  });
}
int hg_adam_rows(hg_ctx* c, hg_tensor w, hg_tensor m, hg_tensor v, const uint32_t* rows, int64_t n, hg_tensor grads,
                 int64_t step, double lr, double beta1, double beta2, double eps) {
  return guard<int>(-1, [&] {
    c->c->adam_rows(dt(w), dt(m), dt(v), rows, n, dt(grads), step, hyper(lr, beta1, beta2, eps));
    return 0;
  });
}

// sample_neighbors (src/sampling.cpp:17-39): copy-all rows on the host, drawn rows on the device
int hg_sample_neighbors(const uint64_t* indptr, uint64_t n_dst, const uint32_t* src, uint32_t dst, int fanout,
                        uint64_t rng_seed, int hop, int rel, uint32_t* out, int* n_out, int device) {
  return guard<int>(-1, [&] {
    if (dst >= n_dst) throw std::invalid_argument("destination id out of range: " + std::to_string(dst));
    if (fanout < 0) throw std::invalid_argument("fanout must be non-negative");
    const std::uint64_t lo = indptr[dst], deg = indptr[dst + 1] - lo;
    if (deg <= static_cast<std::uint64_t>(fanout)) {
      std::copy(src + lo, src + lo + deg, out);
      if (n_out) *n_out = static_cast<int>(deg);
      return 0;
    }
    if (deg > 0xFFFFFFFFull) throw std::invalid_argument("degree beyond the u32 position range");
    HG_CUDA(cudaSetDevice(device));
    const std::uint64_t seed =
        mix_seed(rng_seed, mix_seed((static_cast<std::uint64_t>(hop) << 32) | static_cast<std::uint64_t>(rel), dst));
    std::uint32_t *d_nbr = nullptr, *d_out = nullptr;
    std::uint64_t* d_scr = nullptr;
    HG_CUDA(cudaMalloc(&d_nbr, deg * 4));
    HG_CUDA(cudaMalloc(&d_out, static_cast<std::size_t>(fanout) * 4 + 4));
    HG_CUDA(cudaMalloc(&d_scr, (312 + static_cast<std::size_t>(fanout)) * 8));
    HG_CUDA(cudaMemcpy(d_nbr, src + lo, deg * 4, cudaMemcpyHostToDevice));
    sample_row(d_nbr, deg, fanout, seed, d_out, d_scr, nullptr);
    HG_CUDA(cudaMemcpy(out, d_out, static_cast<std::size_t>(fanout) * 4, cudaMemcpyDeviceToHost));
    cudaFree(d_nbr);
    cudaFree(d_out);
    cudaFree(d_scr);
    if (n_out) *n_out = fanout;
    return 0;
  });
}

}  // extern "C"
