// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the *unmodified* reference library (hetsim, compiled from
// /root/reference/proj/src/*.cpp by oracle/Makefile into oracle/_ref/). It lets
// the Python tests, __graft_entry__.smoke() and bench.py's cpu_baseline leg call
// the reference as the checker. Every result is returned as a "bundle": a
// name -> (dtype, shape, bytes) map that oracle/ref.py turns into numpy arrays.
//
// Reference entry points wrapped (file:line under /root/reference/proj):
//   sample_neighbors / sample_khop / sample_khop_restricted   src/sampling.cpp:17,94,99
//   build_metatree / meta_partition / cacheable_types           src/metapartition.cpp:32,283; src/cache.cpp:143
//   init_model / init_learnable / forward_flat / cross_entropy  src/hgnn.cpp:39,64,215,281
//   backward_flat / adam_update_model / adam_update_rows        src/hgnn.cpp:309,379,392
//   run_raf_batch / check_equivalence                           src/raf.cpp:344,639
//   presample_hotness / allocate_cache / fill_and_serve         src/cache.cpp:39,65,121
//   gen_synthetic / bundled_spec / run_experiment / stats_hash  src/harness.cpp:74,192,342,548
//   random_hetgraph (the reference's own test fixture)          tests/test_util.hpp:17
#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "hetsim/cache.hpp"
#include "hetsim/container.hpp"
#include "hetsim/harness.hpp"
#include "hetsim/hgnn.hpp"
#include "hetsim/metapartition.hpp"
#include "hetsim/raf.hpp"
#include "hetsim/sampling.hpp"
#include "test_util.hpp"

using namespace hetsim;

namespace {

thread_local std::string g_err;

struct Entry {
  std::string dtype;  // numpy dtype string: "<u4", "<u8", "<i4", "<i8", "<f8", "|u1"
  std::vector<long long> shape;
  std::vector<char> data;
};

struct Bundle {
  std::map<std::string, Entry> items;
  std::vector<std::string> order;

  template <typename T>
  void put(const std::string& name, const char* dtype, const std::vector<T>& v,
           std::vector<long long> shape = {}) {
    Entry e;
    e.dtype = dtype;
    e.shape = shape.empty() ? std::vector<long long>{static_cast<long long>(v.size())} : shape;
    e.data.resize(v.size() * sizeof(T));
    if (!v.empty()) std::memcpy(e.data.data(), v.data(), e.data.size());
    if (!items.count(name)) order.push_back(name);
    items[name] = std::move(e);
  }
  void put_u32(const std::string& n, const std::vector<NodeId>& v) { put(n, "<u4", v); }
  void put_i32(const std::string& n, const std::vector<int>& v) { put(n, "<i4", v); }
  void put_u64(const std::string& n, const std::vector<std::uint64_t>& v) { put(n, "<u8", v); }
  void put_f64(const std::string& n, const std::vector<double>& v) { put(n, "<f8", v); }
  void put_scalar_f64(const std::string& n, double x) { put(n, "<f8", std::vector<double>{x}); }
  void put_scalar_i64(const std::string& n, long long x) { put(n, "<i8", std::vector<long long>{x}); }
  void put_matrix(const std::string& n, const Matrix& m) {
    put(n, "<f8", m.data,
        {static_cast<long long>(m.rows), static_cast<long long>(m.cols)});
  }
  void put_string(const std::string& n, const std::string& s) {
    std::vector<char> v(s.begin(), s.end());
    put(n, "|u1", v);
  }
};

template <typename F>
void* guarded(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

std::vector<int> to_vec(const int* p, int n) { return std::vector<int>(p, p + n); }

// hop_relations as a flat list with per-hop counts; counts == nullptr -> unrestricted
std::vector<std::vector<int>> hop_sets(const int* flat, const int* counts, int k) {
  std::vector<std::vector<int>> out(k);
  int off = 0;
  for (int h = 0; h < k; ++h) {
    out[h].assign(flat + off, flat + off + counts[h]);
    off += counts[h];
  }
  return out;
}

void put_blocks(Bundle& b, const SampledBlocks& s, int num_types) {
  b.put_scalar_i64("k", s.k);
  for (int h = 0; h < s.k; ++h) {
    std::vector<int> rels;
    for (std::size_t i = 0; i < s.hops[h].size(); ++i) {
      const Block& blk = s.hops[h][i];
      rels.push_back(blk.rel_index);
      const std::string p = "hop" + std::to_string(h + 1) + ".rel" + std::to_string(blk.rel_index);
      b.put_u32(p + ".dst_ids", blk.dst_ids);
      b.put(p + ".indptr", "<u4", blk.indptr);
      b.put_u32(p + ".src_ids", blk.src_ids);
    }
    b.put_i32("hop" + std::to_string(h + 1) + ".rels", rels);
  }
  for (int h = 0; h <= s.k; ++h)
    for (int t = 0; t < num_types; ++t)
      b.put_u32("frontier" + std::to_string(h) + ".t" + std::to_string(t), s.frontier[h][t]);
}

void put_model(Bundle& b, const HGNNModel& m, const std::string& prefix) {
  for (const auto& [key, w] : m.weights)
    b.put_matrix(prefix + ".r" + std::to_string(key.rel_index) + ".l" + std::to_string(key.layer), w);
}

void put_grads(Bundle& b, const GradientSet& g, const std::string& prefix) {
  for (const auto& [key, w] : g.weight_grads)
    b.put_matrix(prefix + ".w.r" + std::to_string(key.rel_index) + ".l" + std::to_string(key.layer), w);
  for (const auto& [t, fg] : g.feature_grads) {
    b.put_u32(prefix + ".f.t" + std::to_string(t) + ".ids", fg.first);
    b.put_matrix(prefix + ".f.t" + std::to_string(t) + ".rows", fg.second);
  }
}

struct Session {
  HetGraph g;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- bundles ----------------------------------------------------------------
int ref_bundle_size(void* bp) { return static_cast<int>(static_cast<Bundle*>(bp)->order.size()); }
const char* ref_bundle_name(void* bp, int i) { return static_cast<Bundle*>(bp)->order[i].c_str(); }
const char* ref_bundle_dtype(void* bp, int i) {
  auto* b = static_cast<Bundle*>(bp);
  return b->items[b->order[i]].dtype.c_str();
}
int ref_bundle_ndim(void* bp, int i) {
  auto* b = static_cast<Bundle*>(bp);
  return static_cast<int>(b->items[b->order[i]].shape.size());
}
long long ref_bundle_dim(void* bp, int i, int d) {
  auto* b = static_cast<Bundle*>(bp);
  return b->items[b->order[i]].shape[d];
}
long long ref_bundle_nbytes(void* bp, int i) {
  auto* b = static_cast<Bundle*>(bp);
  return static_cast<long long>(b->items[b->order[i]].data.size());
}
const void* ref_bundle_data(void* bp, int i) {
  auto* b = static_cast<Bundle*>(bp);
  return b->items[b->order[i]].data.data();
}
void ref_bundle_free(void* bp) { delete static_cast<Bundle*>(bp); }

// ---- graphs -----------------------------------------------------------------
void* ref_graph_random(unsigned long long seed, int max_types, int max_rels, int max_nodes) {
  return guarded([&]() -> void* {
    auto* s = new Session;
    s->g = testutil::random_hetgraph(seed, max_types, max_rels, static_cast<NodeId>(max_nodes));
    return s;
  });
}

void* ref_graph_bundled(const char* name, unsigned long long seed) {
  return guarded([&]() -> void* {
    auto* s = new Session;
    s->g = gen_synthetic(bundled_spec(name), seed);
    return s;
  });
}

// load_container / save_container (container.cpp:47-154)
void* ref_graph_load(const char* path) {
  return guarded([&]() -> void* {
    auto* s = new Session;
    s->g = load_container(path);
    return s;
  });
}

void* ref_graph_save(void* sp, const char* path) {
  return guarded([&]() -> void* {
    save_container(static_cast<Session*>(sp)->g, path);
    auto* b = new Bundle;
    b->put_u64("ok", std::vector<std::uint64_t>{1});
    return b;
  });
}

void* ref_graph_spec(const char* spec_json, unsigned long long seed) {
  return guarded([&]() -> void* {
    auto* s = new Session;
    s->g = gen_synthetic(parse_spec(nlohmann::json::parse(spec_json)), seed);
    return s;
  });
}

// build_hetgraph from per-relation (src,dst) pairs, then attach features:
// kinds[t] in {0 absent,1 dense,2 learnable}; dense values as f64 row-major.
void* ref_graph_build(int num_types, const unsigned long long* counts, int num_rels,
                      const int* rel_src, const int* rel_dst, const unsigned long long* edge_counts,
                      const unsigned* edge_src, const unsigned* edge_dst, int target,
                      int num_classes, const int* labels, const int* kinds, const int* dims,
                      const double* dense_values) {
  return guarded([&]() -> void* {
    TypeRegistry reg;
    for (int t = 0; t < num_types; ++t) reg.add_node_type("t" + std::to_string(t));
    std::vector<std::uint64_t> cnt(counts, counts + num_types);
    std::vector<Relation> rels;
    std::vector<std::vector<std::pair<NodeId, NodeId>>> edges(num_rels);
    std::size_t off = 0;
    for (int r = 0; r < num_rels; ++r) {
      rels.push_back({rel_src[r], reg.add_edge_type("e" + std::to_string(r)), rel_dst[r]});
      for (unsigned long long e = 0; e < edge_counts[r]; ++e, ++off)
        edges[r].push_back({edge_src[off], edge_dst[off]});
    }
    auto* s = new Session;
    s->g = build_hetgraph(std::move(reg), cnt, std::move(rels), edges, target, num_classes);
    std::size_t voff = 0;
    for (int t = 0; t < num_types; ++t) {
      TypeFeatures& f = s->g.features[t];
      f.dim = dims[t];
      f.kind = kinds[t] == 1 ? StorageKind::Dense
                             : (kinds[t] == 2 ? StorageKind::Learnable : StorageKind::Absent);
      if (f.kind == StorageKind::Dense) {
        f.values = Matrix(cnt[t], static_cast<std::size_t>(dims[t]));
        for (double& x : f.values.data) x = dense_values[voff++];
      }
    }
    s->g.labels.assign(labels, labels + cnt[target]);
    return s;
  });
}

void ref_graph_free(void* sp) { delete static_cast<Session*>(sp); }

// Rounds every dense feature value to the nearest fp16 (mode 1) or bf16 (mode 2)
// value, in place: the "parity mode" inputs of SURVEY §7 (fp16-representable features
// travel losslessly through a half-precision device table).
void* ref_graph_round_features(void* sp, int mode) {
  return guarded([&]() -> void* {
    HetGraph& g = static_cast<Session*>(sp)->g;
    auto round_f16 = [](double x) {
      // IEEE binary16, round to nearest even, via its 11-bit significand (normals;
      // |x| <= 1 here so no overflow; subnormals below 2^-14 use the fixed 2^-24 step)
      const double a = std::fabs(x);
      if (a == 0.0) return x;
      int e;
      std::frexp(a, &e);                       // a = m * 2^e, m in [0.5, 1)
      const int q = std::max(e - 11, -24);     // ulp exponent
      const double ulp = std::ldexp(1.0, q);
      const double r = std::nearbyint(a / ulp) * ulp;  // default rounding mode: to nearest even
      return x < 0 ? -r : r;
    };
    auto round_bf16 = [](double x) {
      float f = static_cast<float>(x);  // the engine rounds the f32 table value
      std::uint32_t u;
      std::memcpy(&u, &f, 4);
      u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
      std::memcpy(&f, &u, 4);
      return static_cast<double>(f);
    };
    for (auto& f : g.features) {
      if (f.kind != StorageKind::Dense) continue;
      for (double& x : f.values.data) {
        const double xf = static_cast<double>(static_cast<float>(x));  // the engine's f32 source value
        x = mode == 1 ? round_f16(xf) : round_bf16(xf);
      }
    }
    return new Bundle;
  });
}

void* ref_graph_export(void* sp) {
  return guarded([&]() -> void* {
    const HetGraph& g = static_cast<Session*>(sp)->g;
    auto* b = new Bundle;
    const int nt = g.reg.num_node_types();
    b->put_u64("node_counts", g.node_counts);
    b->put_scalar_i64("target", g.target);
    b->put_scalar_i64("num_classes", g.num_classes);
    b->put("labels", "<i4", g.labels);
    std::vector<int> rs, re, rd, rev;
    for (std::size_t r = 0; r < g.relations.size(); ++r) {
      rs.push_back(g.relations[r].src);
      re.push_back(g.relations[r].etype);
      rd.push_back(g.relations[r].dst);
      rev.push_back(g.is_reverse[r] ? 1 : 0);
      b->put_u64("rel" + std::to_string(r) + ".indptr", g.adj[r].indptr);
      b->put_u32("rel" + std::to_string(r) + ".src", g.adj[r].src);
    }
    b->put_i32("rel_src", rs);
    b->put_i32("rel_etype", re);
    b->put_i32("rel_dst", rd);
    b->put_i32("rel_reverse", rev);
    std::vector<int> kinds, dims;
    for (int t = 0; t < nt; ++t) {
      kinds.push_back(static_cast<int>(g.features[t].kind));
      dims.push_back(g.features[t].dim);
      if (g.features[t].kind == StorageKind::Dense)
        b->put_matrix("feat.t" + std::to_string(t), g.features[t].values);
    }
    b->put_i32("kinds", kinds);
    b->put_i32("dims", dims);
    std::string names;
    for (int t = 0; t < nt; ++t) names += (t ? "," : "") + g.reg.node_type_names[t];
    b->put_string("type_names", names);
    std::string enames;
    for (std::size_t e = 0; e < g.reg.edge_type_names.size(); ++e)
      enames += (e ? "," : "") + g.reg.edge_type_names[e];
    b->put_string("etype_names", enames);
    return b;
  });
}

// ---- metatree / partitioning -----------------------------------------------
void* ref_meta_partition(void* sp, int k, int p) {
  return guarded([&]() -> void* {
    const HetGraph& g = static_cast<Session*>(sp)->g;
    const Metagraph m = build_metagraph(g);
    const PartitionPlan plan = meta_partition(m, g.target, k, p);
    auto* b = new Bundle;
    std::vector<int> ty, de, pa, re;
    for (const auto& pos : plan.tree.pos) {
      ty.push_back(pos.type);
      de.push_back(pos.depth);
      pa.push_back(pos.parent);
      re.push_back(pos.rel_index);
    }
    b->put_i32("tree.type", ty);
    b->put_i32("tree.depth", de);
    b->put_i32("tree.parent", pa);
    b->put_i32("tree.rel", re);
    std::vector<int> sub_child;
    std::vector<std::uint64_t> sub_w;
    for (const auto& s : plan.subs) {
      sub_child.push_back(s.child_pos);
      sub_w.push_back(s.weight);
    }
    b->put_i32("subs.child_pos", sub_child);
    b->put_u64("subs.weight", sub_w);
    for (std::size_t i = 0; i < plan.parts.size(); ++i) {
      const auto& part = plan.parts[i];
      const std::string pre = "part" + std::to_string(i);
      b->put_i32(pre + ".sub_ids", part.sub_ids);
      b->put_i32(pre + ".relations", part.relations);
      b->put_i32(pre + ".node_types", part.node_types);
      b->put_i32(pre + ".cacheable", cacheable_types(plan, static_cast<int>(i)));
      b->put_i32(pre + ".replica",
                 {part.replica ? 1 : 0, part.replica_index, part.replica_count});
      b->put_u64(pre + ".weight", {part.weight});
      b->put_u32(pre + ".boundary", boundary_nodes(g, plan, static_cast<int>(i)));
    }
    b->put_scalar_i64("p", plan.p);
    const auto hr = hop_relation_sets(plan.tree, k);
    for (int h = 0; h < k; ++h) b->put_i32("hop_rels" + std::to_string(h + 1), hr[h]);
    return b;
  });
}

// ---- sampling ----------------------------------------------------------------
void* ref_sample_neighbors(const unsigned long long* indptr, int n_dst, const unsigned* src,
                           unsigned dst, int fanout, unsigned long long rng_seed, int hop, int rel) {
  return guarded([&]() -> void* {
    Csr a;
    a.indptr.assign(indptr, indptr + n_dst + 1);
    a.src.assign(src, src + indptr[n_dst]);
    auto* b = new Bundle;
    b->put_u32("out", sample_neighbors(a, dst, fanout, rng_seed, hop, rel));
    return b;
  });
}

// hop_counts == nullptr -> sample_khop (unrestricted)
void* ref_sample_khop(void* sp, const unsigned* seeds, int n_seeds, const int* fanouts, int k,
                      unsigned long long rng_seed, const int* hop_flat, const int* hop_counts) {
  return guarded([&]() -> void* {
    const HetGraph& g = static_cast<Session*>(sp)->g;
    std::vector<NodeId> sd(seeds, seeds + n_seeds);
    const auto fo = to_vec(fanouts, k);
    SampledBlocks s = hop_counts ? sample_khop_restricted(g, sd, fo, rng_seed,
                                                          hop_sets(hop_flat, hop_counts, k))
                                 : sample_khop(g, sd, fo, rng_seed);
    auto* b = new Bundle;
    put_blocks(*b, s, g.reg.num_node_types());
    return b;
  });
}

unsigned long long ref_mix_seed(unsigned long long a, unsigned long long b) { return mix_seed(a, b); }

// ---- numerics: one flat training step on the BFS metatree --------------------
// Returns the initial model/learnable state, the sampled blocks, the forward tape
// (per-depth H), logits, loss, dlogits, gradients and post-Adam parameters.
void* ref_flat_step(void* sp, int k, int hidden, unsigned long long model_seed,
                    unsigned long long learn_seed, const unsigned* batch, int n_batch,
                    const int* fanouts, unsigned long long rng_seed, int want_init) {
  return guarded([&]() -> void* {
    const HetGraph& g = static_cast<Session*>(sp)->g;
    const Metatree tree = build_metatree(build_metagraph(g), g.target, k);
    HGNNModel model = init_model(g, tree, hidden, model_seed);
    LearnableStore store = init_learnable(g, learn_seed);
    std::vector<NodeId> bt(batch, batch + n_batch);
    std::vector<NodeId> ids(bt);
    std::sort(ids.begin(), ids.end());
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    const auto fo = to_vec(fanouts, k);
    const SampledBlocks blocks =
        sample_khop_restricted(g, ids, fo, rng_seed, hop_relation_sets(tree, k));
    auto [logits, tape] = forward_flat(g, tree, blocks, model, store);
    Matrix dlogits;
    const double loss = cross_entropy(logits, blocks.frontier[0][g.target], bt, g.labels,
                                      g.num_classes, &dlogits);
    GradientSet grads = backward_flat(g, tree, model, tape, dlogits);

    // want_init: 0 = no initial state, 1 = full learnable tables, 2 = learnable
    // tables only at the rows this batch touches (the gradient ids): the
    // ogbn-mag-shaped tables are ~0.6 GB each in f64.
    const bool rows_only = want_init == 2;
    auto rows_of = [](const Matrix& m, const std::vector<NodeId>& ids) {
      Matrix r(ids.size(), m.cols);
      for (std::size_t i = 0; i < ids.size(); ++i)
        for (std::size_t c = 0; c < m.cols; ++c) r.at(i, c) = m.at(ids[i], c);
      return r;
    };
    auto* b = new Bundle;
    if (want_init) {
      put_model(*b, model, "init");
      for (const auto& [t, tab] : store.tables) {
        if (!rows_only) {
          b->put_matrix("init.learn.t" + std::to_string(t), tab.w);
        } else if (grads.feature_grads.count(t)) {
          b->put_matrix("init.learn_rows.t" + std::to_string(t),
                        rows_of(tab.w, grads.feature_grads.at(t).first));
        }
      }
    }
    put_blocks(*b, blocks, g.reg.num_node_types());
    for (int d = 0; d <= k; ++d)
      for (const auto& [t, h] : tape.H[d])
        b->put_matrix("H" + std::to_string(d) + ".t" + std::to_string(t), h);
    for (const auto& e : tape.entries)
      b->put_matrix("mean.l" + std::to_string(e.layer) + ".r" + std::to_string(e.rel_index) + ".t" +
                        std::to_string(e.dst_type),
                    e.mean);
    b->put_matrix("logits", logits);
    b->put_scalar_f64("loss", loss);
    b->put_matrix("dlogits", dlogits);
    put_grads(*b, grads, "grad");

    ModelAdamState st;
    adam_update_model(model, st, grads);
    for (const auto& [t, fg] : grads.feature_grads)
      adam_update_rows(store.tables.at(t), fg.first, fg.second);
    put_model(*b, model, "post");
    for (const auto& [t, tab] : store.tables) {
      if (rows_only) {
        if (!grads.feature_grads.count(t)) continue;
        const auto& ids = grads.feature_grads.at(t).first;
        b->put_matrix("post.learn_rows.t" + std::to_string(t), rows_of(tab.w, ids));
        b->put_matrix("post.learn_m_rows.t" + std::to_string(t), rows_of(tab.m, ids));
        b->put_matrix("post.learn_v_rows.t" + std::to_string(t), rows_of(tab.v, ids));
        b->put_scalar_i64("post.learn_step.t" + std::to_string(t), tab.step);
        continue;
      }
      b->put_matrix("post.learn.t" + std::to_string(t), tab.w);
      b->put_matrix("post.learn_m.t" + std::to_string(t), tab.m);
      b->put_matrix("post.learn_v.t" + std::to_string(t), tab.v);
      b->put_scalar_i64("post.learn_step.t" + std::to_string(t), tab.step);
    }
    return b;
  });
}

// ---- RAF engine: several consecutive training batches through run_raf_batch ---
// Mirrors the hot loop of run_experiment (harness.cpp:400-423): per batch the
// rng seed is mix_seed(seed, 0xb000 + counter) and designated = counter % p.
// The batches are given explicitly (flat + counts).
void* ref_raf_train(void* sp, int k, int hidden, int p, unsigned long long seed,
                    const unsigned* batches_flat, const int* batch_counts, int n_batches,
                    const int* fanouts, int elem_bytes, int full_tables) {
  return guarded([&]() -> void* {
    const HetGraph& g = static_cast<Session*>(sp)->g;
    const Metagraph m = build_metagraph(g);
    const Metatree tree = build_metatree(m, g.target, k);
    const PartitionPlan plan = meta_partition(m, g.target, k, p);
    const RafPlanView view = raf_view_from_plan(plan);
    HGNNModel model = init_model(g, tree, hidden, mix_seed(seed, 0xd0de1ULL));
    LearnableStore store = init_learnable(g, mix_seed(seed, 0x1ea4aULL));
    ModelAdamState mst;
    const AccountingModel acct{32, 8, elem_bytes};
    const auto fo = to_vec(fanouts, k);
    auto* b = new Bundle;
    std::vector<double> losses;
    std::vector<std::uint64_t> bytes, sync, bound_ok, target_ok;
    const int n_rel = static_cast<int>(g.relations.size());
    int off = 0;
    for (int i = 0; i < n_batches; ++i) {
      std::vector<NodeId> batch(batches_flat + off, batches_flat + off + batch_counts[i]);
      off += batch_counts[i];
      const std::uint64_t rng_seed = mix_seed(seed, 0xb000ULL + i);
      ExecutionReport rep = run_raf_batch(g, view, model, store, batch, fo, rng_seed, i % p, acct);
      losses.push_back(rep.loss);
      bytes.push_back(rep.stats.total_bytes());
      sync.push_back(rep.sync_bytes);
      const CommBoundVerdict v = check_comm_bounds(rep, n_rel, view.meta);  // as harness.cpp:411
      bound_ok.push_back(v.message_bound_ok ? 1 : 0);
      target_ok.push_back(v.target_only_ok ? 1 : 0);
      if (i == 0) {
        b->put_u64("boundary_counts", rep.boundary_counts);
        b->put_u64("boundary_cut_edges", {rep.boundary_cut_edges});
        b->put_matrix("b0.logits", rep.logits);
        put_grads(*b, rep.grads, "b0.grad");
        std::vector<std::uint64_t> dirs;
        for (const auto& [key, e] : rep.stats.per_direction) {
          dirs.push_back(static_cast<std::uint64_t>(std::get<0>(key)));
          dirs.push_back(static_cast<std::uint64_t>(std::get<1>(key)));
          dirs.push_back(static_cast<std::uint64_t>(std::get<2>(key)));
          dirs.push_back(e.count);
          dirs.push_back(e.bytes);
        }
        b->put_u64("b0.comm", dirs);
      }
      adam_update_model(model, mst, rep.grads);
      for (const auto& [t, fg] : rep.grads.feature_grads)
        adam_update_rows(store.tables.at(t), fg.first, fg.second);
    }
    b->put_f64("losses", losses);
    b->put_u64("bytes", bytes);
    b->put_u64("sync_bytes", sync);
    b->put_u64("message_bound_ok", bound_ok);
    b->put_u64("target_only_ok", target_ok);
    put_model(*b, model, "final");
    for (const auto& [t, tab] : store.tables) {
      if (full_tables) b->put_matrix("final.learn.t" + std::to_string(t), tab.w);
      b->put_scalar_i64("final.learn_step.t" + std::to_string(t), tab.step);
    }
    b->put_scalar_i64("final.model_step", mst.step);
    return b;
  });
}

// check_equivalence (raf.cpp:639): RAF vs flat on one batch
void* ref_check_equivalence(void* sp, int k, int hidden, int p, unsigned long long model_seed,
                            unsigned long long learn_seed, const unsigned* batch, int n_batch,
                            const int* fanouts, unsigned long long rng_seed, int designated) {
  return guarded([&]() -> void* {
    const HetGraph& g = static_cast<Session*>(sp)->g;
    const Metagraph m = build_metagraph(g);
    const PartitionPlan plan = meta_partition(m, g.target, k, p);
    const HGNNModel model = init_model(g, plan.tree, hidden, model_seed);
    const LearnableStore store = init_learnable(g, learn_seed);
    std::vector<NodeId> bt(batch, batch + n_batch);
    auto eq = check_equivalence(g, raf_view_from_plan(plan), model, store, bt, to_vec(fanouts, k),
                                rng_seed, designated);
    auto* b = new Bundle;
    b->put_scalar_f64("logit_diff", eq.logit_diff);
    b->put_scalar_f64("grad_diff", eq.grad_diff);
    return b;
  });
}

// ---- cache -------------------------------------------------------------------
void* ref_cache_sim(void* sp, int k, const int* fanouts, int epochs, unsigned long long seed,
                    int batch_size, unsigned long long budget, double read_ns, double write_ns,
                    double overhead_ns, int elem_bytes) {
  return guarded([&]() -> void* {
    const HetGraph& g = static_cast<Session*>(sp)->g;
    const Metatree tree = build_metatree(build_metagraph(g), g.target, k);
    const auto fo = to_vec(fanouts, k);
    const HotnessTable hot =
        presample_hotness(g, tree, fo, epochs, seed, static_cast<std::size_t>(batch_size));
    auto* b = new Bundle;
    for (std::size_t t = 0; t < hot.counts.size(); ++t)
      b->put_u64("hot.t" + std::to_string(t), hot.counts[t]);
    CostModel cm;
    cm.read_ns_per_byte = read_ns;
    cm.write_ns_per_byte = write_ns;
    cm.fixed_overhead_ns = overhead_ns;
    cm.elem_bytes = elem_bytes;
    const MissPenaltyProfile prof = profile_miss_penalty(g, cm);
    std::vector<double> ratio, tns;
    std::vector<std::uint64_t> rb;
    for (const auto& tp : prof.types) {
      ratio.push_back(tp.ratio);
      tns.push_back(tp.transfer_ns);
      rb.push_back(tp.record_bytes);
    }
    b->put_f64("profile.ratio", ratio);
    b->put_f64("profile.transfer_ns", tns);
    b->put_u64("profile.record_bytes", rb);
    if (budget > 0) {
      const CacheAllocation alloc = allocate_cache(budget, hot, prof);
      b->put_u64("alloc.bytes", alloc.bytes);
      b->put_u64("alloc.capacity", alloc.capacity);
      const CacheState cs = fill_and_serve(alloc, hot, prof);
      for (std::size_t t = 0; t < cs.types.size(); ++t)
        b->put_u32("cached.t" + std::to_string(t), cs.types[t].cached);
    }
    return b;
  });
}

// ---- harness -----------------------------------------------------------------
void* ref_run_experiment(const char* config_json) {
  return guarded([&]() -> void* {
    const ExperimentConfig cfg = config_from_json(nlohmann::json::parse(config_json));
    ExperimentResult res = run_experiment(cfg);
    auto* b = new Bundle;
    b->put_string("stats", res.stats.dump());
    b->put_string("hash", stats_hash(res.stats));
    b->put_scalar_i64("checks_ok", res.checks_ok ? 1 : 0);
    return b;
  });
}

// ---- CPU baseline timing ------------------------------------------------------
// Runs `n_threads` independent run_raf_batch calls (disjoint batches of the
// shuffled target order, exactly as make_batches builds them) concurrently and
// reports wall seconds and total sampled edges. The reference is single
// threaded; concurrency comes from independent batches.
void* ref_bench_raf(void* sp, int k, int hidden, int p, unsigned long long seed, int batch_size,
                    const int* fanouts, int first_batch, int n_batches, int n_threads) {
  return guarded([&]() -> void* {
    const HetGraph& g = static_cast<Session*>(sp)->g;
    const Metagraph m = build_metagraph(g);
    const PartitionPlan plan = meta_partition(m, g.target, k, p);
    const RafPlanView view = raf_view_from_plan(plan);
    const HGNNModel model = init_model(g, plan.tree, hidden, mix_seed(seed, 0xd0de1ULL));
    const LearnableStore store = init_learnable(g, mix_seed(seed, 0x1ea4aULL));
    std::vector<NodeId> order(g.node_counts[g.target]);
    std::iota(order.begin(), order.end(), 0);
    std::mt19937_64 rng(mix_seed(seed, 0xba7cULL));
    std::shuffle(order.begin(), order.end(), rng);
    const auto fo = to_vec(fanouts, k);
    std::vector<std::uint64_t> edges(n_batches, 0);
    std::vector<double> losses(n_batches, 0.0);
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int w = 0; w < n_threads; ++w)
      pool.emplace_back([&, w]() {
        for (int i = w; i < n_batches; i += n_threads) {
          const int bi = first_batch + i;
          const std::size_t lo = static_cast<std::size_t>(bi) * batch_size;
          if (lo >= order.size()) continue;
          const std::size_t hi = std::min(order.size(), lo + static_cast<std::size_t>(batch_size));
          std::vector<NodeId> batch(order.begin() + lo, order.begin() + hi);
          const std::uint64_t rs = mix_seed(seed, 0xb000ULL + bi);
          ExecutionReport rep = run_raf_batch(g, view, model, store, batch, fo, rs, bi % p);
          losses[i] = rep.loss;
        }
      });
    for (auto& t : pool) t.join();
    const double secs =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    // sampled edges = Block::src_ids entries of the flat sample (BFS mode),
    // counted outside the timed region
    for (int i = 0; i < n_batches; ++i) {
      const int bi = first_batch + i;
      const std::size_t lo = static_cast<std::size_t>(bi) * batch_size;
      if (lo >= order.size()) continue;
      const std::size_t hi = std::min(order.size(), lo + static_cast<std::size_t>(batch_size));
      std::vector<NodeId> ids(order.begin() + lo, order.begin() + hi);
      std::sort(ids.begin(), ids.end());
      ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
      const SampledBlocks s = sample_khop_restricted(g, ids, fo, mix_seed(seed, 0xb000ULL + bi),
                                                     hop_relation_sets(plan.tree, k));
      std::uint64_t e = 0;
      for (const auto& hop : s.hops)
        for (const auto& blk : hop) e += blk.src_ids.size();
      edges[i] = e;
    }
    auto* b = new Bundle;
    b->put_scalar_f64("seconds", secs);
    b->put_u64("edges", edges);
    b->put_f64("losses", losses);
    return b;
  });
}

}  // extern "C"
