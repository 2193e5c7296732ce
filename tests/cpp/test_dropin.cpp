// C++ drop-in parity test: the reference library (hetsim, compiled from
// /root/reference/proj by oracle/Makefile) and the B200 path (libhetgpu.so via
// include/hetsim_b200.hpp) called side by side through their C++ APIs, the way
// a hetsim user would switch. TEST INFRASTRUCTURE: links the oracle as the
// checker only. Mirrors reference tests:
//   tests/test_sampling.cpp:12-117  (copy-all, determinism, frontiers, restricted == full, errors)
//   tests/test_raf.cpp:35-64         (RAF batch vs the reference's run_raf_batch)
//   tests/acceptance.cpp:336-348     (determinism)
//   tests/test_hgnn.cpp:11-175       (mean/agg_relation/agg_all, CE, backward, Adam) through the
//                                    layer interface (hgnn.hpp:76-130) on the same inputs
//   tests/test_cache.cpp:35-217      (penalty, hotness, allocation, fill, lookup/update, types)
//   raf.hpp:79-103                   (run_raf_batch with caller-owned state at p = 1, 2, 4;
//                                    check_equivalence)
// Prints one line per check; exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <set>
#include <string>
#include <vector>

#include "hetsim/cache.hpp"
#include "hetsim/harness.hpp"
#include "hetsim/hgnn.hpp"
#include "hetsim/metapartition.hpp"
#include "hetsim/raf.hpp"
#include "hetsim/sampling.hpp"
#include "hetsim_b200.hpp"
#include "test_util.hpp"

namespace R = hetsim;       // the reference (oracle)
namespace B = hetsim_b200;  // the B200 path

static int g_fail = 0, g_pass = 0;
#define EXPECT(cond, what)                                        \
  do {                                                            \
    if (cond) {                                                   \
      ++g_pass;                                                   \
    } else {                                                      \
      ++g_fail;                                                   \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, what);   \
    }                                                             \
  } while (0)

// the reference graph handed to the B200 path in CSR form (hetgraph.hpp:41-74)
static B::HetGraph to_b200(const R::HetGraph& g) {
  const int nt = g.reg.num_node_types(), nr = static_cast<int>(g.relations.size());
  std::vector<int> rs, rd, rr, kinds, dims;
  std::vector<std::uint64_t> ip;
  std::vector<std::uint32_t> src;
  std::vector<float> dense;
  for (int r = 0; r < nr; ++r) {
    rs.push_back(g.relations[r].src);
    rd.push_back(g.relations[r].dst);
    rr.push_back(g.is_reverse.empty() ? 0 : static_cast<int>(g.is_reverse[r]));
    ip.insert(ip.end(), g.adj[r].indptr.begin(), g.adj[r].indptr.end());
    src.insert(src.end(), g.adj[r].src.begin(), g.adj[r].src.end());
  }
  for (int t = 0; t < nt; ++t) {
    const auto& f = g.features[t];
    kinds.push_back(f.kind == R::StorageKind::Dense ? 1 : f.kind == R::StorageKind::Learnable ? 2 : 0);
    dims.push_back(f.dim);
    if (f.kind == R::StorageKind::Dense)
      for (double x : f.values.data) dense.push_back(static_cast<float>(x));
  }
  if (src.empty()) src.push_back(0);
  if (dense.empty()) dense.push_back(0.f);
  return B::HetGraph(hg_graph_from_csr(nt, g.node_counts.data(), nr, rs.data(), rd.data(), rr.data(), ip.data(),
                                       src.data(), kinds.data(), dims.data(), dense.data(), g.target,
                                       g.num_classes, g.labels.data()));
}

static bool same_blocks(const R::SampledBlocks& a, const B::SampledBlocks& b) {
  if (a.k != b.k || a.hops.size() != b.hops.size()) return false;
  for (std::size_t h = 0; h < a.hops.size(); ++h) {
    if (a.hops[h].size() != b.hops[h].size()) return false;
    for (std::size_t i = 0; i < a.hops[h].size(); ++i) {
      const auto& x = a.hops[h][i];
      const auto& y = b.hops[h][i];
      if (x.rel_index != y.rel_index || x.hop != y.hop || x.dst_ids != y.dst_ids || x.indptr != y.indptr ||
          x.src_ids != y.src_ids)
        return false;
    }
  }
  for (std::size_t h = 0; h < a.frontier.size(); ++h)
    for (std::size_t t = 0; t < a.frontier[h].size(); ++t)
      if (a.frontier[h][t] != b.frontier[h][t]) return false;
  return true;
}

// ---- reference <-> mirror conversions for the layer interface ------------------------------------
static B::Matrix bm(const R::Matrix& m) {
  B::Matrix o(m.rows, m.cols);
  o.data = m.data;
  return o;
}
static double rel_err(const B::Matrix& a, const R::Matrix& b) {
  if (a.rows != b.rows || a.cols != b.cols) return 1e30;
  double m = 0, r = 1e-30;
  for (std::size_t i = 0; i < a.data.size(); ++i) {
    m = std::max(m, std::fabs(a.data[i] - b.data[i]));
    r = std::max(r, std::fabs(b.data[i]));
  }
  return m / r;
}
static B::Metatree btree(const R::Metatree& t) {
  B::Metatree o;
  o.k = t.k;
  for (const auto& p : t.pos) o.pos.push_back({p.type, p.depth, p.parent, p.rel_index});
  return o;
}
static B::SampledBlocks bblocks(const R::SampledBlocks& s) {
  B::SampledBlocks o;
  o.k = s.k;
  o.seeds = s.seeds;
  o.rng_seed = s.rng_seed;
  o.frontier = s.frontier;
  o.hops.resize(s.hops.size());
  for (std::size_t h = 0; h < s.hops.size(); ++h)
    for (const auto& b : s.hops[h]) o.hops[h].push_back({b.rel_index, b.hop, b.dst_ids, b.indptr, b.src_ids});
  return o;
}
static B::HGNNModel bmodel(const R::HGNNModel& m) {
  B::HGNNModel o;
  o.k = m.k;
  o.hidden = m.hidden;
  o.num_classes = m.num_classes;
  o.input_dims = m.input_dims;
  for (const auto& [key, w] : m.weights) o.weights.emplace(B::SlotKey{key.rel_index, key.layer}, bm(w));
  return o;
}
static B::LearnableStore bstore(const R::LearnableStore& s) {
  B::LearnableStore o;
  for (const auto& [t, tab] : s.tables) {
    B::LearnableFeatureTable b;
    b.w = bm(tab.w);
    b.m = bm(tab.m);
    b.v = bm(tab.v);
    b.step = tab.step;
    o.tables.emplace(t, std::move(b));
  }
  return o;
}
static double grad_rel(const B::GradientSet& a, const R::GradientSet& b) {
  double m = 0, r = 1e-30;
  for (const auto& [key, w] : b.weight_grads) {
    auto it = a.weight_grads.find(B::SlotKey{key.rel_index, key.layer});
    if (it == a.weight_grads.end()) return 1e30;
    for (std::size_t i = 0; i < w.data.size(); ++i) {
      m = std::max(m, std::fabs(it->second.data[i] - w.data[i]));
      r = std::max(r, std::fabs(w.data[i]));
    }
  }
  for (const auto& [t, fg] : b.feature_grads) {
    auto it = a.feature_grads.find(t);
    if (it == a.feature_grads.end() || it->second.first != fg.first) return 1e30;
    for (std::size_t i = 0; i < fg.second.data.size(); ++i) {
      m = std::max(m, std::fabs(it->second.second.data[i] - fg.second.data[i]));
      r = std::max(r, std::fabs(fg.second.data[i]));
    }
  }
  return m / r;
}
// post-Adam parameters: elements with a gradient at fp32 rounding level may take the
// opposite +-lr step (at most 0.2% of them, each within 2 lr); the rest within 1e-3
static bool adam_close(const std::vector<double>& a, const std::vector<double>& b, double lr = 1e-2) {
  double scale = 1e-12;
  for (double x : b) scale = std::max(scale, std::fabs(x));
  std::size_t bad = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    const double d = std::fabs(a[i] - b[i]);
    if (d > 1e-3 * scale) {
      ++bad;
      if (d > 2 * lr * 1.01) return false;
    }
  }
  return bad <= a.size() / 500;
}
static B::SyntheticSpec bspec(const R::SyntheticSpec& rs) {
  B::SyntheticSpec bs;
  bs.name = rs.name;
  bs.target = rs.target;
  bs.num_classes = rs.num_classes;
  bs.label_noise = rs.label_noise;
  for (const auto& t : rs.node_types) bs.node_types.push_back({t.name, t.count, t.dim, t.storage});
  for (const auto& r : rs.relations) bs.relations.push_back({r.src, r.edge, r.dst, r.edges, r.degree, r.alpha});
  bs.add_reverse = rs.add_reverse;
  bs.self_paired = rs.self_paired;
  return bs;
}

int main() {
  // test_sampling.cpp:12-18 — copy-all rows keep CSR order; :20-33 determinism
  {
    std::vector<std::uint64_t> counts = {2, 20};
    std::vector<std::vector<std::pair<B::NodeId, B::NodeId>>> edges(1);
    for (B::NodeId i = 0; i < 3; ++i) edges[0].push_back({std::vector<B::NodeId>{7, 5, 9}[i], 0});
    for (B::NodeId i = 0; i < 20; ++i) edges[0].push_back({i, 1});
    B::HetGraph g = B::build_hetgraph(counts, {{1, 0}}, edges, 0, 2);
    std::vector<B::NodeId> seeds = {0};
    auto s = B::sample_khop(g, seeds, {3}, 42);
    EXPECT(s.hops[0].size() == 1 && s.hops[0][0].src_ids == (std::vector<B::NodeId>{7, 5, 9}), "copy-all row in CSR order");
    std::vector<B::NodeId> s1 = {1};
    auto a = B::sample_khop(g, s1, {8}, 42), b = B::sample_khop(g, s1, {8}, 42), c = B::sample_khop(g, s1, {8}, 43);
    EXPECT(a.hops[0][0].src_ids == b.hops[0][0].src_ids, "identical seeds give identical draws");
    EXPECT(std::set<B::NodeId>(a.hops[0][0].src_ids.begin(), a.hops[0][0].src_ids.end()).size() == 8, "no replacement");
    EXPECT(a.hops[0][0].src_ids != c.hops[0][0].src_ids, "seed changes the draw");
  }

  // random graphs (test_util.hpp:17-75): full and restricted samples bit-exact vs the reference,
  // and restricted rows == full rows (test_sampling.cpp:73-109)
  for (std::uint64_t s = 10; s < 30; ++s) {
    R::HetGraph rg = testutil::random_hetgraph(s);
    B::HetGraph bg = to_b200(rg);
    std::vector<R::NodeId> seeds;
    for (R::NodeId v = 0; v < std::min<R::NodeId>(7, rg.node_counts[rg.target]); ++v) seeds.push_back(v % 5);
    const std::uint64_t rs = s * 31 + 1;
    auto full_r = R::sample_khop(rg, seeds, {3, 3}, rs);
    auto full_b = B::sample_khop(bg, seeds, {3, 3}, rs);
    EXPECT(same_blocks(full_r, full_b), ("sample_khop bit-exact, graph " + std::to_string(s)).c_str());
    std::vector<std::vector<int>> subset(2);
    for (std::size_t r = 0; r < rg.relations.size(); r += 2) {
      subset[0].push_back(static_cast<int>(r));
      subset[1].push_back(static_cast<int>(r));
    }
    auto part_r = R::sample_khop_restricted(rg, seeds, {3, 3}, rs, subset);
    auto part_b = B::sample_khop_restricted(bg, seeds, {3, 3}, rs, subset);
    EXPECT(same_blocks(part_r, part_b), ("sample_khop_restricted bit-exact, graph " + std::to_string(s)).c_str());
    for (const auto& pb : part_b.hops[0]) {
      const B::Block* fb = nullptr;
      for (const auto& cand : full_b.hops[0])
        if (cand.rel_index == pb.rel_index) fb = &cand;
      EXPECT(fb && fb->src_ids == pb.src_ids && fb->indptr == pb.indptr, "restricted hop-1 rows == full rows");
    }
  }

  // test_sampling.cpp:111-117 — errors carry the reference's type and message
  {
    R::HetGraph rg = testutil::random_hetgraph(1);
    B::HetGraph bg = to_b200(rg);
    std::vector<B::NodeId> bad = {static_cast<B::NodeId>(rg.node_counts[rg.target])};
    std::string rmsg, bmsg;
    try {
      R::sample_khop(rg, bad, {2}, 0);
    } catch (const std::invalid_argument& e) {
      rmsg = e.what();
    }
    try {
      B::sample_khop(bg, bad, {2}, 0);
    } catch (const std::invalid_argument& e) {
      bmsg = e.what();
    }
    EXPECT(!rmsg.empty() && rmsg == bmsg, "out-of-range seed: same std::invalid_argument message");
    bool threw = false;
    std::vector<B::NodeId> ok = {0};
    try {
      B::sample_khop(bg, ok, {}, 0);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    EXPECT(threw, "empty fanouts rejected with std::invalid_argument");
  }

  // bundled mag-mini (harness.cpp:192-247): generator, plan and the first RAF batches
  for (int p : {1, 2}) {
    const std::uint64_t seed = 3;
    R::SyntheticSpec rs = R::bundled_spec("mag-mini");
    R::HetGraph rg = R::gen_synthetic(rs, seed);
    B::SyntheticSpec bs;
    bs.name = rs.name;
    bs.target = rs.target;
    bs.num_classes = rs.num_classes;
    bs.label_noise = rs.label_noise;
    for (const auto& t : rs.node_types) bs.node_types.push_back({t.name, t.count, t.dim, t.storage});
    for (const auto& r : rs.relations) bs.relations.push_back({r.src, r.edge, r.dst, r.edges, r.degree, r.alpha});
    bs.add_reverse = rs.add_reverse;
    bs.self_paired = rs.self_paired;
    B::HetGraph bg = B::gen_synthetic(bs, seed);
    EXPECT(bg.node_counts == rg.node_counts, "gen_synthetic node counts");

    const int k = 2;
    R::PartitionPlan rplan = R::meta_partition(R::build_metagraph(rg), rg.target, k, p);
    B::PartitionPlan bplan = B::meta_partition(bg, k, p);
    bool plan_ok = rplan.parts.size() == bplan.parts.size();
    for (std::size_t i = 0; plan_ok && i < rplan.parts.size(); ++i)
      plan_ok = rplan.parts[i].sub_ids == bplan.parts[i].sub_ids && rplan.parts[i].relations == bplan.parts[i].relations;
    EXPECT(plan_ok, ("meta_partition parts, p=" + std::to_string(p)).c_str());
    if (p != 1) continue;  // the multi-partition RAF path needs one GPU per partition (tests/test_gpu_multi.py)

    const int hidden = 16;
    const std::vector<int> fanouts = {25, 20};
    R::RafPlanView view = R::raf_view_from_plan(rplan);
    R::HGNNModel model = R::init_model(rg, rplan.tree, hidden, R::mix_seed(seed, 0xd0de1));
    R::LearnableStore store = R::init_learnable(rg, R::mix_seed(seed, 0x1ea4a));
    B::RafEngine eng(bg, fanouts, hidden, seed, 256, 1, 0, 0);
    auto batches = B::make_batches(bg, 256, 3, R::mix_seed(seed, 0xba7c));
    for (std::size_t i = 0; i < batches.size(); ++i) {
      const std::uint64_t rngs = R::mix_seed(seed, 0xb000 + i);
      auto rrep = R::run_raf_batch(rg, view, model, store, batches[i], fanouts, rngs, 0);
      auto brep = eng.run_raf_batch(batches[i], rngs, 0, /*train=*/false);
      const double rel = std::fabs(brep.loss - rrep.loss) / std::fabs(rrep.loss);
      std::printf("batch %zu loss ref %.9f b200 %.9f rel %.2e\n", i, rrep.loss, brep.loss, rel);
      EXPECT(rel < 1e-3, "run_raf_batch loss within 1e-3");
      EXPECT(brep.boundary_counts == rrep.boundary_counts, "ExecutionReport::boundary_counts");
      EXPECT(brep.boundary_cut_edges == rrep.boundary_cut_edges, "ExecutionReport::boundary_cut_edges");
      EXPECT(brep.sync_bytes == rrep.sync_bytes, "ExecutionReport::sync_bytes");
      EXPECT(brep.cross_ids_target_only == rrep.cross_ids_target_only, "ExecutionReport::cross_ids_target_only");
    }
    // the RGAT layer type behind the same engine interface (no reference counterpart:
    // tests/test_rgat.py holds its parity): training on one batch lowers its loss
    B::RafEngine att(bg, fanouts, hidden, seed, 256, 1, 0, 0, 0, false, B::LayerKind::RGAT, 4);
    double first = 0.0, last = 0.0;
    for (int it = 0; it < 8; ++it) {
      const double l = att.run_raf_batch(batches[0], R::mix_seed(seed, 0xb000), 0).loss;
      if (it == 0) first = l;
      last = l;
    }
    std::printf("RGAT loss %.6f -> %.6f\n", first, last);
    EXPECT(std::isfinite(last) && last < first, "RGAT engine trains");
  }

  // sample_neighbors (sampling.hpp:34-35) on raw CSRs: every row of several relations
  for (std::uint64_t s = 40; s < 46; ++s) {
    R::HetGraph rg = testutil::random_hetgraph(s);
    bool ok = true;
    for (std::size_t r = 0; r < rg.relations.size(); ++r) {
      B::Csr csr{rg.adj[r].indptr, rg.adj[r].src};
      for (R::NodeId d = 0; d + 1 < rg.adj[r].indptr.size(); ++d)
        for (int fo : {1, 3}) {
          const auto want = R::sample_neighbors(rg.adj[r], d, fo, s * 7 + 1, 2, static_cast<int>(r));
          const auto got = B::sample_neighbors(csr, d, fo, s * 7 + 1, 2, static_cast<int>(r));
          ok = ok && want == got;
        }
    }
    EXPECT(ok, ("sample_neighbors bit-exact, graph " + std::to_string(s)).c_str());
  }

  // the layer interface (hgnn.hpp:76-130) on the reference's own inputs: mag-mini, one batch
  {
    const std::uint64_t seed = 3;
    const int k = 2, hidden = 16;
    const std::vector<int> fanouts = {25, 20};
    R::HetGraph rg = R::gen_synthetic(R::bundled_spec("mag-mini"), seed);
    B::HetGraph bg = B::gen_synthetic(bspec(R::bundled_spec("mag-mini")), seed);
    const R::Metatree rt = R::build_metatree(R::build_metagraph(rg), rg.target, k);
    const B::Metatree bt = btree(rt);
    R::HGNNModel rmodel = R::init_model(rg, rt, hidden, 77);
    R::LearnableStore rstore = R::init_learnable(rg, 88);
    B::HGNNModel bmod = B::init_model(bg, bt, hidden, 77);
    B::LearnableStore bst = B::init_learnable(bg, 88);
    bool init_ok = bmod.weights.size() == rmodel.weights.size();
    for (const auto& [key, w] : rmodel.weights) init_ok = init_ok && bmod.weights.at(B::SlotKey{key.rel_index, key.layer}).data == w.data;
    for (const auto& [t, tab] : rstore.tables) init_ok = init_ok && bst.tables.at(t).w.data == tab.w.data;
    EXPECT(init_ok, "init_model / init_learnable bit-identical");

    std::vector<R::NodeId> batch;
    for (R::NodeId v = 0; v < 300; v += 2) batch.push_back(v);
    batch.push_back(4);  // a duplicate seed counts twice in the loss
    std::vector<R::NodeId> ids(batch);
    std::sort(ids.begin(), ids.end());
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    const auto hops = R::hop_relation_sets(rt, k);
    const R::SampledBlocks rb = R::sample_khop_restricted(rg, ids, fanouts, 123, hops);
    const B::SampledBlocks bb = bblocks(rb);
    auto [rlog, rtape] = R::forward_flat(rg, rt, rb, rmodel, rstore);

    // mean_aggregate / agg_relation / agg_all on every hop-2 block (hgnn.cpp:173-203)
    double mean_err = 0, agg_err = 0;
    for (const auto& e : rtape.entries) {
      if (e.layer != 1) continue;
      const R::Block& blk = rb.hops[e.hop - 1][e.block_idx];
      const int src_t = rg.relations[e.rel_index].src;
      const auto& hsrc = rtape.H[e.hop].at(src_t);
      const auto& front = rb.frontier[e.hop][src_t];
      const B::Block bblk{blk.rel_index, blk.hop, blk.dst_ids, blk.indptr, blk.src_ids};
      mean_err = std::max(mean_err, rel_err(B::mean_aggregate(bblk, bm(hsrc), front), R::mean_aggregate(blk, hsrc, front)));
      const auto& w = rmodel.weights.at(R::SlotKey{e.rel_index, 1});
      agg_err = std::max(agg_err, rel_err(B::agg_relation(bblk, bm(hsrc), front, bm(w)), R::agg_relation(blk, hsrc, front, w)));
    }
    std::printf("mean_aggregate rel err %.2e, agg_relation %.2e\n", mean_err, agg_err);
    EXPECT(mean_err < 1e-5, "mean_aggregate within fp32 of the reference");
    EXPECT(agg_err < 1e-4, "agg_relation within 1e-4 of the reference");
    {
      R::Matrix a(5, 7), b2(5, 7), c(5, 7);
      for (std::size_t i = 0; i < a.data.size(); ++i) {
        a.data[i] = 0.25 * i;
        b2.data[i] = -1.0 + i;
        c.data[i] = 3.0;
      }
      const B::Matrix ba = bm(a), bb2 = bm(b2), bc = bm(c);
      EXPECT(rel_err(B::agg_all({&ba, &bb2, &bc}), R::agg_all({&a, &b2, &c})) < 1e-6, "agg_all (hgnn.cpp:194-203)");
      bool threw = false;
      const B::Matrix odd(4, 7);
      try {
        B::agg_all({&ba, &odd});
      } catch (const std::invalid_argument& ex) {
        threw = std::string(ex.what()) == "agg_all partials have mismatched shapes";
      }
      EXPECT(threw, "agg_all shape mismatch: the reference's invalid_argument");
    }
    // a source id missing from its frontier: the reference's message
    {
      const R::Block& blk = rb.hops[1][0];
      const int src_t = rg.relations[blk.rel_index].src;
      std::vector<R::NodeId> front = rb.frontier[2][src_t];
      const R::NodeId gone = blk.src_ids.at(0);
      front.erase(std::find(front.begin(), front.end(), gone));
      std::string rmsg, bmsg;
      const R::Matrix h(front.size(), 4);
      try {
        R::mean_aggregate(blk, h, front);
      } catch (const std::invalid_argument& ex) {
        rmsg = ex.what();
      }
      try {
        B::mean_aggregate(B::Block{blk.rel_index, blk.hop, blk.dst_ids, blk.indptr, blk.src_ids}, bm(h), front);
      } catch (const std::invalid_argument& ex) {
        bmsg = ex.what();
      }
      EXPECT(!rmsg.empty() && rmsg == bmsg, "row_index miss: same std::invalid_argument message");
    }

    // forward_flat / cross_entropy / backward_flat (hgnn.cpp:215-362)
    auto [blog, btape] = B::forward_flat(bg, bt, bb, bmod, bst);
    const double lerr = rel_err(blog, rlog);
    std::printf("forward_flat logits rel err %.2e\n", lerr);
    EXPECT(lerr < 1e-3, "forward_flat logits within 1e-3");
    bool tape_ok = btape.entries.size() == rtape.entries.size();
    for (std::size_t i = 0; tape_ok && i < rtape.entries.size(); ++i)
      tape_ok = btape.entries[i].rel_index == rtape.entries[i].rel_index && btape.entries[i].layer == rtape.entries[i].layer &&
                rel_err(btape.entries[i].mean, rtape.entries[i].mean) < 1e-3;
    EXPECT(tape_ok, "forward tape entries (relation order, means) match");
    R::Matrix rdz;
    B::Matrix bdz;
    const double rloss = R::cross_entropy(rlog, ids, batch, rg.labels, rg.num_classes, &rdz);
    const double bloss = B::cross_entropy(blog, ids, batch, bg.labels(), bg.num_classes, &bdz);
    std::printf("cross_entropy ref %.9f b200 %.9f\n", rloss, bloss);
    EXPECT(std::fabs(rloss - bloss) < 1e-3 * std::fabs(rloss), "cross_entropy loss within 1e-3");
    EXPECT(rel_err(bdz, rdz) < 1e-3, "cross_entropy dlogits within 1e-3");
    const R::GradientSet rg_ = R::backward_flat(rg, rt, rmodel, rtape, rdz);
    const B::GradientSet bg_ = B::backward_flat(bg, bt, bmod, btape, bdz);
    const double gerr = grad_rel(bg_, rg_);
    std::printf("backward_flat gradients rel err %.2e\n", gerr);
    EXPECT(gerr < 1e-3, "backward_flat gradients within 1e-3 (ids exact)");
    {
      std::string rmsg, bmsg;
      std::vector<R::NodeId> bad_batch = {ids[0], static_cast<R::NodeId>(rg.node_counts[rg.target] + 5)};
      try {
        R::cross_entropy(rlog, ids, std::span<const R::NodeId>(bad_batch.data(), 1), rg.labels, rg.num_classes, nullptr);
        std::vector<std::int32_t> labels(rg.labels);
        labels[ids[0]] = rg.num_classes;
        R::cross_entropy(rlog, ids, std::span<const R::NodeId>(bad_batch.data(), 1), labels, rg.num_classes, nullptr);
      } catch (const std::invalid_argument& ex) {
        rmsg = ex.what();
      }
      try {
        std::vector<std::int32_t> labels(bg.labels().begin(), bg.labels().end());
        labels[ids[0]] = bg.num_classes;
        B::cross_entropy(blog, ids, std::span<const B::NodeId>(bad_batch.data(), 1), labels, bg.num_classes, nullptr);
      } catch (const std::invalid_argument& ex) {
        bmsg = ex.what();
      }
      EXPECT(!rmsg.empty() && rmsg == bmsg, "label out of range: same std::invalid_argument message");
    }

    // adam_update_model / adam_update_rows from identical state and gradients (hgnn.cpp:379-410)
    {
      R::ModelAdamState rs;
      B::ModelAdamState bs;
      B::HGNNModel bm2 = bmodel(rmodel);
      B::GradientSet bgr;
      for (const auto& [key, w] : rg_.weight_grads) bgr.weight_grads.emplace(B::SlotKey{key.rel_index, key.layer}, bm(w));
      for (int step = 0; step < 2; ++step) {
        R::adam_update_model(rmodel, rs, rg_);
        B::adam_update_model(bm2, bs, bgr);
      }
      bool ok = bs.step == rs.step;
      for (const auto& [key, w] : rmodel.weights) ok = ok && adam_close(bm2.weights.at(B::SlotKey{key.rel_index, key.layer}).data, w.data);
      EXPECT(ok, "adam_update_model (2 steps) within the one-flip bound");
      bool rows_ok = true;
      for (const auto& [t, fg] : rg_.feature_grads) {
        R::LearnableFeatureTable& rt2 = rstore.tables.at(t);
        B::LearnableFeatureTable bt2 = bst.tables.at(t);
        R::adam_update_rows(rt2, fg.first, fg.second);
        B::adam_update_rows(bt2, fg.first, bm(fg.second));
        rows_ok = rows_ok && bt2.step == rt2.step && adam_close(bt2.w.data, rt2.w.data) &&
                  rel_err(bt2.m, rt2.m) < 1e-3 && rel_err(bt2.v, rt2.v) < 1e-3;
      }
      EXPECT(rows_ok, "adam_update_rows: w within the flip bound, m and v within 1e-3, step advanced");
    }
  }

  // run_raf_batch with caller-owned model / store (raf.hpp:79-82) and check_equivalence
  // (raf.hpp:100-103) at p = 1, 2, 4 (single process, like the reference's workers)
  for (int p : {1, 2, 4}) {
    const std::uint64_t seed = 5;
    const int k = 2, hidden = 32;
    const std::vector<int> fanouts = {25, 20};
    R::HetGraph rg = R::gen_synthetic(R::bundled_spec("mag-mini"), seed);
    B::HetGraph bg = B::gen_synthetic(bspec(R::bundled_spec("mag-mini")), seed);
    R::PartitionPlan rplan = R::meta_partition(R::build_metagraph(rg), rg.target, k, p);
    B::PartitionPlan bplan = B::meta_partition(bg, k, p);
    const R::RafPlanView rview = R::raf_view_from_plan(rplan);
    const B::RafPlanView bview = B::raf_view_from_plan(bplan);
    EXPECT(bview.top_owners == rview.top_owners, ("raf_view_from_plan owners, p=" + std::to_string(p)).c_str());
    R::HGNNModel rmodel = R::init_model(rg, rplan.tree, hidden, 11);
    R::LearnableStore rstore = R::init_learnable(rg, 12);
    B::HGNNModel bmod = bmodel(rmodel);
    B::LearnableStore bst = bstore(rstore);
    auto batches = B::make_batches(bg, 200, 2, R::mix_seed(seed, 0xba7c));
    for (std::size_t i = 0; i < batches.size(); ++i) {
      const std::uint64_t rs = R::mix_seed(seed, 0xb000 + i);
      const int des = static_cast<int>(i) % p;
      const auto rrep = R::run_raf_batch(rg, rview, rmodel, rstore, batches[i], fanouts, rs, des);
      const auto brep = B::run_raf_batch(bg, bview, bmod, bst, batches[i], fanouts, rs, des);
      const std::string tag = " (p=" + std::to_string(p) + ", batch " + std::to_string(i) + ")";
      EXPECT(std::fabs(brep.loss - rrep.loss) < 1e-3 * std::fabs(rrep.loss), ("caller-owned run_raf_batch loss" + tag).c_str());
      EXPECT(brep.logit_ids == rrep.logit_ids && rel_err(brep.logits, rrep.logits) < 1e-3, ("logits" + tag).c_str());
      EXPECT(grad_rel(brep.grads, rrep.grads) < 1e-3, ("gradients" + tag).c_str());
      bool stats_ok = brep.stats.per_direction.size() == rrep.stats.per_direction.size();
      for (const auto& [key, e] : rrep.stats.per_direction) {
        auto it = brep.stats.per_direction.find(key);
        stats_ok = stats_ok && it != brep.stats.per_direction.end() && it->second.count == e.count && it->second.bytes == e.bytes;
      }
      EXPECT(stats_ok && brep.stats.total_bytes() == rrep.stats.total_bytes(), ("CommStats per direction" + tag).c_str());
      bool trace_ok = brep.trace.size() == rrep.trace.size();
      for (std::size_t m = 0; trace_ok && m < rrep.trace.size(); ++m)
        trace_ok = static_cast<int>(brep.trace[m].kind) == static_cast<int>(rrep.trace[m].kind) &&
                   brep.trace[m].sender == rrep.trace[m].sender && brep.trace[m].receiver == rrep.trace[m].receiver &&
                   brep.trace[m].node_ids == rrep.trace[m].node_ids && brep.trace[m].bytes == rrep.trace[m].bytes;
      EXPECT(trace_ok, ("message trace" + tag).c_str());
      EXPECT(brep.sync_bytes == rrep.sync_bytes, ("sync_bytes" + tag).c_str());
      EXPECT(brep.boundary_counts == rrep.boundary_counts && brep.boundary_cut_edges == rrep.boundary_cut_edges,
             ("boundary counts / cut edges" + tag).c_str());
      const auto rv = R::check_comm_bounds(rrep, static_cast<int>(rg.relations.size()), true);
      const auto bv = B::check_comm_bounds(brep, static_cast<int>(bg.relations.size()), true);
      EXPECT(rv.message_bound_ok == bv.message_bound_ok && rv.target_only_ok == bv.target_only_ok,
             ("check_comm_bounds" + tag).c_str());
      std::printf("p=%d batch %zu: loss ref %.9f b200 %.9f, %zu messages, %llu bytes\n", p, i, rrep.loss, brep.loss,
                  rrep.trace.size(), static_cast<unsigned long long>(rrep.stats.total_bytes()));
    }
    const auto eq = B::check_equivalence(bg, bview, bmod, bst, batches[0], fanouts, R::mix_seed(seed, 0xb000), 0);
    double lscale = 0;
    {
      const auto rrep = R::run_raf_batch(rg, rview, rmodel, rstore, batches[0], fanouts, R::mix_seed(seed, 0xb000), 0);
      for (double x : rrep.logits.data) lscale = std::max(lscale, std::fabs(x));
    }
    std::printf("check_equivalence p=%d: logit diff %.2e (scale %.2e), grad diff %.2e\n", p, eq.logit_diff, lscale, eq.grad_diff);
    EXPECT(eq.logit_diff < 1e-4 * lscale && eq.grad_diff < 1e-4, ("check_equivalence engine vs layer primitives, p=" + std::to_string(p)).c_str());
  }

  // feature cache (cache.hpp:36-89) against the reference
  {
    const std::uint64_t seed = 5;
    const int k = 2;
    const std::vector<int> fanouts = {10, 5};
    R::HetGraph rg = R::gen_synthetic(R::bundled_spec("mag-mini"), seed);
    B::HetGraph bg = B::gen_synthetic(bspec(R::bundled_spec("mag-mini")), seed);
    const R::Metatree rt = R::build_metatree(R::build_metagraph(rg), rg.target, k);
    const R::CostModel rcm{};
    const B::CostModel bcm{};
    const auto rprof = R::profile_miss_penalty(rg, rcm);
    const auto bprof = B::profile_miss_penalty(bg, bcm);
    bool prof_ok = rprof.types.size() == bprof.types.size();
    for (std::size_t t = 0; prof_ok && t < rprof.types.size(); ++t)
      prof_ok = rprof.types[t].record_bytes == bprof.types[t].record_bytes && rprof.types[t].transfer_ns == bprof.types[t].transfer_ns &&
                rprof.types[t].learnable == bprof.types[t].learnable;
    EXPECT(prof_ok, "profile_miss_penalty");
    const auto rhot = R::presample_hotness(rg, rt, fanouts, 2, 99, 512);
    const auto bhot = B::presample_hotness(bg, btree(rt), fanouts, 2, 99, 512);
    EXPECT(rhot.counts == bhot.counts, "presample_hotness counts bit-exact");
    const std::uint64_t budget = 4 << 20;
    const auto ralloc = R::allocate_cache(budget, rhot, rprof);
    const auto balloc = B::allocate_cache(budget, bhot, bprof);
    EXPECT(ralloc.capacity == balloc.capacity && ralloc.bytes == balloc.bytes, "allocate_cache");
    R::CacheState rcs = R::fill_and_serve(ralloc, rhot, rprof, 3);
    B::CacheState bcs = B::fill_and_serve(balloc, bhot, bprof, 3);
    bool fill_ok = rcs.types.size() == bcs.types.size();
    for (std::size_t t = 0; fill_ok && t < rcs.types.size(); ++t) fill_ok = rcs.types[t].cached == bcs.types[t].cached;
    EXPECT(fill_ok, "fill_and_serve cached ids");
    std::vector<R::NodeId> ids;
    for (R::NodeId v = 0; v < 512; ++v) ids.push_back(v);
    const auto blocks = R::sample_khop_restricted(rg, ids, fanouts, 7, R::hop_relation_sets(rt, k));
    for (std::size_t t = 0; t < blocks.frontier[k].size(); ++t) {
      if (rprof.types[t].record_bytes == 0) continue;
      for (R::NodeId v : blocks.frontier[k][t]) {
        rcs.lookup(static_cast<int>(t), v);
        bcs.lookup(static_cast<int>(t), v);
        if (rprof.types[t].learnable) {
          rcs.update(static_cast<int>(t), v);
          bcs.update(static_cast<int>(t), v);
        }
      }
    }
    bool hm_ok = true;
    for (std::size_t t = 0; t < rcs.types.size(); ++t)
      hm_ok = hm_ok && rcs.types[t].hits == bcs.types[t].hits && rcs.types[t].misses == bcs.types[t].misses &&
              rcs.types[t].penalty_ns == bcs.types[t].penalty_ns && rcs.hit_rate(static_cast<int>(t)) == bcs.hit_rate(static_cast<int>(t));
    EXPECT(hm_ok && rcs.placement_rank(7) == bcs.placement_rank(7), "CacheState lookup / update / hit_rate / placement");
    for (int p : {2, 4}) {
      R::PartitionPlan rplan = R::meta_partition(R::build_metagraph(rg), rg.target, k, p);
      B::PartitionPlan bplan = B::meta_partition(bg, k, p);
      bool ct_ok = true;
      for (int part = 0; part < p; ++part) {
        ct_ok = ct_ok && R::cacheable_types(rplan, part) == B::cacheable_types(bplan, part);
        for (int t = 0; t < static_cast<int>(rg.node_counts.size()); ++t)
          ct_ok = ct_ok && R::partition_aware_space(rplan, part, t) == B::partition_aware_space(bplan, part, t);
      }
      EXPECT(ct_ok, ("cacheable_types / partition_aware_space, p=" + std::to_string(p)).c_str());
    }
  }

  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail;
}
