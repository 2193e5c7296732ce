// C++ drop-in parity test: the reference library (hetsim, compiled from
// /root/reference/proj by oracle/Makefile) and the B200 path (libhetgpu.so via
// include/hetsim_b200.hpp) called side by side through their C++ APIs, the way
// a hetsim user would switch. TEST INFRASTRUCTURE: links the oracle as the
// checker only. Mirrors reference tests:
//   tests/test_sampling.cpp:12-117  (copy-all, determinism, frontiers, restricted == full, errors)
//   tests/test_raf.cpp:35-64         (RAF batch vs the reference's run_raf_batch)
//   tests/acceptance.cpp:336-348     (determinism)
// Prints one line per check; exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <set>
#include <string>
#include <vector>

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
  }

  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail;
}
