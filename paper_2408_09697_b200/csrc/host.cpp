// Host-side algorithms that stay on the CPU; see host.hpp for the reference map.
#include "host.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <random>
#include <atomic>
#include <exception>
#include <functional>
#include <memory>
#include <map>
#include <set>
#include <thread>

namespace hetgpu {

namespace {

int index_of(const std::vector<std::string>& names, const std::string& n) {
  for (std::size_t i = 0; i < names.size(); ++i)
    if (names[i] == n) return static_cast<int>(i);
  return -1;
}

template <typename T>
void sort_unique(std::vector<T>& v) {
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
}

template <typename T>
bool contains(const std::vector<T>& v, const T& x) {
  return std::find(v.begin(), v.end(), x) != v.end();
}

// Counting-sort the pairs of one relation into dst-major order, keeping the
// insertion order inside every destination row.
// Runs independent tasks on up to hardware_concurrency host threads; the first
// exception (in task order) is rethrown after all tasks finish.
void run_parallel(std::vector<std::function<void()>>& tasks) {
  const std::size_t nthreads =
      std::max<std::size_t>(1, std::min<std::size_t>(tasks.size(), std::thread::hardware_concurrency()));
  std::vector<std::exception_ptr> errs(tasks.size());
  std::atomic<std::size_t> next{0};
  auto worker = [&] {
    for (std::size_t i = next++; i < tasks.size(); i = next++) {
      try {
        tasks[i]();
      } catch (...) {
        errs[i] = std::current_exception();
      }
    }
  };
  std::vector<std::thread> pool;
  for (std::size_t t = 1; t < nthreads; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

// n values of std::uniform_real_distribution<double>(lo, hi) over std::mt19937_64(seed)
// (one engine output per value): the stream cut into chunks whose engines are jumped
// ahead (mt64_jump_engines), generated as tasks; bit-identical to the serial stream.
// HG_FEAT_CHUNK (values per chunk) is a test knob.
template <typename T>
void uniform_stream_tasks(std::uint64_t seed, double lo, double hi, T* out, std::uint64_t n,
                          std::vector<std::function<void()>>& tasks) {
  const char* chunk_env = std::getenv("HG_FEAT_CHUNK");
  const std::uint64_t chunk = std::max<std::uint64_t>(1, chunk_env ? std::stoull(chunk_env) : 1ULL << 26);
  std::vector<std::uint64_t> starts;
  for (std::uint64_t c = 0; c < n; c += chunk) starts.push_back(c);
  auto engines = std::make_shared<std::vector<std::mt19937_64>>(
      starts.size() > 1 ? mt64_jump_engines(seed, starts) : std::vector<std::mt19937_64>{std::mt19937_64(seed)});
  for (std::size_t c = 0; c < starts.size(); ++c)
    tasks.emplace_back([=] {
      std::mt19937_64& eng = (*engines)[c];
      std::uniform_real_distribution<double> u(lo, hi);
      const std::uint64_t end = std::min(n, starts[c] + chunk);
      for (std::uint64_t i = starts[c]; i < end; ++i) out[i] = static_cast<T>(u(eng));
    });
}

Adjacency dst_major(std::uint64_t n_dst, const std::vector<std::pair<NodeId, NodeId>>& pairs) {
  Adjacency a;
  a.offsets.assign(n_dst + 1, 0);
  for (const auto& pr : pairs) ++a.offsets[pr.second + 1];
  std::partial_sum(a.offsets.begin(), a.offsets.end(), a.offsets.begin());
  a.sources.resize(pairs.size());
  std::vector<std::uint64_t> fill(a.offsets.begin(), a.offsets.end() - 1);
  for (const auto& pr : pairs) a.sources[fill[pr.second]++] = pr.first;
  return a;
}

}  // namespace

std::uint64_t Graph::total_edges() const {
  std::uint64_t n = 0;
  for (const auto& r : rels) n += r.adj.sources.size();
  return n;
}

void Graph::validate() const {
  if (target < 0 || target >= num_types()) throw std::invalid_argument("target node type out of range");
  for (std::size_t r = 0; r < rels.size(); ++r) {
    const RelationInfo& rel = rels[r];
    if (rel.adj.offsets.size() != types[rel.dst_type].count + 1)
      throw std::invalid_argument("adjacency indptr size mismatch for relation " + std::to_string(r));
    if (!std::is_sorted(rel.adj.offsets.begin(), rel.adj.offsets.end()))
      throw std::invalid_argument("adjacency offsets not monotone");
    const std::uint64_t ns = types[rel.src_type].count;
    for (NodeId s : rel.adj.sources)
      if (s >= ns) throw std::invalid_argument("edge endpoint out of range");
    for (std::size_t q = r + 1; q < rels.size(); ++q)
      if (rels[q].src_type == rel.src_type && rels[q].edge_type == rel.edge_type &&
          rels[q].dst_type == rel.dst_type)
        throw std::invalid_argument("duplicate relation triple");
  }
}

Graph assemble(std::vector<std::string> type_names, std::vector<std::uint64_t> counts,
               std::vector<std::string> edge_names, const std::vector<int>& rel_src,
               const std::vector<int>& rel_dst,
               const std::vector<std::vector<std::pair<NodeId, NodeId>>>& pairs, int target,
               int num_classes) {
  Graph g;
  for (std::size_t t = 0; t < type_names.size(); ++t) {
    NodeTypeInfo nt;
    nt.name = type_names[t];
    nt.count = counts[t];
    g.types.push_back(std::move(nt));
  }
  g.edge_type_names = std::move(edge_names);
  g.rels.resize(rel_src.size());
  std::vector<std::function<void()>> tasks;
  for (std::size_t r = 0; r < rel_src.size(); ++r)
    tasks.emplace_back([&, r] {
      RelationInfo& rel = g.rels[r];
      rel.src_type = rel_src[r];
      rel.edge_type = static_cast<int>(r);
      rel.dst_type = rel_dst[r];
      const std::uint64_t ns = counts[rel.src_type], nd = counts[rel.dst_type];
      for (const auto& pr : pairs[r])
        if (pr.first >= ns || pr.second >= nd)
          throw std::invalid_argument("edge endpoint out of range in relation " + std::to_string(r));
      rel.adj = dst_major(nd, pairs[r]);
    });
  run_parallel(tasks);
  g.target = target;
  g.num_classes = num_classes;
  g.labels.assign(counts[target], -1);
  return g;
}

void append_reverse(Graph& g, const std::vector<int>& self_paired) {
  for (const auto& r : g.rels)
    if (r.reverse) throw std::invalid_argument("graph already contains reverse relations");
  const std::size_t n_fwd = g.rels.size();
  std::vector<std::size_t> todo;
  std::vector<int> name_idx;
  for (std::size_t r = 0; r < n_fwd; ++r) {
    if (contains(self_paired, static_cast<int>(r))) continue;
    const std::string name = "rev_" + g.edge_type_names[g.rels[r].edge_type];
    if (contains(g.edge_type_names, name))
      throw std::invalid_argument("reverse edge type name already exists: " + name);
    g.edge_type_names.push_back(name);
    todo.push_back(r);
    name_idx.push_back(static_cast<int>(g.edge_type_names.size()) - 1);
  }
  // transposes (independent per relation, built on host threads): rows become
  // the old sources, each listing old destinations in ascending order
  std::vector<Adjacency> tr(todo.size());
  std::vector<std::function<void()>> tasks;
  for (std::size_t i = 0; i < todo.size(); ++i)
    tasks.emplace_back([&, i] {
      const Adjacency& fwd = g.rels[todo[i]].adj;
      const std::uint64_t n_new_dst = g.types[g.rels[todo[i]].src_type].count;
      Adjacency& t = tr[i];
      t.offsets.assign(n_new_dst + 1, 0);
      for (NodeId s : fwd.sources) ++t.offsets[s + 1];
      std::partial_sum(t.offsets.begin(), t.offsets.end(), t.offsets.begin());
      t.sources.resize(fwd.sources.size());
      std::vector<std::uint64_t> fill(t.offsets.begin(), t.offsets.end() - 1);
      const std::uint64_t n_old_dst = fwd.offsets.size() - 1;
      for (std::uint64_t d = 0; d < n_old_dst; ++d)
        for (std::uint64_t e = fwd.offsets[d]; e < fwd.offsets[d + 1]; ++e)
          t.sources[fill[fwd.sources[e]]++] = static_cast<NodeId>(d);
    });
  run_parallel(tasks);
  for (std::size_t i = 0; i < todo.size(); ++i) {
    RelationInfo rev;
    rev.src_type = g.rels[todo[i]].dst_type;
    rev.dst_type = g.rels[todo[i]].src_type;
    rev.edge_type = name_idx[i];
    rev.reverse = true;
    rev.adj = std::move(tr[i]);
    g.rels.push_back(std::move(rev));
  }
}

Graph generate(const Spec& spec, std::uint64_t seed) {
  std::vector<std::string> names;
  for (const auto& t : spec.node_types) names.push_back(t.name);
  std::vector<std::string> problems;
  if (spec.node_types.empty()) problems.push_back("no node types");
  const int tgt = index_of(names, spec.target);
  if (tgt < 0)
    problems.push_back("target type not declared: " + spec.target);
  else if (spec.node_types[tgt].count < 1)
    problems.push_back("target type has no nodes");
  for (const auto& r : spec.relations) {
    if (index_of(names, r.src) < 0) problems.push_back("relation src not declared: " + r.src);
    if (index_of(names, r.dst) < 0) problems.push_back("relation dst not declared: " + r.dst);
    if (r.edges == 0) problems.push_back("relation has no edges: " + r.edge);
  }
  if (!problems.empty()) {
    std::string msg = "invalid synthetic spec:";
    for (const auto& p : problems) msg += " " + p + ";";
    throw std::invalid_argument(msg);
  }
  for (std::size_t i = 0; i < names.size(); ++i)
    for (std::size_t j = i + 1; j < names.size(); ++j)
      if (names[i] == names[j]) throw std::invalid_argument("duplicate node type name: " + names[i]);

  std::vector<std::uint64_t> counts;
  for (const auto& t : spec.node_types) counts.push_back(t.count);
  std::vector<std::string> edge_names;
  std::vector<int> rs, rd;
  std::vector<std::vector<std::pair<NodeId, NodeId>>> pairs(spec.relations.size());
  for (std::size_t ri = 0; ri < spec.relations.size(); ++ri) {
    const SpecRelation& sr = spec.relations[ri];
    if (contains(edge_names, sr.edge)) throw std::invalid_argument("duplicate edge type name: " + sr.edge);
    edge_names.push_back(sr.edge);
    rs.push_back(index_of(names, sr.src));
    rd.push_back(index_of(names, sr.dst));
  }
  // Every stochastic part draws from its own mt19937_64 stream (per relation
  // mix_seed(seed, 0x9e0 + ri), per feature type mix_seed(seed, 0xf0 + t), the
  // labels mix_seed(seed, 0x1abe1); harness.cpp:113-166), so the streams run on
  // separate host threads with bit-identical results.
  std::vector<std::function<void()>> tasks;
  for (std::size_t ri = 0; ri < spec.relations.size(); ++ri) tasks.emplace_back([&, ri] {
    const SpecRelation& sr = spec.relations[ri];
    const int s = rs[ri], d = rd[ri];
    std::mt19937_64 eng(mix_seed(seed, 0x9e0ULL + ri));
    std::uniform_int_distribution<std::uint64_t> src_pick(0, counts[s] - 1);
    auto& out = pairs[ri];
    out.reserve(sr.edges);
    if (!sr.powerlaw) {
      std::uniform_int_distribution<std::uint64_t> dst_pick(0, counts[d] - 1);
      for (std::uint64_t e = 0; e < sr.edges; ++e) {
        const auto a = static_cast<NodeId>(src_pick(eng));  // source drawn first
        const auto b = static_cast<NodeId>(dst_pick(eng));
        out.emplace_back(a, b);
      }
    } else {
      // in-degree of destination i proportional to (i+1)^-alpha, floored, then
      // topped up round-robin from destination 0 to the exact edge count
      const std::uint64_t nd = counts[d];
      std::vector<double> w(nd);
      double total = 0.0;
      for (std::uint64_t i = 0; i < nd; ++i) {
        w[i] = std::pow(static_cast<double>(i + 1), -sr.alpha);
        total += w[i];
      }
      std::vector<std::uint64_t> deg(nd);
      std::uint64_t placed = 0;
      for (std::uint64_t i = 0; i < nd; ++i) {
        deg[i] = static_cast<std::uint64_t>(static_cast<double>(sr.edges) * w[i] / total);
        placed += deg[i];
      }
      for (std::uint64_t i = 0; placed < sr.edges; i = (i + 1) % nd, ++placed) ++deg[i];
      for (std::uint64_t dd = 0; dd < nd; ++dd)
        for (std::uint64_t e = 0; e < deg[dd]; ++e)
          out.emplace_back(static_cast<NodeId>(src_pick(eng)), static_cast<NodeId>(dd));
    }
  });
  // A feature stream draws one engine output per value (generate_canonical<double, 53>
  // over 64-bit words); a long one is cut into jumped-ahead chunks generated on many
  // threads, bit-identical to the serial stream (uniform_stream_tasks).
  std::vector<std::vector<float>> dense(spec.node_types.size());
  for (std::size_t t = 0; t < spec.node_types.size(); ++t) {
    if (spec.node_types[t].storage != Storage::Dense) continue;
    const std::uint64_t n = spec.node_types[t].count * static_cast<std::uint64_t>(spec.node_types[t].dim);
    dense[t].resize(n);
    uniform_stream_tasks(mix_seed(seed, 0xf0ULL + t), -1.0, 1.0, dense[t].data(), n, tasks);
  }
  std::vector<std::int32_t> labels(counts[tgt]);
  tasks.emplace_back([&] {
    std::mt19937_64 leng(mix_seed(seed, 0x1abe1ULL));
    std::uniform_real_distribution<double> coin(0.0, 1.0);
    std::uniform_int_distribution<int> any_class(0, spec.num_classes - 1);
    for (NodeId v = 0; v < counts[tgt]; ++v) {
      labels[v] = static_cast<std::int32_t>(v % spec.num_classes);
      if (coin(leng) < spec.label_noise) labels[v] = any_class(leng);
    }
  });
  run_parallel(tasks);

  Graph g = assemble(names, counts, edge_names, rs, rd, pairs, tgt, spec.num_classes);
  for (std::size_t t = 0; t < spec.node_types.size(); ++t) {
    NodeTypeInfo& nt = g.types[t];
    nt.dim = spec.node_types[t].dim;
    nt.storage = spec.node_types[t].storage;
    if (nt.storage == Storage::Dense) nt.dense = std::move(dense[t]);
  }
  g.labels = std::move(labels);
  if (spec.add_reverse) {
    std::vector<int> paired;
    for (const auto& n : spec.self_paired) {
      const int et = index_of(g.edge_type_names, n);
      if (et < 0) throw std::invalid_argument("self_paired edge type not found: " + n);
      for (std::size_t r = 0; r < g.rels.size(); ++r)
        if (g.rels[r].edge_type == et) paired.push_back(static_cast<int>(r));
    }
    append_reverse(g, paired);
  }
  g.validate();
  return g;
}

// ---- metatree / partition ------------------------------------------------------

int Tree::root_child_ancestor(int p) const {
  if (p <= 0) return -1;
  while (pos[p].parent != 0) p = pos[p].parent;
  return p;
}

std::vector<int> Plan::owners_of_sub(int sub_id) const {
  std::vector<int> out;
  for (std::size_t i = 0; i < parts.size(); ++i)
    if (contains(parts[i].sub_ids, sub_id)) out.push_back(static_cast<int>(i));
  return out;
}

RafAccounting raf_accounting(const Graph& g, const Tree& t, const std::vector<std::vector<int>>& top_owners, int p) {
  RafAccounting a;
  a.boundary_counts.assign(static_cast<std::size_t>(std::max(p, 1)), 0);
  const auto& root_kids = t.pos.at(0).children;
  if (top_owners.size() != root_kids.size()) throw std::invalid_argument("one owner list per root child expected");
  auto owners_of = [&](int pos) -> const std::vector<int>& {
    const int anc = t.root_child_ancestor(pos);
    for (std::size_t ci = 0; ci < root_kids.size(); ++ci)
      if (root_kids[ci] == anc) return top_owners[ci];
    throw std::logic_error("position outside every root subtree");
  };
  // sender-side boundary per worker: the parent-type nodes with at least one
  // in-edge of a crossing (depth-1) relation, as a set over (type, node)
  std::vector<std::vector<std::uint64_t>> marks(a.boundary_counts.size());
  for (std::size_t pos = 1; pos < t.pos.size(); ++pos) {
    const TreePos& tp = t.pos[pos];
    const std::vector<int>& own = owners_of(static_cast<int>(pos));
    std::set<int> who(own.begin(), own.end());
    auto& c = a.slot_contributors[SlotId{tp.rel, t.k - tp.depth + 1}];
    for (int w : c) who.insert(w);
    c.assign(who.begin(), who.end());
    if (tp.depth == t.k && g.types[tp.type].storage == Storage::Learnable) {
      auto& lo = a.leaf_owners[tp.type];
      std::set<int> lw(lo.begin(), lo.end());
      lw.insert(own.begin(), own.end());
      lo.assign(lw.begin(), lw.end());
    }
    if (tp.depth != 1) continue;  // meta plans: inner positions never cross workers
    const Adjacency& adj = g.rels[tp.rel].adj;
    a.boundary_cut_edges += adj.sources.size();
    const int parent_type = t.pos[tp.parent].type;
    const std::uint64_t n = g.types[parent_type].count;
    for (int w : own) {
      auto& m = marks[w];
      if (m.empty()) m.assign(static_cast<std::size_t>((n + 63) / 64), 0);  // one parent type: the root
      for (std::uint64_t v = 0; v < n; ++v)
        if (adj.offsets[v + 1] > adj.offsets[v]) m[v >> 6] |= 1ull << (v & 63);
    }
  }
  for (std::size_t w = 0; w < marks.size(); ++w)
    for (std::uint64_t x : marks[w]) a.boundary_counts[w] += static_cast<std::uint64_t>(__builtin_popcountll(x));
  return a;
}

RafAccounting plan_accounting(const Graph& g, const Plan& plan) {
  std::vector<std::vector<int>> top;
  for (int c : plan.tree.pos.at(0).children) {
    bool found = false;
    for (const auto& sub : plan.subs)
      if (sub.child_pos == c) {
        top.push_back(plan.owners_of_sub(sub.id));
        found = true;
        break;
      }
    if (!found) throw std::invalid_argument("plan has no sub-metatree for a root child");
  }
  return raf_accounting(g, plan.tree, top, plan.p);
}

Schema schema_of(const Graph& g) {
  Schema s;
  for (const auto& t : g.types) s.vertex_weight.push_back(t.count);
  for (std::size_t r = 0; r < g.rels.size(); ++r)
    s.links.push_back({static_cast<int>(r), g.rels[r].src_type, g.rels[r].dst_type,
                       static_cast<std::uint64_t>(g.rels[r].adj.sources.size())});
  return s;
}

Tree bfs_tree(const Schema& s, int root, int k) {
  if (root < 0 || root >= static_cast<int>(s.vertex_weight.size()))
    throw std::invalid_argument("metatree root not in metagraph");
  Tree t;
  t.k = k;
  t.root_type = root;
  t.pos.push_back({root, 0, -1, -1, {}});
  std::size_t level_begin = 0;
  for (int depth = 1; depth <= k; ++depth) {
    const std::size_t level_end = t.pos.size();
    for (std::size_t p = level_begin; p < level_end; ++p)
      for (const auto& l : s.links) {
        if (l.dst != t.pos[p].type) continue;
        t.pos[p].children.push_back(static_cast<int>(t.pos.size()));
        t.pos.push_back({l.src, depth, static_cast<int>(p), l.rel, {}});
      }
    level_begin = level_end;
  }
  return t;
}

Tree metapath_tree(const Schema& s, int root, const std::vector<std::vector<int>>& paths) {
  if (root < 0 || root >= static_cast<int>(s.vertex_weight.size()))
    throw std::invalid_argument("metatree root not in metagraph");
  Tree t;
  t.root_type = root;
  t.pos.push_back({root, 0, -1, -1, {}});
  for (const auto& path : paths) {
    int at = 0;
    for (int rel : path) {
      const Schema::Link* link = nullptr;
      for (const auto& l : s.links)
        if (l.rel == rel) link = &l;
      if (!link || link->dst != t.pos[at].type)
        throw std::invalid_argument("invalid metapath step: relation " + std::to_string(rel) +
                                    " does not leave node type " + std::to_string(t.pos[at].type));
      int next = -1;
      for (int c : t.pos[at].children)
        if (t.pos[c].rel == rel) next = c;
      if (next < 0) {
        next = static_cast<int>(t.pos.size());
        t.pos.push_back({link->src, t.pos[at].depth + 1, at, rel, {}});
        t.pos[at].children.push_back(next);
      }
      at = next;
      t.k = std::max(t.k, t.pos[at].depth);
    }
  }
  return t;
}

namespace {

std::vector<SubTree> split(const Tree& t, const Schema& s) {
  std::vector<SubTree> subs;
  for (std::size_t i = 0; i < t.pos[0].children.size(); ++i) {
    SubTree st;
    st.id = static_cast<int>(i);
    st.child_pos = t.pos[0].children[i];
    st.positions.push_back(0);
    // pre-order walk of the subtree, children in tree order
    std::vector<int> todo{st.child_pos};
    while (!todo.empty()) {
      const int p = todo.back();
      todo.pop_back();
      st.positions.push_back(p);
      st.rel_multiset.push_back(t.pos[p].rel);
      const auto& ch = t.pos[p].children;
      for (auto it = ch.rbegin(); it != ch.rend(); ++it) todo.push_back(*it);
    }
    for (int p : st.positions) st.types_unique.push_back(t.pos[p].type);
    sort_unique(st.types_unique);
    st.rel_unique = st.rel_multiset;
    sort_unique(st.rel_unique);
    for (int ty : st.types_unique) st.weight += s.vertex_weight[ty];
    for (int r : st.rel_unique) {
      bool found = false;
      for (const auto& l : s.links)
        if (l.rel == r) {
          st.weight += l.weight;
          found = true;
          break;
        }
      if (!found) throw std::invalid_argument("relation not in metagraph: " + std::to_string(r));
    }
    subs.push_back(std::move(st));
  }
  return subs;
}

// endpoint types of each relation, recovered from the tree itself
void dedup_part(Part& part, const Plan& plan) {
  part.relations.clear();
  for (int sid : part.sub_ids)
    for (int r : plan.subs[sid].rel_multiset)
      if (!contains(part.relations, r)) part.relations.push_back(r);
  part.node_types.assign(1, plan.tree.root_type);
  for (int r : part.relations)
    for (const auto& p : plan.tree.pos)
      if (p.rel == r) {
        part.node_types.push_back(p.type);
        part.node_types.push_back(plan.tree.pos[p.parent].type);
        break;
      }
  sort_unique(part.node_types);
  part.weight = 0;
  for (int sid : part.sub_ids) part.weight += plan.subs[sid].weight;
}

}  // namespace

std::vector<int> lpt(const std::vector<std::uint64_t>& weights, int p) {
  if (p <= 0) throw std::invalid_argument("partition count must be positive");
  std::vector<int> order(weights.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return weights[a] > weights[b]; });
  std::vector<std::uint64_t> load(p, 0);
  std::vector<int> where(weights.size(), -1);
  for (int item : order) {
    const int lightest = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
    where[item] = lightest;
    load[lightest] += weights[item];
  }
  return where;
}

Plan meta_partition(const Schema& s, int root, int k, int p) {
  Plan plan;
  plan.p = p;
  plan.tree = bfs_tree(s, root, k);
  if (plan.tree.pos.empty()) throw std::invalid_argument("empty metatree");
  plan.subs = split(plan.tree, s);
  std::vector<std::uint64_t> w;
  for (const auto& st : plan.subs) w.push_back(st.weight);
  const std::vector<int> where = lpt(w, p);
  plan.parts.resize(p);
  for (std::size_t i = 0; i < where.size(); ++i) plan.parts[where[i]].sub_ids.push_back(static_cast<int>(i));
  for (auto& part : plan.parts) dedup_part(part, plan);
  plan.deduplicated = true;

  // more workers than sub-metatrees: heaviest subs first, round robin into
  // the empty partitions; owners of a shared sub become replicas
  const int n_subs = static_cast<int>(plan.subs.size());
  if (p > n_subs && n_subs > 0) {
    std::vector<int> heavy(n_subs);
    std::iota(heavy.begin(), heavy.end(), 0);
    std::stable_sort(heavy.begin(), heavy.end(),
                     [&](int a, int b) { return plan.subs[a].weight > plan.subs[b].weight; });
    std::size_t rr = 0;
    for (auto& part : plan.parts)
      if (part.sub_ids.empty()) part.sub_ids.push_back(heavy[rr++ % heavy.size()]);
    for (int sid = 0; sid < n_subs; ++sid) {
      const auto owners = plan.owners_of_sub(sid);
      if (owners.size() < 2) continue;
      for (std::size_t i = 0; i < owners.size(); ++i) {
        Part& part = plan.parts[owners[i]];
        part.replica = true;
        part.replica_index = static_cast<int>(i);
        part.replica_count = static_cast<int>(owners.size());
      }
    }
    for (auto& part : plan.parts) dedup_part(part, plan);
  }
  return plan;
}

// Work-aware meta-partitioning (not the reference's policy; the reference plan stays
// the parity mode). The same metatree and sub-metatrees as meta_partition, but the p
// workers are split into groups that each replicate a set of sub-metatrees, chosen to
// minimise the busiest worker's cost. A group g of r_g workers splits the batch
// (raf.cpp:390-391): each worker samples and trains sum(work[S_g]) / r_g; replicas also
// merge their learnable-row gradients every step (the union of the replicas' rows gets
// one summed Adam update, raf.cpp:496-510), which costs ~merge_cost x learn_rows[S_g]
// (a row's w, m, v read-modify-write ~ that many sampled edges' gather bytes). Every set
// partition of the subs and every split of p over its blocks is scored (the bundled
// schemas' metatrees have <= 6 subs); ties go to fewer groups.
Plan work_aware_partition(const Schema& s, int root, int k, int p, const std::vector<double>& work,
                          const std::vector<double>& learn_rows, double merge_cost,
                          const std::vector<bool>& learnable_types) {
  Plan plan;
  plan.p = p;
  plan.tree = bfs_tree(s, root, k);
  if (plan.tree.pos.empty()) throw std::invalid_argument("empty metatree");
  plan.subs = split(plan.tree, s);
  const int n = static_cast<int>(plan.subs.size());
  if (static_cast<int>(work.size()) != n || (!learn_rows.empty() && static_cast<int>(learn_rows.size()) != n))
    throw std::invalid_argument("work-aware plan: one work value per sub-metatree expected (" + std::to_string(n) + ")");
  if (n > 8) throw std::invalid_argument("work-aware plan: more than 8 sub-metatrees");
  if (p < 1) throw std::invalid_argument("p must be >= 1");
  // what each sub-metatree trains: its weight slots (rel, layer) and learnable leaf types.
  // Groups must not share either (the engine exchanges gradients only inside a replica
  // group), which deep metatrees (a relation at several depths: MAG240M at k = 3) make
  // binding; the single all-subs group (data parallel) is always feasible.
  std::vector<std::set<std::pair<int, int>>> sub_slots(n);
  std::vector<std::set<int>> sub_leaves(n);
  for (int sid = 0; sid < n; ++sid)
    for (std::size_t q = 1; q < plan.tree.pos.size(); ++q) {
      if (plan.tree.root_child_ancestor(static_cast<int>(q)) != plan.subs[sid].child_pos) continue;
      const TreePos& tp = plan.tree.pos[q];
      sub_slots[sid].insert({tp.rel, k - tp.depth + 1});
      if (tp.depth == k && tp.type < static_cast<int>(learnable_types.size()) && learnable_types[tp.type])
        sub_leaves[sid].insert(tp.type);
    }
  auto feasible = [&](const std::vector<std::vector<int>>& groups) {
    std::map<std::pair<int, int>, int> slot_owner;
    std::map<int, int> leaf_owner;
    for (int g = 0; g < static_cast<int>(groups.size()); ++g)
      for (int sid : groups[g]) {
        for (const auto& key : sub_slots[sid]) {
          auto it = slot_owner.emplace(key, g).first;
          if (it->second != g) return false;
        }
        for (int t : sub_leaves[sid]) {
          auto it = leaf_owner.emplace(t, g).first;
          if (it->second != g) return false;
        }
      }
    return true;
  };
  double best = -1.0;
  std::vector<std::vector<int>> best_groups;
  std::vector<int> best_r;
  std::vector<int> label(n, 0);  // restricted-growth string: subs -> group
  std::function<void(int, int)> each_partition = [&](int i, int ng) {
    if (i == n) {
      if (ng > p) return;
      std::vector<std::vector<int>> groups(ng);
      std::vector<double> w(ng, 0.0), m(ng, 0.0);
      for (int q = 0; q < n; ++q) {
        groups[label[q]].push_back(q);
        w[label[q]] += work[q];
        m[label[q]] += learn_rows.empty() ? 0.0 : merge_cost * learn_rows[q];
      }
      if (!feasible(groups)) return;
      auto cost = [&](int g, int r) { return w[g] / r + (r > 1 ? m[g] : 0.0); };
      // every extra worker goes to the group whose cost it lowers the most, while any does
      std::vector<int> r(ng, 1);
      for (int extra = p - ng; extra > 0; --extra) {
        int arg = -1;
        double gain = 0.0;
        for (int g = 0; g < ng; ++g) {
          const double d = cost(g, r[g]) - cost(g, r[g] + 1);
          if (d > gain) {
            gain = d;
            arg = g;
          }
        }
        if (arg < 0) {  // no worker lowers a cost: the one that raises it least
          double least = 0.0;
          for (int g = 0; g < ng; ++g) {
            const double d = cost(g, r[g] + 1) - cost(g, r[g]);
            if (arg < 0 || d < least) {
              least = d;
              arg = g;
            }
          }
        }
        ++r[arg];
      }
      double worst = 0.0;
      for (int g = 0; g < ng; ++g) worst = std::max(worst, cost(g, r[g]));
      if (best < 0 || worst < best * (1.0 - 1e-12) ||
          (std::abs(worst - best) <= 1e-12 * best && groups.size() < best_groups.size())) {
        best = worst;
        best_groups = groups;
        best_r = r;
      }
      return;
    }
    for (int g = 0; g <= ng && g < p; ++g) {
      label[i] = g;
      each_partition(i + 1, std::max(ng, g + 1));
    }
  };
  if (n > 0) each_partition(0, 0);
  for (std::size_t g = 0; g < best_groups.size(); ++g)
    for (int q = 0; q < best_r[g]; ++q) {
      Part part;
      part.sub_ids = best_groups[g];
      part.replica = best_r[g] > 1;
      part.replica_index = q;
      part.replica_count = best_r[g];
      plan.parts.push_back(part);
    }
  for (auto& part : plan.parts) dedup_part(part, plan);
  plan.deduplicated = true;
  return plan;
}

std::vector<int> cacheable_types(const Plan& plan, int part) {
  const Tree& t = plan.tree;
  std::vector<int> leaves, kept;
  // first relation occurrence wins: subs in id order, depth-first inside a sub
  auto walk = [&](auto&& self, int p) -> void {
    bool any = false;
    for (int c : t.pos[p].children) {
      if (contains(kept, t.pos[c].rel)) continue;
      kept.push_back(t.pos[c].rel);
      any = true;
      self(self, c);
    }
    if (!any && t.pos[p].depth > 0 && !contains(leaves, t.pos[p].type)) leaves.push_back(t.pos[p].type);
  };
  for (int sid : plan.parts.at(part).sub_ids) {
    const int cp = plan.subs[sid].child_pos;
    if (contains(kept, t.pos[cp].rel)) continue;
    kept.push_back(t.pos[cp].rel);
    walk(walk, cp);
  }
  std::sort(leaves.begin(), leaves.end());
  return leaves;
}

std::vector<std::vector<int>> hop_relations(const Tree& t, int k) {
  std::vector<std::vector<int>> out(k);
  for (const auto& p : t.pos)
    if (p.rel >= 0 && p.depth >= 1 && p.depth <= k && !contains(out[p.depth - 1], p.rel))
      out[p.depth - 1].push_back(p.rel);
  for (auto& v : out) std::sort(v.begin(), v.end());
  return out;
}

std::map<int, std::vector<int>> relations_into_at_depth(const Tree& t, int depth) {
  std::map<int, std::vector<int>> out;
  for (const auto& p : t.pos) {
    if (p.depth != depth || p.rel < 0) continue;
    auto& v = out[t.pos[p.parent].type];
    if (!contains(v, p.rel)) v.push_back(p.rel);
  }
  for (auto& kv : out) std::sort(kv.second.begin(), kv.second.end());
  return out;
}

// ---- parameters ----------------------------------------------------------------

ModelInit init_model(const Graph& g, const Tree& t, int hidden, std::uint64_t seed) {
  ModelInit m;
  m.k = std::max(t.k, 1);
  m.hidden = hidden;
  m.num_classes = g.num_classes;
  for (const auto& nt : g.types) m.input_dims.push_back(nt.dim);
  for (const auto& p : t.pos) {
    if (p.rel < 0) continue;
    const int layer = m.k - p.depth + 1;
    const SlotId id{p.rel, layer};
    if (m.weights.count(id)) continue;
    WeightInit w;
    w.in_dim = layer == 1 ? m.input_dims[p.type] : hidden;
    w.out_dim = m.out_dim(layer);
    const double scale = w.in_dim > 0 ? 1.0 / std::sqrt(static_cast<double>(w.in_dim)) : 0.0;
    std::mt19937_64 eng(mix_seed(seed, (static_cast<std::uint64_t>(p.rel) << 8) | layer));
    std::uniform_real_distribution<double> u(-scale, scale);
    w.values.resize(static_cast<std::size_t>(w.in_dim) * w.out_dim);
    for (double& x : w.values) x = u(eng);
    m.weights.emplace(id, std::move(w));
  }
  return m;
}

std::map<int, std::vector<double>> init_learnable(const Graph& g, std::uint64_t seed) {
  std::map<int, std::vector<double>> out;
  for (int t = 0; t < g.num_types(); ++t) {
    if (g.types[t].storage != Storage::Learnable) continue;
    const int d = g.types[t].dim;
    out.emplace(t, std::vector<double>(g.types[t].count * static_cast<std::uint64_t>(d)));
  }
  // one uniform stream per table (hgnn.cpp:64-81), in jumped-ahead chunks on host threads
  std::vector<std::function<void()>> tasks;
  for (auto& [t, w] : out) {
    const int d = g.types[t].dim;
    const double scale = d > 0 ? 1.0 / std::sqrt(static_cast<double>(d)) : 0.0;
    uniform_stream_tasks(mix_seed(seed, 0xfeedULL + t), -scale, scale, w.data(), w.size(), tasks);
  }
  run_parallel(tasks);
  return out;
}

std::vector<std::vector<NodeId>> make_batches(const Graph& g, int batch_size, int max_batches,
                                              std::uint64_t seed) {
  std::vector<NodeId> ids(g.types[g.target].count);
  std::iota(ids.begin(), ids.end(), 0);
  std::mt19937_64 eng(seed);
  std::shuffle(ids.begin(), ids.end(), eng);
  std::vector<std::vector<NodeId>> out;
  for (std::size_t lo = 0; lo < ids.size(); lo += batch_size) {
    if (max_batches > 0 && static_cast<int>(out.size()) >= max_batches) break;
    const std::size_t hi = std::min(ids.size(), lo + static_cast<std::size_t>(batch_size));
    out.emplace_back(ids.begin() + lo, ids.begin() + hi);
  }
  return out;
}

// ---- cache planning --------------------------------------------------------------

std::vector<TypePenalty> miss_penalty(const Graph& g, const CostModel& cm) {
  std::vector<TypePenalty> out(g.num_types());
  for (int t = 0; t < g.num_types(); ++t) {
    const NodeTypeInfo& nt = g.types[t];
    if (nt.storage == Storage::Absent) continue;
    TypePenalty& tp = out[t];
    tp.learnable = nt.storage == Storage::Learnable;
    const std::uint64_t row = static_cast<std::uint64_t>(nt.dim) * cm.elem_bytes;
    if (row == 0) throw std::invalid_argument("zero record size for node type " + nt.name);
    if (tp.learnable) {
      // feature row + Adam m + Adam v, each read and written back
      tp.record_bytes = 3 * row;
      tp.transfer_ns = 3.0 * (cm.fixed_overhead_ns + cm.read_ns_per_byte * row) +
                       3.0 * (cm.fixed_overhead_ns + cm.write_ns_per_byte * row);
    } else {
      tp.record_bytes = row;
      tp.transfer_ns = cm.fixed_overhead_ns + cm.read_ns_per_byte * row;
    }
    tp.ratio = tp.transfer_ns / static_cast<double>(tp.record_bytes);
  }
  return out;
}

CacheAlloc allocate_cache(std::uint64_t budget, const std::vector<std::vector<std::uint64_t>>& counts,
                          const std::vector<TypePenalty>& prof) {
  CacheAlloc a;
  a.budget = budget;
  a.bytes.assign(prof.size(), 0);
  a.capacity.assign(prof.size(), 0);
  std::vector<double> mass(prof.size(), 0.0);
  double denom = 0.0;
  for (std::size_t t = 0; t < prof.size(); ++t) {
    if (prof[t].record_bytes == 0) continue;
    const std::uint64_t tot = std::accumulate(counts[t].begin(), counts[t].end(), std::uint64_t{0});
    mass[t] = static_cast<double>(tot) * prof[t].ratio;
    denom += mass[t];
  }
  if (denom <= 0.0) throw std::invalid_argument("nothing to cache: all count*ratio products are zero");
  for (std::size_t t = 0; t < prof.size(); ++t) {
    if (prof[t].record_bytes == 0) continue;
    const double share = static_cast<double>(budget) * mass[t] / denom;
    a.capacity[t] = static_cast<std::uint64_t>(share) / prof[t].record_bytes;
    a.bytes[t] = a.capacity[t] * prof[t].record_bytes;
  }
  return a;
}

}  // namespace hetgpu
