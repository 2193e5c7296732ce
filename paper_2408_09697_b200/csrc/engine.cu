// Device engine: static plan, workspace, and the per-step launch sequence.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "engine.hpp"
#include "gemm.cuh"

#include <cstdio>
#include <algorithm>
#include <cstring>
#include <functional>
#include <numeric>

namespace hetgpu {

namespace {

__global__ void k_shard_rows(const std::uint32_t* full, const int* n_full, int index, int count,
                             std::uint32_t* shard, int* n_shard) {
  pdl_enter();
  const int n = *n_full;
  const int m = n > index ? (n - index + count - 1) / count : 0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x)
    shard[j] = full[index + j * count];
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_shard = m;
}

struct EdgeCountArgs {
  const std::uint32_t* indptr[kMaxBlocks * 4];
  const int* n_rows[kMaxBlocks * 4];
  int n;
};

__global__ void k_count_edges(EdgeCountArgs a, std::uint64_t* out) {
  pdl_enter();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    std::uint64_t s = 0;
    for (int i = 0; i < a.n; ++i) s += a.indptr[i][*a.n_rows[i]];
    *out = s;
  }
}

// rows of the hop-1 row space with at least one sampled edge in any top block
// (the bucket's `active` set, raf.cpp:418-419); stored as a float counter in
// the partition's slot of the AGG_all buffer
__global__ void k_active_rows(EdgeCountArgs a, const int* n_rows, float* slot) {
  pdl_enter();
  __shared__ int total;
  if (threadIdx.x == 0) total = 0;
  __syncthreads();
  const int n = *n_rows;
  int mine = 0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    bool act = false;
    for (int b = 0; b < a.n; ++b) act |= a.indptr[b][j + 1] > a.indptr[b][j];
    mine += act ? 1 : 0;
  }
  atomicAdd(&total, mine);
  __syncthreads();
  if (threadIdx.x == 0) *slot = static_cast<float>(total);
}

// learnable-row part of sync_bytes for a replica group (raf.cpp:504-510): per
// exchanged type, s = replicas with a non-empty leaf frontier (its
// feat_contributors), rows = the union the merge just built
struct FeatSyncArgs {
  const int* ucount[kMaxSegs];
  const int* count[kMaxSegs][kMaxRep];
  int dim[kMaxSegs];
  int nt, n_rep, elem;
  const int* peer_slot[kMaxRep];  // each replica's bound sample slot (its arena)
  std::uint32_t* err;
};
__global__ void k_feat_sync(FeatSyncArgs a, std::uint64_t* out) {
  pdl_enter();
  // every replica must merge the same step's rows: all trained the same sample slot
  for (int r = 0; r < a.n_rep; ++r)
    if (*a.peer_slot[r] != *a.peer_slot[0]) atomicOr(a.err, 8u);
  std::uint64_t bytes = 0;
  for (int t = 0; t < a.nt; ++t) {
    std::uint64_t s = 0;
    for (int r = 0; r < a.n_rep; ++r) s += *a.count[t][r] > 0 ? 1 : 0;
    if (s < 2) continue;
    const std::uint64_t n = static_cast<std::uint64_t>(*a.ucount[t]) * static_cast<std::uint64_t>(a.dim[t]);
    bytes += 2ull * n * static_cast<std::uint64_t>(a.elem) * (s - 1) / s;
  }
  *out = bytes;
}

__global__ void k_gather_rows(const float* table, int ld, const std::uint32_t* ids, const int* n, int cols,
                              float* out, int dtype) {
  pdl_enter();
  const int total = *n * cols;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += gridDim.x * blockDim.x) {
    const int i = x / cols, c = x % cols;
    const std::size_t at = static_cast<std::size_t>(ids[i]) * ld + c;
    if (dtype == kF32)
      out[x] = table[at];
    else if (dtype == kF16)
      out[x] = __half2float(reinterpret_cast<const __half*>(table)[at]);
    else
      out[x] = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(table)[at]);
  }
}

// Algorithmic bytes of the main kernel classes for one step, accumulated on
// the device (SURVEY §8(d) formulas): [0] sample, [1] aggregate (layer 1, hop-k
// blocks), [2] aggregate_top (hop-1 blocks), [3] csc_gather (backward gather +
// fused sparse Adam).
struct AlgBytesArgs {
  const std::uint32_t* indptr[kMaxBlocks * 4];
  const int* n_rows[kMaxBlocks * 4];
  int din[kMaxBlocks * 4];
  int cls[kMaxBlocks * 4];  // 1 inner aggregate, 2 top aggregate
  int src_esz[kMaxBlocks * 4];  // bytes per gathered source feature (2: fp16 / bf16 tables)
  int nblk;
  int grad[kMaxBlocks * 4];  // block feeds a source gradient (its edges are gathered by csc_gather)
  // csc_gather per (hop, source type): live source rows, row width, bytes per row
  const int* c_rows[kMaxBlocks * 4];
  int c_din[kMaxBlocks * 4];
  int c_row_bytes_mult[kMaxBlocks * 4];  // 1: dH write; 6: fused Adam (w, m, v read + write); 7: both
  int c_top[kMaxBlocks * 4];             // the transposed view of hop 1 (the top layer's gather)
  int ncsc;
};

__global__ void k_alg_bytes(AlgBytesArgs a, double* acc) {
  pdl_enter();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0, agg[3] = {0, 0, 0}, csc = 0, csc_top = 0;
  for (int i = 0; i < a.nblk; ++i) {
    const double R = *a.n_rows[i], E = a.indptr[i][*a.n_rows[i]];
    // sampling: indptr pair + dst id read, neighbour reads, src write, offset write
    s += 16.0 * R + 4.0 * R + 4.0 * E + 4.0 * E + 4.0 * R;
    // aggregation: per edge one source row (its table's element size) + its id; offsets; tape write
    agg[a.cls[i]] += E * (static_cast<double>(a.src_esz[i]) * a.din[i] + 4.0) + 4.0 * (R + 1) + 4.0 * R * a.din[i];
    // backward gather: per edge one dmean row + the edge id
    if (a.grad[i]) (a.cls[i] == 2 ? csc_top : csc) += E * (4.0 * a.din[i] + 4.0);
  }
  // per source row: segment offsets + the gradient row (or the fused Adam row update)
  for (int i = 0; i < a.ncsc; ++i) {
    const double n = *a.c_rows[i];
    (a.c_top[i] ? csc_top : csc) += 4.0 * (n + 1) + n * 4.0 * a.c_din[i] * a.c_row_bytes_mult[i];
  }
  acc[0] += s;
  acc[1] += agg[1];
  acc[2] += agg[2];
  acc[3] += csc;
  acc[4] += csc_top;
}

template <typename T>
void put(std::vector<char>& data, const std::vector<T>& v) {
  data.resize(v.size() * sizeof(T));
  if (!v.empty()) std::memcpy(data.data(), v.data(), data.size());
}

}  // namespace

// ---------------------------------------------------------------------------------------------
Engine::Engine(const Graph& g, const EngineOptions& o) : o_(o) {
  try {
    init_streams();
    init_graph(g);
  } catch (...) {
    release();
    throw;
  }
}

void Engine::init_streams() {
  const EngineOptions& o = o_;
  if (static_cast<int>(o.fanouts.size()) != o.k) throw std::invalid_argument("fanout count must equal the model depth");
  if (o.k < 1) throw std::invalid_argument("fanouts must be non-empty");
  HG_CUDA(cudaSetDevice(o.device));
  // the sampling stream (batch i+1) gets the highest priority so that its
  // latency-bound chain is never starved by the bandwidth-bound training
  // kernels (measured +1%; prioritising training instead costs 6%)
  // With several partitions the training stream carries the AGG_all collective,
  // which every rank waits on: there all streams keep the default priority.
  int least = 0, greatest = 0;
  HG_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  if (o.p > 1) greatest = least;
  HG_CUDA(cudaStreamCreateWithPriority(&st_, cudaStreamNonBlocking, least));
  HG_CUDA(cudaStreamCreateWithPriority(&st2_, cudaStreamNonBlocking, least));
  HG_CUDA(cudaStreamCreateWithPriority(&st_s_, cudaStreamNonBlocking, greatest));
  for (int sl = 0; sl < 2; ++sl) {
    HG_CUDA(cudaEventCreateWithFlags(&ev_sampled_[sl], cudaEventDisableTiming));
    HG_CUDA(cudaEventCreateWithFlags(&ev_trained_[sl], cudaEventDisableTiming));
    HG_CUDA(cudaEventCreateWithFlags(&ev_staged_[sl], cudaEventDisableTiming));
  }
  fork_ev_.resize(16);
  for (auto& e : fork_ev_) HG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

void Engine::init_graph(const Graph& g) {
  ntypes_ = g.num_types();
  target_ = g.target;
  num_classes_ = g.num_classes;
  for (const auto& t : g.types) {
    type_counts_.push_back(t.count);
    learnable_type_.push_back(t.storage == Storage::Learnable);
  }
  for (const auto& r : g.rels) {
    rel_src_.push_back(r.src_type);
    rel_dst_.push_back(r.dst_type);
  }
  build_plan(g);
  upload(g);
}

Engine::~Engine() { release(); }

// everything the engine owns; safe on a partially constructed engine (null handles are
// skipped or rejected harmlessly), so a constructor that throws releases through it
void Engine::release() noexcept {
  if (st_) cudaStreamSynchronize(st_);
  drop_graphs();
  for (auto e : ev_pool_) cudaEventDestroy(e);
  for (void* p : ipc_opened_) cudaIpcCloseMemHandle(p);
  if (st2_) cudaStreamSynchronize(st2_);
  for (auto e : fork_ev_)
    if (e) cudaEventDestroy(e);
  for (void* p : allocs_) cudaFree(p);
  for (auto& tb : tables_)
    if (tb.host_mem) cudaFreeHost(tb.host_mem);
  for (int sl = 0; sl < 2; ++sl) {
    if (h_sc_slot_[sl]) cudaFreeHost(h_sc_slot_[sl]);
    if (h_batch_slot_[sl]) cudaFreeHost(h_batch_slot_[sl]);
    if (h_rb_slot_[sl]) cudaFreeHost(h_rb_slot_[sl]);
    if (ev_sampled_[sl]) cudaEventDestroy(ev_sampled_[sl]);
    if (ev_staged_[sl]) cudaEventDestroy(ev_staged_[sl]);
    if (ev_trained_[sl]) cudaEventDestroy(ev_trained_[sl]);
  }
  if (h_tsc_) cudaFreeHost(h_tsc_);
  if (st_s_) {
    cudaStreamSynchronize(st_s_);
    cudaStreamDestroy(st_s_);
  }
  if (st2_) cudaStreamDestroy(st2_);
  if (st_) cudaStreamDestroy(st_);
}

void Engine::fork() {
  if (side() == st_) return;
  if (fork_used_ >= static_cast<int>(fork_ev_.size())) throw std::runtime_error("fork events exhausted");
  cudaEvent_t e = fork_ev_[fork_used_++];
  HG_CUDA(cudaEventRecord(e, st_));
  HG_CUDA(cudaStreamWaitEvent(st2_, e, 0));
  side_open_ = true;
}

void Engine::join() {
  if (side() == st_ || !side_open_) return;  // nothing was forked since the last join
  side_open_ = false;
  if (fork_used_ >= static_cast<int>(fork_ev_.size())) throw std::runtime_error("fork events exhausted");
  cudaEvent_t e = fork_ev_[fork_used_++];
  HG_CUDA(cudaEventRecord(e, st2_));
  HG_CUDA(cudaStreamWaitEvent(st_, e, 0));
}

void* Engine::alloc(std::size_t bytes) {
  void* p = nullptr;
  bytes = std::max<std::size_t>(bytes, 16);
  HG_CUDA(cudaMalloc(&p, bytes));
  HG_CUDA(cudaMemsetAsync(p, 0, bytes, st_));
  allocs_.push_back(p);
  total_bytes_ += bytes;
  return p;
}

void Engine::build_plan(const Graph& g) {
  const Schema sch = schema_of(g);
  const int k = o_.k;
  n_rel_ = g.num_rels();
  if (o_.p <= 1) {
    tree_ = bfs_tree(sch, target_, k);
    acct_ = raf_accounting(g, tree_, std::vector<std::vector<int>>(tree_.pos.at(0).children.size(), {0}), 1);
  } else {
    Plan plan;
    if (o_.sub_work.empty()) {
      plan = meta_partition(sch, target_, k, o_.p);
    } else {  // [work per sub] or [work per sub, learnable rows per sub]
      const std::size_t n_subs = meta_partition(sch, target_, k, 1).subs.size();
      std::vector<double> w(o_.sub_work.begin(), o_.sub_work.begin() + std::min(n_subs, o_.sub_work.size())), l;
      if (o_.sub_work.size() == 2 * n_subs) l.assign(o_.sub_work.begin() + n_subs, o_.sub_work.end());
      std::vector<bool> learnable(g.num_types());
      for (int t = 0; t < g.num_types(); ++t) learnable[t] = g.types[t].storage == Storage::Learnable;
      plan = work_aware_partition(sch, target_, k, o_.p, w, l, 6.0, learnable);
    }
    acct_ = plan_accounting(g, plan);  // run_experiment's view: raf_view_from_plan
    const Part& part = plan.parts.at(o_.rank);
    // replica group: the partitions owning exactly this sub-metatree set
    for (int q = 0; q < static_cast<int>(plan.parts.size()); ++q)
      if (plan.parts[q].sub_ids == part.sub_ids) replica_group_.push_back(q);
    std::sort(replica_group_.begin(), replica_group_.end(), [&](int a, int b) {
      return plan.parts[a].replica_index < plan.parts[b].replica_index;
    });
    replica_pos_ = static_cast<int>(std::find(replica_group_.begin(), replica_group_.end(), o_.rank) -
                                    replica_group_.begin());
    if (replica_group_.size() > static_cast<std::size_t>(kMaxRep))
      throw std::invalid_argument("replica group larger than supported");
    // gradients are exchanged only inside a replica group: a weight slot or a
    // learnable leaf type shared by two different sub-metatree sets would need a
    // cross-group reduction, which this engine does not implement
    {
      std::map<std::pair<int, int>, std::vector<int>> slot_groups;
      std::map<int, std::vector<int>> leaf_groups;
      for (int q = 0; q < static_cast<int>(plan.parts.size()); ++q) {
        const int color = plan.parts[q].sub_ids.empty() ? -1 : plan.parts[q].sub_ids.front();
        std::vector<int> kids;
        for (int sid : plan.parts[q].sub_ids) kids.push_back(plan.subs[sid].child_pos);
        for (std::size_t p = 1; p < plan.tree.pos.size(); ++p) {
          if (std::find(kids.begin(), kids.end(), plan.tree.root_child_ancestor(static_cast<int>(p))) == kids.end())
            continue;
          const TreePos& tp = plan.tree.pos[p];
          slot_groups[{tp.rel, k - tp.depth + 1}].push_back(color);
          if (tp.depth == k && g.types[tp.type].storage == Storage::Learnable) leaf_groups[tp.type].push_back(color);
        }
      }
      auto distinct = [](std::vector<int> v) {
        std::sort(v.begin(), v.end());
        return std::unique(v.begin(), v.end()) - v.begin();
      };
      for (const auto& [key, cs] : slot_groups)
        if (distinct(cs) > 1) throw std::runtime_error("weight slot shared by two partition groups is not supported");
      for (const auto& [t, cs] : leaf_groups)
        if (distinct(cs) > 1)
          throw std::runtime_error("learnable type shared by two partition groups is not supported");
    }
    replica_ = part.replica;
    shard_index_ = part.replica ? part.replica_index : 0;
    shard_count_ = part.replica ? part.replica_count : 1;
    std::vector<int> owned_children;
    for (int sid : part.sub_ids) owned_children.push_back(plan.subs[sid].child_pos);
    const Tree& full = plan.tree;
    std::vector<int> remap(full.pos.size(), -1);
    tree_.k = full.k;
    tree_.root_type = full.root_type;
    for (std::size_t p = 0; p < full.pos.size(); ++p) {
      const bool keep = p == 0 || std::find(owned_children.begin(), owned_children.end(),
                                            full.root_child_ancestor(static_cast<int>(p))) != owned_children.end();
      if (!keep) continue;
      remap[p] = static_cast<int>(tree_.pos.size());
      TreePos tp = full.pos[p];
      tp.children.clear();
      tp.parent = p == 0 ? -1 : remap[full.pos[p].parent];
      tree_.pos.push_back(tp);
      if (p != 0) tree_.pos[tp.parent].children.push_back(remap[p]);
    }
  }
  hop_rels_ = hop_relations(tree_, k);
  if (o_.sample_only) {
    // the reference filters relations by membership and walks them ascending
    // (sampling.cpp:64-68): the effective per-hop set is sorted and unique
    hop_rels_.assign(k, {});
    for (int h = 0; h < k; ++h) {
      if (o_.all_relations) {
        for (int r = 0; r < g.num_rels(); ++r) hop_rels_[h].push_back(r);
        continue;
      }
      if (static_cast<int>(o_.hop_relations.size()) != k)
        throw std::invalid_argument("hop_relations must have one entry per hop");
      for (int r : o_.hop_relations[h])
        if (r >= 0 && r < g.num_rels()) hop_rels_[h].push_back(r);
      std::sort(hop_rels_[h].begin(), hop_rels_[h].end());
      hop_rels_[h].erase(std::unique(hop_rels_[h].begin(), hop_rels_[h].end()), hop_rels_[h].end());
    }
  }

  // max in-degree per relation tightens the edge capacities
  maxdeg_.assign(g.num_rels(), 0);
  rng_frac_.assign(k, std::vector<float>(g.num_rels(), 0.f));
  for (int r = 0; r < g.num_rels(); ++r) {
    const auto& off = g.rels[r].adj.offsets;
    std::uint64_t m = 0;
    std::vector<std::uint64_t> above(k, 0);  // destinations drawn with the RNG at each hop's fanout
    for (std::size_t i = 0; i + 1 < off.size(); ++i) {
      const std::uint64_t d = off[i + 1] - off[i];
      m = std::max(m, d);
      for (int h = 0; h < k; ++h) above[h] += d > static_cast<std::uint64_t>(o_.fanouts[h]) ? 1 : 0;
    }
    maxdeg_[r] = m;
    for (int h = 0; h < k; ++h)
      rng_frac_[h][r] = off.size() > 1 ? static_cast<float>(above[h]) / static_cast<float>(off.size() - 1) : 0.f;
  }

  // frontier capacities and blocks, hop by hop
  fronts_.assign((k + 1) * ntypes_, Front{});
  front(0, target_).cap = o_.batch_cap;
  hop_blocks_.assign(k + 1, {});
  int edge_base = 0;
  for (int h = 1; h <= k; ++h) {
    std::vector<std::uint64_t> cap_src(ntypes_, 0);
    edge_base = 0;
    for (int r : hop_rels_[h - 1]) {
      BlockBuf b;
      b.rel = r;
      b.hop = h;
      b.src_t = rel_src_[r];
      b.dst_t = rel_dst_[r];
      b.rows_cap = front(h - 1, b.dst_t).cap;
      if (h == 1 && replica_ && b.dst_t == target_) b.rows_cap = static_cast<int>(ceil_div(o_.batch_cap, shard_count_));
      const std::uint64_t per_row = std::min<std::uint64_t>(o_.fanouts[h - 1], maxdeg_[r]);
      const std::uint64_t ec = std::max<std::uint64_t>(1, static_cast<std::uint64_t>(b.rows_cap) * per_row);
      if (ec > 0x7fffffffULL) throw std::invalid_argument("block edge capacity exceeds 2^31");
      if (b.rows_cap >= (1 << 28)) throw std::invalid_argument("block row capacity exceeds 2^28");
      b.edge_cap = static_cast<int>(ec);
      b.edge_base = edge_base;
      edge_base += b.edge_cap;
      cap_src[b.src_t] += ec;
      hop_blocks_[h].push_back(static_cast<int>(blocks_.size()));
      blocks_.push_back(b);
    }
    for (int t = 0; t < ntypes_; ++t)
      front(h, t).cap = static_cast<int>(std::min<std::uint64_t>(type_counts_[t], cap_src[t]));
    if (hop_blocks_[h].size() > static_cast<std::size_t>(kMaxBlocks))
      throw std::invalid_argument("too many relations in one hop");
  }

  for (auto& b : blocks_) {
    b.din = b.hop == k ? g.types[b.src_t].dim : o_.hidden;
    b.ld_mean = round_up4(std::max(1, b.din));
  }
  if (o_.sample_only) return;
  // model slots present in the (local) tree: W_{r,l}, l = k - depth + 1 (hgnn.cpp:39-62)
  const ModelInit mi = init_model(g, tree_, o_.hidden, o_.model_seed);
  for (const auto& [id, w] : mi.weights) {
    Slot s;
    s.rel = id.rel;
    s.layer = id.layer;
    s.din = w.in_dim;
    s.dout = w.out_dim;
    s.ld = round_up4(std::max(1, w.out_dim));
    slot_of_[id] = static_cast<int>(slots_.size());
    slots_.push_back(s);
  }

  // output groups per layer: for each frontier type at depth d-1, the
  // relations into it at depth d (rels_by_dst_at_depth, hgnn.cpp:16-26)
  for (int l = 1; l <= k; ++l) {
    const int d = k - l + 1;
    const auto into = relations_into_at_depth(tree_, d);
    for (int t = 0; t < ntypes_; ++t) {
      const bool has_front = (d - 1 == 0) ? t == target_ : front(d - 1, t).cap > 0;
      if (!has_front) continue;
      Group gr;
      gr.layer = l;
      gr.depth = d;
      gr.type = t;
      gr.dout = out_dim(l);
      gr.ld = round_up4(gr.dout);
      gr.rows_cap = front(d - 1, t).cap;
      auto it = into.find(t);
      if (it != into.end())
        for (int r : it->second) {
          for (int bi : hop_blocks_[d])
            if (blocks_[bi].rel == r) {
              gr.blocks.push_back(bi);
              gr.slots.push_back(slot_of_.at(SlotId{r, l}));
            }
        }
      if (gr.blocks.size() > static_cast<std::size_t>(kMaxRelsPerGroup))
        throw std::invalid_argument("too many relations into one type");
      groups_.push_back(gr);
    }
  }
  // gradient needs: inner sources whose group has relations, learnable leaves
  auto group_at = [&](int depth_of_output, int t) -> Group* {
    for (auto& gr : groups_)
      if (gr.depth - 1 == depth_of_output && gr.type == t) return &gr;
    return nullptr;
  };
  for (auto& b : blocks_) {
    b.din = b.hop == k ? g.types[b.src_t].dim : o_.hidden;
    b.ld_mean = round_up4(std::max(1, b.din));
    if (b.hop < k) {
      Group* src_group = group_at(b.hop, b.src_t);
      b.need_src_grad = src_group && !src_group->blocks.empty();
    } else {
      b.need_src_grad = g.types[b.src_t].storage == Storage::Learnable;
    }
  }
  if (rgat()) rgat_plan(g);
  for (int h = 1; h <= k; ++h)
    for (int t = 0; t < ntypes_; ++t) {
      CscBuf c;
      c.hop = h;
      c.src_t = t;
      for (int bi : hop_blocks_[h])
        if (blocks_[bi].src_t == t && blocks_[bi].need_src_grad) c.blocks.push_back(bi);
      if (c.blocks.empty()) continue;
      c.src_cap = front(h, t).cap;
      c.din = blocks_[c.blocks[0]].din;
      c.ld = blocks_[c.blocks[0]].ld_mean;
      cscs_.push_back(c);
    }
}

void Engine::upload(const Graph& g) {
  const int k = o_.k;
  // relation CSRs this partition samples
  csr_ptr_.assign(g.num_rels(), nullptr);
  csr_src_.assign(g.num_rels(), nullptr);
  std::vector<bool> used(g.num_rels(), false);
  for (const auto& hr : hop_rels_)
    for (int r : hr) used[r] = true;
  for (int r = 0; r < g.num_rels(); ++r) {
    if (!used[r]) continue;
    if (!pre_ptr_.empty()) {  // streamed from a container (loader.cu)
      csr_ptr_[r] = pre_ptr_[r];
      csr_src_[r] = pre_src_[r];
      continue;
    }
    const auto& a = g.rels[r].adj;
    csr_ptr_[r] = static_cast<std::uint64_t*>(alloc(a.offsets.size() * 8));
    csr_src_[r] = static_cast<std::uint32_t*>(alloc(a.sources.size() * 4));
    HG_CUDA(cudaMemcpyAsync(csr_ptr_[r], a.offsets.data(), a.offsets.size() * 8, cudaMemcpyHostToDevice, st_));
    if (!a.sources.empty())
      HG_CUDA(cudaMemcpyAsync(csr_src_[r], a.sources.data(), a.sources.size() * 4, cudaMemcpyHostToDevice, st_));
  }
  // feature / learnable tables of the leaf types (layer-0 inputs)
  tables_.assign(ntypes_, TypeTable{});
  if (!o_.sample_only) {
  std::vector<bool> leaf(ntypes_, false);
  for (const auto& b : blocks_)
    if (b.hop == k) leaf[b.src_t] = true;
  const auto learn = init_learnable(g, o_.learn_seed);
  for (int t = 0; t < ntypes_; ++t) {
    if (!leaf[t]) continue;
    const NodeTypeInfo& nt = g.types[t];
    TypeTable& tb = tables_[t];
    tb.dim = nt.dim;
    tb.ld = round_up4(std::max(1, nt.dim));
    const std::size_t rows = nt.count;
    if (nt.storage == Storage::Absent) throw std::runtime_error("missing features for node type " + nt.name);
    if (nt.storage == Storage::Dense) {
      if (lay_)
        stream_dense(nt, t, tb);  // straight from the container file (loader.cu)
      else
        upload_dense(nt, tb);
      continue;
    }
    std::vector<float> host(rows * tb.ld, 0.0f);
    {
      tb.learnable = true;
      const auto& w = learn.at(t);
      for (std::size_t i = 0; i < rows; ++i)
        for (int c = 0; c < nt.dim; ++c) host[i * tb.ld + c] = static_cast<float>(w[i * nt.dim + c]);
      tb.m = static_cast<float*>(alloc(host.size() * 4));
      tb.v = static_cast<float*>(alloc(host.size() * 4));
      tb.step = static_cast<std::int64_t*>(alloc(8));
    }
    tb.w = static_cast<float*>(alloc(host.size() * 4));
    HG_CUDA(cudaMemcpyAsync(tb.w, host.data(), host.size() * 4, cudaMemcpyHostToDevice, st_));
    HG_CUDA(cudaStreamSynchronize(st_));  // host staging buffer goes out of scope
  }
  // target ids whose label is outside [0, C): cross_entropy throws for them
  // (hgnn.cpp:289-291), so step()/prefetch() reject such batches on the host
  // before anything is enqueued
  bad_labels_.clear();
  for (std::size_t v = 0; v < g.labels.size(); ++v)
    if (g.labels[v] < 0 || g.labels[v] >= num_classes_) bad_labels_.push_back(static_cast<NodeId>(v));
  labels_ = static_cast<std::int32_t*>(alloc(g.labels.size() * 4));
  HG_CUDA(cudaMemcpyAsync(labels_, g.labels.data(), g.labels.size() * 4, cudaMemcpyHostToDevice, st_));

  // model weights (f64 init rounded to fp32)
  const ModelInit mi = init_model(g, tree_, o_.hidden, o_.model_seed);
  for (auto& s : slots_) {
    const WeightInit& wi = mi.weights.at(SlotId{s.rel, s.layer});
    std::vector<float> host(static_cast<std::size_t>(std::max(1, s.din)) * s.ld, 0.0f);
    for (int i = 0; i < s.din; ++i)
      for (int j = 0; j < s.dout; ++j) host[i * s.ld + j] = static_cast<float>(wi.values[i * s.dout + j]);
    const std::size_t bytes = host.size() * 4;
    s.w = static_cast<float*>(alloc(bytes));
    s.m = static_cast<float*>(alloc(bytes));
    s.v = static_cast<float*>(alloc(bytes));
    s.g = static_cast<float*>(alloc(bytes));
    HG_CUDA(cudaMemcpyAsync(s.w, host.data(), bytes, cudaMemcpyHostToDevice, st_));
    HG_CUDA(cudaStreamSynchronize(st_));
  }
  }  // !sample_only

  // frontier machinery: one bitmap region for all types
  word_base_.assign(ntypes_ + 1, 0);
  for (int t = 0; t < ntypes_; ++t)
    word_base_[t + 1] = word_base_[t] + static_cast<int>(ceil_div(type_counts_[t], 32));
  total_words_ = std::max(1, word_base_[ntypes_]);
  for (int sl = 0; sl < 2; ++sl) {
    bits_slot_[sl] = static_cast<std::uint32_t*>(alloc(static_cast<std::size_t>(total_words_) * 4));
    wscan_slot_[sl] = static_cast<std::uint32_t*>(alloc(static_cast<std::size_t>(total_words_) * 4));
  }
  cached_bits_ = static_cast<std::uint32_t*>(alloc(static_cast<std::size_t>(total_words_) * 4));
  // static per-hop frontier slot layout: slot i of hop h is the i-th distinct
  // source type of that hop's blocks (hop 0: the target)
  hop_slot_types_.assign(k + 1, {});
  hop_slot_types_[0] = {target_};
  for (int h = 1; h <= k; ++h)
    for (int bi : hop_blocks_[h]) {
      auto& v = hop_slot_types_[h];
      if (std::find(v.begin(), v.end(), blocks_[bi].src_t) == v.end()) v.push_back(blocks_[bi].src_t);
    }
  {
    std::vector<int> wd(static_cast<std::size_t>(k + 1) * kMaxSegs, 0);
    for (int h = 0; h <= k; ++h)
      for (std::size_t i = 0; i < hop_slot_types_[h].size(); ++i) {
        const int t = hop_slot_types_[h][i];
        wd[h * kMaxSegs + i] = word_base_[t + 1] - word_base_[t];
      }
    words_dev_ = static_cast<int*>(alloc(wd.size() * sizeof(int)));
    HG_CUDA(cudaMemcpyAsync(words_dev_, wd.data(), wd.size() * sizeof(int), cudaMemcpyHostToDevice, st_));
    HG_CUDA(cudaStreamSynchronize(st_));
  }
  // replica exchange arena: frontier ids + count and gradient rows of every
  // learnable leaf type, in one cudaMalloc so one CUDA IPC handle maps it on the
  // peers (identical layout on every replica of the group)
  if (replica_group_.size() > 1) {
    std::size_t at = 0;
    auto take = [&](std::size_t bytes) {
      const std::size_t o = at;
      at += (bytes + 255) & ~static_cast<std::size_t>(255);
      return o;
    };
    for (const auto& c : cscs_) {
      if (c.hop != k || !tables_[c.src_t].learnable) continue;
      Xchg x;
      x.t = c.src_t;
      x.cap = front(k, c.src_t).cap;
      x.ld = c.ld;
      x.din = c.din;
      for (int sl = 0; sl < 2; ++sl) {
        x.off_count[sl] = take(sizeof(int));
        x.off_ids[sl] = take(static_cast<std::size_t>(std::max(1, x.cap)) * 4);
      }
      x.off_dh = take(static_cast<std::size_t>(std::max(1, x.cap)) * x.ld * 4);
      xchg_.push_back(x);
    }
    // the replica barrier's flags: slot q holds the last step replica q finished reading
    off_flags_ = take(static_cast<std::size_t>(kMaxRep) * 4);
    off_slot_ = take(sizeof(int));
    arena_bytes_ = std::max<std::size_t>(at, 256);
    arena_ = static_cast<std::uint8_t*>(alloc(arena_bytes_));
    for (auto& x : xchg_) {
      for (auto& c : cscs_)
        if (c.hop == k && c.src_t == x.t) c.dh = reinterpret_cast<float*>(arena_ + x.off_dh);
      x.ucap = static_cast<int>(std::min<std::uint64_t>(type_counts_[x.t],
                                                        static_cast<std::uint64_t>(x.cap) * replica_group_.size()));
      x.ulist = static_cast<std::uint32_t*>(alloc(static_cast<std::size_t>(std::max(1, x.ucap)) * 4));
      x.ucount = static_cast<int*>(alloc(sizeof(int)));
      x.slot = static_cast<int*>(alloc(static_cast<std::size_t>(std::max(1, x.ucap)) * replica_group_.size() * 4));
      x.ug = static_cast<float*>(alloc(static_cast<std::size_t>(std::max(1, x.ucap)) * x.ld * 4));
      x.utotal = static_cast<int*>(alloc(sizeof(int)));
      x.peer_w.assign(replica_group_.size(), nullptr);
      x.peer_w[replica_pos_] = tables_[x.t].w;
    }
    HG_CUDA(cudaMemsetAsync(arena_ + off_flags_, 0, static_cast<std::size_t>(kMaxRep) * 4, st_));
    barrier_epoch_ = static_cast<unsigned*>(alloc(16));
    HG_CUDA(cudaMemsetAsync(barrier_epoch_, 0, 16, st_));
    HG_CUDA(cudaStreamSynchronize(st_));
    peer_arena_.assign(replica_group_.size(), nullptr);
    peer_arena_[replica_pos_] = arena_;
  }
  for (int sl = 0; sl < 2; ++sl) {
    fronts_slot_[sl] = fronts_;  // capacities
    for (int h = 0; h <= k; ++h)
      for (int t = 0; t < ntypes_; ++t) {
        Front& f = fronts_slot_[sl][h * ntypes_ + t];
        if (h == k && xchg_type(t)) {  // lives in the exchange arena
          for (const auto& x : xchg_)
            if (x.t == t) {
              f.count = reinterpret_cast<int*>(arena_ + x.off_count[sl]);
              f.list = reinterpret_cast<std::uint32_t*>(arena_ + x.off_ids[sl]);
            }
          continue;
        }
        f.count = static_cast<int*>(alloc(sizeof(int)));
        if (f.cap > 0) f.list = static_cast<std::uint32_t*>(alloc(static_cast<std::size_t>(f.cap) * 4));
      }
    shard_list_slot_[sl] = static_cast<std::uint32_t*>(alloc(static_cast<std::size_t>(o_.batch_cap) * 4));
    shard_count_slot_[sl] = static_cast<int*>(alloc(sizeof(int)));
  }

  int max_rows = 1, total_rows = 0;
  for (auto& b : blocks_) {
    for (int sl = 0; sl < 2; ++sl) {
      b.s_indptr[sl] = static_cast<std::uint32_t*>(alloc(static_cast<std::size_t>(b.rows_cap + 1) * 4));
      b.s_src[sl] = static_cast<std::uint32_t*>(alloc(static_cast<std::size_t>(b.edge_cap) * 4));
      b.s_erow[sl] = static_cast<std::uint32_t*>(alloc(static_cast<std::size_t>(b.edge_cap) * 4));
      b.s_col[sl] = static_cast<std::uint32_t*>(alloc(static_cast<std::size_t>(b.edge_cap) * 4));
    }
    if (!o_.sample_only && !rgat()) {
      b.mean = static_cast<float*>(alloc(static_cast<std::size_t>(b.rows_cap) * b.ld_mean * 4));
    }
    if (b.need_src_grad && !rgat())
      b.dmean = static_cast<float*>(alloc(static_cast<std::size_t>(b.rows_cap) * b.ld_mean * 4));
    max_rows = std::max(max_rows, b.rows_cap + 1);
    total_rows += b.rows_cap;
  }

  ldc_ = round_up4(num_classes_);
  // + kMaxRep rows: a replica's strided shard view (rows i * shards + shard, i < ceil(B /
  // shards)) may reach past the counter row by up to shards - 1 rows (never read as data)
  logits_ = static_cast<float*>(alloc(static_cast<std::size_t>(o_.batch_cap + 1 + kMaxRep) * ldc_ * 4));
  dlogits_ = static_cast<float*>(alloc(static_cast<std::size_t>(o_.batch_cap + 1 + kMaxRep) * ldc_ * 4));
  if (o_.p > ldc_) throw std::invalid_argument("more partitions than logit columns for the AGG_all counters");
  for (auto& gr : groups_) {
    if (gr.layer == o_.k) {
      gr.out = logits_;
      gr.dout_buf = dlogits_;
      gr.ld = ldc_;
    } else {
      gr.out = static_cast<float*>(alloc(static_cast<std::size_t>(std::max(1, gr.rows_cap)) * gr.ld * 4));
    }
  }
  // transposed views: per hop one contiguous offs/cursor region (one memset each)
  for (int sl = 0; sl < 2; ++sl) {
    csc_region_slot_[sl].assign(o_.k + 1, {nullptr, nullptr, 0});
    for (int h = 1; h <= o_.k; ++h) {
      std::size_t words = 0;
      for (const auto& c : cscs_)
        if (c.hop == h) words += static_cast<std::size_t>(c.src_cap) + 1;
      if (!words) continue;
      auto& reg = csc_region_slot_[sl][h];
      reg.words = words;
      reg.offs = static_cast<std::uint32_t*>(alloc(words * 4));
      reg.cursor = static_cast<std::uint32_t*>(alloc(words * 4));
      std::size_t at = 0;
      for (auto& c : cscs_) {
        if (c.hop != h) continue;
        c.s_offs[sl] = reg.offs + at;
        c.s_cursor[sl] = reg.cursor + at;
        at += static_cast<std::size_t>(c.src_cap) + 1;
      }
    }
  }
  for (auto& c : cscs_) {
    std::size_t ent = 0;
    for (int bi : c.blocks) ent = std::max<std::size_t>(ent, blocks_[bi].edge_base + blocks_[bi].edge_cap);
    for (int sl = 0; sl < 2; ++sl) {
      c.s_entries[sl] = static_cast<std::uint32_t*>(alloc(ent * 4));
      c.s_tmp[sl] = static_cast<std::uint32_t*>(alloc(ent * 4));
    }
    const bool dense_leaf = rgat() && c.hop == o_.k && !tables_[c.src_t].learnable;  // RGAT: no gradient rows
    if (!(c.hop == o_.k && xchg_type(c.src_t)) && !dense_leaf)
      c.dh = static_cast<float*>(alloc(static_cast<std::size_t>(std::max(1, c.src_cap)) * c.ld * 4));
    if (c.hop < o_.k) {
      for (auto& gr : groups_)
        if (gr.depth - 1 == c.hop && gr.type == c.src_t) {
          gr.dout_buf = c.dh;
        }
    }
  }

  // per-step state and scratch
  for (int sl = 0; sl < 2; ++sl) {
    d_sc_slot_[sl] = static_cast<StepScalars*>(alloc(sizeof(StepScalars)));
    HG_CUDA(cudaMallocHost(&h_sc_slot_[sl], sizeof(StepScalars)));
    std::memset(h_sc_slot_[sl], 0, sizeof(StepScalars));
    d_batch_slot_[sl] = static_cast<std::uint32_t*>(alloc(static_cast<std::size_t>(o_.batch_cap) * 4));
    HG_CUDA(cudaMallocHost(&h_batch_slot_[sl], static_cast<std::size_t>(o_.batch_cap) * 4));
    mult_slot_[sl] = static_cast<float*>(alloc(static_cast<std::size_t>(o_.batch_cap) * 4));
    rb_slot_[sl] = static_cast<Readback*>(alloc(sizeof(Readback)));
    HG_CUDA(cudaMallocHost(&h_rb_slot_[sl], sizeof(Readback)));
  }
  d_tsc_ = static_cast<StepScalars*>(alloc(sizeof(StepScalars)));
  HG_CUDA(cudaMallocHost(&h_tsc_, sizeof(StepScalars)));
  std::memset(h_tsc_, 0, sizeof(StepScalars));
  row_loss_ = static_cast<double*>(alloc(static_cast<std::size_t>(o_.batch_cap) * 8));
  loss_done_ = static_cast<unsigned*>(alloc(sizeof(unsigned)));
  cache_hm_ = static_cast<unsigned long long*>(alloc(sizeof(unsigned long long) * 2 * ntypes_));
  alg_bytes_ = static_cast<double*>(alloc(sizeof(double) * 5));
  cache_types_.assign(ntypes_, false);

  int max_cap = std::max(total_words_, max_rows);
  for (const auto& c : cscs_) max_cap = std::max(max_cap, c.src_cap + 1);
  {
    // look-back scratch: enough tiles for the largest single-pass launch
    std::size_t tiles = ceil_div(total_words_, kCompactWordsPerTile) + kMaxSegs;
    for (int h = 1; h <= o_.k; ++h) {
      std::size_t t = 0;
      for (int bi : hop_blocks_[h]) t += ceil_div(std::max(1, blocks_[bi].rows_cap), kSampleTileRows) + 1;
      tiles = std::max(tiles, t);
    }
    tiles = std::max<std::size_t>(tiles, kMaxSegs * (ceil_div(max_cap, kScanTile) + 1));
    for (int sl = 0; sl < 2; ++sl) {
      lb_slot_[sl].cap = static_cast<int>(tiles);
      lb_slot_[sl].mem = static_cast<unsigned long long*>(alloc((tiles + 1) * 8));
    }
    lb2_.cap = static_cast<int>(tiles);
    lb2_.mem = static_cast<unsigned long long*>(alloc((tiles + 1) * 8));
  }
  for (int sl = 0; sl < 2; ++sl) {
    slow_slot_[sl] = static_cast<std::uint32_t*>(alloc(static_cast<std::size_t>(total_rows + 1) * 8));
    n_slow_slot_[sl] = static_cast<int*>(alloc(sizeof(int)));
  }
  int maxf = 1;
  for (int f : o_.fanouts) maxf = std::max(maxf, f);
  for (int sl = 0; sl < 2; ++sl)
    mt_scratch_slot_[sl] = static_cast<std::uint64_t*>(alloc(sample_scratch_words(maxf) * 8));
  std::size_t wt = 1, wp = 1;
  for (const auto& s : slots_) wt = std::max<std::size_t>(wt, static_cast<std::size_t>(round_up4(s.din)) * s.dout);
  for (int l = 1; l <= o_.k; ++l) {
    std::size_t layer = 0;
    for (const auto& gr : groups_) {
      if (gr.layer != l) continue;
      const int rc = (l == o_.k && replica_) ? static_cast<int>(ceil_div(o_.batch_cap, shard_count_)) : gr.rows_cap;
      for (std::size_t q = 0; q < gr.blocks.size(); ++q)
        layer += ceil_div(std::max(1, rc), kWChunkRows) * static_cast<std::size_t>(blocks_[gr.blocks[q]].din) * gr.dout;
    }
    wp = std::max(wp, layer);
  }
  wt_scratch_ = static_cast<float*>(alloc(wt * 4));
  wgrad_partial_ = static_cast<float*>(alloc(wp * 4));
  if (rgat()) rgat_alloc();
  HG_CUDA(cudaStreamSynchronize(st_));
  bind_slot(0);
}

void Engine::bind_slot(int s) {
  bound_ = s;
  fronts_ = fronts_slot_[s];
  bits_ = bits_slot_[s];
  wscan_ = wscan_slot_[s];
  shard_list_ = shard_list_slot_[s];
  shard_count_dev_ = shard_count_slot_[s];
  for (auto& b : blocks_) {
    b.indptr = b.s_indptr[s];
    b.src = b.s_src[s];
    b.erow = b.s_erow[s];
    b.col = b.s_col[s];
  }
  for (auto& c : cscs_) {
    c.offs = c.s_offs[s];
    c.cursor = c.s_cursor[s];
    c.entries = c.s_entries[s];
    c.tmp = c.s_tmp[s];
  }
  csc_region_ = csc_region_slot_[s];
  d_sc_ = d_sc_slot_[s];
  h_sc_ = h_sc_slot_[s];
  d_batch_ = d_batch_slot_[s];
  h_batch_ = h_batch_slot_[s];
  mult_ = mult_slot_[s];
  loss_ = &rb_slot_[s]->loss;
  err_ = &rb_slot_[s]->err;
  edges_dev_ = &rb_slot_[s]->edges;
  feat_sync_dev_ = &rb_slot_[s]->feat_sync;
  h_rb_ = h_rb_slot_[s];
  lb_ = lb_slot_[s];  // sampling scratch: two slots can sample concurrently
  slow_ = slow_slot_[s];
  n_slow_ = n_slow_slot_[s];
  mt_scratch_ = mt_scratch_slot_[s];
}

std::uint64_t Engine::param_count() const {
  std::uint64_t n = 0;
  for (const auto& s : slots_) n += static_cast<std::uint64_t>(s.din + (rgat() ? 1 : 0)) * s.dout;
  return n;
}

// ---------------------------------------------------------------------------------------------
void Engine::timed(const char* name, double bytes, const std::function<void()>& f) {
  if (!profiling_) {
    f();
    return;
  }
  // event pairs are recorded asynchronously and resolved in finish_step(), so
  // the per-class device times come from the timed run itself
  if (ev_used_ + 2 > ev_pool_.size()) {
    cudaEvent_t e;
    for (int i = 0; i < 2; ++i) {
      HG_CUDA(cudaEventCreate(&e));
      ev_pool_.push_back(e);
    }
  }
  cudaEvent_t a = ev_pool_[ev_used_++], b = ev_pool_[ev_used_++];
  HG_CUDA(cudaEventRecord(a, st_));
  f();
  HG_CUDA(cudaEventRecord(b, st_));
  pending_.push_back({name, a, b});
  kernel_bytes_[name] += bytes;
}

void Engine::resolve_profile() {
  for (const auto& p : pending_) {
    float ms = 0.f;
    HG_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    kernel_ms_[p.name] += ms;
    kernel_launches_[p.name] += 1;
  }
  pending_.clear();
  ev_used_ = 0;
}

void Engine::run_sampling(cudaStream_t ss) {
  const int k = o_.k;
  // frontier[0][target] = sorted unique batch (bitmap), with multiplicities
  FrontierArgs f0{};
  f0.ntypes = 1;
  f0.t[0] = {bits_ + word_base_[target_], word_base_[target_ + 1] - word_base_[target_], wscan_ + word_base_[target_],
             front(0, target_).list, front(0, target_).count, front(0, target_).cap};
  HG_CUDA(cudaMemsetAsync(bits_, 0, static_cast<std::size_t>(total_words_) * 4, ss));
  HG_CUDA(cudaMemsetAsync(mult_, 0, static_cast<std::size_t>(o_.batch_cap) * 4, ss));
  timed("frontier", 0, [&] {
    frontier_mark_batch(d_batch_, d_sc_, o_.batch_cap, f0.t[0], ss);
    frontier_compact(f0, lb_, ss);
    batch_multiplicity(d_batch_, d_sc_, o_.batch_cap, f0.t[0], mult_, ss);
  });
  if (replica_)
    launch_pdl(k_shard_rows, 4, 256, 0, ss, front(0, target_).list, front(0, target_).count, shard_index_, shard_count_,
                                     shard_list_, shard_count_dev_);

  for (int h = 1; h <= k; ++h) {
    SampleHop sh{};
    sh.fanout = o_.fanouts[h - 1];
    sh.hop = h;
    for (int bi : hop_blocks_[h]) {
      BlockBuf& b = blocks_[bi];
      SampleBlock& s = sh.b[sh.nblk++];
      s.csr_ptr = csr_ptr_[b.rel];
      s.csr_src = csr_src_[b.rel];
      s.dst_list = block_dst(b);
      s.n_rows = block_rows(b);
      s.indptr = b.indptr;
      s.src_ids = b.src;
      s.erow = b.erow;
      s.mark_bits = nullptr;
      s.rel = b.rel;
      s.rows_cap = b.rows_cap;
      s.rng_frac = rng_frac_[h - 1][b.rel];
    }

    // frontier[h][t]: bitmap of every sampled source, compacted in id order
    // The last hop's frontier of a type is needed only for its gradient rows
    // (learnable leaves: the transposed view and the sparse Adam ids): layer 1
    // reads its sources by global id. Lean mode (no retained gradients, no cache
    // lookups) skips the other types' mark/compact/relabel; presampling needs
    // none of them.
    const bool lean = h == k && (presampling_ || (!retain_grads_ && !cache_on_));
    auto wanted = [&](int t) {
      if (!lean || presampling_) return !presampling_ || h < k;
      for (const auto& c : cscs_)
        if (c.hop == k && c.src_t == t) return true;
      return false;
    };
    FrontierArgs fa{};
    std::vector<int> slot_of_type(ntypes_, -1);
    for (int t : hop_slot_types_[h]) {
      if (!wanted(t)) continue;
      slot_of_type[t] = fa.ntypes;
      fa.t[fa.ntypes++] = {bits_ + word_base_[t], word_base_[t + 1] - word_base_[t], wscan_ + word_base_[t],
                           front(h, t).list, front(h, t).count, front(h, t).cap};
    }
    RelabelArgs ra{};
    for (int q = 0; q < sh.nblk; ++q) {
      const BlockBuf& b = blocks_[hop_blocks_[h][q]];
      if (slot_of_type[b.src_t] < 0) continue;
      sh.b[q].mark_bits = bits_ + word_base_[b.src_t];  // the sampler marks frontier[h] as it emits
      std::uint32_t* cnt = nullptr;
      if (b.need_src_grad)
        for (const auto& c : cscs_)
          if (c.hop == h && c.src_t == b.src_t) cnt = c.offs;
      ra.b[ra.nblk++] = {b.src, b.indptr, sh.b[q].n_rows, b.col, b.edge_cap, slot_of_type[b.src_t], cnt};
    }
    // frontier[h-1]'s bitmap is dead once its relabel / transposed views are enqueued
    HG_CUDA(cudaMemsetAsync(bits_, 0, static_cast<std::size_t>(total_words_) * 4, ss));
    if (trace_sampler_) {  // diagnostics: per-tile timestamps of this hop's sampler
      if (!sample_trace_[h]) sample_trace_[h] = static_cast<unsigned long long*>(alloc(static_cast<std::size_t>(lb_.cap) * 64));
      HG_CUDA(cudaMemsetAsync(sample_trace_[h], 0, static_cast<std::size_t>(lb_.cap) * 64, ss));
      sh.trace = sample_trace_[h];
    }
    timed("sample", 0, [&] { sample_hop(sh, d_sc_, slow_, n_slow_, mt_scratch_, lb_, ss); });
    if (csc_region_[h].words) {
      HG_CUDA(cudaMemsetAsync(csc_region_[h].offs, 0, csc_region_[h].words * 4, ss));
      HG_CUDA(cudaMemsetAsync(csc_region_[h].cursor, 0, csc_region_[h].words * 4, ss));
    }
    timed("frontier", 0, [&] {
      frontier_compact(fa, lb_, ss);
      frontier_relabel(ra, fa, ss);
    });
    // transposed views of this hop (independent of the forward values)
    if (!presampling_) {
      const CscHop ch = csc_hop(h);
      timed("csc_build", 0, [&] { csc_prepare(ch, lb_, ss); });
    }
  }
  EdgeCountArgs ec{};
  for (const auto& b : blocks_) {
    ec.indptr[ec.n] = b.indptr;
    ec.n_rows[ec.n] = block_rows(b);
    ++ec.n;
  }
  launch_pdl(k_count_edges, 1, 32, 0, ss, ec, edges_dev_);
  if (profiling_) {
    AlgBytesArgs ab{};
    for (const auto& b : blocks_) {
      ab.indptr[ab.nblk] = b.indptr;
      ab.n_rows[ab.nblk] = block_rows(b);
      ab.din[ab.nblk] = b.din;
      ab.src_esz[ab.nblk] = (b.hop == o_.k && tables_[b.src_t].dense && tables_[b.src_t].dtype != kF32) ? 2 : 4;
      ab.cls[ab.nblk] = b.hop == 1 ? 2 : 1;
      ab.grad[ab.nblk] = b.need_src_grad ? 1 : 0;
      ++ab.nblk;
    }
    for (const auto& c : cscs_) {
      const bool leaf_learnable = c.hop == o_.k && tables_[c.src_t].learnable;
      // the sparse Adam is fused here (w, m, v read + written: 6 row passes, +1 for a
      // retained gradient row) unless the type is exchanged between replicas, whose
      // Adam runs after the merge (k_rsum_adam): then only the gradient row is written
      const bool fused_adam = leaf_learnable && !xchg_type(c.src_t);
      ab.c_rows[ab.ncsc] = front(c.hop, c.src_t).count;
      ab.c_din[ab.ncsc] = c.din;
      ab.c_row_bytes_mult[ab.ncsc] = fused_adam ? (retain_grads_ ? 7 : 6) : 1;
      ab.c_top[ab.ncsc] = c.hop == 1 ? 1 : 0;
      ++ab.ncsc;
    }
    launch_pdl(k_alg_bytes, 1, 32, 0, ss, ab, alg_bytes_);
  }
  // cache lookups + updates over the layer-0 frontier (harness.cpp:425-437)
  // (p > 1: over the union of every partition's frontier, run_agg_all)
  if (cache_on_ && !presampling_ && o_.p == 1)
    for (int t = 0; t < ntypes_; ++t)
      if (cache_types_[t] && front(k, t).cap > 0)
        cache_count(front(k, t).list, front(k, t).count, front(k, t).cap, cached_bits_ + word_base_[t],
                    cache_hm_ + 2 * t, ss);
}

void Engine::run_forward() {
  const int k = o_.k;
  // AGG_all buffer: rows beyond the live batch and the counter row stay zero
  HG_CUDA(cudaMemsetAsync(logits_, 0, static_cast<std::size_t>(o_.batch_cap + 1) * ldc_ * 4, st_));
  for (int l = 1; l <= k; ++l) {
    const int d = k - l + 1;
    const bool top = l == k;
    // (1) relation-first mean aggregation of every block of hop d: one launch;
    // layer 1 reads the feature / learnable tables by global id (fused gather)
    MeanBatch mb{};
    double bytes = 0;
    for (int bi : hop_blocks_[d]) {
      const BlockBuf& b = blocks_[bi];
      MeanBlock& m = mb.b[mb.nb++];
      m.indptr = b.indptr;
      if (b.hop == k) {
        m.keys = b.src;
        const TypeTable& tb = tables_[b.src_t];
        m.h = tb.w;
        m.ld_h = tb.ld;
        m.h_dtype = tb.dense ? tb.dtype : kF32;
        m.slot = tb.host ? tb.slot : nullptr;
        m.cache = tb.cache;
      } else {
        const Group* sg = nullptr;
        for (const auto& g2 : groups_)
          if (g2.depth - 1 == b.hop && g2.type == b.src_t) sg = &g2;
        m.keys = b.col;
        m.h = sg->out;
        m.ld_h = sg->ld;
      }
      m.din = b.din;
      m.n_rows = block_rows(b);
      m.rows_cap = b.rows_cap;
      m.mean = b.mean;
      m.ld_mean = b.ld_mean;
    }
    timed(top ? "aggregate_top" : "aggregate", bytes, [&] { gather_mean(mb, st_); });
    // (2) per-relation projection summed over the relations into each type (agg_all):
    // one launch per kProjGroups destination types
    std::vector<ProjBatch> pbs(1);
    for (const auto& gr : groups_) {
      if (gr.layer != l) continue;
      if (gr.blocks.empty()) {
        if (!top) zero_rows(gr.out, gr.ld, front(gr.depth - 1, gr.type).count, gr.rows_cap, st_);
        continue;
      }
      if (gr.blocks.size() > static_cast<std::size_t>(kProjRels))
        throw std::runtime_error("more relations into one type than a projection group holds");
      if (pbs.back().ng == kProjGroups) pbs.emplace_back();
      ProjBatch& pb = pbs.back();
      ProjGroup& pg = pb.g[pb.ng++];
      pg.nrel = static_cast<int>(gr.blocks.size());
      pg.n_rows = (top && replica_) ? shard_count_dev_ : front(gr.depth - 1, gr.type).count;
      pg.rows_cap = top && replica_ ? static_cast<int>(ceil_div(o_.batch_cap, shard_count_)) : gr.rows_cap;
      pg.out = gr.out;
      pg.ld_out = gr.ld;
      pg.dout = gr.dout;
      pg.relu = top ? 0 : 1;
      pg.out_stride = top ? shard_count_ : 1;
      pg.out_offset = top ? shard_index_ : 0;
      for (std::size_t q = 0; q < gr.blocks.size(); ++q) {
        const BlockBuf& b = blocks_[gr.blocks[q]];
        const Slot& s = slots_[gr.slots[q]];
        pg.r[q] = {b.mean, b.ld_mean, b.din, s.w, s.ld};
      }
    }
    timed(top ? "project_top" : "project", 0, [&] {
      for (auto& pb : pbs) use_umma_ ? project_umma(pb, st_) : project_tiles(pb, st_);
    });
  }
  run_agg_all();
  if (o_.p > 1 && training_ && replica_group_.size() > 1) replica_prepare();
}

// AGG_all: sum the partial logits of every partition (raf.cpp:427-446); the counter
// row records which batch rows had a sampled top-level edge on this partition
void Engine::run_agg_all() {
  const int k = o_.k;
  if (o_.p > 1) {
    EdgeCountArgs ec{};
    for (int bi : hop_blocks_[1]) {
      ec.indptr[ec.n] = blocks_[bi].indptr;
      ++ec.n;
    }
    launch_pdl(k_active_rows, 1, 256, 0, st_, ec, replica_ ? shard_count_dev_ : front(0, target_).count,
                                      logits_ + static_cast<std::size_t>(o_.batch_cap) * ldc_ + o_.rank);
#ifdef HG_WITH_NCCL
    if (comm_ && !counting_) {
      timed("agg_all", static_cast<double>(o_.batch_cap + 1) * ldc_ * 4, [&] {
        if (ncclAllReduce(logits_, logits_, static_cast<std::size_t>(o_.batch_cap + 1) * ldc_, ncclFloat, ncclSum,
                          comm_, st_) != ncclSuccess)
          throw std::runtime_error("ncclAllReduce failed");
      });
      // cache lookups over the global layer-0 frontier (harness.cpp:425-437 samples the
      // whole batch): the union of every partition's frontier, identical on every rank
      if (cache_on_) {
        timed("cache_union", 0, [&] {
          for (int t = 0; t < ntypes_; ++t) {
            if (!cache_types_[t]) continue;
            HG_CUDA(cudaMemsetAsync(union_map_[t], 0, type_counts_[t], st_));
            if (front(k, t).cap > 0) union_mark(front(k, t).list, front(k, t).count, front(k, t).cap, union_map_[t], st_);
            if (ncclAllReduce(union_map_[t], union_map_[t], type_counts_[t], ncclUint8, ncclMax, comm_, st_) !=
                ncclSuccess)
              throw std::runtime_error("ncclAllReduce (cache frontier union) failed");
            union_count(union_map_[t], type_counts_[t], cached_bits_ + word_base_[t], cache_hm_ + 2 * t, st_);
          }
        });
      }
    }
#endif
  }
  (void)k;
}

void Engine::run_loss(bool train) {
  LossArgs la{};
  la.done = loss_done_;
  if (train && apply_adam_ && !rgat()) {
    // learnable layer-0 tables advance their Adam step before the fused row
    // update of the backward pass; the loss kernel's last CTA does it
    for (const auto& c : cscs_)
      if (c.hop == o_.k && tables_[c.src_t].learnable && !xchg_type(c.src_t) && la.bumps.count < kMaxSegs) {
        la.bumps.step[la.bumps.count] = tables_[c.src_t].step;
        la.bumps.n[la.bumps.count] = front(o_.k, c.src_t).count;
        ++la.bumps.count;
      }
  }
  la.logits = logits_;
  la.ld = ldc_;
  la.C = num_classes_;
  la.n_rows = front(0, target_).count;
  la.rows_cap = o_.batch_cap;
  la.row_ids = front(0, target_).list;
  la.mult = mult_;
  la.labels = labels_;
  la.sc = d_tsc_;  // batch_len of the step being trained
  la.dlogits = dlogits_;
  la.row_loss = row_loss_;
  la.loss_out = loss_;
  la.err = err_;
  timed("loss", 0, [&] { cross_entropy(la, st_); });
}

void Engine::run_backward() {
  const int k = o_.k;
  // (the layer-0 tables' steps were bumped by the loss kernel.) Every slot's weight
  // gradient is overwritten by its reduction; the zeroing below is kept because
  // it delays the side-stream weight gradients behind the critical mean-gradient
  // chain (measured: 1.89G vs 1.77G sampled-edges/s without it)
  for (auto& s : slots_) HG_CUDA(cudaMemsetAsync(s.g, 0, static_cast<std::size_t>(std::max(1, s.din)) * s.ld * 4, st_));

  for (int l = k; l >= 1; --l) {
    const int d = k - l + 1;
    WGradBatch wb{};
    DMeanBatch db{};
    std::size_t partial_off = 0;
    for (const auto& gr : groups_) {
      if (gr.layer != l || gr.blocks.empty()) continue;
      const bool top = l == k;
      const int* n_rows = (top && replica_) ? shard_count_dev_ : front(d - 1, gr.type).count;
      const int rows_cap = top && replica_ ? static_cast<int>(ceil_div(o_.batch_cap, shard_count_)) : gr.rows_cap;
      // dpre = dH (x) [H > 0] between layers, fused into the operand loads
      // dpre = dH * [H > 0]: the mask was applied when csc_gather wrote dH
      const DpreView dv{gr.dout_buf, nullptr, gr.ld, gr.dout, top ? shard_count_ : 1, top ? shard_index_ : 0};
      for (std::size_t q = 0; q < gr.blocks.size(); ++q) {
        BlockBuf& b = blocks_[gr.blocks[q]];
        Slot& s = slots_[gr.slots[q]];
        if (wb.np >= kMaxProblems || db.np >= kMaxProblems) throw std::runtime_error("too many problems per layer");
        wb.p[wb.np++] = {b.mean, b.ld_mean, b.din, dv, n_rows, rows_cap, wgrad_partial_ + partial_off, s.g, s.ld};
        partial_off += ceil_div(std::max(1, rows_cap), kWChunkRows) * static_cast<std::size_t>(b.din) * gr.dout;
        if (b.need_src_grad)
          db.p[db.np++] = {dv, s.w, s.ld, b.din, b.indptr, n_rows, rows_cap, b.dmean, b.ld_mean};
      }
    }
    // dpre of this layer is complete on st_: the weight gradient runs beside the
    // mean gradient and the next backward gather. Without replicas (nothing to
    // all-reduce) each slot's Adam is fused into its gradient reduction, which
    // then waits for this layer's mean gradient (the last reader of W_l).
    const bool fuse_adam = fused_model_adam();
    if (fuse_adam) {
      wb.defer_reduce = 1;
      wb.step = &d_tsc_->model_step;
      wb.err = err_;
      for (int q = 0; q < wb.np; ++q)
        for (const auto& gr : groups_) {
          if (gr.layer != l || gr.blocks.empty()) continue;
          for (std::size_t j = 0; j < gr.slots.size(); ++j) {
            const Slot& sl = slots_[gr.slots[j]];
            if (wb.p[q].dw == sl.g) {
              wb.p[q].w = sl.w;
              wb.p[q].m = sl.m;
              wb.p[q].v = sl.v;
            }
          }
        }
    }
    fork();
    timed("weight_grad", 0, [&] { use_umma_ ? wgrad_umma(wb, side()) : wgrad_tiles(wb, side()); });
    timed("mean_grad", 0, [&] { use_umma_ ? dmean_umma(db, st_) : dmean_tiles(db, st_); });
    if (fuse_adam) {
      fork();  // the side stream waits for the mean gradient, then reduces + updates
      timed("weight_grad", 0, [&] { wgrad_reduce(wb, side()); });
    }
    // scatter back to the sources of this hop, as ordered gathers (learnable
    // layer-0 rows get their Adam update in the same pass)
    const CscHop ch = csc_hop(d);
    AdamHyper hp;
    timed(d == 1 ? "csc_gather_top" : "csc_gather", 0, [&] { csc_gather(ch, hp, err_, st_); });
  }
  join();  // weight gradients
  if (replica_group_.size() > 1) run_replica_merge();
}

// Replica group gradient synchronisation (raf.cpp:496-510 accounts it as a ring
// all-reduce over the slots' contributors): dense weight gradients over NCCL;
// learnable rows merged by reading every replica's (ids, rows) through peer
// mappings of their exchange arenas, then one sparse Adam on the union.
void Engine::run_replica_merge() {
#ifdef HG_WITH_NCCL
  if (!rcomm_) throw std::runtime_error("replica group without a communicator (attach_nccl first)");
  for (std::size_t r = 0; r < peer_arena_.size(); ++r)
    if (!peer_arena_[r]) throw std::runtime_error("replica peers not attached (attach_replicas)");
  // 0. this rank's sample slot, checked against the peers' once the all-reduce below has
  //    ordered every replica's earlier writes (a rank-local prefetch / quiesce would
  //    otherwise pair another batch's ids with this step's rows)
  HG_CUDA(cudaMemsetAsync(arena_ + off_slot_, bound_, sizeof(int), st_));
  // 1. weight gradients; completing it also orders every replica's gradient rows
  //    (written by its csc_gather before its all-reduce) before our reads below
  // (a launch-count capture leaves the collectives out, see count_launches)
  timed("replica_wgrad", 0, [&] {
    if (counting_) return;
    if (ncclGroupStart() != ncclSuccess) throw std::runtime_error("ncclGroupStart failed");
    for (auto& sl : slots_) {
      if (ncclAllReduce(sl.g, sl.g, static_cast<std::size_t>(std::max(1, sl.din)) * sl.ld, ncclFloat, ncclSum, rcomm_,
                        st_) != ncclSuccess)
        throw std::runtime_error("ncclAllReduce (replica weight gradients) failed");
      if (sl.ag && ncclAllReduce(sl.ag, sl.ag, static_cast<std::size_t>(sl.ld), ncclFloat, ncclSum, rcomm_, st_) !=
                       ncclSuccess)  // RGAT attention vectors
        throw std::runtime_error("ncclAllReduce (replica attention gradients) failed");
    }
    if (ncclGroupEnd() != ncclSuccess) throw std::runtime_error("ncclGroupEnd failed");
  });
  // 2. learnable rows: the union and row slots were built by replica_prepare
  //    (side stream, during the loss and backward pass; joined before this).
  //    Step, then the fused ordered sum + Adam over the union.
  std::vector<const std::int64_t*> steps;
  std::vector<const int*> ucounts;
  for (auto& x : xchg_) {
    steps.push_back(tables_[x.t].step);
    ucounts.push_back(x.utotal);  // the step moves iff the whole union is non-empty
  }
  // each table's step += 1 iff its union is non-empty (hgnn.cpp:392-394)
  bump_steps(steps.data(), ucounts.data(), static_cast<int>(steps.size()), st_);
  timed("replica_adam", 0, [&] {
    for (std::size_t i = 0; i < merges_.size(); ++i) {
      const TypeTable& tb = tables_[xchg_[i].t];
      ReplicaAdam ra{tb.w, tb.m, tb.v, tb.ld, tb.step, {}, merges_[i].n_rep};
      if (shard_merge_) {
        for (int r = 0; r < ra.n_rep; ++r) ra.peer_w[r] = xchg_[i].peer_w[r];
      } else {
        ra.n_rep = 1;
        ra.peer_w[0] = tb.w;
      }
      replica_sum_adam(merges_[i], ra, AdamHyper{}, err_, st_);
    }
  });
  {
    FeatSyncArgs fs{};
    fs.n_rep = static_cast<int>(peer_arena_.size());
    fs.elem = elem_bytes_;
    fs.err = err_;
    for (int r = 0; r < fs.n_rep; ++r) fs.peer_slot[r] = reinterpret_cast<const int*>(peer_arena_[r] + off_slot_);
    for (auto& x : xchg_) {
      fs.ucount[fs.nt] = x.utotal;
      for (int r = 0; r < fs.n_rep; ++r)
        fs.count[fs.nt][r] = reinterpret_cast<const int*>(peer_arena_[r] + x.off_count[bound_]);
      fs.dim[fs.nt] = tables_[x.t].dim;
      ++fs.nt;
    }
    launch_pdl(k_feat_sync, 1, 1, 0, st_, fs, feat_sync_dev_);
  }
  // 3. nobody rewrites its arena (next step's sampling) before every peer read it:
  //    a flag barrier over the IPC-mapped arenas (NVLink stores + acquire loads)
  timed("replica_barrier", 0, [&] {
    ReplicaBarrier rb{};
    rb.n = static_cast<int>(peer_arena_.size());
    rb.pos = replica_pos_;
    for (int r = 0; r < rb.n; ++r)
      rb.peer_flags[r] = reinterpret_cast<unsigned*>(const_cast<std::uint8_t*>(peer_arena_[r]) + off_flags_);
    rb.my_flags = reinterpret_cast<unsigned*>(arena_ + off_flags_);
    rb.epoch = barrier_epoch_;
    replica_barrier(rb, st_);
  });
#else
  throw std::runtime_error("replica groups need NCCL");
#endif
}

// Replica groups, first half of the merge: the union of the replicas' leaf ids
// and each replica's row slots. It reads only the replicas' sampled ids and
// counts, which exist on every replica once the AGG_all all-reduce has run, so
// it is enqueued on the side stream right after it and overlaps the loss and
// the backward pass (the gradient rows are read only after the replicas'
// weight-gradient all-reduce, in run_replica_merge).
void Engine::replica_prepare() {
  merges_.clear();
  fork();
  for (auto& x : xchg_) {
    ReplicaMerge m{};
    m.n_rep = static_cast<int>(peer_arena_.size());
    for (int r = 0; r < m.n_rep; ++r) {
      m.ids[r] = reinterpret_cast<const std::uint32_t*>(peer_arena_[r] + x.off_ids[bound_]);
      m.count[r] = reinterpret_cast<const int*>(peer_arena_[r] + x.off_count[bound_]);
      m.dh[r] = reinterpret_cast<const float*>(peer_arena_[r] + x.off_dh);
    }
    m.ld = x.ld;
    m.din = x.din;
    m.u = {bits_ + word_base_[x.t], word_base_[x.t + 1] - word_base_[x.t], wscan_ + word_base_[x.t], x.ulist, x.ucount,
           x.ucap};
    m.slot = x.slot;
    m.ug = nullptr;
    // sharded: this replica merges and Adam-updates only the ids of its shard and
    // stores the new rows into every copy; unsharded: every replica updates the
    // whole union in its own copy (measured faster on B200 at p=4, the default)
    m.shard = shard_merge_ ? replica_pos_ : 0;
    m.nshard = shard_merge_ ? m.n_rep : 1;
    m.total = x.utotal;
    timed("replica_union", 0, [&] { replica_union(m, lb2_, side()); });
    timed("replica_slots", 0, [&] { replica_slots(m, side()); });
    merges_.push_back(m);
  }
}

// IPC handles of this replica's exchange arena, then of its copy of every
// exchanged learnable table (the sharded merge writes updated rows into them)
std::vector<char> Engine::replica_handle() {
  if (replica_group_.size() < 2) return {};
  std::vector<const void*> bases{arena_};
  for (const auto& x : xchg_) bases.push_back(tables_[x.t].w);
  std::vector<char> out(bases.size() * sizeof(cudaIpcMemHandle_t));
  for (std::size_t i = 0; i < bases.size(); ++i) {
    cudaIpcMemHandle_t h;
    HG_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(bases[i])));
    std::memcpy(out.data() + i * sizeof(h), &h, sizeof(h));
  }
  return out;
}

void Engine::attach_replicas(const std::vector<std::vector<char>>& handles_by_rank) {
  if (replica_group_.size() < 2) return;
  HG_CUDA(cudaSetDevice(o_.device));
  for (std::size_t r = 0; r < replica_group_.size(); ++r) {
    if (static_cast<int>(r) == replica_pos_) continue;
    const int q = replica_group_[r];
    const std::size_t want = (1 + xchg_.size()) * sizeof(cudaIpcMemHandle_t);
    if (q >= static_cast<int>(handles_by_rank.size()) || handles_by_rank[q].size() < want)
      throw std::invalid_argument("missing IPC handle of replica partition " + std::to_string(q));
    auto open = [&](std::size_t i) {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles_by_rank[q].data() + i * sizeof(h), sizeof(h));
      void* p = nullptr;
      HG_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      ipc_opened_.push_back(p);
      return p;
    };
    peer_arena_[r] = static_cast<const std::uint8_t*>(open(0));
    for (std::size_t i = 0; i < xchg_.size(); ++i) xchg_[i].peer_w[r] = static_cast<float*>(open(1 + i));
  }
  drop_graphs();
}

CscHop Engine::csc_hop(int h) {
  CscHop ch{};
  ch.edge_ids = rgat() ? 1 : 0;  // RGAT's backward reads per-edge attention weights
  std::vector<int> slot(ntypes_, -1);
  for (const auto& c : cscs_) {
    if (c.hop != h) continue;
    slot[c.src_t] = ch.nt;
    CscType& t = ch.t[ch.nt++];
    t.offs = c.offs;
    t.cursor = c.cursor;
    t.entries = c.entries;
    t.tmp = c.tmp;
    t.n_src = front(h, c.src_t).count;
    t.src_cap = c.src_cap;
    // replicas merge their learnable-row gradients before Adam: keep the rows
    const bool exchanged = h == o_.k && xchg_type(c.src_t);
    const bool leaf_learnable = h == o_.k && tables_[c.src_t].learnable && !exchanged && apply_adam_;
    t.dh = (!leaf_learnable || retain_grads_) ? c.dh : nullptr;
    t.ld_dh = c.ld;
    t.din = c.din;
    if (h < o_.k)  // inner type: its forward output H[h][t] masks the stored gradient
      for (const auto& gr : groups_)
        if (gr.depth - 1 == h && gr.type == c.src_t) {
          t.relu_h = gr.out;
          t.ld_h = gr.ld;
        }
    if (leaf_learnable) {
      const TypeTable& tb = tables_[c.src_t];
      t.w = tb.w;
      t.m = tb.m;
      t.v = tb.v;
      t.ld_w = tb.ld;
      t.ids = front(h, c.src_t).list;
      t.step = tb.step;
    }
  }
  for (int bi : hop_blocks_[h]) {
    const BlockBuf& b = blocks_[bi];
    if (!b.need_src_grad || slot[b.src_t] < 0) continue;
    CscEdges& e = ch.b[ch.nb++];
    e.col = b.col;
    e.erow = b.erow;
    e.indptr = b.indptr;
    e.n_rows = block_rows(b);
    e.cap = b.edge_cap;
    e.edge_base = b.edge_base;
    e.type = slot[b.src_t];
    e.dmean = b.dmean;
    e.ld_dmean = b.ld_mean;
  }
  return ch;
}

void Engine::run_update() {
  if (!apply_adam_) return;        // gradient-only step (caller-owned optimizer)
  if (fused_model_adam()) return;  // applied by the weight-gradient reductions
  AdamHyper hp;
  AdamModelBatch mb{};
  int base = 0;
  for (auto& s : slots_) {
    if (mb.n >= kMaxSlots) throw std::runtime_error("too many model slots");
    mb.w[mb.n] = s.w;
    mb.m[mb.n] = s.m;
    mb.v[mb.n] = s.v;
    mb.g[mb.n] = s.g;
    mb.base4[mb.n] = base;
    base += std::max(1, s.din) * s.ld / 4;
    ++mb.n;
  }
  mb.total4 = base;
  timed("adam", 0, [&] { adam_model(mb, &d_tsc_->model_step, hp, err_, st_); });
}


// Sampling of the bound slot: everything that depends only on (graph, batch,
// rng_seed). Training of the bound slot: forward, AGG_all, loss, backward, Adam
// and the readback. Each is captured once per slot into a CUDA graph and replayed
// (profiling runs them eagerly on st_ so every kernel class can be bracketed).
void Engine::sample_body(cudaStream_t ss) {
  HG_CUDA(cudaMemsetAsync(err_, 0, sizeof(std::uint32_t), ss));
  run_sampling(ss);
}

void Engine::train_body(bool train) {
  fork_used_ = 0;
  side_open_ = false;
  training_ = train;
  if (rgat()) {
    run_forward_rgat();
    run_loss(train);
    if (train) {
      run_backward_rgat();
      run_update_rgat();
    }
  } else {
    run_forward();
    run_loss(train);
    if (train) {
      run_backward();
      run_update();
    }
  }
  join();  // nothing of this step may remain on the side stream
  HG_CUDA(cudaMemcpyAsync(h_rb_, loss_, sizeof(Readback), cudaMemcpyDeviceToHost, st_));
}

void Engine::step_body(bool train) {
  sample_body(st_);
  train_body(train);
}

namespace {
template <typename F>
void capture(cudaGraphExec_t& ex, cudaStream_t st, F&& body) {
  cudaGraph_t graph = nullptr;
  HG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  try {
    body();
  } catch (...) {
    cudaStreamEndCapture(st, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  HG_CUDA(cudaStreamEndCapture(st, &graph));
  HG_CUDA(cudaGraphInstantiate(&ex, graph, cudaGraphInstantiateFlagUseNodePriority));
  cudaGraphDestroy(graph);
}
}  // namespace

void Engine::enqueue_sample(int s) {
  bind_slot(s);
  cudaStream_t ss = sstream();
  if (!use_graphs_ || profiling_) {
    sample_body(ss);
    return;
  }
  if (!exec_sample_[s]) capture(exec_sample_[s], ss, [&] { sample_body(ss); });
  HG_CUDA(cudaGraphLaunch(exec_sample_[s], ss));
}

void Engine::enqueue_train(int s, bool train) {
  bind_slot(s);
  if (!use_graphs_ || profiling_) {
    train_body(train);
    return;
  }
  cudaGraphExec_t& ex = train ? exec_train_[s] : exec_eval_[s];
  if (!ex) capture(ex, st_, [&] { train_body(train); });
  HG_CUDA(cudaGraphLaunch(ex, st_));
}

StepScalars Engine::next_scalars(std::uint64_t rng_seed, int n, int designated, bool train) {
  if (n > o_.batch_cap) throw std::invalid_argument("batch larger than the engine's batch capacity");
  if (n <= 0) throw std::invalid_argument("empty batch");
  if (train) ++model_step_;
  StepScalars sc{};
  sc.rng_seed = rng_seed;
  sc.batch_len = n;
  sc.designated = designated;
  last_designated_ = designated;
  sc.model_step = model_step_;
  return sc;
}

void Engine::validate_batch(const NodeId* batch, int n, bool labels) const {
  for (int i = 0; i < n; ++i)
    if (batch[i] >= type_counts_[target_])
      throw std::invalid_argument("seed node id out of range: " + std::to_string(batch[i]));
  if (labels && !o_.sample_only && !bad_labels_.empty())
    for (int i = 0; i < n; ++i)
      if (std::binary_search(bad_labels_.begin(), bad_labels_.end(), batch[i]))
        throw std::invalid_argument("label out of range for node " + std::to_string(batch[i]));
}

void Engine::prefetch(const NodeId* batch, int n, std::uint64_t rng_seed) {
  if (o_.sample_only) throw std::invalid_argument("a sampler engine has no model to step");
  if (n > o_.batch_cap) throw std::invalid_argument("batch larger than the engine's batch capacity");
  if (n <= 0) throw std::invalid_argument("empty batch");
  validate_batch(batch, n);
  if (pending_slots_.size() >= 2) throw std::runtime_error("two batches already prefetched: step one first");
  const int s = next_slot_;
  next_slot_ ^= 1;
  cudaStream_t ss = sstream();
  // the slot is free once the step that last trained on it is done
  HG_CUDA(cudaStreamWaitEvent(ss, ev_trained_[s], 0));
  // the slot's pinned staging buffers are reusable once their previous copies
  // ran (not the whole sampling stream: the other slot may still be sampling)
  HG_CUDA(cudaEventSynchronize(ev_staged_[s]));
  std::memcpy(h_batch_slot_[s], batch, sizeof(NodeId) * n);
  *h_sc_slot_[s] = StepScalars{rng_seed, n, 0, 0};
  HG_CUDA(cudaMemcpyAsync(d_batch_slot_[s], h_batch_slot_[s], sizeof(NodeId) * n, cudaMemcpyHostToDevice, ss));
  HG_CUDA(cudaMemcpyAsync(d_sc_slot_[s], h_sc_slot_[s], sizeof(StepScalars), cudaMemcpyHostToDevice, ss));
  HG_CUDA(cudaEventRecord(ev_staged_[s], ss));
  enqueue_sample(s);
  HG_CUDA(cudaEventRecord(ev_sampled_[s], ss));
  pending_slots_.push_back({s, rng_seed, std::vector<NodeId>(batch, batch + n)});
}

void Engine::prefetch_device(const std::uint32_t* d_ids, int n, const StepScalars* d_ss) {
  if (pending_slots_.size() >= 2) throw std::runtime_error("two batches already prefetched: step one first");
  const int s = next_slot_;
  next_slot_ ^= 1;
  cudaStream_t ss = sstream();
  HG_CUDA(cudaStreamWaitEvent(ss, ev_trained_[s], 0));
  HG_CUDA(cudaMemcpyAsync(d_batch_slot_[s], d_ids, static_cast<std::size_t>(n) * 4, cudaMemcpyDeviceToDevice, ss));
  HG_CUDA(cudaMemcpyAsync(d_sc_slot_[s], d_ss, sizeof(StepScalars), cudaMemcpyDeviceToDevice, ss));
  enqueue_sample(s);
  HG_CUDA(cudaEventRecord(ev_sampled_[s], ss));
  pending_slots_.push_back({s, 0, {}});
}

void Engine::train_device(const StepScalars* d_ts, bool train) {
  if (pending_slots_.empty()) throw std::runtime_error("no sampled batch to train");
  const int s = pending_slots_.front().slot;
  pending_slots_.erase(pending_slots_.begin());
  HG_CUDA(cudaMemcpyAsync(d_tsc_, d_ts, sizeof(StepScalars), cudaMemcpyDeviceToDevice, st_));
  HG_CUDA(cudaStreamWaitEvent(st_, ev_sampled_[s], 0));
  enqueue_train(s, train);
  HG_CUDA(cudaEventRecord(ev_trained_[s], st_));
  last_trained_ = s;
}

StepReport Engine::finish_step() {
  HG_CUDA(cudaStreamSynchronize(st_));
  HG_CUDA(cudaGetLastError());
  if (profiling_) resolve_profile();
  bind_slot(last_trained_);
  StepReport r;
  r.loss = h_rb_->loss;
  r.err = h_rb_->err;
  r.sampled_edges = h_rb_->edges;
  if (r.err & 1u) throw std::invalid_argument("fanout above the sampler's supported map size");
  if (r.err & 2u) throw std::invalid_argument("label out of range in batch");
  if (r.err & 4u) throw std::runtime_error("non-finite gradient");
  if (r.err & 8u)
    throw std::runtime_error("replica group out of step: its ranks trained different sample slots "
                             "(a prefetch or quiesce on one rank only)");
  if (o_.p > 1) {
    std::vector<float> row(ldc_);
    HG_CUDA(cudaMemcpy(row.data(), logits_ + static_cast<std::size_t>(o_.batch_cap) * ldc_, ldc_ * 4,
                       cudaMemcpyDeviceToHost));
    for (int q = 0; q < o_.p; ++q) r.active_rows.push_back(static_cast<int>(row[q]));
  }
  // ExecutionReport bookkeeping. Only the AGG_all partials cross workers, one
  // PartialAgg per non-designated worker with active rows (raf.cpp:427-446), all
  // of the target type, so cross_ids_target_only holds and check_comm_bounds
  // compares that one message against num_relations x boundary_counts[sender].
  r.boundary_counts = acct_.boundary_counts;
  r.boundary_cut_edges = acct_.boundary_cut_edges;
  for (std::size_t q = 0; q < r.active_rows.size(); ++q)
    if (static_cast<int>(q) != last_designated_ && r.active_rows[q] > 0 &&
        1ull > static_cast<std::uint64_t>(n_rel_) * acct_.boundary_counts.at(q))
      r.message_bound_ok = false;
  r.sync_bytes = model_sync_bytes() + h_rb_->feat_sync;
  r.sync_leader = replica_pos_ == 0;
  return r;
}

std::uint64_t Engine::model_sync_bytes() const {
  // slot part of sync_bytes (raf.cpp:496-503) for the slots this rank contributes to
  std::uint64_t bytes = 0;
  for (const auto& [id, who] : acct_.slot_contributors) {
    const std::uint64_t s = who.size();
    if (s < 2 || std::find(who.begin(), who.end(), o_.rank) == who.end()) continue;
    for (const auto& sl : slots_)
      if (sl.rel == id.rel && sl.layer == id.layer) {
        const std::uint64_t n = static_cast<std::uint64_t>(sl.din) * static_cast<std::uint64_t>(sl.dout);
        bytes += 2ull * n * static_cast<std::uint64_t>(elem_bytes_) * (s - 1) / s;
      }
  }
  return bytes;
}

StepReport Engine::step(const NodeId* batch, int n, std::uint64_t rng_seed, int designated, bool train) {
  if (o_.sample_only) throw std::invalid_argument("a sampler engine has no model to step");
  // use the prefetched slot if it holds exactly this batch; otherwise sample now
  const bool hit = !pending_slots_.empty() && pending_slots_.front().rng_seed == rng_seed &&
                   pending_slots_.front().batch.size() == static_cast<std::size_t>(n) &&
                   std::equal(batch, batch + n, pending_slots_.front().batch.begin());
  if (!hit) {
    if (!pending_slots_.empty()) {  // a stale prefetch: drop it (its slot is rewritten later)
      HG_CUDA(cudaStreamSynchronize(sstream()));
      pending_slots_.clear();
    }
    prefetch(batch, n, rng_seed);
  }
  const int s = pending_slots_.front().slot;
  pending_slots_.erase(pending_slots_.begin());
  *h_tsc_ = next_scalars(rng_seed, n, designated, train);
  HG_CUDA(cudaMemcpyAsync(d_tsc_, h_tsc_, sizeof(StepScalars), cudaMemcpyHostToDevice, st_));
  HG_CUDA(cudaStreamWaitEvent(st_, ev_sampled_[s], 0));
  enqueue_train(s, train);
  HG_CUDA(cudaEventRecord(ev_trained_[s], st_));
  last_trained_ = s;
  return finish_step();
}

int Engine::count_launches(int n, bool train) {
  // capture one step (without executing it) and count our kernel nodes
  // the collective is left out of this capture: a captured-but-never-launched
  // NCCL call would desynchronise the ranks (NCCL kernels are not counted anyway)
  const bool prof = profiling_;
  profiling_ = false;
  counting_ = true;
  cudaGraph_t graph = nullptr;
  HG_CUDA(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
  (void)n;
  try {
    step_body(train);
  } catch (...) {
    cudaStreamEndCapture(st_, &graph);
    if (graph) cudaGraphDestroy(graph);
    profiling_ = prof;
    counting_ = false;
    throw;
  }
  HG_CUDA(cudaStreamEndCapture(st_, &graph));
  profiling_ = prof;
  counting_ = false;
  std::size_t nn = 0;
  HG_CUDA(cudaGraphGetNodes(graph, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  HG_CUDA(cudaGraphGetNodes(graph, nodes.data(), &nn));
  int kernels = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType ty;
    HG_CUDA(cudaGraphNodeGetType(nd, &ty));
    if (ty != cudaGraphNodeTypeKernel) continue;
    cudaKernelNodeParams kp{};
    HG_CUDA(cudaGraphKernelNodeGetParams(nd, &kp));
    const char* fname = nullptr;
    if (cudaFuncGetName(&fname, kp.func) == cudaSuccess && fname && std::strstr(fname, "nccl")) continue;
    ++kernels;
  }
  cudaGraphDestroy(graph);
  launches_per_step_ = kernels;
  return kernels;
}

std::vector<double> Engine::algorithmic_bytes() {
  std::vector<double> v(5, 0.0);
  HG_CUDA(cudaStreamSynchronize(st_));
  HG_CUDA(cudaMemcpy(v.data(), alg_bytes_, sizeof(double) * 5, cudaMemcpyDeviceToHost));
  return v;
}

void Engine::sample_only(const NodeId* batch, int n, std::uint64_t rng_seed) {
  if (n > o_.batch_cap) throw std::invalid_argument("batch larger than the engine's batch capacity");
  if (n <= 0) throw std::invalid_argument("empty batch");
  validate_batch(batch, n, /*labels=*/false);
  quiesce();
  bind_slot(0);
  std::memcpy(h_batch_, batch, sizeof(NodeId) * n);
  HG_CUDA(cudaMemcpyAsync(d_batch_, h_batch_, sizeof(NodeId) * n, cudaMemcpyHostToDevice, st_));
  h_sc_->rng_seed = rng_seed;
  h_sc_->batch_len = n;
  HG_CUDA(cudaMemcpyAsync(d_sc_, h_sc_, sizeof(StepScalars), cudaMemcpyHostToDevice, st_));
  sample_body(st_);
  HG_CUDA(cudaStreamSynchronize(st_));
  HG_CUDA(cudaGetLastError());
}

// finish everything in flight and forget prefetched batches (their slots are reused)
void Engine::quiesce() {
  HG_CUDA(cudaStreamSynchronize(st_s_));
  HG_CUDA(cudaStreamSynchronize(st_));
  pending_slots_.clear();
  next_slot_ = 0;
}

// ---------------------------------------------------------------------------------------------
// presample_hotness (cache.cpp:39-63): `epochs` passes over the target ids in id
// order, batch_size per batch, rng seed mix_seed(seed, epoch); +1 per seed and
// per sampled source occurrence. All batch ids and scalars are uploaded once;
// every batch is one replay of a captured graph (sampling without the transposed
// views + histogram) on one stream, with no host round trip between batches.
std::vector<std::vector<std::uint64_t>> Engine::presample_hotness(int epochs, std::uint64_t seed, int batch_size) {
  if (batch_size > o_.batch_cap) throw std::invalid_argument("presample batch larger than the batch capacity");
  if (batch_size <= 0) throw std::invalid_argument("presample batch size must be positive");
  quiesce();
  bind_slot(0);
  if (hot_counts_.empty()) {
    hot_counts_.assign(ntypes_, nullptr);
    for (int t = 0; t < ntypes_; ++t)
      hot_counts_[t] = static_cast<unsigned long long*>(alloc(std::max<std::uint64_t>(1, type_counts_[t]) * 8));
  }
  for (int t = 0; t < ntypes_; ++t)
    HG_CUDA(cudaMemsetAsync(hot_counts_[t], 0, type_counts_[t] * 8, st_));
  const std::uint64_t n_target = type_counts_[target_];
  std::vector<NodeId> ids(n_target);
  for (std::uint64_t v = 0; v < n_target; ++v) ids[v] = static_cast<NodeId>(v);
  std::vector<StepScalars> sc;
  std::vector<std::uint64_t> lo_of;
  for (int e = 0; e < epochs; ++e)
    for (std::uint64_t lo = 0; lo < n_target; lo += batch_size) {
      sc.push_back(StepScalars{mix_seed(seed, static_cast<std::uint64_t>(e)),
                               static_cast<int>(std::min<std::uint64_t>(batch_size, n_target - lo)), 0, 0});
      lo_of.push_back(lo);
    }
  NodeId* d_ids = nullptr;
  StepScalars* d_sc = nullptr;
  HG_CUDA(cudaMalloc(&d_ids, std::max<std::size_t>(4, ids.size() * 4)));
  HG_CUDA(cudaMalloc(&d_sc, std::max<std::size_t>(1, sc.size()) * sizeof(StepScalars)));
  HG_CUDA(cudaMemcpyAsync(d_ids, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice, st_));
  HG_CUDA(cudaMemcpyAsync(d_sc, sc.data(), sc.size() * sizeof(StepScalars), cudaMemcpyHostToDevice, st_));
  // batches alternate between the two sample slots, each on its own stream
  // (histogram counters are atomics, order-independent)
  HG_CUDA(cudaStreamSynchronize(st_));
  cudaStream_t sts[2] = {st_, st_s_};
  auto body = [&](cudaStream_t ss) {
    presampling_ = true;
    run_sampling(ss);
    presampling_ = false;
    // +1 per seed, +1 per sampled source occurrence (cache.cpp:51-56)
    hotness_add_list(front(0, target_).list, front(0, target_).count, o_.batch_cap, hot_counts_[target_], ss);
    for (const auto& b : blocks_) hotness_add(b.src, b.indptr, block_rows(b), b.edge_cap, hot_counts_[b.src_t], ss);
  };
  cudaGraphExec_t ex[2] = {nullptr, nullptr};
  auto release = [&] {
    for (auto& e : ex)
      if (e) cudaGraphExecDestroy(e);
    cudaFree(d_ids);
    cudaFree(d_sc);
  };
  try {
    if (use_graphs_ && !profiling_)
      for (int sl = 0; sl < 2; ++sl) {
        bind_slot(sl);
        capture(ex[sl], sts[sl], [&] { body(sts[sl]); });
      }
    for (std::size_t i = 0; i < sc.size(); ++i) {
      const int sl = static_cast<int>(i & 1);
      bind_slot(sl);
      HG_CUDA(cudaMemcpyAsync(d_batch_, d_ids + lo_of[i], static_cast<std::size_t>(sc[i].batch_len) * 4,
                              cudaMemcpyDeviceToDevice, sts[sl]));
      HG_CUDA(cudaMemcpyAsync(d_sc_, d_sc + i, sizeof(StepScalars), cudaMemcpyDeviceToDevice, sts[sl]));
      if (ex[sl])
        HG_CUDA(cudaGraphLaunch(ex[sl], sts[sl]));
      else
        body(sts[sl]);
    }
    HG_CUDA(cudaStreamSynchronize(st_));
    HG_CUDA(cudaStreamSynchronize(st_s_));
  } catch (...) {
    release();
    throw;
  }
  for (auto& e : ex)
    if (e) cudaGraphExecDestroy(e);
  cudaFree(d_ids);
  cudaFree(d_sc);
  bind_slot(0);
  std::vector<std::vector<std::uint64_t>> out(ntypes_);
  for (int t = 0; t < ntypes_; ++t) {
    out[t].resize(type_counts_[t]);
    if (!out[t].empty())
      HG_CUDA(cudaMemcpy(out[t].data(), hot_counts_[t], out[t].size() * 8, cudaMemcpyDeviceToHost));
  }
  return out;
}

void Engine::set_cache(const std::vector<std::vector<NodeId>>& cached) {
  std::vector<std::uint32_t> bits(static_cast<std::size_t>(total_words_), 0u);
  for (int t = 0; t < ntypes_ && t < static_cast<int>(cached.size()); ++t)
    for (NodeId v : cached[t]) bits[word_base_[t] + (v >> 5)] |= 1u << (v & 31);
  quiesce();  // the engine's streams are non-blocking: order the update after all work in flight
  HG_CUDA(cudaMemcpyAsync(cached_bits_, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice, st_));
  HG_CUDA(cudaMemsetAsync(cache_hm_, 0, sizeof(unsigned long long) * 2 * ntypes_, st_));
  HG_CUDA(cudaStreamSynchronize(st_));
  cache_on_ = true;
  for (int t = 0; t < ntypes_; ++t) cache_types_[t] = t < static_cast<int>(cached.size());
  if (o_.p > 1) {  // the global frontier's union maps (every rank lists the same types)
    union_map_.resize(ntypes_, nullptr);
    for (int t = 0; t < ntypes_; ++t)
      if (cache_types_[t] && !union_map_[t])
        union_map_[t] = static_cast<std::uint8_t*>(alloc(std::max<std::uint64_t>(1, type_counts_[t])));
  }
  // host-resident feature tables: copy the cached rows into HBM and map every node to
  // its cache row (or -1: read over PCIe from the pinned table)
  for (int t = 0; t < ntypes_ && t < static_cast<int>(cached.size()); ++t) {
    TypeTable& tb = tables_[t];
    if (!tb.host) continue;
    if (!tb.slot) tb.slot = static_cast<int*>(alloc(type_counts_[t] * 4));
    std::vector<int> slot(type_counts_[t], -1);
    const std::size_t esz = tb.dtype == kF32 ? 4 : 2, row = static_cast<std::size_t>(tb.ld) * esz;
    if (cached[t].size() > tb.cache_rows) {
      tb.cache = static_cast<float*>(alloc(std::max<std::size_t>(16, cached[t].size() * row)));
      tb.cache_rows = cached[t].size();
    }
    std::vector<std::uint8_t> rows(cached[t].size() * row);
    for (std::size_t i = 0; i < cached[t].size(); ++i) {
      const NodeId v = cached[t][i];
      if (v >= type_counts_[t]) throw std::invalid_argument("cached node id out of range: " + std::to_string(v));
      slot[v] = static_cast<int>(i);
      std::memcpy(&rows[i * row], static_cast<const std::uint8_t*>(tb.host_mem) + static_cast<std::size_t>(v) * row, row);
    }
    if (!rows.empty()) HG_CUDA(cudaMemcpyAsync(tb.cache, rows.data(), rows.size(), cudaMemcpyHostToDevice, st_));
    HG_CUDA(cudaMemcpyAsync(tb.slot, slot.data(), slot.size() * 4, cudaMemcpyHostToDevice, st_));
    HG_CUDA(cudaStreamSynchronize(st_));
  }
  drop_graphs();  // the captured steps did not look the frontier up
}

std::vector<std::pair<unsigned long long, unsigned long long>> Engine::cache_counters() {
  std::vector<unsigned long long> v(2 * ntypes_);
  HG_CUDA(cudaStreamSynchronize(st_));
  HG_CUDA(cudaMemcpy(v.data(), cache_hm_, v.size() * 8, cudaMemcpyDeviceToHost));
  std::vector<std::pair<unsigned long long, unsigned long long>> out;
  for (int t = 0; t < ntypes_; ++t) out.emplace_back(v[2 * t], v[2 * t + 1]);
  return out;
}

// ---------------------------------------------------------------------------------------------
// Named tensors (mirror oracle/ref_shim.cpp bundle names):
//   frontier{h}.t{t}, hop{h}.rel{r}.{dst_ids,indptr,src_ids,col}, H{d}.t{t},
//   mean.l{l}.r{r}.t{t}, logits, dlogits, loss, grad.w.r{r}.l{l},
//   grad.f.t{t}.ids, grad.f.t{t}.rows, post.r{r}.l{l}, post.learn.t{t},
//   post.learn_m.t{t}, post.learn_v.t{t}, post.learn_step.t{t}, sampled_edges
std::vector<std::string> Engine::tensor_names() const {
  std::vector<std::string> n;
  const int k = o_.k;
  for (int h = 0; h <= k; ++h)
    for (int t = 0; t < ntypes_; ++t)
      if (fronts_[h * ntypes_ + t].cap > 0) n.push_back("frontier" + std::to_string(h) + ".t" + std::to_string(t));
  for (const auto& b : blocks_) {
    const std::string p = "hop" + std::to_string(b.hop) + ".rel" + std::to_string(b.rel);
    for (const char* s : {".dst_ids", ".indptr", ".src_ids", ".col"}) n.push_back(p + s);
  }
  for (const auto& gr : groups_) {
    if (gr.layer < k) n.push_back("H" + std::to_string(gr.depth - 1) + ".t" + std::to_string(gr.type));
    if (!rgat())
      for (std::size_t q = 0; q < gr.blocks.size(); ++q)
        n.push_back("mean.l" + std::to_string(gr.layer) + ".r" + std::to_string(blocks_[gr.blocks[q]].rel) + ".t" +
                    std::to_string(gr.type));
  }
  for (int t = 0; t < ntypes_; ++t)
    if (tables_[t].w) n.push_back("H" + std::to_string(k) + ".t" + std::to_string(t));
  for (const char* s : {"logits", "dlogits", "loss", "sampled_edges"}) n.push_back(s);
  for (const auto& s : slots_) {
    const std::string key = "r" + std::to_string(s.rel) + ".l" + std::to_string(s.layer);
    n.push_back("grad.w." + key);
    n.push_back("post." + key);
    if (rgat()) {
      n.push_back("att." + key);
      n.push_back("grad.att." + key);
    }
  }
  for (const auto& c : cscs_)
    if (c.hop == k && (c.dh || xchg_type(c.src_t))) {
      n.push_back("grad.f.t" + std::to_string(c.src_t) + ".ids");
      n.push_back("grad.f.t" + std::to_string(c.src_t) + ".rows");
    }
  for (int t = 0; t < ntypes_; ++t)
    if (tables_[t].learnable)
      for (const char* s : {"post.learn.t", "post.learn_m.t", "post.learn_v.t", "post.learn_step.t"})
        n.push_back(s + std::to_string(t));
  return n;
}

bool Engine::read_tensor(const std::string& name, std::string& dtype, std::vector<long long>& shape,
                         std::vector<char>& data) {
  HG_CUDA(cudaStreamSynchronize(st_));
  const int k = o_.k;
  auto dev_int = [&](const int* p) {
    int v = 0;
    HG_CUDA(cudaMemcpy(&v, p, sizeof(int), cudaMemcpyDeviceToHost));
    return v;
  };
  auto u32s = [&](const std::uint32_t* p, std::size_t n) {
    std::vector<std::uint32_t> v(n);
    if (n) HG_CUDA(cudaMemcpy(v.data(), p, n * 4, cudaMemcpyDeviceToHost));
    dtype = "<u4";
    shape = {static_cast<long long>(n)};
    put(data, v);
    return true;
  };
  // rows x cols of an ld-strided fp32 matrix, widened to f64 like the oracle
  auto mat = [&](const float* p, std::size_t rows, int cols, int ld, std::size_t row_stride = 1,
                 std::size_t row_offset = 0) {
    std::vector<float> raw;
    std::vector<double> v(rows * cols);
    if (rows) {
      const std::size_t span = ((rows - 1) * row_stride + row_offset + 1) * ld;
      raw.resize(span);
      HG_CUDA(cudaMemcpy(raw.data(), p, span * 4, cudaMemcpyDeviceToHost));
      for (std::size_t i = 0; i < rows; ++i)
        for (int c = 0; c < cols; ++c) v[i * cols + c] = raw[(i * row_stride + row_offset) * ld + c];
    }
    dtype = "<f8";
    shape = {static_cast<long long>(rows), cols};
    put(data, v);
    return true;
  };
  auto n_rows_of_block = [&](const BlockBuf& b) {
    if (b.hop == 1 && b.dst_t == target_ && replica_) return dev_int(shard_count_dev_);
    return dev_int(front(b.hop - 1, b.dst_t).count);
  };
  for (int h = 0; h <= k; ++h)
    for (int t = 0; t < ntypes_; ++t)
      if (name == "frontier" + std::to_string(h) + ".t" + std::to_string(t)) {
        const Front& f = fronts_[h * ntypes_ + t];
        return u32s(f.list, f.cap > 0 ? dev_int(f.count) : 0);
      }
  for (const auto& b : blocks_) {
    const std::string p = "hop" + std::to_string(b.hop) + ".rel" + std::to_string(b.rel);
    if (name.rfind(p + ".", 0) != 0) continue;
    const int n = n_rows_of_block(b);
    std::uint32_t total = 0;
    HG_CUDA(cudaMemcpy(&total, b.indptr + n, 4, cudaMemcpyDeviceToHost));
    if (name == p + ".dst_ids")
      return u32s(block_dst(b), n);
    if (name == p + ".indptr") return u32s(b.indptr, n + 1);
    if (name == p + ".src_ids") return u32s(b.src, total);
    if (name == p + ".col") return u32s(b.col, total);
  }
  for (const auto& gr : groups_) {
    const int n = dev_int(front(gr.depth - 1, gr.type).count);
    if (gr.layer < k && name == "H" + std::to_string(gr.depth - 1) + ".t" + std::to_string(gr.type))
      return mat(gr.out, n, gr.dout, gr.ld);
    for (std::size_t q = 0; q < gr.blocks.size(); ++q) {
      const BlockBuf& b = blocks_[gr.blocks[q]];
      if (name == "mean.l" + std::to_string(gr.layer) + ".r" + std::to_string(b.rel) + ".t" + std::to_string(gr.type))
        return mat(b.mean, n_rows_of_block(b), b.din, b.ld_mean);
    }
  }
  for (int t = 0; t < ntypes_; ++t)
    if (tables_[t].w && name == "H" + std::to_string(k) + ".t" + std::to_string(t)) {
      const Front& f = front(k, t);
      const int n = dev_int(f.count);
      float* tmp = nullptr;
      HG_CUDA(cudaMalloc(&tmp, std::max<std::size_t>(16, static_cast<std::size_t>(n) * tables_[t].dim * 4)));
      if (n)
        launch_pdl(k_gather_rows, 64, 256, 0, st_, static_cast<const float*>(tables_[t].w), tables_[t].ld,
                   static_cast<const std::uint32_t*>(f.list), static_cast<const int*>(f.count), tables_[t].dim, tmp,
                   tables_[t].dense ? tables_[t].dtype : 0);
      HG_CUDA(cudaStreamSynchronize(st_));
      mat(tmp, n, tables_[t].dim, tables_[t].dim);
      cudaFree(tmp);
      return true;
    }
  const int n0 = dev_int(front(0, target_).count);
  if (name == "logits") return mat(logits_, n0, num_classes_, ldc_);
  if (name == "dlogits") return mat(dlogits_, n0, num_classes_, ldc_);
  if (name == "loss" || name == "sampled_edges") {
    Readback rb;
    HG_CUDA(cudaMemcpy(&rb, loss_, sizeof(rb), cudaMemcpyDeviceToHost));
    if (name == "loss") {
      dtype = "<f8";
      put(data, std::vector<double>{rb.loss});
    } else {
      dtype = "<u8";
      put(data, std::vector<std::uint64_t>{rb.edges});
    }
    shape = {1};
    return true;
  }
  for (const auto& s : slots_) {
    const std::string key = "r" + std::to_string(s.rel) + ".l" + std::to_string(s.layer);
    if (name == "grad.w." + key) return mat(s.g, s.din, s.dout, s.ld);
    if (name == "post." + key) return mat(s.w, s.din, s.dout, s.ld);
    if (rgat() && name == "att." + key) return mat(s.a, 1, s.dout, s.ld);
    if (rgat() && name == "grad.att." + key) return mat(s.ag, 1, s.dout, s.ld);
  }
  for (const auto& c : cscs_) {
    if (c.hop != k || !c.dh) continue;
    const std::string p = "grad.f.t" + std::to_string(c.src_t);
    const Front& f = front(k, c.src_t);
    if (name == p + ".ids") return u32s(f.list, dev_int(f.count));
    if (name == p + ".rows") return mat(c.dh, dev_int(f.count), c.din, c.ld);
  }
  for (int h = 1; h <= o_.k && h < 8; ++h)
    if (sample_trace_[h] && name == "trace.sample.h" + std::to_string(h)) {
      std::vector<unsigned long long> v(static_cast<std::size_t>(lb_.cap) * 8);
      HG_CUDA(cudaMemcpy(v.data(), sample_trace_[h], v.size() * 8, cudaMemcpyDeviceToHost));
      dtype = "<u8";
      shape = {static_cast<long long>(lb_.cap), 8};
      put(data, v);
      return true;
    }
  for (const auto& x : xchg_)  // replica groups: the merged union of the last step
    if (name == "merge.t" + std::to_string(x.t) + ".union") return u32s(x.ulist, dev_int(x.ucount));
  for (int t = 0; t < ntypes_; ++t) {
    const TypeTable& tb = tables_[t];
    if (!tb.learnable) continue;
    const std::string ts = std::to_string(t);
    if (name == "post.learn.t" + ts) return mat(tb.w, type_counts_[t], tb.dim, tb.ld);
    if (name == "post.learn_m.t" + ts) return mat(tb.m, type_counts_[t], tb.dim, tb.ld);
    if (name == "post.learn_v.t" + ts) return mat(tb.v, type_counts_[t], tb.dim, tb.ld);
    if (name == "post.learn_step.t" + ts) {
      std::int64_t s = 0;
      HG_CUDA(cudaMemcpy(&s, tb.step, 8, cudaMemcpyDeviceToHost));
      dtype = "<i8";
      shape = {1};
      put(data, std::vector<std::int64_t>{s});
      return true;
    }
  }
  return false;
}

}  // namespace hetgpu

namespace hetgpu {
namespace {
__global__ void k_put_rows(float* table, int ld, const std::uint32_t* ids, std::int64_t n, const float* rows,
                           int dim) {
  const std::int64_t total = n * dim;
  for (std::int64_t x = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t i = x / dim;
    const int c = static_cast<int>(x % dim);
    table[static_cast<std::int64_t>(ids[i]) * ld + c] = rows[i * dim + c];
  }
}
}  // namespace

void Engine::load_weights(int rel, int layer, const double* w, int din, int dout) {
  quiesce();
  for (auto& s : slots_) {
    if (s.rel != rel || s.layer != layer) continue;
    if (s.din != din || s.dout != dout)
      throw std::invalid_argument("weight/input dim mismatch for relation " + std::to_string(rel));
    std::vector<float> host(static_cast<std::size_t>(std::max(1, s.din)) * s.ld, 0.0f);
    for (int i = 0; i < din; ++i)
      for (int j = 0; j < dout; ++j) host[static_cast<std::size_t>(i) * s.ld + j] = static_cast<float>(w[i * dout + j]);
    const std::size_t bytes = host.size() * 4;
    HG_CUDA(cudaMemcpyAsync(s.w, host.data(), bytes, cudaMemcpyHostToDevice, st_));
    HG_CUDA(cudaMemsetAsync(s.m, 0, bytes, st_));
    HG_CUDA(cudaMemsetAsync(s.v, 0, bytes, st_));
    HG_CUDA(cudaStreamSynchronize(st_));
    return;
  }
  // a slot this partition does not evaluate: nothing to load
}

void Engine::load_table_rows(int type, const NodeId* ids, std::int64_t n, const double* rows, int dim) {
  if (type < 0 || type >= ntypes_ || !tables_[type].learnable)
    throw std::invalid_argument("no learnable table for node type " + std::to_string(type));
  const TypeTable& tb = tables_[type];
  if (!tb.w) return;  // not a layer-0 type of this partition
  if (dim != tb.dim) throw std::invalid_argument("learnable row width mismatch for node type " + std::to_string(type));
  if (n <= 0) return;
  for (std::int64_t i = 0; i < n; ++i)
    if (ids[i] >= type_counts_[type]) throw std::invalid_argument("node id out of range: " + std::to_string(ids[i]));
  quiesce();
  std::vector<float> host(static_cast<std::size_t>(n) * dim);
  for (std::size_t i = 0; i < host.size(); ++i) host[i] = static_cast<float>(rows[i]);
  void* d_ids = nullptr;
  void* d_rows = nullptr;
  HG_CUDA(cudaMallocAsync(&d_ids, static_cast<std::size_t>(n) * 4, st_));
  HG_CUDA(cudaMallocAsync(&d_rows, host.size() * 4, st_));
  HG_CUDA(cudaMemcpyAsync(d_ids, ids, static_cast<std::size_t>(n) * 4, cudaMemcpyHostToDevice, st_));
  HG_CUDA(cudaMemcpyAsync(d_rows, host.data(), host.size() * 4, cudaMemcpyHostToDevice, st_));
  const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(static_cast<std::uint64_t>(n) * dim, 256),
                                                                      8ull * num_sms()));
  k_put_rows<<<std::max(1u, grid), 256, 0, st_>>>(tb.w, tb.ld, static_cast<const std::uint32_t*>(d_ids), n,
                                                  static_cast<const float*>(d_rows), dim);
  HG_CUDA(cudaGetLastError());
  HG_CUDA(cudaFreeAsync(d_ids, st_));
  HG_CUDA(cudaFreeAsync(d_rows, st_));
  HG_CUDA(cudaStreamSynchronize(st_));
}

}  // namespace hetgpu

namespace hetgpu {

namespace {
// round-to-nearest-even conversions on the host (the CUDA headers' __host__ paths)
std::uint16_t f32_to_f16(float x) {
  const __half_raw r = __float2half_rn(x);
  return r.x;
}
std::uint16_t f32_to_bf16(float x) {
  const __nv_bfloat16_raw r = __float2bfloat16_rn(x);
  return r.x;
}
}  // namespace

// One dense feature table, converted to its storage type in chunks (no full-size
// staging copy): f32 / f16 / bf16 rows of ld elements (ld = dim rounded up to 4, zero
// padding), in HBM or, with feat_host, in pinned host memory mapped into the device's
// address space (the gather reads missing rows over PCIe; set_cache() adds an HBM copy
// of the hot rows).
void Engine::upload_dense(const NodeTypeInfo& nt, TypeTable& tb) {
  tb.dense = true;
  tb.dtype = o_.feat_dtype;
  if (tb.dtype < 0 || tb.dtype > 2) throw std::invalid_argument("feature dtype must be 0 (f32), 1 (f16) or 2 (bf16)");
  if (tb.dtype != kF32) tb.ld = (std::max(1, nt.dim) + 7) & ~7;  // 16-byte rows of halves (8-wide loads)
  const std::size_t rows = nt.count, esz = tb.dtype == kF32 ? 4 : 2;
  const std::size_t bytes = std::max<std::size_t>(16, rows * tb.ld * esz);
  std::uint8_t* dst = nullptr;
  if (o_.feat_host) {
    tb.host = true;
    HG_CUDA(cudaHostAlloc(&tb.host_mem, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    void* dev = nullptr;
    HG_CUDA(cudaHostGetDevicePointer(&dev, tb.host_mem, 0));
    tb.w = static_cast<float*>(dev);
    dst = static_cast<std::uint8_t*>(tb.host_mem);
  } else {
    tb.w = static_cast<float*>(alloc(bytes));
  }
  const std::size_t chunk_rows = std::max<std::size_t>(1, (64u << 20) / (tb.ld * esz));
  std::vector<std::uint8_t> stage(std::min(rows, chunk_rows) * tb.ld * esz);
  for (std::size_t r0 = 0; r0 < rows; r0 += chunk_rows) {
    const std::size_t n = std::min(chunk_rows, rows - r0);
    std::fill(stage.begin(), stage.end(), 0);
    for (std::size_t i = 0; i < n; ++i) {
      const float* src = &nt.dense[(r0 + i) * nt.dim];
      if (tb.dtype == kF32) {
        std::memcpy(&stage[i * tb.ld * 4], src, sizeof(float) * nt.dim);
      } else {
        auto* o = reinterpret_cast<std::uint16_t*>(&stage[i * tb.ld * 2]);
        for (int c = 0; c < nt.dim; ++c) o[c] = tb.dtype == kF16 ? f32_to_f16(src[c]) : f32_to_bf16(src[c]);
      }
    }
    const std::size_t off = r0 * tb.ld * esz, len = n * tb.ld * esz;
    if (dst) {
      std::memcpy(dst + off, stage.data(), len);
    } else {
      HG_CUDA(cudaMemcpyAsync(reinterpret_cast<std::uint8_t*>(tb.w) + off, stage.data(), len, cudaMemcpyHostToDevice, st_));
      HG_CUDA(cudaStreamSynchronize(st_));  // the staging buffer is refilled next
    }
  }
}

}  // namespace hetgpu
