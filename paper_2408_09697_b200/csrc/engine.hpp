// Device engine for the mini-batch hot path of one meta-partition (one GPU).
//
// It replaces, for the relations and node types this partition owns, the
// reference's per-batch pipeline run_raf_batch (raf.cpp:344-530):
//   sample_khop_restricted (sampling.cpp:41-103)  -> sample_count/sample_draw + bitmap frontier
//   layer-0 gather + mean_aggregate + matmul + agg_all (hgnn.cpp:215-279, raf.cpp:167-248)
//                                                 -> aggregate_project (fused, gather by id)
//   AGG_all across partitions (raf.cpp:427-446)   -> ncclAllReduce of the [B x C] partial logits
//   cross_entropy (hgnn.cpp:281-307)              -> cross_entropy
//   backward (hgnn.cpp:309-362, raf.cpp:250-304) -> weight_grad / mean_grad / csc gather
//   adam_update_model / adam_update_rows          -> adam_dense / adam_rows
// Every live size stays on the device; a step is one stream of launches.
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "host.hpp"
#include "kernels.cuh"
#include "rgat.cuh"

#ifdef HG_WITH_NCCL
#include <nccl.h>
#endif

namespace hetgpu {

struct EngineOptions {
  int k = 2;
  std::vector<int> fanouts{25, 20};
  int hidden = 64;
  int batch_cap = 1024;
  int p = 1;      // meta-partition count
  int rank = 0;   // which partition this engine evaluates
  std::uint64_t model_seed = 0;  // init_model seed
  std::uint64_t learn_seed = 0;  // init_learnable seed
  int device = 0;
  int elem_bytes = 4;  // byte accounting of partial messages (AccountingModel)
  // storage of the dense layer-0 feature tables: 0 f32 (parity), 1 f16, 2 bf16 (C4's
  // fp16 paper features); feat_host = 1 keeps them in pinned host memory (read over
  // PCIe, zero-copy) with an HBM cache of the rows set_cache() installs
  int feat_dtype = 0;
  int feat_host = 0;
  // layer type: 0 RGCN (the reference's, hgnn.cpp:173-362), 1 RGAT (rgat.cuh: relational
  // attention with `heads` heads below the top layer, one head at the top)
  int model = 0;
  int heads = 4;
  // non-empty: the work-aware plan (work_aware_partition, one value per sub-metatree)
  // instead of the reference's meta_partition; the numbers are the flat pass's either way
  std::vector<double> sub_work;
  // sampler-only engines (sample_khop / sample_khop_restricted, sampling.cpp:94-103):
  // explicit per-hop relation sets replace the metatree's; no model state is built
  bool sample_only = false;
  bool all_relations = false;                  // sample_khop: every relation at every hop
  std::vector<std::vector<int>> hop_relations; // sample_khop_restricted: allowed set per hop
};

// Host-visible outputs of one step (one small D2H copy).
struct StepReport {
  double loss = 0.0;
  std::uint64_t sampled_edges = 0;   // Block::src_ids entries, all hops (this partition)
  std::uint32_t err = 0;
  std::vector<int> active_rows;      // per rank: batch rows with >= 1 sampled top edge
  // ExecutionReport bookkeeping (raf.hpp:66-77), see Engine::accounting
  std::uint64_t sync_bytes = 0;      // this rank's replica group: ring all-reduce model (raf.cpp:496-510)
  bool sync_leader = true;           // sum sync_bytes over leaders = the reference's run-wide number
  std::vector<std::uint64_t> boundary_counts;  // per worker (raf.cpp:306-340)
  std::uint64_t boundary_cut_edges = 0;        // raf.cpp:521-528
  bool message_bound_ok = true;      // check_comm_bounds (raf.cpp:662-676)
  bool target_only_ok = true;        // only target-type rows cross workers (raf.cpp:511-514)
};

struct DeviceBuffer {
  void* ptr = nullptr;
  std::size_t bytes = 0;
};

class Engine {
 public:
  Engine(const Graph& g, const EngineOptions& o);
  // streaming loader (loader.cu): CSR and dense tables go from an HGC1 file straight into
  // HBM (container.cpp:92-154 semantics, no host graph)
  Engine(const std::string& container_path, const EngineOptions& o);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

#ifdef HG_WITH_NCCL
  // comm: all partitions (AGG_all); rcomm: this partition's replica group (or null)
  void attach_comm(ncclComm_t comm, ncclComm_t rcomm) {
    comm_ = comm;
    rcomm_ = rcomm;
    drop_graphs();
  }
#endif
  // ---- replica groups (p > #sub-metatrees, metapartition.cpp:206-236) ----------------
  // partitions owning the same sub-metatrees split the batch rows (raf.cpp:390-391);
  // their weight gradients are all-reduced (NCCL) and their learnable-row gradients
  // merged by a kernel that reads the peers' gradient rows over NVLink (IPC-mapped).
  const std::vector<int>& replica_group() const { return replica_group_; }
  int replica_color() const { return replica_group_.size() > 1 ? replica_group_.front() : -1; }
  int replica_pos() const { return replica_pos_; }
  std::vector<char> replica_handle();  // CUDA IPC handle of the exchange arena (empty: none)
  void attach_replicas(const std::vector<std::vector<char>>& handles_by_rank);

  // Full training step: sample, forward, AGG_all, loss, backward, Adam.
  // `batch` is host memory (copied to the device inside the call). If the same
  // (batch, rng_seed) was handed to prefetch() before, its sampled blocks are used.
  StepReport step(const NodeId* batch, int n, std::uint64_t rng_seed, int designated, bool train = true);
  // Sampling is a pure function of (graph, batch, rng_seed): prefetch() samples a
  // future batch into the other of two sample slots on the sampling stream, so it
  // runs while the current step trains (at most two batches in flight).
  void prefetch(const NodeId* batch, int n, std::uint64_t rng_seed);
  // seed ids in range and (labels) every seed's label in [0, C): the reference's
  // std::invalid_argument cases (sampling.cpp:44-47, hgnn.cpp:289-291), raised
  // on the host before anything is enqueued
  void validate_batch(const NodeId* batch, int n, bool labels = true) const;
  // Benchmark inner loop, inputs resident in HBM: sample a batch into the next
  // slot (d_ss: its sampling scalars), then train the oldest sampled slot.
  void prefetch_device(const std::uint32_t* d_ids, int n, const StepScalars* d_ss);
  void train_device(const StepScalars* d_ts, bool train);
  StepScalars next_scalars(std::uint64_t rng_seed, int n, int designated, bool train);
  cudaStream_t sample_stream() const { return st_s_; }
  void quiesce();  // finish everything in flight, drop prefetched batches
  void drop_pending() { pending_slots_.clear(); }  // bench phase timing: sampled slots never trained
  void set_graphs(bool on) { use_graphs_ = on; }
  void set_side_stream(bool on) {
    if (on != use_side_) {
      use_side_ = on;
      drop_graphs();
    }
  }
  void set_umma(bool on) {
    if (on != use_umma_) {
      use_umma_ = on;
      drop_graphs();
    }
  }
  // keep the learnable-row gradients in memory (grad.f.* tensors); the bench
  // turns this off so the sparse Adam update consumes them in registers
  void set_retain_grads(bool on) {
    if (on != retain_grads_) {
      retain_grads_ = on;
      drop_graphs();
    }
  }
  // train steps compute gradients but leave the model and tables untouched (the
  // caller owns the optimizer state: run_raf_batch with a caller's HGNNModel,
  // raf.hpp:79-82, followed by the caller's own adam_update_* calls)
  void set_apply_adam(bool on) {
    if (on != apply_adam_) {
      if (!on && replica_group_.size() > 1) throw std::invalid_argument("gradient-only steps need p = 1 or no replicas");
      apply_adam_ = on;
      drop_graphs();
    }
  }
  // caller-owned parameters: one weight slot (f64 [din x dout] row-major; its Adam
  // moments are reset) and rows of a learnable table (f64 [n x dim]; with
  // apply_adam off the engine's moments are never read)
  void load_weights(int rel, int layer, const double* w, int din, int dout);
  void load_table_rows(int type, const NodeId* ids, std::int64_t n, const double* rows, int dim);
  StepReport finish_step();  // waits for the last trained step and reads its report
  // payload element width of the accounting model (AccountingModel::elem_bytes, raf.hpp:15-19)
  void set_trace_sampler(bool on) {
    trace_sampler_ = on;
    drop_graphs();
  }
  void set_shard_merge(bool on) {
    if (on != shard_merge_) {
      shard_merge_ = on;
      drop_graphs();
    }
  }
  void set_elem_bytes(int b) {
    if (b != 2 && b != 4 && b != 8) throw std::invalid_argument("elem_bytes must be 2, 4 or 8");
    elem_bytes_ = b;
  }
  // Sampling only (parity of the sampler; presample_hotness).
  void sample_only(const NodeId* batch, int n, std::uint64_t rng_seed);

  // Read any named tensor (see engine.cu: tensor names mirror the oracle's).
  // Returns false if the name is unknown.
  bool read_tensor(const std::string& name, std::string& dtype, std::vector<long long>& shape,
                   std::vector<char>& data);
  std::vector<std::string> tensor_names() const;

  // cache: hotness presample over `epochs` id-ordered passes (cache.cpp:39-63)
  std::vector<std::vector<std::uint64_t>> presample_hotness(int epochs, std::uint64_t seed, int batch_size);
  // mark the cached ids per type (sorted lists from fill_and_serve); lookups
  // then run on every step for the layer-0 frontier (harness.cpp:425-437)
  void set_cache(const std::vector<std::vector<NodeId>>& cached);
  std::vector<std::pair<unsigned long long, unsigned long long>> cache_counters();

  // per-kernel-class device time accumulated with events (profiling on)
  void set_profiling(bool on) { profiling_ = on; }
  std::map<std::string, double> kernel_ms() const { return kernel_ms_; }
  std::map<std::string, double> kernel_bytes() const { return kernel_bytes_; }
  void reset_profile() {
    kernel_ms_.clear();
    kernel_bytes_.clear();
    kernel_launches_.clear();
    if (alg_bytes_) cudaMemsetAsync(alg_bytes_, 0, sizeof(double) * 5, st_);
  }
  // kernel launches of one step, counted from a captured (not executed) step
  int count_launches(int n, bool train);
  // cumulative algorithmic bytes since reset_profile (profiling on):
  // [0] sample, [1] aggregate, [2] aggregate_top, [3] csc_gather
  std::vector<double> algorithmic_bytes();
  std::map<std::string, int> kernel_launches() const { return kernel_launches_; }
  int launches_per_step() const { return launches_per_step_; }

  cudaStream_t stream() const { return st_; }
  std::uint32_t* device_batch() { return d_batch_; }
  std::uint64_t param_count() const;
  std::uint64_t device_bytes() const { return total_bytes_; }

  // static description (for CommStats / tests)
  const Tree& local_tree() const { return tree_; }
  const std::vector<std::vector<int>>& hop_rels() const { return hop_rels_; }
  int model_step() const { return static_cast<int>(model_step_); }
  int batch_cap() const { return o_.batch_cap; }
  // rows of the last sample's layer-0 (hop k) frontier over the learnable types
  std::uint64_t learnable_leaf_rows() {
    HG_CUDA(cudaStreamSynchronize(st_));
    std::uint64_t n = 0;
    for (int t = 0; t < ntypes_; ++t) {
      if (!learnable_type_[t] || !front(o_.k, t).count) continue;
      int v = 0;
      HG_CUDA(cudaMemcpy(&v, front(o_.k, t).count, sizeof(int), cudaMemcpyDeviceToHost));
      n += static_cast<std::uint64_t>(v);
    }
    return n;
  }
  // sampled edges of the last sample_only / step (all hops, this partition)
  std::uint64_t sampled_edges() {
    HG_CUDA(cudaStreamSynchronize(st_));
    std::uint64_t v = 0;
    HG_CUDA(cudaMemcpy(&v, edges_dev_, sizeof(v), cudaMemcpyDeviceToHost));
    return v;
  }

 private:
  struct BlockBuf {
    int rel = -1, hop = 0, src_t = -1, dst_t = -1;
    int rows_cap = 0, edge_cap = 0, edge_base = 0;
    std::uint32_t *indptr = nullptr, *src = nullptr, *erow = nullptr, *col = nullptr;  // bound sample slot
    std::uint32_t *s_indptr[2] = {}, *s_src[2] = {}, *s_erow[2] = {}, *s_col[2] = {};
    float* mean = nullptr;   // tape: rows_cap x ld_mean (only for blocks feeding a layer)
    float* dmean = nullptr;  // rows_cap x ld_mean (only if the source needs a gradient)
    int din = 0, ld_mean = 0;
    bool need_src_grad = false;
    // RGAT (rgat.cuh): projected source rows, scores, softmax state and gradients
    float *lse = nullptr, *alpha = nullptr, *dt = nullptr;
    float *dz = nullptr, *tsum = nullptr;
    int ld_z = 0, heads = 1, src_cap = 0;
    // RGAT layer 1 (aggregate first, rgat.cuh): per-head aggregates of the table rows and
    // the block-diagonal weight; din_p = round_up4(din)
    float *agg = nullptr, *dagg = nullptr, *te = nullptr, *qv = nullptr, *wbd = nullptr, *wbdt = nullptr;
    float *dwfull = nullptr, *dq_part = nullptr, *dqv = nullptr;
    int din_p = 0;
  };
  struct Front {
    std::uint32_t* list = nullptr;
    int* count = nullptr;  // device
    int cap = 0;
  };
  struct Slot {
    int rel = -1, layer = 0, din = 0, dout = 0, ld = 0;
    float *w = nullptr, *m = nullptr, *v = nullptr, *g = nullptr;
    // RGAT: attention vector [dout] (+ Adam state, gradient) and W^T [dout x ld_wt]
    float *a = nullptr, *am = nullptr, *av = nullptr, *ag = nullptr, *wt = nullptr;
    int ld_wt = 0;
  };
  struct Group {  // one output type of one layer
    int layer = 0, depth = 0, type = -1, dout = 0, ld = 0, rows_cap = 0;
    std::vector<int> blocks;  // indices into blocks_
    std::vector<int> slots;   // matching slot indices
    float* out = nullptr;     // H[depth-1][type] (logits for layer k)
    float* dout_buf = nullptr;  // dH for it
  };
  struct CscBuf {
    int hop = 0, src_t = -1, src_cap = 0, din = 0, ld = 0;
    std::vector<int> blocks;
    std::uint32_t *offs = nullptr, *cursor = nullptr, *entries = nullptr;  // bound sample slot
    std::uint32_t *s_offs[2] = {}, *s_cursor[2] = {}, *s_entries[2] = {};
    std::uint32_t *tmp = nullptr, *s_tmp[2] = {};  // scratch of the long-segment sort
    float* dh = nullptr;  // gradient of H[hop][src_t] (or learnable rows)
  };
  struct TypeTable {
    int dim = 0, ld = 0;
    bool learnable = false, dense = false;
    int dtype = 0;               // dense tables: FeatDtype of the rows w points at
    bool host = false;           // dense rows in pinned host memory (w = its device mapping)
    void* host_mem = nullptr;    // the pinned allocation (host pointer)
    int* slot = nullptr;         // host tables: per node its HBM cache row or -1
    float* cache = nullptr;      // HBM cache rows (dtype elements)
    std::uint64_t cache_rows = 0;
    float *w = nullptr, *m = nullptr, *v = nullptr;
    std::int64_t* step = nullptr;  // device
    std::int64_t host_step = 0;
  };

  void* alloc(std::size_t bytes);
  void release() noexcept;  // the destructor's work (also for a constructor that throws)
  void init_streams();
  void init_graph(const Graph& g);  // plan + upload
  void stream_csr(ContainerLayout& lay, const std::string& path);
  void stream_dense(const NodeTypeInfo& nt, int t, TypeTable& tb);
  const ContainerLayout* lay_ = nullptr;  // set while a container-streamed engine uploads
  std::string lay_path_;
  std::vector<std::uint64_t*> pre_ptr_;  // streamed CSR per relation (device)
  std::vector<std::uint32_t*> pre_src_;
  void build_plan(const Graph& g);
  void upload(const Graph& g);
  void upload_dense(const NodeTypeInfo& nt, TypeTable& tb);
  void run_sampling(cudaStream_t ss);  // everything of one sample slot, on stream ss
  void run_forward();
  void run_agg_all();  // AGG_all of the partial logits (p > 1)
  void run_loss(bool train);
  void run_backward();
  void run_update();
  // RGAT layer type (rgat.cu)
  bool rgat() const { return o_.model == 1; }
  int heads_of(int layer) const { return layer == o_.k ? 1 : o_.heads; }
  void rgat_plan(const Graph& g);
  void rgat_alloc();
  void run_forward_rgat();
  void run_backward_rgat();
  void run_update_rgat();
  const float* rgat_src(const BlockBuf& b, int& ld);  // source-frontier rows of an inner block's layer input
  AttLeafJob rgat_leaf_job(const BlockBuf& b);  // a block's aggregate-first attention job
  float* rgat_wpart_ = nullptr;  // weight-gradient split-K partials
  std::size_t rgat_wpart_floats_ = 0;
  void timed(const char* name, double bytes, const std::function<void()>& f);
  Front& front(int h, int t) { return fronts_[h * ntypes_ + t]; }
  // destination rows of a block: frontier[hop-1][dst type]; hop-1 blocks into the
  // target read the replica's shard of the batch when the partition is a replica
  const int* block_rows(const BlockBuf& b) {
    if (b.hop == 1 && b.dst_t == target_ && replica_) return shard_count_dev_;
    return front(b.hop - 1, b.dst_t).count;
  }
  const std::uint32_t* block_dst(const BlockBuf& b) {
    if (b.hop == 1 && b.dst_t == target_ && replica_) return shard_list_;
    return front(b.hop - 1, b.dst_t).list;
  }
  int out_dim(int layer) const { return layer == o_.k ? num_classes_ : o_.hidden; }

  EngineOptions o_;
  Tree tree_;
  std::vector<std::vector<int>> hop_rels_;
  int ntypes_ = 0, target_ = 0, num_classes_ = 0;
  std::vector<std::uint64_t> type_counts_;
  std::vector<bool> learnable_type_;  // Storage::Learnable per node type
  std::vector<int> rel_src_, rel_dst_;
  bool replica_ = false;
  int shard_index_ = 0, shard_count_ = 1;

  cudaStream_t st_ = nullptr;
  // side stream for work off the critical path (captured as parallel graph
  // branches): the hop-k frontier + transposed views overlap the forward pass,
  // weight gradients overlap the mean gradients and backward gathers
  cudaStream_t st2_ = nullptr;
  std::vector<cudaEvent_t> fork_ev_;
  int fork_used_ = 0;
  bool side_open_ = false;  // the side stream has work forked since the last join
  bool presampling_ = false;  // run_sampling for presample_hotness: no transposed views, no cache lookups
  std::vector<unsigned long long*> hot_counts_;  // presample_hotness histograms, u64 (allocated once)
  LbScratch lb2_;  // look-back scratch of the side stream
  bool use_side_ = true;
  cudaStream_t side() const { return (profiling_ || !use_side_) ? st_ : st2_; }
  void fork();  // side stream waits for everything queued on st_ so far
  void join();  // st_ waits for everything queued on the side stream so far
  std::vector<void*> allocs_;
  std::size_t total_bytes_ = 0;

  // graph on device
  std::vector<std::uint64_t*> csr_ptr_;
  std::vector<std::uint32_t*> csr_src_;
  std::vector<std::uint64_t> maxdeg_;
  std::vector<std::vector<float>> rng_frac_;  // [hop-1][rel]: share of destinations drawn with the RNG
  std::vector<TypeTable> tables_;
  std::int32_t* labels_ = nullptr;
  std::vector<NodeId> bad_labels_;  // target ids with labels outside [0, C), sorted

  // ---- two sample slots: everything sampling writes exists twice; bind_slot(s)
  // points the working pointers below at slot s (host-side rebinding: each
  // captured graph is for one slot)
  void bind_slot(int s);
  int bound_ = 0;
  std::vector<Front> fronts_slot_[2];
  std::uint32_t *bits_slot_[2] = {}, *wscan_slot_[2] = {};
  std::uint32_t* shard_list_slot_[2] = {};
  int* shard_count_slot_[2] = {};
  StepScalars *d_sc_slot_[2] = {}, *h_sc_slot_[2] = {};
  std::uint32_t *d_batch_slot_[2] = {}, *h_batch_slot_[2] = {};
  float* mult_slot_[2] = {};
  struct Readback;
  Readback *rb_slot_[2] = {}, *h_rb_slot_[2] = {};
  LbScratch lb_slot_[2];
  std::uint32_t* slow_slot_[2] = {};
  int* n_slow_slot_[2] = {};
  std::uint64_t* mt_scratch_slot_[2] = {};
  // slots sampled and not trained yet (FIFO), with the host batch they hold
  struct Pending {
    int slot;
    std::uint64_t rng_seed;
    std::vector<NodeId> batch;
  };
  std::vector<Pending> pending_slots_;
  int next_slot_ = 0, last_trained_ = 0;
  cudaStream_t st_s_ = nullptr;  // sampling stream
  cudaEvent_t ev_sampled_[2] = {}, ev_trained_[2] = {};
  cudaEvent_t ev_staged_[2] = {};  // the slot's pinned batch staging copy has been consumed
  StepScalars* d_tsc_ = nullptr;  // scalars of the step being trained
  StepScalars* h_tsc_ = nullptr;  // pinned
  cudaStream_t sstream() const { return profiling_ ? st_ : st_s_; }
  void enqueue_sample(int s);   // graph or eager sampling of slot s on sstream()
  void enqueue_train(int s, bool train);
  void sample_body(cudaStream_t ss);
  void train_body(bool train);

  // frontier machinery
  std::vector<Front> fronts_;       // [(k+1) x ntypes], bound slot
  std::vector<int> word_base_;      // per type, offset in words
  std::uint32_t *bits_ = nullptr, *wscan_ = nullptr, *cached_bits_ = nullptr;
  int total_words_ = 0;
  int* words_dev_ = nullptr;        // per hop, per frontier slot: word counts (device)
  std::vector<std::vector<int>> hop_slot_types_;  // per hop: types in slot order
  std::uint32_t* shard_list_ = nullptr;
  int* shard_count_dev_ = nullptr;

  std::vector<BlockBuf> blocks_;
  std::vector<std::vector<int>> hop_blocks_;  // per hop: block indices
  std::vector<Group> groups_;                 // ordered by layer
  std::vector<Slot> slots_;
  std::map<SlotId, int> slot_of_;
  std::vector<CscBuf> cscs_;

  // per-step state
  StepScalars* d_sc_ = nullptr;
  StepScalars* h_sc_ = nullptr;      // pinned
  std::uint32_t* d_batch_ = nullptr;
  std::uint32_t* h_batch_ = nullptr;  // pinned
  float* mult_ = nullptr;
  float* logits_ = nullptr;   // [batch_cap + 1 rows x ldC] (+1: partition counters)
  float* dlogits_ = nullptr;
  int ldc_ = 0;
  double* row_loss_ = nullptr;
  double* loss_ = nullptr;
  std::uint32_t* err_ = nullptr;
  std::int64_t* model_step_dev_ = nullptr;
  std::int64_t model_step_ = 0;
  struct Readback {
    double loss;
    std::uint32_t err;
    std::uint32_t pad;
    std::uint64_t edges;
    std::uint64_t feat_sync;  // learnable-row part of sync_bytes (replica groups)
  };
  // batch-invariant RAF bookkeeping of the whole plan (host, once)
  RafAccounting acct_;
  int elem_bytes_ = 4;
  bool shard_merge_ = false;  // replica merge: each replica updates only its id shard
  bool trace_sampler_ = false;  // diagnostics: per-tile sampler timestamps
  unsigned long long* sample_trace_[8] = {};
  int n_rel_ = 0;
  std::uint64_t model_sync_bytes() const;
  Readback* h_rb_ = nullptr;  // pinned, bound slot
  std::uint64_t* edges_dev_ = nullptr;
  std::uint64_t* feat_sync_dev_ = nullptr;
  unsigned* loss_done_ = nullptr;  // CTA completion counter of the loss kernel
  int last_designated_ = 0;
  unsigned long long* cache_hm_ = nullptr;  // [ntypes x 2]

  // scratch
  LbScratch lb_;
  std::uint32_t* slow_ = nullptr;
  int* n_slow_ = nullptr;
  std::uint64_t* mt_scratch_ = nullptr;
  float* wt_scratch_ = nullptr;
  float* wgrad_partial_ = nullptr;

  bool cache_on_ = false;
  std::vector<bool> cache_types_;
  std::vector<std::uint8_t*> union_map_;  // p > 1: per cached type, the global frontier's 0/1 map
  bool profiling_ = false;
  struct PendingEvent {
    std::string name;
    cudaEvent_t a, b;
  };
  std::vector<PendingEvent> pending_;
  std::vector<cudaEvent_t> ev_pool_;
  std::size_t ev_used_ = 0;
  double* alg_bytes_ = nullptr;
  void resolve_profile();
  void step_body(bool train);  // sample_body + train_body on st_ (launch counting)
  bool use_graphs_ = true;
  bool use_umma_ = true;
  bool counting_ = false;  // count_launches capture in progress (no collectives)  // tcgen05 contractions (0: SIMT fp32 tiles, kept for A/B checks)
  bool retain_grads_ = true;
  bool apply_adam_ = true;
  struct CscRegion {
    std::uint32_t *offs, *cursor;
    std::size_t words;
  };
  std::vector<CscRegion> csc_region_;  // bound slot
  std::vector<CscRegion> csc_region_slot_[2];
  CscHop csc_hop(int h);
  void drop_graphs() {
    for (int s = 0; s < 2; ++s) {
      if (exec_train_[s]) cudaGraphExecDestroy(exec_train_[s]);
      if (exec_eval_[s]) cudaGraphExecDestroy(exec_eval_[s]);
      if (exec_sample_[s]) cudaGraphExecDestroy(exec_sample_[s]);
      exec_train_[s] = exec_eval_[s] = exec_sample_[s] = nullptr;
    }
  }
  cudaGraphExec_t exec_train_[2] = {}, exec_eval_[2] = {}, exec_sample_[2] = {};
  std::map<std::string, double> kernel_ms_, kernel_bytes_;
  std::map<std::string, int> kernel_launches_;
  int launches_per_step_ = 0;
#ifdef HG_WITH_NCCL
  ncclComm_t comm_ = nullptr;
  ncclComm_t rcomm_ = nullptr;
#endif
  std::vector<int> replica_group_;  // partition ranks, ordered by replica index
  int replica_pos_ = 0;
  // learnable leaf types exchanged between replicas: local views into the IPC
  // arena (frontier ids + count, gradient rows) and the merge scratch
  struct Xchg {
    int t = -1, cap = 0, ld = 0, din = 0;
    std::size_t off_count[2] = {}, off_ids[2] = {}, off_dh = 0;  // offsets in every replica's arena (per slot)
    std::uint32_t* ulist = nullptr;
    int* ucount = nullptr;
    int ucap = 0;
    int* slot = nullptr;  // [n_rep x ucap]: row of union entry u in replica r (-1: absent)
    float* ug = nullptr;  // merged gradient rows [ucap x ld]
    int* utotal = nullptr;  // size of the whole union (every shard)
    std::vector<float*> peer_w;  // per group member: its copy of this table (self: ours)
  };
  std::vector<Xchg> xchg_;
  std::uint8_t* arena_ = nullptr;
  std::size_t arena_bytes_ = 0;
  std::vector<const std::uint8_t*> peer_arena_;  // per group member (self: arena_)
  std::vector<void*> ipc_opened_;
  unsigned* barrier_epoch_ = nullptr;  // steps this replica has passed the barrier (device)
  std::size_t off_flags_ = 0;          // barrier flags in the exchange arena
  std::size_t off_slot_ = 0;           // this replica's bound sample slot (checked by the peers)
  bool xchg_type(int t) const {
    for (const auto& x : xchg_)
      if (x.t == t) return true;
    return false;
  }
  void run_replica_merge();
  void replica_prepare();
  bool fused_model_adam() const { return replica_group_.size() <= 1 && apply_adam_; }
  std::vector<ReplicaMerge> merges_;  // built by replica_prepare for run_replica_merge
  bool training_ = false;
};

}  // namespace hetgpu
