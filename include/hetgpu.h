/*
 * hetgpu — C-ABI of the B200-native mini-batch hot path of Heta (arXiv 2408.09697).
 *
 * Drop-in boundary for the reference simulator "hetsim" (/root/reference/proj).
 * The reference has no FFI layer of its own: callers link its C++ library
 * directly. Each entry point below names the reference interface it replaces
 * (file:line under /root/reference/proj). Plain pointers and sizes only; no
 * C++ or torch types cross the ABI. Every function returns 0 / a non-NULL
 * handle on success; on failure it returns -1 / NULL and hg_last_error()
 * holds the message (the reference's exception text where one exists).
 * Errors are classified by hg_last_error_kind(): 1 = std::invalid_argument,
 * 2 = std::runtime_error (mirrors the reference's exception types).
 */
#ifndef HETGPU_H
#define HETGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hg_graph hg_graph;
typedef struct hg_engine hg_engine;
typedef struct hg_bundle hg_bundle;

const char* hg_last_error(void);
int hg_last_error_kind(void);
const char* hg_version(void);

/* ---- bundles: named arrays returned by the query functions ------------------ */
int hg_bundle_size(const hg_bundle* b);
const char* hg_bundle_name(const hg_bundle* b, int i);
const char* hg_bundle_dtype(const hg_bundle* b, int i); /* numpy dtype string */
int hg_bundle_ndim(const hg_bundle* b, int i);
long long hg_bundle_dim(const hg_bundle* b, int i, int d);
long long hg_bundle_nbytes(const hg_bundle* b, int i);
const void* hg_bundle_data(const hg_bundle* b, int i);
void hg_bundle_free(hg_bundle* b);

/* ---- graphs (host) ---------------------------------------------------------------- */
typedef struct {
  const char* name;
  uint64_t count;
  int dim;
  int storage; /* 1 dense, 2 learnable */
} hg_spec_node_type;

typedef struct {
  const char* src;
  const char* edge;
  const char* dst;
  uint64_t edges;
  int powerlaw; /* 0 uniform, 1 powerlaw */
  double alpha;
} hg_spec_relation;

typedef struct {
  const char* target;
  int num_classes;
  double label_noise;
  int n_types;
  const hg_spec_node_type* types;
  int n_rels;
  const hg_spec_relation* rels;
  int add_reverse;
  int n_self_paired;
  const char* const* self_paired;
} hg_spec;

/* gen_synthetic (src/harness.cpp:74-186), bit-exact with the reference. */
hg_graph* hg_graph_generate(const hg_spec* spec, uint64_t seed);

/* A HetGraph given directly in CSR form (dst-major per relation, hetgraph.hpp:41-74).
 * indptr: concatenation of per-relation indptr arrays (n_dst(r)+1 each);
 * src: concatenation of per-relation source arrays; kinds: 0 absent, 1 dense,
 * 2 learnable; dense: concatenated row-major f32 tables of the dense types. */
hg_graph* hg_graph_from_csr(int n_types, const uint64_t* counts, int n_rels, const int* rel_src,
                            const int* rel_dst, const int* rel_reverse, const uint64_t* indptr,
                            const uint32_t* src, const int* kinds, const int* dims, const float* dense,
                            int target, int num_classes, const int32_t* labels);

/* build_hetgraph (src/hetgraph.cpp:126-156) from (src,dst) pairs per relation. */
hg_graph* hg_graph_from_pairs(int n_types, const uint64_t* counts, int n_rels, const int* rel_src,
                              const int* rel_dst, const uint64_t* pair_counts, const uint32_t* pair_src,
                              const uint32_t* pair_dst, int target, int num_classes);

/* HGC1 container (save_container / load_container, src/container.cpp:47-154): the
 * writer produces the reference's exact bytes; failures are runtime_error. */
hg_graph* hg_graph_load(const char* path);
int hg_graph_save(const hg_graph* g, const char* path);

void hg_graph_free(hg_graph* g);
/* node_counts, labels, rel_src/rel_dst/rel_reverse, rel{r}.indptr, rel{r}.src, feat.t{t}, kinds, dims */
hg_bundle* hg_graph_export(const hg_graph* g);
/* schema only (no edges or features): node_counts, kinds, dims, target, num_classes, rel_src, rel_dst */
hg_bundle* hg_graph_schema(const hg_graph* g);

/* ---- planning (host; meta-partitioner stays on the CPU) ------------------------------- */
/* meta_partition (src/metapartition.cpp:283-295) + cacheable_types (src/cache.cpp:143-177)
 * + hop_relation_sets (src/hgnn.cpp:28-37). Names: tree.{type,depth,parent,rel},
 * subs.{child_pos,weight}, part{i}.{sub_ids,relations,node_types,cacheable,replica,weight},
 * hop_rels{h}. */
hg_bundle* hg_meta_partition(const hg_graph* g, int k, int p);
/* Work-aware meta-partitioning (NOT the reference's policy, which stays the parity mode):
 * the same metatree and sub-metatrees, with the p workers split into groups that each
 * replicate a set of sub-metatrees so the busiest worker's share of the sampled work is
 * smallest. work: the sampled work of every sub-metatree, optionally followed by its learnable
 * leaf rows per batch (both from hg_sub_work; rows weigh the replicas' gradient merge).
 * Same bundle as hg_meta_partition. */
hg_bundle* hg_meta_partition_work_aware(const hg_graph* g, int k, int p, const double* work, int n_work);
/* sampled work per sub-metatree: mean sampled edges per batch of a device sampler restricted
 * to the sub's relations, over n_batches make_batches(batch_size, seed) batches ("work" f64),
 * and its learnable layer-0 rows per batch ("learn_rows" f64) */
hg_bundle* hg_sub_work(const hg_graph* g, const int* fanouts, int k, int n_batches, int batch_size, uint64_t seed,
                       int device);
/* make_batches (src/harness.cpp:327-340): batch{i} arrays */
hg_bundle* hg_make_batches(const hg_graph* g, int batch_size, int max_batches, uint64_t seed);
uint64_t hg_mix_seed(uint64_t a, uint64_t b); /* src/sampling.cpp:9-15 */
/* n raw outputs of std::mt19937_64(seed) from output index start on, reached by polynomial
 * jump-ahead (the feature streams of src/harness.cpp:153-162 are generated in jumped chunks);
 * returns 0, or -1 with hg_last_error set */
int hg_mt64_outputs(uint64_t seed, uint64_t start, uint64_t n, uint64_t* out);

/* ---- device engine (one meta-partition per GPU) ---------------------------------------- */
typedef struct {
  int k;
  const int* fanouts;
  int hidden;
  int batch_cap;
  int p;       /* meta-partition count */
  int rank;    /* partition evaluated by this engine */
  uint64_t model_seed; /* init_model seed (src/hgnn.cpp:39) */
  uint64_t learn_seed; /* init_learnable seed (src/hgnn.cpp:64) */
  int device;
  /* storage of the dense layer-0 feature tables: 0 f32 (parity), 1 f16, 2 bf16 */
  int feat_dtype;
  /* 1: dense feature tables stay in pinned host memory (read over PCIe, zero-copy);
   * hg_engine_set_cache installs an HBM copy of the cached rows (cache.cpp:121-141) */
  int feat_host;
  /* layer type: 0 RGCN (src/hgnn.cpp:173-362), 1 RGAT (relational attention, no reference
   * counterpart: DESIGN.md §3, oracle/rgat.py); heads below the top layer (0: 4) */
  int model;
  int heads;
} hg_engine_opts;

typedef struct {
  double loss;
  uint64_t sampled_edges;
  int n_active; /* entries filled in active_rows (p > 1) */
  int active_rows[64];
  /* ExecutionReport bookkeeping (raf.hpp:66-77). sync_bytes is this rank's replica
   * group's share of the ring all-reduce model (raf.cpp:496-510); summing it over
   * the ranks with sync_leader = 1 gives the reference's run-wide number. */
  uint64_t sync_bytes;
  int sync_leader;
  int message_bound_ok; /* check_comm_bounds (raf.cpp:662-676) */
  int target_only_ok;   /* cross_ids_target_only (raf.cpp:511-514) */
  int n_boundary;       /* entries filled in boundary_counts (= p) */
  uint64_t boundary_cut_edges;   /* raf.cpp:521-528 */
  uint64_t boundary_counts[64];  /* structural_boundaries (raf.cpp:306-340), per worker */
} hg_step_report;

hg_engine* hg_engine_create(const hg_graph* g, const hg_engine_opts* opts);
/* streaming loader: an engine whose graph comes straight from an HGC1 container file
 * (src/container.cpp:92-154 format): relations' dst-major pairs and dense feature rows
 * stream through pinned buffers into the device CSR and tables (no host graph) */
hg_engine* hg_engine_create_from_container(const char* path, const hg_engine_opts* o);
/* An engine of the work-aware plan (hg_meta_partition_work_aware) instead of the reference's */
hg_engine* hg_engine_create_work_aware(const hg_graph* g, const hg_engine_opts* opts, const double* work, int n_work);
/* Sampler-only engine for sample_khop (hop_rel_flat == NULL: every relation at
 * every hop; src/sampling.cpp:94-97) and sample_khop_restricted (per-hop allowed
 * relation lists, concatenated, hop_rel_counts[h] entries each; sampling.cpp:99-103).
 * Use hg_engine_sample + hg_engine_read; hg_engine_step is rejected. */
hg_engine* hg_sampler_create(const hg_graph* g, const int* fanouts, int k, const int* hop_rel_flat,
                             const int* hop_rel_counts, int batch_cap, int device);
void hg_engine_free(hg_engine* e);

/* One RAF training batch: run_raf_batch (src/raf.cpp:344-530) followed by
 * adam_update_model / adam_update_rows (src/hgnn.cpp:379-410), exactly as the
 * hot loop of run_experiment (src/harness.cpp:403-423). `batch` is host memory.
 * train = 0 runs forward + loss only. */
int hg_engine_step(hg_engine* e, const uint32_t* batch, int n, uint64_t rng_seed, int designated,
                   int train, hg_step_report* out);
/* Sampling depends only on (graph, batch, rng_seed): hg_engine_prefetch samples a future
 * batch into the engine's second sample slot on its sampling stream and returns at once;
 * a later hg_engine_step with the same (batch, rng_seed) trains on it, so the sampling of
 * batch i+1 overlaps the training of batch i. At most two batches may be in flight. */
int hg_engine_prefetch(hg_engine* e, const uint32_t* batch, int n, uint64_t rng_seed);
/* sample_khop_restricted (src/sampling.cpp:99-103) with the engine's hop relation sets. */
int hg_engine_sample(hg_engine* e, const uint32_t* batch, int n, uint64_t rng_seed);
/* Named device tensors after the last call (comma-separated names, NULL = all):
 * frontier{h}.t{t}, hop{h}.rel{r}.{dst_ids,indptr,src_ids,col}, H{d}.t{t},
 * mean.l{l}.r{r}.t{t}, logits, dlogits, loss, grad.w.r{r}.l{l}, grad.f.t{t}.{ids,rows},
 * post.r{r}.l{l}, post.learn{,_m,_v,_step}.t{t}, sampled_edges */
hg_bundle* hg_engine_read(hg_engine* e, const char* names);

/* Device-resident benchmark loop: uploads all batches first, then times
 * n_steps steps back to back with CUDA events on the engine's stream.
 * out_ms = device milliseconds for all steps; out_edges = sampled edges. */
int hg_engine_bench(hg_engine* e, const uint32_t* batches, const int* lens, const uint64_t* seeds,
                    int n_steps, int train, double* out_ms, uint64_t* out_edges, double* out_loss);
void hg_engine_profile(hg_engine* e, int on);
/* per kernel class: kernel.<name>.ms / .launches; alg_bytes = cumulative algorithmic
 * bytes [sample, aggregate, aggregate_top, csc_gather, csc_gather_top] since profiling
 * was switched on (the *_top classes are the top layer's launches: hop-1 blocks) */
hg_bundle* hg_engine_profile_read(hg_engine* e);
int hg_engine_info(hg_engine* e, uint64_t* param_count, uint64_t* device_bytes, int* model_step);
/* options: "retain_grads" (keep learnable-row gradients readable as grad.f.*; default 1),
 * "graphs" (replay the step as a CUDA graph; default 1), "umma" (dense contractions on
 * tcgen05 tensor cores, 3xTF32; 0 = SIMT fp32 tiles for A/B checks; default 1),
 * "elem_bytes" (AccountingModel::elem_bytes of the sync_bytes model: 2, 4 or 8; default 4),
 * "shard_merge" (replica groups: each replica Adam-updates only its id shard of the merged
 * learnable rows and stores them into every copy; default 0), "apply_adam" (0: training
 * steps compute every gradient but leave parameters and Adam state untouched — the caller
 * owns the optimizer; p = 1 or partitions without replicas; default 1) */
int hg_engine_set_option(hg_engine* e, const char* name, int value);
/* Device self-test of the tcgen05 contractions against the fp32 SIMT tiles on random
 * problems: cases = n_cases x (rows, nrel, din, dout); err = [n_cases x 3] relative
 * errors of (projection, mean gradient, weight gradient). */
hg_bundle* hg_selftest_contractions(const int* cases, int n_cases, int device);
/* kernel launches of one step (a captured, never executed step; NCCL kernels excluded) */
int hg_engine_count_launches(hg_engine* e, int n, int train);

/* ---- cache (src/cache.cpp) -------------------------------------------------------------- */
/* presample_hotness (src/cache.cpp:39-63) on the device: hot.t{t} u64 counts */
hg_bundle* hg_engine_presample_hotness(hg_engine* e, int epochs, uint64_t seed, int batch_size);
/* profile_miss_penalty + allocate_cache + fill_and_serve (src/cache.cpp:11-141):
 * counts are the hot.t{t} arrays concatenated in type order. Names: profile.*,
 * alloc.bytes, alloc.capacity, cached.t{t} (sorted). */
hg_bundle* hg_cache_plan(const hg_graph* g, const uint64_t* counts, uint64_t budget, double read_ns,
                         double write_ns, double overhead_ns, int elem_bytes);
/* Install the cached sets (concatenated sorted ids, per-type lengths) for the
 * per-batch lookup/update accounting (CacheState::lookup/update, cache.cpp:87-113;
 * hook harness.cpp:425-437). */
int hg_engine_set_cache(hg_engine* e, const uint32_t* ids, const uint64_t* lens, int n_types);
/* per type: hits, misses of the layer-0 frontier lookups so far (cache.t{t} = [hits, misses]) */
hg_bundle* hg_engine_cache_counters(hg_engine* e);

/* ---- multi-GPU: AGG_all over NCCL (one engine per rank) --------------------------------- */
int hg_nccl_unique_id(void* out, int cap);
int hg_engine_attach_nccl(hg_engine* e, const void* unique_id, int id_bytes, int nranks, int rank);
/* Replica groups (p larger than the number of sub-metatrees; metapartition.cpp:206-236):
 * hg_engine_replica_handle writes this engine's CUDA IPC handles (its gradient-exchange
 * arena, then its copy of every exchanged learnable table; returns the byte count, 0 if
 * the partition has no replicas). Every rank passes the handles of all ranks (nranks x
 * handle_bytes, rank order, each zero-padded to handle_bytes; any bytes for ranks without
 * replicas) to hg_engine_attach_replicas after hg_engine_attach_nccl. */
int hg_engine_replica_handle(hg_engine* e, void* out, int cap);
int hg_engine_attach_replicas(hg_engine* e, const void* handles, int handle_bytes, int nranks);

/* sample_neighbors (src/sampling.cpp:17-39) on a host CSR (indptr u64 [n_dst+1], src u32):
 * min(fanout, deg) sources of `dst` in draw order into out (capacity >= fanout); rows with
 * deg > fanout are drawn on the device (exact mt19937_64 + Lemire + partial Fisher-Yates) */
int hg_sample_neighbors(const uint64_t* indptr, uint64_t n_dst, const uint32_t* src, uint32_t dst, int fanout,
                        uint64_t rng_seed, int hop, int rel, uint32_t* out, int* n_out, int device);

/* ---- model state for caller-owned models (hgnn.hpp:34-62) ------------------------------- */
/* init_model (src/hgnn.cpp:39-62) on the BFS metatree of depth k: w.r{r}.l{l} f64
 * [din x dout], input_dims, k. init_learnable (src/hgnn.cpp:64-81): learn.t{t} f64
 * [count x dim]. Both bit-identical to the reference (same libstdc++ engines). */
hg_bundle* hg_init_model(const hg_graph* g, int k, int hidden, uint64_t seed);
hg_bundle* hg_init_learnable(const hg_graph* g, uint64_t seed);
/* Borrowed views of the host graph: a type's dense f32 features ([rows x dim] row-major,
 * NULL unless kind == 1) and the labels (hetgraph.hpp:58-74). */
int hg_graph_dense(const hg_graph* g, int type, const float** data, uint64_t* rows, int* dim, int* kind);
int hg_graph_labels(const hg_graph* g, const int32_t** labels, uint64_t* n);
/* Caller-owned parameters for an engine (run_raf_batch with the caller's HGNNModel /
 * LearnableStore, raf.hpp:79-82): one weight slot (f64 [din x dout]) and rows of a
 * learnable table (f64 [n x dim]). With the option "apply_adam" = 0 a training step
 * computes every gradient (grad.w.*, grad.f.*) and leaves the parameters untouched. */
int hg_engine_load_weights(hg_engine* e, int rel, int layer, const double* w, int din, int dout);
int hg_engine_load_table_rows(hg_engine* e, int type, const uint32_t* ids, int64_t n, const double* rows, int dim);

/* ---- layer interface on device tensors (hgnn.hpp:76-130) ----------------------------------
 * A context owns a device stream; every primitive is stream-ordered on it and returns at
 * once. Device-side errors are raised by hg_ctx_sync with the reference's exception type
 * and message ("node id not in frontier: <id>" = invalid_argument, "non-finite gradient" =
 * runtime_error). Tensors are row-major fp32 device matrices whose row stride `ld` is a
 * multiple of 4 with zero padding; index arrays are device u32 unless stated otherwise. */
typedef struct hg_ctx hg_ctx;
typedef struct {
  float* data;
  int64_t rows;
  int32_t cols;
  int32_t ld;
} hg_tensor;
hg_ctx* hg_ctx_create(int device);
void hg_ctx_free(hg_ctx* c);
int hg_ctx_sync(hg_ctx* c);
void* hg_ctx_malloc(hg_ctx* c, size_t bytes); /* zero-filled device memory */
int hg_ctx_mfree(hg_ctx* c, void* p);
int hg_ctx_copy(hg_ctx* c, void* dst, const void* src, size_t bytes); /* any direction, synchronous */
/* row_index (src/hgnn.cpp:166-171): rows[i] = position of ids[i] in the sorted list */
int hg_rows_in(hg_ctx* c, const uint32_t* ids, int64_t n, const uint32_t* sorted, int64_t n_sorted, uint32_t* rows);
/* mean_aggregate (src/hgnn.cpp:173-187): out[i] = mean of h_src[src_rows[e]] over the
 * block's segment i (u32 indptr), zero rows for empty segments; out [n_dst x h_src.cols] */
int hg_mean_aggregate(hg_ctx* c, const uint32_t* indptr, int64_t n_dst, const uint32_t* src_rows, hg_tensor h_src,
                      hg_tensor out);
/* agg_relation + agg_all (src/hgnn.cpp:189-203): out (+)= sum_r means[r] . ws[r], ReLU
 * optional (src/hgnn.cpp:271-272); 1-16 relations; tcgen05 kind::tf32 3xTF32 */
int hg_project(hg_ctx* c, const hg_tensor* means, const hg_tensor* ws, int nrel, hg_tensor out, int relu,
               int accumulate);
/* agg_all (src/hgnn.cpp:194-203): ordered elementwise sum of 1..32 partials */
int hg_agg_all(hg_ctx* c, const hg_tensor* partials, int n, hg_tensor out);
/* x = max(x, 0), or with a mask: x *= [mask > 0] (dpre = dH (x) [H > 0], src/hgnn.cpp:326-328) */
int hg_relu(hg_ctx* c, hg_tensor x, const hg_tensor* mask);
/* the layer-0 gather of forward_flat (src/hgnn.cpp:223-242): out[i] = table[ids[i]] */
int hg_gather_rows(hg_ctx* c, hg_tensor table, const uint32_t* ids, int64_t n, hg_tensor out);
/* cross_entropy (src/hgnn.cpp:281-307) on device logits; row_ids (sorted), batch and
 * labels (indexed by node id) are HOST arrays; dlogits may be NULL; synchronous */
int hg_cross_entropy(hg_ctx* c, hg_tensor logits, const uint32_t* row_ids, int64_t n_rows, const uint32_t* batch,
                     int64_t n_batch, const int32_t* labels, int64_t n_labels, int num_classes,
                     const hg_tensor* dlogits, double* loss);
/* matmul_tn_acc (src/matrix.hpp:49-61): dw (+)= mean^T . dpre (tcgen05, ordered split-K) */
int hg_weight_grad(hg_ctx* c, hg_tensor mean, hg_tensor dpre, hg_tensor dw, int accumulate);
/* matmul_nt (src/matrix.hpp:64-78) with the scatter's 1/deg (src/hgnn.cpp:337-353):
 * dmean[i] = (dpre[i] . W^T) / deg_i, deg from the block's u32 indptr */
int hg_mean_grad(hg_ctx* c, hg_tensor dpre, hg_tensor w, const uint32_t* indptr, hg_tensor dmean);
/* the backward scatter (src/hgnn.cpp:344-353): dh_src[src_rows[e]] += dmean[row(e)] for
 * every edge e, as a source-major ordered gather (deterministic) */
int hg_scatter_rows(hg_ctx* c, const uint32_t* indptr, int64_t n_dst, int64_t n_edges, const uint32_t* src_rows,
                    hg_tensor dmean, hg_tensor dh_src);
/* adam_step (src/hgnn.cpp:364-377) over n elements at Adam step `step` (adam_update_model
 * calls it per slot); adam_update_rows (src/hgnn.cpp:392-410) on listed table rows at the
 * table's advanced step */
int hg_adam_dense(hg_ctx* c, float* w, float* m, float* v, const float* g, int64_t n, int64_t step, double lr,
                  double beta1, double beta2, double eps);
int hg_adam_rows(hg_ctx* c, hg_tensor w, hg_tensor m, hg_tensor v, const uint32_t* rows, int64_t n, hg_tensor grads,
                 int64_t step, double lr, double beta1, double beta2, double eps);

#ifdef __cplusplus
}
#endif

#endif /* HETGPU_H */
