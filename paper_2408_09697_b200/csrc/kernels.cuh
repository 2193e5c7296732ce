// Kernel interfaces of the mini-batch hot path (sm_100a). All sizes that
// depend on the sampled data live in device memory: kernels are launched with
// grids sized from host-known capacities and read their live counts on the
// device, so a whole training step is one stream of launches with no host
// round trip (and capturable into a CUDA graph).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace hetgpu {

constexpr int kMaxBlocks = 16;  // sampled blocks per hop (relations)
constexpr int kMaxSegs = 16;
constexpr int kMaxRelsPerGroup = 16;

// Per-step scalars written by one small H2D copy (the only per-batch upload
// besides the batch ids).
struct StepScalars {
  std::uint64_t rng_seed;
  int batch_len;       // |batch| including duplicates
  int designated;
  std::int64_t model_step;  // Adam step after this batch's increment
};

// ---- segmented inclusive scan of u32 (in place) --------------------------------
struct ScanSeg {
  std::uint32_t* data;
  const int* n;  // live length (device)
  int cap;       // capacity (host)
};
struct ScanArgs {
  ScanSeg s[kMaxSegs];
  int nseg;
};
constexpr int kScanTile = 4096;
// look-back scratch for the single-pass scans: word 0 is the ticket counter,
// words 1.. the per-tile (flag, value) states; reset with one memset per use
struct LbScratch {
  unsigned long long* mem = nullptr;
  int cap = 0;  // tiles
  unsigned long long* state = nullptr;
  int* ticket = nullptr;
  void reset(int tiles, cudaStream_t st) {
    if (tiles > cap) throw std::runtime_error("look-back scratch too small");
    ticket = reinterpret_cast<int*>(mem);
    state = mem + 1;
    HG_CUDA(cudaMemsetAsync(mem, 0, (static_cast<std::size_t>(tiles) + 1) * 8, st));
  }
};
// rows per sampler tile (= threads per CTA of k_sample_fused); 128 measured best
// (the RNG-row tiles are the long pole: smaller tiles spread them over more SMs)
#ifndef HG_SAMPLE_TILE
#define HG_SAMPLE_TILE 128
#endif
constexpr int kSampleTileRows = HG_SAMPLE_TILE;
// bitmap words per frontier-compaction tile (one word per thread)
constexpr int kCompactWordsPerTile = 256;
// single-pass (decoupled look-back) segmented inclusive scan
void scan_inclusive(const ScanArgs& a, LbScratch& lb, cudaStream_t st);

// ---- sampling ---------------------------------------------------------------------
struct SampleBlock {
  const std::uint64_t* csr_ptr;  // relation CSR (dst-major), full graph
  const std::uint32_t* csr_src;
  const std::uint32_t* dst_list;  // frontier[h-1][rel.dst]
  const int* n_rows;              // its live size
  std::uint32_t* indptr;          // [rows_cap + 1] block offsets (u32)
  std::uint32_t* src_ids;         // [edge_cap] sampled sources in draw order
  std::uint32_t* erow;            // [edge_cap] block row of every sampled edge
  std::uint32_t* mark_bits;       // frontier[h][src type] bitmap (marked as sampled), or null
  int rel;
  int rows_cap;
  float rng_frac;  // expected share of RNG rows: blocks with more get the earliest tiles
};
struct SampleHop {
  SampleBlock b[kMaxBlocks];
  int nblk;
  int fanout;
  int hop;
  // diagnostics (null normally): per tile [start, scanned, drawn, end] %globaltimer
  // ns, the segment, and the SM
  unsigned long long* trace;
};
// One pass per hop: per-row counts min(fanout, deg), the block offsets (single-pass
// scan) and the draws (exact mt19937_64 + Lemire + partial Fisher-Yates). Rows
// whose draw overflows the streaming engine go to `slow` ((block,row) pairs,
// capacity = total rows) and are replayed with the full-state engine on
// `scratch` (sample_scratch_words(fanout) u64).
std::size_t sample_scratch_words(int fanout);
// one row drawn on the device (sample_neighbors, sampling.cpp:17-39, for deg > fanout):
// seed = mix_seed(rng_seed, mix_seed(hop << 32 | rel, dst)); scratch: 312 u64 + fanout u64
void sample_row(const std::uint32_t* d_nbr, std::uint64_t deg, int fanout, std::uint64_t seed, std::uint32_t* d_out,
                std::uint64_t* d_scratch, cudaStream_t st);
void sample_hop(const SampleHop& h, const StepScalars* sc, std::uint32_t* slow, int* n_slow,
                std::uint64_t* scratch, LbScratch& lb, cudaStream_t st);

// ---- frontier: bitmap set -> sorted unique ids + rank -----------------------------
struct BitmapType {
  std::uint32_t* bits;   // words of this type's id space
  int words;
  std::uint32_t* wscan;  // inclusive scan of per-word popcounts
  std::uint32_t* list;   // out: sorted unique ids
  int* count;            // out: live size
  int cap;
};
struct FrontierArgs {
  BitmapType t[kMaxSegs];
  int ntypes;
};
void frontier_mark_batch(const std::uint32_t* ids, const StepScalars* sc, int cap, const BitmapType& t,
                         cudaStream_t st);
// popcount + single-pass scan + emit of every type's bitmap (sorted unique ids)
void frontier_compact(const FrontierArgs& f, LbScratch& lb, cudaStream_t st);
struct RelabelBlock {
  const std::uint32_t* ids;
  const std::uint32_t* indptr;
  const int* n_rows;
  std::uint32_t* col;
  int cap;
  int slot;
  std::uint32_t* csc_count;  // optional: per-source-row edge counts for the transposed view
};
struct RelabelArgs {
  RelabelBlock b[kMaxBlocks];
  int nblk;
};
void frontier_relabel(const RelabelArgs& r, const FrontierArgs& f, cudaStream_t st);
// multiplicity of every unique batch row (duplicates in the batch)
void batch_multiplicity(const std::uint32_t* ids, const StepScalars* sc, int cap, const BitmapType& t,
                        float* mult, cudaStream_t st);

// ---- dense: relation-first aggregation + projection -------------------------------

// ---- loss ------------------------------------------------------------------------
// per table: step += 1 iff its gradient row count is non-zero (hgnn.cpp:392-394)
struct StepBumps {
  std::int64_t* step[kMaxSegs];
  const int* n[kMaxSegs];
  int count;
};
struct LossArgs {
  const float* logits;
  int ld;
  int C;
  const int* n_rows;
  int rows_cap;
  const std::uint32_t* row_ids;  // frontier[0][target]
  const float* mult;
  const std::int32_t* labels;
  const StepScalars* sc;
  float* dlogits;
  double* row_loss;   // scratch [rows_cap]
  double* loss_out;   // [1]
  std::uint32_t* err;
  unsigned* done;     // CTA completion counter (zero between launches)
  StepBumps bumps;    // applied by the last CTA (training steps)
};
// softmax cross-entropy per row, then the batch loss as an ordered sum over the
// rows by the last CTA to finish (one launch)
void cross_entropy(const LossArgs& a, cudaStream_t st);

// ---- backward ------------------------------------------------------------------------
// Transposed (src-major) view of one hop's blocks per source type: turns the
// backward scatter (hgnn.cpp:344-353) into an ordered gather (deterministic).
// Counts come from the relabel kernel; csc_prepare scans, fills and sorts
// every segment by (block, edge); csc_gather sums dmean rows per source row and,
// for learnable layer-0 types, applies the sparse Adam row update in place
// (adam_update_rows, hgnn.cpp:392-410) without materialising the gradient.
struct CscType {
  std::uint32_t* offs;     // [src_cap + 1]: counts, then inclusive prefix
  std::uint32_t* cursor;   // [src_cap]
  std::uint32_t* entries;  // packed (block << 28 | destination row, or edge) of every edge, grouped by source row
  const int* n_src;
  int src_cap;
  float* dh;               // gradient rows (nullptr: not materialised)
  int ld_dh;
  int din;
  // fused Adam (learnable leaf types only; w == nullptr otherwise)
  float *w, *m, *v;
  int ld_w;
  const std::uint32_t* ids;  // frontier[k][t]: global row of every source row
  const std::int64_t* step;
  // inner types: dH is stored already masked by the ReLU of its forward output
  // (dpre = dH * [H > 0], hgnn.cpp:326-328), so the backward contractions read it plain
  const float* relu_h;
  int ld_h;
  std::uint32_t* tmp;  // entries-sized scratch: merges of long (hub) segments
};
struct CscEdges {
  const std::uint32_t* col;
  const std::uint32_t* erow;
  const std::uint32_t* indptr;
  const int* n_rows;
  int cap;
  int edge_base;
  int type;  // index into CscHop::t
  const float* dmean;
  int ld_dmean;
};
struct CscHop {
  CscType t[kMaxSegs];
  int nt;
  CscEdges b[kMaxBlocks];
  int nb;
  int edge_ids;  // entries hold (block, edge) instead of (block, destination row)
};
void csc_prepare(const CscHop& h, LbScratch& lb, cudaStream_t st);

// ---- optimizer ------------------------------------------------------------------------
struct AdamHyper {  // hgnn.hpp:16-21
  double lr = 1e-2, beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
};
constexpr int kMaxSlots = 64;
// all model slots (adam_update_model, hgnn.cpp:379-390); base4 = prefix of rows*ld/4
struct AdamModelBatch {
  float* w[kMaxSlots];
  float* m[kMaxSlots];
  float* v[kMaxSlots];
  const float* g[kMaxSlots];
  int base4[kMaxSlots];
  int n;
  int total4;
};
void adam_model(AdamModelBatch& b, const std::int64_t* step, AdamHyper hp, std::uint32_t* err, cudaStream_t st);
// sparse learnable rows (adam_update_rows, hgnn.cpp:392-410): ids = frontier[k][t]
struct AdamRowsTable {
  float *w, *m, *v;
  int ld;
  const std::uint32_t* ids;
  const float* g;
  int ld_g;
  const int* n_rows;
  std::int64_t* step;
};
struct AdamRowsBatch {
  AdamRowsTable t[kMaxSegs];
  int base4[kMaxSegs];  // prefix of rows_cap * ld / 4
  int n;
  int total4;
};
void adam_rows(AdamRowsBatch& b, AdamHyper hp, std::uint32_t* err, cudaStream_t st);
// gather (+ fused sparse Adam for learnable leaves) of every type of one hop
void csc_gather(const CscHop& h, AdamHyper hp, std::uint32_t* err, cudaStream_t st);
// per table: step += 1 iff it has gradient rows (hgnn.cpp:392-394)
void bump_steps(const std::int64_t* const* steps, const int* const* counts, int n, cudaStream_t st);

// ---- replica groups: merge of the learnable-row gradients of every replica ----------
// ids/count/dh of replica r may live in a peer GPU's memory (CUDA IPC over NVLink).
// Union of the replicas' sorted id lists (bitmap + compaction, sorted), then per
// union row the ordered sum over replicas (r = 0..n-1) of their gradient rows:
// deterministic and identical on every replica, so the replicated tables stay equal.
constexpr int kMaxRep = 8;
// replica barrier (the end of the replica merge): every replica stores its step count
// into flag slot `pos` of every peer's IPC-mapped arena (release, system scope), then
// waits until all flags of its own arena reached the count (acquire)
struct ReplicaBarrier {
  unsigned* peer_flags[kMaxRep];  // flags of replica r's arena (ours included)
  unsigned* my_flags;
  unsigned* epoch;                // steps passed (device)
  int n;
  int pos;
};
void replica_barrier(const ReplicaBarrier& b, cudaStream_t st);
struct ReplicaMerge {
  const std::uint32_t* ids[kMaxRep];
  const int* count[kMaxRep];
  const float* dh[kMaxRep];
  int n_rep;
  int ld;       // row stride of dh and ug
  int din;
  BitmapType u; // union over the type's id space: list/count/wscan = this shard's ids
  int* slot;    // [n_rep x u.cap]
  float* ug;    // [u.cap x ld] merged gradient rows
  int shard, nshard;  // ids with id % nshard == shard are merged (and Adam-updated) here
  int* total;         // size of the whole union (all shards)
};
// stages: union (bitmap of every replica's ids, compaction of this shard's) and
// per-replica row slots of the shard's union rows
void replica_union(const ReplicaMerge& m, LbScratch& lb, cudaStream_t st);
void replica_slots(const ReplicaMerge& m, cudaStream_t st);
// ordered sum fused with the sparse Adam of the union rows (one pass instead of
// sum -> ug -> adam_rows); ug is still written when m.ug is set (retained grads).
// The table's step must already be bumped (bump_steps).
struct ReplicaAdam {
  float *w, *m, *v;
  int ld_w;
  const std::int64_t* step;
  float* peer_w[kMaxRep];  // every replica's copy of the table (IPC-mapped; ours included)
  int n_rep;
};
void replica_sum_adam(const ReplicaMerge& m, const ReplicaAdam& a, AdamHyper hp, std::uint32_t* err,
                      cudaStream_t st);

// ---- misc --------------------------------------------------------------------------------
void zero_rows(float* p, int ld, const int* n_rows, int rows_cap, cudaStream_t st);
// cache lookups: hits of frontier ids against a cached-id bitmap, accumulated
void cache_count(const std::uint32_t* ids, const int* n, int cap, const std::uint32_t* cached_bits,
                 unsigned long long* hits_misses, cudaStream_t st);
// p > 1: the global layer-0 frontier of a type as the union of every partition's (a 0/1
// byte per node, OR-ed across ranks with an ncclMax all-reduce), then its cache lookups
void union_mark(const std::uint32_t* ids, const int* n, int cap, std::uint8_t* map, cudaStream_t st);
void union_count(const std::uint8_t* map, std::uint64_t n, const std::uint32_t* cached_bits, unsigned long long* hm,
                 cudaStream_t st);
// histogram for presample_hotness
void hotness_add(const std::uint32_t* ids, const std::uint32_t* indptr, const int* n_rows, int cap,
                 unsigned long long* counts, cudaStream_t st);
void hotness_add_list(const std::uint32_t* ids, const int* n, int cap, unsigned long long* counts,
                      cudaStream_t st);

}  // namespace hetgpu
