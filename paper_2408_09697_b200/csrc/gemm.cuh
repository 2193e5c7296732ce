// Multi-problem tile kernels for the dense contractions (gemm_kernels.cu).
#pragma once

#include <vector>

#include "kernels.cuh"

namespace hetgpu {

constexpr int kMaxProblems = 16;
#ifndef HG_WCHUNK
#define HG_WCHUNK 512
#endif
constexpr int kWChunkRows = HG_WCHUNK;  // split-K rows per weight-gradient partial (512 measured best)

// dpre rows: g[(i*stride + offset) * ld + c], masked by H > 0 when h != nullptr
struct DpreView {
  const float* g;
  const float* h;
  int ld;
  int cols;
  int stride;
  int offset;
};

struct WGradProblem {
  const float* mean;
  int ld_mean;
  int din;
  DpreView d;
  const int* n_rows;
  int rows_cap;
  float* partial;  // [chunks x din x cols]
  float* dw;
  int ld_dw;
  // optional Adam of the slot fused into the reduction (stride ld_dw): each
  // gradient element is final there, so it is applied to w / m / v at once
  float *w, *m, *v;
};
struct WGradBatch {
  WGradProblem p[kMaxProblems];
  int tile_base[kMaxProblems];
  int np;
  int defer_reduce;            // the caller runs wgrad_reduce itself (after an event)
  const std::int64_t* step;    // model Adam step (fused update)
  AdamHyper hp;
  std::uint32_t* err;
};

struct DMeanProblem {
  DpreView d;
  const float* w;  // [din x dout], ld_w
  int ld_w;
  int din;
  const std::uint32_t* indptr;
  const int* n_rows;
  int rows_cap;
  float* dmean;
  int ld_dmean;
};
struct DMeanBatch {
  DMeanProblem p[kMaxProblems];
  int tile_base[kMaxProblems];
  int np;
};

// ---- split forward: gather-mean of every block of a hop, then projection ------------------
// storage of a layer-0 dense feature table (fp16 features)
enum FeatDtype : int { kF32 = 0, kF16 = 1, kBF16 = 2 };
struct MeanBlock {
  const std::uint32_t* indptr;
  const std::uint32_t* keys;  // global ids (by_id) or frontier rows
  const float* h;             // rows of h_dtype elements (h_dtype != kF32: reinterpret)
  int ld_h;
  int h_dtype;                // FeatDtype of h (layer-0 dense tables; inner layers are f32)
  // device cache of a host-resident table (cache.cpp:121-141 fill): slot[key] >= 0 reads
  // row slot of `cache` (HBM), otherwise row key of h (pinned host memory, read over PCIe)
  const int* slot;
  const float* cache;
  int din;
  const int* n_rows;
  int rows_cap;
  float* mean;
  int ld_mean;  // rows live..next multiple of 32 are zero-filled (weight-gradient K chunks)
};
struct MeanBatch {
  MeanBlock b[kMaxBlocks];
  int item_base[kMaxBlocks + 1];  // prefix of rows_cap * ceil(din/64)
  int nb;
};
void gather_mean(MeanBatch& m, cudaStream_t st);

struct ProjRel {
  const float* mean;
  int ld_mean;
  int din;
  const float* w;
  int ld_w;
  int row_stride;  // elements between consecutive A rows (0: ld_mean); a replica's shard of the logits
};
constexpr int kProjRels = 16;   // relations into one destination type (concatenated along K)
constexpr int kProjGroups = 4;  // destination types per projection launch
struct ProjGroup {
  ProjRel r[kProjRels];
  int nrel;
  const int* n_rows;
  int rows_cap;
  float* out;
  int ld_out;
  int dout;
  int relu;
  int out_stride, out_offset;
};
struct ProjBatch {
  ProjGroup g[kProjGroups];
  int tile_base[kProjGroups + 1];
  int ng;
};
void project_tiles(ProjBatch& p, cudaStream_t st);
void wgrad_tiles(WGradBatch& b, cudaStream_t st);
void dmean_tiles(DMeanBatch& b, cudaStream_t st);
// ordered (deterministic) sum of the split-K weight-gradient partials into dW
void wgrad_reduce(WGradBatch& b, cudaStream_t st);

// tcgen05 (kind::tf32, 3xTF32 split) versions of the three contractions (umma_kernels.cu)
void project_umma(ProjBatch& p, cudaStream_t st);
void wgrad_umma(WGradBatch& b, cudaStream_t st);
void dmean_umma(DMeanBatch& b, cudaStream_t st);

// self-test (selftest.cu): cases (rows, nrel, din, dout) -> {project, dmean, wgrad}
// max|tcgen05 - fp32 tiles| / max|fp32 tiles|
std::vector<std::vector<double>> selftest_contractions(const std::vector<std::vector<int>>& cases);

}  // namespace hetgpu
