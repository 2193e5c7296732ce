// Device primitives of the reference's layer interface (hgnn.hpp:76-130); see layers.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "kernels.cuh"

namespace hetgpu {

constexpr int kMaxLayerParts = 32;  // partials per agg_all call

// Row-major fp32 device matrix; the row stride `ld` is a multiple of 4 floats
// (16-byte rows for vector loads and TMA) and padding columns are zero.
struct DevTensor {
  float* data = nullptr;
  std::int64_t rows = 0;
  int cols = 0;
  int ld = 0;
};

class LayerCtx {
 public:
  explicit LayerCtx(int device);
  ~LayerCtx();
  LayerCtx(const LayerCtx&) = delete;
  LayerCtx& operator=(const LayerCtx&) = delete;

  cudaStream_t stream() const { return st_; }
  int device() const { return device_; }
  // waits for the stream and raises the reference's exceptions for device-side errors
  void sync();

  // row_index (hgnn.cpp:166-171) of every id in a sorted frontier
  void rows_in(const std::uint32_t* ids, std::int64_t n, const std::uint32_t* sorted, std::int64_t m,
               std::uint32_t* rows);
  // mean_aggregate (hgnn.cpp:173-187): block (u32 indptr, source rows) over h_src
  void mean_aggregate(const std::uint32_t* indptr, std::int64_t n_dst, const std::uint32_t* src_rows,
                      const DevTensor& h_src, const DevTensor& out);
  // out (+)= sum_r means[r] . ws[r] (+ReLU): agg_relation + agg_all (hgnn.cpp:189-203), tcgen05
  void project(const DevTensor* means, const DevTensor* ws, int nrel, const DevTensor& out, bool relu,
               bool accumulate);
  // agg_all (hgnn.cpp:194-203): ordered elementwise sum
  void agg_all(const DevTensor* parts, int n, const DevTensor& out);
  // x = ReLU(x), or x *= [mask > 0] (hgnn.cpp:271-272, 326-328)
  void relu(const DevTensor& x, const DevTensor* mask);
  // out[i] = table[ids[i]] (the layer-0 gather, hgnn.cpp:223-242)
  void gather_rows(const DevTensor& table, const std::uint32_t* ids, std::int64_t n, const DevTensor& out);
  // a += b
  void add(const DevTensor& a, const DevTensor& b);
  // cross_entropy (hgnn.cpp:281-307); row_ids / batch / labels are host arrays
  double cross_entropy(const DevTensor& logits, const std::uint32_t* row_ids, std::int64_t n_rows,
                       const std::uint32_t* batch, std::int64_t n_batch, const std::int32_t* labels,
                       std::int64_t n_labels, int num_classes, const DevTensor* dlogits);
  // dw (+)= mean^T . dpre (matmul_tn_acc, matrix.hpp:49-61), tcgen05 split-K, ordered reduction
  void weight_grad(const DevTensor& mean, const DevTensor& dpre, const DevTensor& dw, bool accumulate);
  // dmean = dpre . W^T / deg (matmul_nt, matrix.hpp:64-78, with the scatter's 1/deg, hgnn.cpp:344-353)
  void mean_grad(const DevTensor& dpre, const DevTensor& w, const std::uint32_t* indptr, const DevTensor& dmean);
  // dh_src[src_rows[e]] += dmean[row(e)] over every edge (hgnn.cpp:344-353): transposed, ordered gather
  void scatter_rows(const std::uint32_t* indptr, std::int64_t n_dst, std::int64_t n_edges,
                    const std::uint32_t* src_rows, const DevTensor& dmean, const DevTensor& dh_src);
  // adam_step on a dense array (hgnn.cpp:364-377) at Adam step `step`
  void adam_dense(float* w, float* m, float* v, const float* g, std::int64_t n, std::int64_t step,
                  const AdamHyper& hp);
  // adam_update_rows (hgnn.cpp:392-410) at the table's (already advanced) step
  void adam_rows(const DevTensor& w, const DevTensor& m, const DevTensor& v, const std::uint32_t* rows,
                 std::int64_t n, const DevTensor& grads, std::int64_t step, const AdamHyper& hp);

  // stream-ordered scratch, released at the next sync()
  void* scratch(std::size_t bytes);

 private:
  static constexpr int kIntSlots = 4096;
  const int* dev_int(long long v);
  void reset_err();
  int device_;
  cudaStream_t st_ = nullptr;
  std::uint32_t* err_ = nullptr;  // [flags, smallest offending id]
  int* ints_ = nullptr;
  int* ints_h_ = nullptr;
  int next_int_ = 0;
  unsigned* done_ = nullptr;
  std::vector<void*> scratch_;
};

}  // namespace hetgpu
