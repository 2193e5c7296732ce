// The reference's layer interface (hgnn.hpp:76-130) as device primitives over
// caller-owned device tensors: one call per reference function, composing the
// hot path's own kernels (gather-mean, the tcgen05 contractions, the loss, the
// ordered CSC gather, Adam). The fused training step lives in Engine; these are
// the drop-in building blocks (include/hetgpu.h "layer interface", and the
// Matrix-level mirrors in include/hetsim_b200.hpp).
//
// Every primitive is stream-ordered on the context's stream; device-side errors
// (an id absent from its frontier, a non-finite gradient) are raised by
// LayerCtx::sync() with the reference's exception type and message.
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "adam.cuh"
#include "gemm.cuh"
#include "layers.hpp"

namespace hetgpu {

namespace {

constexpr std::uint32_t kErrMissing = 1u;  // an id is not in its sorted frontier
constexpr std::uint32_t kErrNonFinite = 4u;  // adam4 / adam1 flag

// row_index (hgnn.cpp:166-171): binary search of every id in a sorted list
__global__ void k_rows_in(const std::uint32_t* ids, std::int64_t n, const std::uint32_t* sorted, std::int64_t m,
                          std::uint32_t* rows, std::uint32_t* err) {
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::uint32_t v = ids[i];
    std::int64_t lo = 0, hi = m;
    while (lo < hi) {
      const std::int64_t mid = (lo + hi) >> 1;
      if (sorted[mid] < v) lo = mid + 1; else hi = mid;
    }
    if (lo < m && sorted[lo] == v) {
      rows[i] = static_cast<std::uint32_t>(lo);
    } else {
      rows[i] = 0;
      atomicOr(err, kErrMissing);
      atomicMin(err + 1, v);  // the smallest offending id is reported
    }
  }
}

// out[i] = sum_{q < n} parts[q][i] in the fixed order q = 0, 1, ... (agg_all, hgnn.cpp:194-203)
struct PartList {
  const float* p[kMaxLayerParts];
  int ld[kMaxLayerParts];
  int n;
};
__global__ void k_agg_all(PartList pl, float* out, int ld_out, std::int64_t rows, int cols) {
  const std::int64_t total = rows * cols;
  for (std::int64_t x = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t i = x / cols;
    const int c = static_cast<int>(x % cols);
    float s = pl.p[0][i * pl.ld[0] + c];
    for (int q = 1; q < pl.n; ++q) s += pl.p[q][i * pl.ld[q] + c];
    out[i * ld_out + c] = s;
  }
}

// x = max(x, 0); dpre = dh * [h > 0] (hgnn.cpp:271-272, 326-328)
__global__ void k_relu(float* x, int ld, std::int64_t rows, int cols, const float* mask, int ld_mask) {
  const std::int64_t total = rows * cols;
  for (std::int64_t t = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t i = t / cols;
    const int c = static_cast<int>(t % cols);
    float& v = x[i * ld + c];
    if (mask) {
      if (mask[i * ld_mask + c] <= 0.f) v = 0.f;
    } else {
      v = v > 0.f ? v : 0.f;
    }
  }
}

// out[i] = table[ids[i]] (the layer-0 gather of forward_flat, hgnn.cpp:223-242)
__global__ void k_gather_rows(const float* table, int ld_t, std::int64_t n_table, const std::uint32_t* ids,
                              std::int64_t n, int cols, float* out, int ld_out, std::uint32_t* err) {
  const std::int64_t total = n * cols;
  for (std::int64_t t = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t i = t / cols;
    const int c = static_cast<int>(t % cols);
    const std::uint32_t id = ids[i];
    if (id >= n_table) {
      atomicOr(err, kErrMissing);
      atomicMin(err + 1, id);
      continue;
    }
    out[i * ld_out + c] = table[static_cast<std::int64_t>(id) * ld_t + c];
  }
}

// a += b (accumulating contractions: matmul_tn_acc, hgnn.cpp:334; the scatter's dH +=)
__global__ void k_add(float* a, int ld_a, const float* b, int ld_b, std::int64_t rows, int cols) {
  const std::int64_t total = rows * cols;
  for (std::int64_t t = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t i = t / cols;
    const int c = static_cast<int>(t % cols);
    a[i * ld_a + c] += b[i * ld_b + c];
  }
}

// block row of every edge, and per-source-row edge counts (the transposed view)
__global__ void k_edge_rows(const std::uint32_t* indptr, std::int64_t n_dst, const std::uint32_t* src_rows,
                            std::uint32_t* erow, std::uint32_t* counts) {
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n_dst;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    for (std::uint32_t e = indptr[i]; e < indptr[i + 1]; ++e) {
      erow[e] = static_cast<std::uint32_t>(i);
      atomicAdd(counts + src_rows[e], 1u);
    }
  }
}

// Adam on a dense array (adam_step, hgnn.cpp:364-377) and on listed table rows
// (adam_update_rows, hgnn.cpp:392-410); the step's bias corrections come from the host
__global__ void k_adam_dense(float* w, float* m, float* v, const float* g, std::int64_t n, AdamHyper hp, double t,
                             std::uint32_t* err) {
  const AdamStep k = adam_step_of(hp, t);
  for (std::int64_t x = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; x < n;
       x += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    float wv = w[x], mv = m[x], vv = v[x];
    adam1(wv, mv, vv, g[x], k, err);
    w[x] = wv;
    m[x] = mv;
    v[x] = vv;
  }
}
__global__ void k_adam_rows(float* w, float* m, float* v, int ld, std::int64_t n_table, const std::uint32_t* rows,
                            std::int64_t n, const float* g, int ld_g, int cols, AdamHyper hp, double t,
                            std::uint32_t* err) {
  const AdamStep k = adam_step_of(hp, t);
  const std::int64_t total = n * cols;
  for (std::int64_t x = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t i = x / cols;
    const int c = static_cast<int>(x % cols);
    const std::uint32_t r = rows[i];
    if (r >= n_table) {
      atomicOr(err, kErrMissing);
      atomicMin(err + 1, r);
      continue;
    }
    const std::int64_t at = static_cast<std::int64_t>(r) * ld + c;
    float wv = w[at], mv = m[at], vv = v[at];
    adam1(wv, mv, vv, g[i * ld_g + c], k, err);
    w[at] = wv;
    m[at] = mv;
    v[at] = vv;
  }
}

unsigned grid_for(std::int64_t n, int threads = 256) {
  return static_cast<unsigned>(std::max<std::int64_t>(1, std::min<std::int64_t>((n + threads - 1) / threads,
                                                                                  8LL * num_sms())));
}

void check_tensor(const DevTensor& t, const char* what) {
  if (t.rows < 0 || t.cols < 0) throw std::invalid_argument(std::string(what) + ": negative shape");
  if (t.rows > 0 && t.cols > 0 && !t.data) throw std::invalid_argument(std::string(what) + ": null data");
  if (t.ld < t.cols || t.ld % 4 != 0)
    throw std::invalid_argument(std::string(what) + ": row stride must be >= cols and a multiple of 4");
  if (reinterpret_cast<std::uintptr_t>(t.data) % 16 != 0)
    throw std::invalid_argument(std::string(what) + ": data must be 16-byte aligned");
}

}  // namespace

// ---- context -----------------------------------------------------------------------------------
LayerCtx::LayerCtx(int device) : device_(device) {
  HG_CUDA(cudaSetDevice(device));
  HG_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  HG_CUDA(cudaMalloc(&err_, 2 * sizeof(std::uint32_t)));
  HG_CUDA(cudaMalloc(&ints_, kIntSlots * sizeof(int)));
  HG_CUDA(cudaMallocHost(&ints_h_, kIntSlots * sizeof(int)));
  HG_CUDA(cudaMalloc(&done_, sizeof(unsigned)));
  HG_CUDA(cudaMemsetAsync(done_, 0, sizeof(unsigned), st_));
  reset_err();  // also synchronises the stream
}

LayerCtx::~LayerCtx() {
  cudaSetDevice(device_);
  cudaStreamSynchronize(st_);
  for (void* p : scratch_) cudaFreeAsync(p, st_);
  cudaStreamSynchronize(st_);
  cudaFree(err_);
  cudaFree(ints_);
  cudaFreeHost(ints_h_);
  cudaFree(done_);
  cudaStreamDestroy(st_);
}

void LayerCtx::reset_err() {
  const std::uint32_t init[2] = {0u, 0xFFFFFFFFu};
  HG_CUDA(cudaMemcpyAsync(err_, init, sizeof(init), cudaMemcpyHostToDevice, st_));
  HG_CUDA(cudaStreamSynchronize(st_));
}

void LayerCtx::sync() {
  HG_CUDA(cudaSetDevice(device_));
  HG_CUDA(cudaStreamSynchronize(st_));
  HG_CUDA(cudaGetLastError());
  std::uint32_t e[2];
  HG_CUDA(cudaMemcpy(e, err_, sizeof(e), cudaMemcpyDeviceToHost));
  for (void* p : scratch_) HG_CUDA(cudaFreeAsync(p, st_));
  scratch_.clear();
  HG_CUDA(cudaStreamSynchronize(st_));
  if (e[0]) {
    reset_err();
    if (e[0] & kErrMissing) throw std::invalid_argument("node id not in frontier: " + std::to_string(e[1]));
    if (e[0] & kErrNonFinite) throw std::runtime_error("non-finite gradient");
    throw std::runtime_error("device error flag " + std::to_string(e[0]));
  }
}

void* LayerCtx::scratch(std::size_t bytes) {
  void* p = nullptr;
  HG_CUDA(cudaMallocAsync(&p, std::max<std::size_t>(bytes, 16), st_));
  HG_CUDA(cudaMemsetAsync(p, 0, std::max<std::size_t>(bytes, 16), st_));
  scratch_.push_back(p);
  return p;
}

const int* LayerCtx::dev_int(long long v) {
  if (v > 0x7FFFFFFF) throw std::invalid_argument("size exceeds the device counters' int range");
  if (next_int_ == kIntSlots) {  // recycle once everything queued so far has run
    HG_CUDA(cudaStreamSynchronize(st_));
    next_int_ = 0;
  }
  // pinned staging slot: the copy is stream-ordered and the slot is not reused
  // before the stream has passed it (the ring wraps only after a sync)
  const int i = next_int_++;
  ints_h_[i] = static_cast<int>(v);
  HG_CUDA(cudaMemcpyAsync(ints_ + i, ints_h_ + i, sizeof(int), cudaMemcpyHostToDevice, st_));
  return ints_ + i;
}

// ---- primitives --------------------------------------------------------------------------------
void LayerCtx::rows_in(const std::uint32_t* ids, std::int64_t n, const std::uint32_t* sorted, std::int64_t m,
                       std::uint32_t* rows) {
  if (n <= 0) return;
  k_rows_in<<<grid_for(n), 256, 0, st_>>>(ids, n, sorted, m, rows, err_);
  HG_CUDA(cudaGetLastError());
}

void LayerCtx::mean_aggregate(const std::uint32_t* indptr, std::int64_t n_dst, const std::uint32_t* src_rows,
                              const DevTensor& h_src, const DevTensor& out) {
  check_tensor(h_src, "mean_aggregate h_src");
  check_tensor(out, "mean_aggregate out");
  if (out.rows != n_dst || out.cols != h_src.cols || out.ld != h_src.ld)
    throw std::invalid_argument("mean_aggregate: out must be [n_dst x cols of h_src] with the same row stride");
  if (n_dst == 0) return;
  MeanBatch mb{};
  MeanBlock& b = mb.b[mb.nb++];
  b.indptr = indptr;
  b.keys = src_rows;
  b.h = h_src.data;
  b.ld_h = h_src.ld;
  b.din = h_src.cols;
  b.n_rows = dev_int(n_dst);
  b.rows_cap = static_cast<int>(n_dst);
  b.mean = out.data;
  b.ld_mean = out.ld;
  gather_mean(mb, st_);
}

void LayerCtx::project(const DevTensor* means, const DevTensor* ws, int nrel, const DevTensor& out, bool relu,
                       bool accumulate) {
  if (nrel < 1 || nrel > kProjRels) throw std::invalid_argument("project: 1..16 relations per call");
  check_tensor(out, "project out");
  for (int r = 0; r < nrel; ++r) {
    check_tensor(means[r], "project mean");
    check_tensor(ws[r], "project w");
    if (means[r].rows != out.rows || ws[r].cols != out.cols)
      throw std::invalid_argument("agg_all partials have mismatched shapes");
    if (ws[r].rows != means[r].cols)
      throw std::invalid_argument("weight/input dim mismatch for relation " + std::to_string(r));
  }
  if (out.rows == 0) return;
  const DevTensor tgt = accumulate ? DevTensor{static_cast<float*>(scratch(static_cast<std::size_t>(out.rows) *
                                                                              out.ld * 4)),
                                               out.rows, out.cols, out.ld}
                                   : out;
  ProjBatch pb{};
  pb.ng = 1;
  ProjGroup& g = pb.g[0];
  g.nrel = nrel;
  for (int r = 0; r < nrel; ++r) g.r[r] = {means[r].data, means[r].ld, means[r].cols, ws[r].data, ws[r].ld};
  g.n_rows = dev_int(out.rows);
  g.rows_cap = static_cast<int>(out.rows);
  g.out = tgt.data;
  g.ld_out = tgt.ld;
  g.dout = out.cols;
  g.relu = relu ? 1 : 0;
  g.out_stride = 1;
  g.out_offset = 0;
  project_umma(pb, st_);
  if (accumulate) add(out, tgt);
}

void LayerCtx::agg_all(const DevTensor* parts, int n, const DevTensor& out) {
  if (n <= 0) throw std::invalid_argument("agg_all needs at least one partial");
  if (n > kMaxLayerParts) throw std::invalid_argument("agg_all: too many partials for one call");
  check_tensor(out, "agg_all out");
  PartList pl{};
  pl.n = n;
  for (int q = 0; q < n; ++q) {
    if (parts[q].rows != out.rows || parts[q].cols != out.cols)
      throw std::invalid_argument("agg_all partials have mismatched shapes");
    pl.p[q] = parts[q].data;
    pl.ld[q] = parts[q].ld;
  }
  if (out.rows * out.cols == 0) return;
  k_agg_all<<<grid_for(out.rows * out.cols), 256, 0, st_>>>(pl, out.data, out.ld, out.rows, out.cols);
  HG_CUDA(cudaGetLastError());
}

void LayerCtx::relu(const DevTensor& x, const DevTensor* mask) {
  if (x.rows * x.cols == 0) return;
  if (mask && (mask->rows != x.rows || mask->cols != x.cols))
    throw std::invalid_argument("relu mask shape mismatch");
  k_relu<<<grid_for(x.rows * x.cols), 256, 0, st_>>>(x.data, x.ld, x.rows, x.cols, mask ? mask->data : nullptr,
                                                     mask ? mask->ld : 0);
  HG_CUDA(cudaGetLastError());
}

void LayerCtx::gather_rows(const DevTensor& table, const std::uint32_t* ids, std::int64_t n, const DevTensor& out) {
  if (out.rows != n || out.cols != table.cols) throw std::invalid_argument("gather_rows: out must be [n x cols]");
  if (n * out.cols == 0) return;
  k_gather_rows<<<grid_for(n * out.cols), 256, 0, st_>>>(table.data, table.ld, table.rows, ids, n, out.cols,
                                                         out.data, out.ld, err_);
  HG_CUDA(cudaGetLastError());
}

void LayerCtx::add(const DevTensor& a, const DevTensor& b) {
  if (a.rows * a.cols == 0) return;
  k_add<<<grid_for(a.rows * a.cols), 256, 0, st_>>>(a.data, a.ld, b.data, b.ld, a.rows, a.cols);
  HG_CUDA(cudaGetLastError());
}

double LayerCtx::cross_entropy(const DevTensor& logits, const std::uint32_t* row_ids, std::int64_t n_rows,
                               const std::uint32_t* batch, std::int64_t n_batch, const std::int32_t* labels,
                               std::int64_t n_labels, int num_classes, const DevTensor* dlogits) {
  // host-side checks in the reference's order (hgnn.cpp:284-293)
  if (n_batch <= 0) throw std::invalid_argument("empty batch");
  if (logits.rows != n_rows || logits.cols < num_classes)
    throw std::invalid_argument("cross_entropy: logits must have one row per row id and num_classes columns");
  std::vector<float> mult(static_cast<std::size_t>(std::max<std::int64_t>(1, n_rows)), 0.f);
  std::vector<std::int32_t> row_label(mult.size(), 0);
  for (std::int64_t b = 0; b < n_batch; ++b) {
    const std::uint32_t v = batch[b];
    if (v >= n_labels) throw std::invalid_argument("label out of range for node " + std::to_string(v));
    const std::int32_t y = labels[v];
    if (y < 0 || y >= num_classes) throw std::invalid_argument("label out of range for node " + std::to_string(v));
    const std::uint32_t* it = std::lower_bound(row_ids, row_ids + n_rows, v);
    if (it == row_ids + n_rows || *it != v) throw std::invalid_argument("node id not in frontier: " + std::to_string(v));
    const std::size_t r = static_cast<std::size_t>(it - row_ids);
    mult[r] += 1.f;
    row_label[r] = y;
  }
  if (dlogits) {
    check_tensor(*dlogits, "cross_entropy dlogits");
    if (dlogits->rows != n_rows || dlogits->cols != logits.cols || dlogits->ld != logits.ld)
      throw std::invalid_argument("cross_entropy: dlogits must match the logits' shape and stride");
  }
  auto* d_mult = static_cast<float*>(scratch(mult.size() * 4));
  auto* d_lab = static_cast<std::int32_t*>(scratch(row_label.size() * 4));
  auto* d_ids = static_cast<std::uint32_t*>(scratch(mult.size() * 4));
  std::vector<std::uint32_t> iota(mult.size());
  for (std::size_t i = 0; i < iota.size(); ++i) iota[i] = static_cast<std::uint32_t>(i);
  HG_CUDA(cudaMemcpyAsync(d_mult, mult.data(), mult.size() * 4, cudaMemcpyHostToDevice, st_));
  HG_CUDA(cudaMemcpyAsync(d_lab, row_label.data(), row_label.size() * 4, cudaMemcpyHostToDevice, st_));
  HG_CUDA(cudaMemcpyAsync(d_ids, iota.data(), iota.size() * 4, cudaMemcpyHostToDevice, st_));
  StepScalars sc{};
  sc.batch_len = static_cast<int>(n_batch);
  auto* d_sc = static_cast<StepScalars*>(scratch(sizeof(StepScalars)));
  HG_CUDA(cudaMemcpyAsync(d_sc, &sc, sizeof(sc), cudaMemcpyHostToDevice, st_));
  auto* d_loss = static_cast<double*>(scratch(8));
  auto* d_rowloss = static_cast<double*>(scratch(mult.size() * 8));
  float* dz = dlogits ? dlogits->data : static_cast<float*>(scratch(static_cast<std::size_t>(n_rows) * logits.ld * 4));
  LossArgs la{};
  la.logits = logits.data;
  la.ld = logits.ld;
  la.C = num_classes;
  la.n_rows = dev_int(n_rows);
  la.rows_cap = static_cast<int>(n_rows);
  la.row_ids = d_ids;
  la.mult = d_mult;
  la.labels = d_lab;
  la.sc = d_sc;
  la.dlogits = dz;
  la.row_loss = d_rowloss;
  la.loss_out = d_loss;
  la.err = err_;
  la.done = done_;
  hetgpu::cross_entropy(la, st_);
  double loss = 0.0;
  HG_CUDA(cudaMemcpyAsync(&loss, d_loss, 8, cudaMemcpyDeviceToHost, st_));
  sync();
  return loss;
}

void LayerCtx::weight_grad(const DevTensor& mean, const DevTensor& dpre, const DevTensor& dw, bool accumulate) {
  check_tensor(mean, "weight_grad mean");
  check_tensor(dpre, "weight_grad dpre");
  check_tensor(dw, "weight_grad dw");
  if (mean.rows != dpre.rows || dw.rows != mean.cols || dw.cols != dpre.cols)
    throw std::invalid_argument("matmul_tn_acc shape mismatch");
  if (dw.rows * dw.cols == 0) return;
  if (mean.rows == 0) {
    if (!accumulate) HG_CUDA(cudaMemsetAsync(dw.data, 0, static_cast<std::size_t>(dw.rows) * dw.ld * 4, st_));
    return;
  }
  const DevTensor tgt = accumulate ? DevTensor{static_cast<float*>(scratch(static_cast<std::size_t>(dw.rows) * dw.ld * 4)),
                                               dw.rows, dw.cols, dw.ld}
                                   : dw;
  WGradBatch wb{};
  wb.np = 1;
  WGradProblem& P = wb.p[0];
  P.mean = mean.data;
  P.ld_mean = mean.ld;
  P.din = mean.cols;
  P.d = DpreView{dpre.data, nullptr, dpre.ld, dpre.cols, 1, 0};
  P.n_rows = dev_int(mean.rows);
  P.rows_cap = static_cast<int>(mean.rows);
  P.partial = static_cast<float*>(
      scratch(ceil_div(static_cast<std::uint64_t>(mean.rows), kWChunkRows) * mean.cols * dpre.cols * 4));
  P.dw = tgt.data;
  P.ld_dw = tgt.ld;
  wgrad_umma(wb, st_);
  if (accumulate) add(dw, tgt);
}

void LayerCtx::mean_grad(const DevTensor& dpre, const DevTensor& w, const std::uint32_t* indptr, const DevTensor& dmean) {
  check_tensor(dpre, "mean_grad dpre");
  check_tensor(w, "mean_grad w");
  check_tensor(dmean, "mean_grad dmean");
  if (w.cols != dpre.cols || dmean.rows != dpre.rows || dmean.cols != w.rows)
    throw std::invalid_argument("matmul_nt shape mismatch");
  if (dmean.rows == 0) return;
  DMeanBatch db{};
  db.np = 1;
  db.p[0] = {DpreView{dpre.data, nullptr, dpre.ld, dpre.cols, 1, 0}, w.data, w.ld, static_cast<int>(w.rows), indptr,
             dev_int(dpre.rows), static_cast<int>(dpre.rows), dmean.data, dmean.ld};
  dmean_umma(db, st_);
}

void LayerCtx::scatter_rows(const std::uint32_t* indptr, std::int64_t n_dst, std::int64_t n_edges,
                            const std::uint32_t* src_rows, const DevTensor& dmean, const DevTensor& dh_src) {
  check_tensor(dmean, "scatter dmean");
  check_tensor(dh_src, "scatter dh_src");
  if (dmean.rows != n_dst || dmean.cols != dh_src.cols || dmean.ld != dh_src.ld)
    throw std::invalid_argument("scatter: dmean must be [n_dst x cols of dh_src] with the same row stride");
  if (n_dst >= (1LL << 28)) throw std::invalid_argument("scatter: block too large");
  if (n_edges == 0 || dh_src.rows == 0) return;
  // transposed view of the block (source-major, each segment in edge order) and an
  // ordered gather-sum per source row: the scatter of hgnn.cpp:344-353, deterministic
  const std::int64_t n_src = dh_src.rows;
  auto* erow = static_cast<std::uint32_t*>(scratch(static_cast<std::size_t>(n_edges) * 4));
  auto* offs = static_cast<std::uint32_t*>(scratch(static_cast<std::size_t>(n_src + 1) * 4));
  auto* cursor = static_cast<std::uint32_t*>(scratch(static_cast<std::size_t>(n_src + 1) * 4));
  auto* entries = static_cast<std::uint32_t*>(scratch(static_cast<std::size_t>(n_edges) * 4));
  auto* sum = static_cast<float*>(scratch(static_cast<std::size_t>(n_src) * dh_src.ld * 4));
  k_edge_rows<<<grid_for(n_dst), 256, 0, st_>>>(indptr, n_dst, src_rows, erow, offs);
  HG_CUDA(cudaGetLastError());
  CscHop h{};
  h.nt = 1;
  CscType& t = h.t[0];
  t.offs = offs;
  t.cursor = cursor;
  t.entries = entries;
  t.tmp = static_cast<std::uint32_t*>(scratch(static_cast<std::size_t>(n_edges) * 4));
  t.n_src = dev_int(n_src);
  t.src_cap = static_cast<int>(n_src);
  t.dh = sum;
  t.ld_dh = dh_src.ld;
  t.din = dh_src.cols;
  h.nb = 1;
  CscEdges& b = h.b[0];
  b.col = src_rows;
  b.erow = erow;
  b.indptr = indptr;
  b.n_rows = dev_int(n_dst);
  b.cap = static_cast<int>(n_edges);
  b.edge_base = 0;
  b.type = 0;
  b.dmean = dmean.data;
  b.ld_dmean = dmean.ld;
  LbScratch lb;
  lb.cap = static_cast<int>(ceil_div(static_cast<std::uint64_t>(n_src), kScanTile)) + 1;
  lb.mem = static_cast<unsigned long long*>(scratch((static_cast<std::size_t>(lb.cap) + 1) * 8));
  csc_prepare(h, lb, st_);
  csc_gather(h, AdamHyper{}, err_, st_);
  add(dh_src, DevTensor{sum, dh_src.rows, dh_src.cols, dh_src.ld});
}

void LayerCtx::adam_dense(float* w, float* m, float* v, const float* g, std::int64_t n, std::int64_t step,
                          const AdamHyper& hp) {
  if (n <= 0) return;
  if (step < 1) throw std::invalid_argument("adam: step must be >= 1");
  k_adam_dense<<<grid_for(n), 256, 0, st_>>>(w, m, v, g, n, hp, static_cast<double>(step), err_);
  HG_CUDA(cudaGetLastError());
}

void LayerCtx::adam_rows(const DevTensor& w, const DevTensor& m, const DevTensor& v, const std::uint32_t* rows,
                         std::int64_t n, const DevTensor& grads, std::int64_t step, const AdamHyper& hp) {
  if (n <= 0) return;
  if (step < 1) throw std::invalid_argument("adam: step must be >= 1");
  if (grads.rows != n || grads.cols != w.cols || m.ld != w.ld || v.ld != w.ld)
    throw std::invalid_argument("adam_update_rows: gradient rows must be [n x dim]");
  k_adam_rows<<<grid_for(n * w.cols), 256, 0, st_>>>(w.data, m.data, v.data, w.ld, w.rows, rows, n, grads.data,
                                                     grads.ld, w.cols, hp, static_cast<double>(step), err_);
  HG_CUDA(cudaGetLastError());
}

}  // namespace hetgpu
