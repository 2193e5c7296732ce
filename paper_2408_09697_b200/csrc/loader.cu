// Streaming HGC1 loader (the reference's load_container,
// container.cpp:92-154, builds a host HetGraph first). Here the file goes straight
// into HBM: every relation's dst-major (src, dst) u32 pairs are read in 64 MB chunks
// into two pinned buffers, copied asynchronously and split on the device into the
// CSR source array (file order = the reference's insertion order) and the offsets
// (destinations ascend, so every offset is the index of its row's first edge: written
// once, no atomics; the host keeps a copy for the plan's degree statistics). Dense feature rows stream the same way and
// are converted on the device to the table's storage type (f32 / f16 / bf16, padded
// rows). The disk read of chunk i+1 overlaps the copy and split of chunk i. Range
// and ordering checks run on the device and raise the host path's exceptions.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>

#include "engine.hpp"
#include "gemm.cuh"

namespace hetgpu {

namespace {

constexpr std::size_t kChunkBytes = 64u << 20;

// pairs[i] = (src, dst), dst-major: sources[e0 + i] = src, and since destinations ascend,
// offsets[d] = e0 + i for every d in (dst of the previous edge, dst] (no atomics: each
// offset is written once). flags: 1 = endpoint out of range, 2 = destinations descend.
// prev_dst = the relation's previous edge's destination, or -1 before its first edge.
__global__ void k_split_pairs(const uint2* pairs, std::uint32_t n, std::uint64_t e0, std::int64_t prev_dst,
                              std::uint32_t* sources, std::uint64_t* offsets, std::uint64_t n_src,
                              std::uint64_t n_dst, std::uint32_t* err) {
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint2 p = pairs[i];
    if (p.x >= n_src || p.y >= n_dst) {
      atomicOr(err, 1u);
      continue;
    }
    sources[e0 + i] = p.x;
    const std::int64_t prev = i ? static_cast<std::int64_t>(pairs[i - 1].y) : prev_dst;
    if (static_cast<std::int64_t>(p.y) < prev) {
      atomicOr(err, 2u);
      continue;
    }
    for (std::int64_t d = prev + 1; d <= static_cast<std::int64_t>(p.y); ++d) offsets[d] = e0 + i;
  }
}

// offsets[d] = E for every destination after the last edge's
__global__ void k_offsets_tail(std::uint64_t* offsets, std::int64_t from, std::uint64_t n_dst, std::uint64_t E) {
  for (std::uint64_t d = from + blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; d <= n_dst;
       d += static_cast<std::uint64_t>(gridDim.x) * blockDim.x)
    offsets[d] = E;
}

// f32 rows [n x dim] -> table rows of ld elements of `dtype` (zero padding)
__global__ void k_rows_convert(const float* src, std::uint64_t n, int dim, void* dst, int ld, int dtype) {
  const std::uint64_t total = n * static_cast<std::uint64_t>(ld);
  for (std::uint64_t x = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
    const std::uint64_t i = x / ld;
    const int c = static_cast<int>(x % ld);
    const float v = c < dim ? src[i * dim + c] : 0.f;
    if (dtype == kF32)
      static_cast<float*>(dst)[x] = v;
    else if (dtype == kF16)
      static_cast<__half*>(dst)[x] = __float2half_rn(v);
    else
      static_cast<__nv_bfloat16*>(dst)[x] = __float2bfloat16_rn(v);
  }
}

struct File {
  std::FILE* f = nullptr;
  explicit File(const std::string& path) : f(std::fopen(path.c_str(), "rb")) {
    if (!f) throw std::runtime_error("cannot open: " + path);
  }
  ~File() {
    if (f) std::fclose(f);
  }
  void seek(std::uint64_t at) {
    if (fseeko(f, static_cast<off_t>(at), SEEK_SET) != 0) throw std::runtime_error("container truncated");
  }
  void read(void* p, std::size_t bytes) {
    if (std::fread(p, 1, bytes, f) != bytes) throw std::runtime_error("container truncated");
  }
};

// two pinned host buffers + two device staging buffers, reused round robin; a buffer is
// refilled only after the copy (and kernel) that consumed it has finished
struct Stage {
  void* host[2] = {};
  void* dev[2] = {};
  cudaEvent_t done[2] = {};
  bool used[2] = {};
  explicit Stage(std::size_t bytes) {
    for (int b = 0; b < 2; ++b) {
      HG_CUDA(cudaMallocHost(&host[b], bytes));
      HG_CUDA(cudaMalloc(&dev[b], bytes));
      HG_CUDA(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
    }
  }
  ~Stage() {
    for (int b = 0; b < 2; ++b) {
      if (used[b]) cudaEventSynchronize(done[b]);
      cudaFreeHost(host[b]);
      cudaFree(dev[b]);
      cudaEventDestroy(done[b]);
    }
  }
  void* acquire(int b) {
    if (used[b]) HG_CUDA(cudaEventSynchronize(done[b]));
    used[b] = true;
    return host[b];
  }
};

unsigned grid_for(std::uint64_t items) {
  return static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(ceil_div(items, 256), 8 * num_sms())));
}

}  // namespace

Engine::Engine(const std::string& container_path, const EngineOptions& o) : o_(o) {
  const bool trace = std::getenv("HG_LOAD_TRACE") != nullptr;  // phase times on stderr
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!trace) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "loader %s %.3f s\n", what, std::chrono::duration<double>(t1 - t0).count());
    t0 = t1;
  };
  ContainerLayout lay = container_layout(container_path);
  lap("header");
  try {
    init_streams();
    lap("streams");
    stream_csr(lay, container_path);
    lap("csr");
    lay_ = &lay;
    lay_path_ = container_path;
    init_graph(lay.meta);
    lay_ = nullptr;
    lap("plan+tables");
  } catch (...) {  // a malformed file: release what was built
    lay_ = nullptr;
    release();
    throw;
  }
}

void Engine::stream_csr(ContainerLayout& lay, const std::string& path) {
  Graph& g = lay.meta;
  File file(path);
  const std::size_t chunk = kChunkBytes / 8;  // pairs per chunk
  Stage st(kChunkBytes);
  std::uint32_t* d_err = nullptr;
  HG_CUDA(cudaMalloc(&d_err, 4));
  std::unique_ptr<std::uint32_t, decltype(&cudaFree)> err_guard(d_err, &cudaFree);
  pre_ptr_.assign(g.num_rels(), nullptr);
  pre_src_.assign(g.num_rels(), nullptr);
  int turn = 0;
  for (int r = 0; r < g.num_rels(); ++r) {
    RelationInfo& rel = g.rels[r];
    const std::uint64_t n_src = g.types[rel.src_type].count, n_dst = g.types[rel.dst_type].count;
    const std::uint64_t E = lay.rel_edges[r];
    if (E >= (1ULL << 32)) throw std::invalid_argument("relation with 2^32 or more edges");
    HG_CUDA(cudaMemsetAsync(d_err, 0, 4, st_));
    pre_src_[r] = static_cast<std::uint32_t*>(alloc(std::max<std::uint64_t>(1, E) * 4));
    pre_ptr_[r] = static_cast<std::uint64_t*>(alloc((n_dst + 1) * 8));
    file.seek(lay.rel_offset[r]);
    std::int64_t prev_dst = -1;
    for (std::uint64_t e0 = 0; e0 < E; e0 += chunk) {
      const int b = turn++ & 1;
      const std::uint32_t n = static_cast<std::uint32_t>(std::min<std::uint64_t>(chunk, E - e0));
      auto* h = static_cast<uint2*>(st.acquire(b));
      file.read(h, static_cast<std::size_t>(n) * 8);
      HG_CUDA(cudaMemcpyAsync(st.dev[b], h, static_cast<std::size_t>(n) * 8, cudaMemcpyHostToDevice, st_));
      launch_pdl(k_split_pairs, grid_for(n), 256, 0, st_, static_cast<const uint2*>(st.dev[b]), n, e0, prev_dst,
                 pre_src_[r], pre_ptr_[r], n_src, n_dst, d_err);
      HG_CUDA(cudaEventRecord(st.done[b], st_));
      prev_dst = std::max<std::int64_t>(prev_dst, h[n - 1].y);
    }
    const std::int64_t tail = std::min<std::int64_t>(prev_dst + 1, static_cast<std::int64_t>(n_dst) + 1);
    if (tail <= static_cast<std::int64_t>(n_dst))
      launch_pdl(k_offsets_tail, grid_for(n_dst + 1 - static_cast<std::uint64_t>(tail)), 256, 0, st_, pre_ptr_[r],
                 tail, n_dst, E);
    // the host keeps the offsets (the plan's degree statistics)
    std::uint32_t err = 0;
    auto& off = rel.adj.offsets;
    off.assign(n_dst + 1, 0);
    HG_CUDA(cudaMemcpyAsync(off.data(), pre_ptr_[r], (n_dst + 1) * 8, cudaMemcpyDeviceToHost, st_));
    HG_CUDA(cudaMemcpyAsync(&err, d_err, 4, cudaMemcpyDeviceToHost, st_));
    HG_CUDA(cudaStreamSynchronize(st_));
    if (err & 1u) throw std::invalid_argument("edge endpoint out of range in relation " + std::to_string(r));
    if (err & 2u) throw std::runtime_error("container relation " + std::to_string(r) + " is not in dst-major order");
    if (off[0] != 0 || off[n_dst] != E)
      throw std::runtime_error("container relation " + std::to_string(r) + ": edge count mismatch");
  }
}

// One dense feature table streamed from the container into its storage (HBM, or pinned
// host memory with feat_host), converted to f32 / f16 / bf16 rows of tb.ld elements
void Engine::stream_dense(const NodeTypeInfo& nt, int t, TypeTable& tb) {
  tb.dense = true;
  tb.dtype = o_.feat_dtype;
  if (tb.dtype < 0 || tb.dtype > 2) throw std::invalid_argument("feature dtype must be 0 (f32), 1 (f16) or 2 (bf16)");
  if (tb.dtype != kF32) tb.ld = (std::max(1, nt.dim) + 7) & ~7;
  const std::size_t rows = nt.count, esz = tb.dtype == kF32 ? 4 : 2, dim = static_cast<std::size_t>(nt.dim);
  const std::size_t bytes = std::max<std::size_t>(16, rows * tb.ld * esz);
  File file(lay_path_);
  file.seek(lay_->dense_offset[t]);
  const std::size_t chunk_rows = std::max<std::size_t>(1, kChunkBytes / std::max<std::size_t>(4, dim * 4));
  if (o_.feat_host) {  // pinned host table, converted on the host (no device copy)
    tb.host = true;
    HG_CUDA(cudaHostAlloc(&tb.host_mem, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    void* dev = nullptr;
    HG_CUDA(cudaHostGetDevicePointer(&dev, tb.host_mem, 0));
    tb.w = static_cast<float*>(dev);
    std::vector<float> buf(std::min(rows, chunk_rows) * dim);
    auto* out = static_cast<std::uint8_t*>(tb.host_mem);
    for (std::size_t r0 = 0; r0 < rows; r0 += chunk_rows) {
      const std::size_t n = std::min(chunk_rows, rows - r0);
      file.read(buf.data(), n * dim * 4);
      std::memset(out + r0 * tb.ld * esz, 0, n * tb.ld * esz);
      for (std::size_t i = 0; i < n; ++i) {
        const float* src = &buf[i * dim];
        if (tb.dtype == kF32) {
          std::memcpy(out + (r0 + i) * tb.ld * 4, src, dim * 4);
        } else {
          auto* o = reinterpret_cast<std::uint16_t*>(out + (r0 + i) * tb.ld * 2);
          for (std::size_t c = 0; c < dim; ++c) {
            if (tb.dtype == kF16) {
              const __half_raw h = __float2half_rn(src[c]);
              o[c] = h.x;
            } else {
              const __nv_bfloat16_raw h = __float2bfloat16_rn(src[c]);
              o[c] = h.x;
            }
          }
        }
      }
    }
    return;
  }
  tb.w = static_cast<float*>(alloc(bytes));
  Stage st(std::min(rows, chunk_rows) * dim * 4 + 16);
  int turn = 0;
  for (std::size_t r0 = 0; r0 < rows; r0 += chunk_rows) {
    const int b = turn++ & 1;
    const std::size_t n = std::min(chunk_rows, rows - r0);
    void* h = st.acquire(b);
    file.read(h, n * dim * 4);
    HG_CUDA(cudaMemcpyAsync(st.dev[b], h, n * dim * 4, cudaMemcpyHostToDevice, st_));
    launch_pdl(k_rows_convert, grid_for(n * tb.ld), 256, 0, st_, static_cast<const float*>(st.dev[b]),
               static_cast<std::uint64_t>(n), nt.dim, static_cast<void*>(reinterpret_cast<std::uint8_t*>(tb.w) + r0 * tb.ld * esz),
               tb.ld, tb.dtype);
    HG_CUDA(cudaEventRecord(st.done[b], st_));
  }
  HG_CUDA(cudaStreamSynchronize(st_));
}

}  // namespace hetgpu
