// Floating-point work of the hot path (fp32 storage, fp32 accumulate):
// relation-first mean aggregation fused with the per-relation projection and
// the AGG_all sum over relations (hgnn.cpp:173-203, 215-279), the softmax
// cross-entropy (hgnn.cpp:281-307), the backward pass (hgnn.cpp:309-362) with a
// deterministic transposed gather instead of the scatter, and Adam
// (hgnn.cpp:364-410). This file is the portable SIMT path: any dims, any
// shape. (The tcgen05 projection lives in umma_kernels.cu.)
#include <cfloat>

#include "kernels.cuh"

namespace hetgpu {

namespace {

constexpr int kThreads = 256;
constexpr int kTM = 32;        // rows per tile
constexpr int kKC = 128;       // staged K chunk (columns of the mean)
constexpr int kAPad = kTM + 4; // padded row length of the transposed A tile

// acc[8][NJ] += At[k][rg*8 + 0..7] * B[k][col + 64*j] over k in [0, K)
template <int NJ>
__device__ __forceinline__ void tile_fma(const float* __restrict__ At, int K, const float* __restrict__ B,
                                         int ldb, int N, int col, int rg, float (&acc)[8][NJ]) {
  for (int k = 0; k < K; ++k) {
    const float4 a0 = *reinterpret_cast<const float4*>(At + k * kAPad + rg * 8);
    const float4 a1 = *reinterpret_cast<const float4*>(At + k * kAPad + rg * 8 + 4);
    const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    const float* brow = B + static_cast<std::size_t>(k) * ldb;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int c = col + 64 * j;
      const float b = c < N ? __ldg(brow + c) : 0.0f;
#pragma unroll
      for (int r = 0; r < 8; ++r) acc[r][j] = fmaf(a[r], b, acc[r][j]);
    }
  }
}

// Mean over the sampled neighbours of kTM block rows, K columns [c0, c0+kKC),
// into the transposed smem tile At[k][row] and the tape.
__device__ __forceinline__ void gather_mean_tile(const AggRel& r, int row0, int n, int c0, float* At) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ncol = min(kKC, r.din - c0);
  for (int rr = warp; rr < kTM; rr += kThreads / 32) {
    const int i = row0 + rr;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    const int c = c0 + 4 * lane;
    if (i < n) {
      const std::uint32_t lo = r.indptr[i], hi = r.indptr[i + 1];
      if (4 * lane < ncol) {
        const std::uint32_t* keys = r.by_id ? r.src : r.col;
        std::uint32_t e = lo;
        // 4 independent row reads in flight per lane
        for (; e + 4 <= hi; e += 4) {
          float4 v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            v[q] = __ldg(reinterpret_cast<const float4*>(r.h + static_cast<std::size_t>(keys[e + q]) * r.ld_h + c));
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            s.x += v[q].x;
            s.y += v[q].y;
            s.z += v[q].z;
            s.w += v[q].w;
          }
        }
        for (; e < hi; ++e) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(r.h + static_cast<std::size_t>(keys[e]) * r.ld_h + c));
          s.x += v.x;
          s.y += v.y;
          s.z += v.z;
          s.w += v.w;
        }
        if (hi > lo) {
          const float inv = 1.0f / static_cast<float>(hi - lo);
          s.x *= inv;
          s.y *= inv;
          s.z *= inv;
          s.w *= inv;
        }
        // padded columns of the source rows are zero, so s is zero past din
        *reinterpret_cast<float4*>(r.mean + static_cast<std::size_t>(i) * r.ld_mean + c) = s;
      }
    }
    const int kc = 4 * lane;
    if (kc < kKC) {
      At[(kc + 0) * kAPad + rr] = s.x;
      At[(kc + 1) * kAPad + rr] = s.y;
      At[(kc + 2) * kAPad + rr] = s.z;
      At[(kc + 3) * kAPad + rr] = s.w;
    }
  }
}

template <int NJ>
__global__ void __launch_bounds__(kThreads) k_aggregate_project(AggGroup g) {
  __shared__ __align__(16) float At[kKC * kAPad];
  const int n = *g.n_rows;
  const int tid = threadIdx.x;
  const int col = tid & 63, rg = tid >> 6;
  for (int row0 = blockIdx.x * kTM; row0 < n; row0 += gridDim.x * kTM) {
    float acc[8][NJ];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[r][j] = 0.f;
    for (int q = 0; q < g.nrel; ++q) {
      const AggRel& r = g.r[q];
      for (int c0 = 0; c0 < r.din; c0 += kKC) {
        __syncthreads();
        gather_mean_tile(r, row0, n, c0, At);
        __syncthreads();
        tile_fma<NJ>(At, min(kKC, r.din - c0), r.w + static_cast<std::size_t>(c0) * r.ld_w, r.ld_w, g.dout,
                     col, rg, acc);
      }
    }
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      const int i = row0 + rg * 8 + rr;
      if (i >= n) break;
      float* orow = g.out + static_cast<std::size_t>(i * g.out_stride + g.out_offset) * g.ld_out;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int c = col + 64 * j;
        if (c < g.dout) orow[c] = g.relu ? fmaxf(acc[rr][j], 0.f) : acc[rr][j];
      }
    }
  }
}

}  // namespace

void aggregate_project(const AggGroup& g, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::max<std::uint64_t>(
      1, std::min<std::uint64_t>(ceil_div(g.rows_cap, kTM), 8 * kNumSMs)));
  const int nj = static_cast<int>(ceil_div(g.dout, 64));
  switch (nj) {
    case 1: k_aggregate_project<1><<<grid, kThreads, 0, st>>>(g); break;
    case 2: k_aggregate_project<2><<<grid, kThreads, 0, st>>>(g); break;
    case 3: k_aggregate_project<3><<<grid, kThreads, 0, st>>>(g); break;
    case 4: k_aggregate_project<4><<<grid, kThreads, 0, st>>>(g); break;
    case 5: k_aggregate_project<5><<<grid, kThreads, 0, st>>>(g); break;
    case 6: k_aggregate_project<6><<<grid, kThreads, 0, st>>>(g); break;
    case 7: k_aggregate_project<7><<<grid, kThreads, 0, st>>>(g); break;
    case 8: k_aggregate_project<8><<<grid, kThreads, 0, st>>>(g); break;
    default: throw std::invalid_argument("output dim above 512 is not supported");
  }
}

// ---- cross entropy ---------------------------------------------------------------------

namespace {

__global__ void __launch_bounds__(kThreads) k_cross_entropy(LossArgs a) {
  const int n = *a.n_rows;
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (kThreads / 32);
  const double invb = 1.0 / static_cast<double>(a.sc->batch_len);
  for (int i = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); i < n; i += warps) {
    const float* z = a.logits + static_cast<std::size_t>(i) * a.ld;
    float* dz = a.dlogits + static_cast<std::size_t>(i) * a.ld;
    const float m = a.mult[i];
    const std::int32_t y = a.labels[a.row_ids[i]];
    if (m == 0.0f) {
      for (int c = lane; c < a.C; c += 32) dz[c] = 0.f;
      if (lane == 0) a.row_loss[i] = 0.0;
      continue;
    }
    if (y < 0 || y >= a.C) {
      if (lane == 0) atomicOr(a.err, 2u);
      continue;
    }
    float zmax = -FLT_MAX;
    for (int c = lane; c < a.C; c += 32) zmax = fmaxf(zmax, z[c]);
    for (int o = 16; o > 0; o >>= 1) zmax = fmaxf(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
    double sum = 0.0;
    for (int c = lane; c < a.C; c += 32) sum += exp(static_cast<double>(z[c]) - zmax);
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const double lse = zmax + log(sum);
    const double scale = m * invb;
    for (int c = lane; c < a.C; c += 32)
      dz[c] = static_cast<float>((exp(static_cast<double>(z[c]) - lse) - (c == y ? 1.0 : 0.0)) * scale);
    if (lane == 0) a.row_loss[i] = (lse - static_cast<double>(z[y])) * scale;
  }
}

// ordered single-CTA reduction: fixed per-thread striding and a fixed tree
__global__ void __launch_bounds__(1024) k_sum_rows(const double* v, const int* n, double* out) {
  __shared__ double part[1024];
  double s = 0.0;
  for (int i = threadIdx.x; i < *n; i += 1024) s += v[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = part[0];
}

}  // namespace

void cross_entropy(const LossArgs& a, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::max<std::uint64_t>(
      1, std::min<std::uint64_t>(ceil_div(a.rows_cap, kThreads / 32), 4 * kNumSMs)));
  k_cross_entropy<<<grid, kThreads, 0, st>>>(a);
  k_sum_rows<<<1, 1024, 0, st>>>(a.row_loss, a.n_rows, a.loss_out);
}

// ---- backward ------------------------------------------------------------------------------

namespace {

__global__ void k_relu_mask(float* dh, const float* h, int ld, int cols, const int* n_rows, int stride,
                            int offset) {
  const int n = *n_rows;
  const std::size_t total = static_cast<std::size_t>(n) * cols;
  for (std::size_t x = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const std::size_t i = x / cols, c = x % cols;
    const std::size_t at = (i * stride + offset) * ld + c;
    if (h[i * ld + c] <= 0.0f) dh[at] = 0.0f;
  }
}

constexpr int kWChunk = 256;  // rows per dW partial

// partial[chunk][i][j] = sum_{rows of chunk} mean[r][i] * dpre[r][j]
template <int NJ>
__global__ void __launch_bounds__(kThreads) k_wgrad_partial(WGradArgs a) {
  __shared__ __align__(16) float At[kKC * kAPad];
  const int n = *a.n_rows;
  const int chunk = blockIdx.x;
  const int r0 = chunk * kWChunk;
  if (r0 >= n) return;
  const int r1 = min(n, r0 + kWChunk);
  const int tid = threadIdx.x, col = tid & 63, rg = tid >> 6;
  // output tile: i in [i0, i0 + 32) (blockIdx.y), all j
  const int i0 = blockIdx.y * kTM;
  float acc[8][NJ];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[r][j] = 0.f;
  for (int k0 = r0; k0 < r1; k0 += kKC) {
    const int kn = min(kKC, r1 - k0);
    __syncthreads();
    // At[k][m] = mean[k0 + k][i0 + m]
    for (int x = tid; x < kKC * kTM; x += kThreads) {
      const int k = x / kTM, m = x % kTM;
      const int i = i0 + m;
      At[k * kAPad + m] = (k < kn && i < a.din) ? a.mean[static_cast<std::size_t>(k0 + k) * a.ld_mean + i] : 0.f;
    }
    __syncthreads();
    tile_fma<NJ>(At, kn, a.dpre + static_cast<std::size_t>(k0 * a.dpre_stride + a.dpre_offset) * a.ld_dpre,
                 a.ld_dpre * a.dpre_stride, a.dout, col, rg, acc);
  }
  float* p = a.partial + static_cast<std::size_t>(chunk) * a.din * a.dout;
#pragma unroll
  for (int rr = 0; rr < 8; ++rr) {
    const int i = i0 + rg * 8 + rr;
    if (i >= a.din) break;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int c = col + 64 * j;
      if (c < a.dout) p[static_cast<std::size_t>(i) * a.dout + c] = acc[rr][j];
    }
  }
}

__global__ void k_wgrad_reduce(WGradArgs a) {
  const int n = *a.n_rows;
  const int chunks = (n + kWChunk - 1) / kWChunk;
  const int total = a.din * a.dout;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < chunks; ++c) s += a.partial[static_cast<std::size_t>(c) * total + x];
    a.dw[static_cast<std::size_t>(x / a.dout) * a.ld_dw + x % a.dout] += s;
  }
}

// dmean[r][c0+i] = sum_j dpre[r][j] * W[c0+i][j] / deg(r): At holds dpre^T for
// 32 rows; wt is W^T ([dout x din], ld ldt)
template <int NJ>
__global__ void __launch_bounds__(kThreads) k_mean_grad(DMeanArgs a, const float* wt, int ldt, int c0,
                                                        int ncols) {
  __shared__ __align__(16) float At[kKC * kAPad];
  const int n = *a.n_rows;
  const int tid = threadIdx.x, col = tid & 63, rg = tid >> 6;
  for (int row0 = blockIdx.x * kTM; row0 < n; row0 += gridDim.x * kTM) {
    float acc[8][NJ];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[r][j] = 0.f;
    for (int k0 = 0; k0 < a.dout; k0 += kKC) {
      const int kn = min(kKC, a.dout - k0);
      __syncthreads();
      for (int x = tid; x < kKC * kTM; x += kThreads) {
        const int m = x / kKC, k = x % kKC;  // k fastest: coalesced reads of a dpre row
        const int i = row0 + m;
        At[k * kAPad + m] = (k < kn && i < n)
                                ? a.dpre[static_cast<std::size_t>(i * a.dpre_stride + a.dpre_offset) * a.ld_dpre + k0 + k]
                                : 0.f;
      }
      __syncthreads();
      tile_fma<NJ>(At, kn, wt + static_cast<std::size_t>(k0) * ldt + c0, ldt, ncols, col, rg, acc);
    }
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      const int i = row0 + rg * 8 + rr;
      if (i >= n) break;
      const std::uint32_t deg = a.indptr[i + 1] - a.indptr[i];
      const float inv = deg ? 1.0f / static_cast<float>(deg) : 0.0f;
      float* orow = a.dmean + static_cast<std::size_t>(i) * a.ld_dmean + c0;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int c = col + 64 * j;
        if (c < ncols) orow[c] = acc[rr][j] * inv;
      }
    }
  }
}

__global__ void k_transpose(const float* w, int rows, int cols, int ldw, float* wt, int ldt) {
  const int total = rows * cols;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += gridDim.x * blockDim.x) {
    const int i = x / cols, j = x % cols;
    wt[static_cast<std::size_t>(j) * ldt + i] = w[static_cast<std::size_t>(i) * ldw + j];
  }
}

}  // namespace

void relu_mask(float* dh, const float* h, int ld, int cols, const int* n_rows, int rows_cap, int in_stride,
               int in_offset, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::max<std::uint64_t>(
      1, std::min<std::uint64_t>(ceil_div(static_cast<std::uint64_t>(rows_cap) * cols, 256), 4 * kNumSMs)));
  k_relu_mask<<<grid, 256, 0, st>>>(dh, h, ld, cols, n_rows, in_stride, in_offset);
}

void weight_grad(const WGradArgs& a, cudaStream_t st) {
  const int chunks = static_cast<int>(std::max<std::uint64_t>(1, ceil_div(a.rows_cap, kWChunk)));
  dim3 grid(chunks, static_cast<unsigned>(ceil_div(a.din, kTM)));
  const int nj = static_cast<int>(ceil_div(a.dout, 64));
  switch (nj) {
    case 1: k_wgrad_partial<1><<<grid, kThreads, 0, st>>>(a); break;
    case 2: k_wgrad_partial<2><<<grid, kThreads, 0, st>>>(a); break;
    case 3: k_wgrad_partial<3><<<grid, kThreads, 0, st>>>(a); break;
    case 4: k_wgrad_partial<4><<<grid, kThreads, 0, st>>>(a); break;
    case 5: k_wgrad_partial<5><<<grid, kThreads, 0, st>>>(a); break;
    case 6: k_wgrad_partial<6><<<grid, kThreads, 0, st>>>(a); break;
    case 7: k_wgrad_partial<7><<<grid, kThreads, 0, st>>>(a); break;
    case 8: k_wgrad_partial<8><<<grid, kThreads, 0, st>>>(a); break;
    default: throw std::invalid_argument("output dim above 512 is not supported");
  }
  const unsigned g2 = static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(
                                                                          ceil_div(a.din * a.dout, 256), 2 * kNumSMs)));
  k_wgrad_reduce<<<g2, 256, 0, st>>>(a);
}

void mean_grad(const DMeanArgs& a, float* wt_scratch, cudaStream_t st) {
  const int ldt = round_up4(a.din);
  const unsigned gt = static_cast<unsigned>(std::max<std::uint64_t>(1, ceil_div(a.din * a.dout, 256)));
  k_transpose<<<std::min(gt, 1024u), 256, 0, st>>>(a.w, a.din, a.dout, a.ld_w, wt_scratch, ldt);
  const unsigned grid = static_cast<unsigned>(std::max<std::uint64_t>(
      1, std::min<std::uint64_t>(ceil_div(a.rows_cap, kTM), 8 * kNumSMs)));
  // up to 512 input columns per launch (wide features take several)
  for (int c0 = 0; c0 < a.din; c0 += 512) {
    const int ncols = std::min(512, a.din - c0);
    switch (static_cast<int>(ceil_div(ncols, 64))) {
      case 1: k_mean_grad<1><<<grid, kThreads, 0, st>>>(a, wt_scratch, ldt, c0, ncols); break;
      case 2: k_mean_grad<2><<<grid, kThreads, 0, st>>>(a, wt_scratch, ldt, c0, ncols); break;
      case 3: k_mean_grad<3><<<grid, kThreads, 0, st>>>(a, wt_scratch, ldt, c0, ncols); break;
      case 4: k_mean_grad<4><<<grid, kThreads, 0, st>>>(a, wt_scratch, ldt, c0, ncols); break;
      case 5: k_mean_grad<5><<<grid, kThreads, 0, st>>>(a, wt_scratch, ldt, c0, ncols); break;
      case 6: k_mean_grad<6><<<grid, kThreads, 0, st>>>(a, wt_scratch, ldt, c0, ncols); break;
      case 7: k_mean_grad<7><<<grid, kThreads, 0, st>>>(a, wt_scratch, ldt, c0, ncols); break;
      default: k_mean_grad<8><<<grid, kThreads, 0, st>>>(a, wt_scratch, ldt, c0, ncols); break;
    }
  }
}

// ---- transposed gather for the backward scatter ------------------------------------------------

namespace {

__global__ void k_csc_count(CscArgs a) {
  const CscBlock& b = a.b[blockIdx.y];
  const std::uint32_t total = b.indptr[*b.n_rows];
  for (std::uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x)
    atomicAdd(a.offs + b.col[e], 1u);
}

__global__ void k_csc_fill(CscArgs a) {
  const CscBlock& b = a.b[blockIdx.y];
  const std::uint32_t total = b.indptr[*b.n_rows];
  for (std::uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const std::uint32_t c = b.col[e];
    const std::uint32_t pos = atomicAdd(a.cursor + c, 1u);
    a.entries[a.offs[c] - 1 - pos] = static_cast<std::uint32_t>(b.edge_base) + e;
  }
}

// make every segment ascending in (block, edge): deterministic summation order
__global__ void k_csc_sort(CscArgs a) {
  const int n = *a.n_src;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const std::uint32_t lo = c ? a.offs[c - 1] : 0u, hi = a.offs[c];
    for (std::uint32_t x = lo + 1; x < hi; ++x) {
      const std::uint32_t v = a.entries[x];
      std::uint32_t y = x;
      while (y > lo && a.entries[y - 1] > v) {
        a.entries[y] = a.entries[y - 1];
        --y;
      }
      a.entries[y] = v;
    }
  }
}

// one warp per source row: dh[c] = sum over its sampled edges of dmean[row(e)]
__global__ void __launch_bounds__(256) k_csc_gather(CscArgs a) {
  const int n = *a.n_src;
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x / 32);
  for (int c = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); c < n; c += warps) {
    const std::uint32_t lo = c ? a.offs[c - 1] : 0u, hi = a.offs[c];
    for (int c0 = 0; c0 < a.din; c0 += 128) {
      const int f = c0 + 4 * lane;
      if (f >= round_up4(a.din)) continue;
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
      for (std::uint32_t x = lo; x < hi; ++x) {
        const std::uint32_t id = a.entries[x];
        int bi = 0;
        while (bi + 1 < a.nblk && id >= static_cast<std::uint32_t>(a.b[bi + 1].edge_base)) ++bi;
        const CscBlock& b = a.b[bi];
        const std::uint32_t row = b.erow[id - b.edge_base];
        const float4 v = *reinterpret_cast<const float4*>(b.dmean + static_cast<std::size_t>(row) * b.ld_dmean + f);
        s.x += v.x;
        s.y += v.y;
        s.z += v.z;
        s.w += v.w;
      }
      *reinterpret_cast<float4*>(a.dh + static_cast<std::size_t>(c) * a.ld_dh + f) = s;
    }
  }
}

}  // namespace

void csc_build(const CscArgs& a, std::uint32_t* partials, cudaStream_t st) {
  HG_CUDA(cudaMemsetAsync(a.offs, 0, sizeof(std::uint32_t) * (a.src_cap + 1), st));
  HG_CUDA(cudaMemsetAsync(a.cursor, 0, sizeof(std::uint32_t) * (a.src_cap + 1), st));
  int cap = 1;
  for (int i = 0; i < a.nblk; ++i) cap = std::max(cap, a.b[i].cap);
  dim3 grid(static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(cap, 256), 4 * kNumSMs)), a.nblk);
  k_csc_count<<<grid, 256, 0, st>>>(a);
  ScanArgs sa{};
  sa.nseg = 1;
  sa.s[0] = {a.offs, a.n_src, a.src_cap};
  scan_inclusive(sa, partials, st);
  k_csc_fill<<<grid, 256, 0, st>>>(a);
  const unsigned g2 = static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(
                                                                          ceil_div(a.src_cap, 256), 4 * kNumSMs)));
  k_csc_sort<<<g2, 256, 0, st>>>(a);
}

void csc_gather(const CscArgs& a, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::max<std::uint64_t>(
      1, std::min<std::uint64_t>(ceil_div(a.src_cap, 8), 8 * kNumSMs)));
  k_csc_gather<<<grid, 256, 0, st>>>(a);
}

// ---- Adam ---------------------------------------------------------------------------------------

namespace {

__device__ __forceinline__ void adam_elem(float& w, float& m, float& v, float g, double bc1, double bc2,
                                          const AdamHyper& hp, std::uint32_t* err) {
  if (!isfinite(g)) {
    atomicOr(err, 4u);
    return;
  }
  // moments and update in f64 like the reference (hgnn.cpp:364-377); fp32 storage
  const double md = hp.beta1 * m + (1.0 - hp.beta1) * g;
  const double vd = hp.beta2 * v + (1.0 - hp.beta2) * static_cast<double>(g) * g;
  m = static_cast<float>(md);
  v = static_cast<float>(vd);
  w = static_cast<float>(w - hp.lr * (md / bc1) / (sqrt(vd / bc2) + hp.eps));
}

__global__ void k_adam_dense(float* w, float* m, float* v, const float* g, int rows, int cols, int ld,
                             const std::int64_t* step, AdamHyper hp, std::uint32_t* err) {
  const double t = static_cast<double>(*step);
  const double bc1 = 1.0 - pow(hp.beta1, t), bc2 = 1.0 - pow(hp.beta2, t);
  const int total = rows * cols;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += gridDim.x * blockDim.x) {
    const std::size_t at = static_cast<std::size_t>(x / cols) * ld + x % cols;
    adam_elem(w[at], m[at], v[at], g[at], bc1, bc2, hp, err);
  }
}

__global__ void k_bump_step(const int* n_rows, std::int64_t* step) {
  if (*n_rows > 0) ++*step;
}

__global__ void k_adam_rows(float* w, float* m, float* v, int ld, int cols, const std::uint32_t* ids,
                            const float* g, int ld_g, const int* n_rows, const std::int64_t* step, AdamHyper hp,
                            std::uint32_t* err) {
  const int n = *n_rows;
  const double t = static_cast<double>(*step);
  const double bc1 = 1.0 - pow(hp.beta1, t), bc2 = 1.0 - pow(hp.beta2, t);
  const std::size_t total = static_cast<std::size_t>(n) * cols;
  for (std::size_t x = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const std::size_t i = x / cols, c = x % cols;
    const std::size_t at = static_cast<std::size_t>(ids[i]) * ld + c;
    adam_elem(w[at], m[at], v[at], g[i * ld_g + c], bc1, bc2, hp, err);
  }
}

__global__ void k_zero_rows(float* p, int ld, const int* n_rows) {
  const std::size_t total = static_cast<std::size_t>(*n_rows) * ld;
  for (std::size_t x = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<std::size_t>(gridDim.x) * blockDim.x)
    p[x] = 0.f;
}

}  // namespace

void adam_dense(float* w, float* m, float* v, const float* g, int rows, int cols, int ld, const std::int64_t* step,
                AdamHyper hp, std::uint32_t* err, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(
                                                                            ceil_div(rows * cols, 256), 2 * kNumSMs)));
  k_adam_dense<<<grid, 256, 0, st>>>(w, m, v, g, rows, cols, ld, step, hp, err);
}

void adam_rows(float* w, float* m, float* v, int ld, int cols, const std::uint32_t* ids, const float* g, int ld_g,
               const int* n_rows, int rows_cap, std::int64_t* step, AdamHyper hp, std::uint32_t* err,
               cudaStream_t st) {
  k_bump_step<<<1, 1, 0, st>>>(n_rows, step);
  const unsigned grid = static_cast<unsigned>(std::max<std::uint64_t>(
      1, std::min<std::uint64_t>(ceil_div(static_cast<std::uint64_t>(rows_cap) * cols, 256), 4 * kNumSMs)));
  k_adam_rows<<<grid, 256, 0, st>>>(w, m, v, ld, cols, ids, g, ld_g, n_rows, step, hp, err);
}

void zero_rows(float* p, int ld, const int* n_rows, int rows_cap, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::max<std::uint64_t>(
      1, std::min<std::uint64_t>(ceil_div(static_cast<std::uint64_t>(rows_cap) * ld, 256), 4 * kNumSMs)));
  k_zero_rows<<<grid, 256, 0, st>>>(p, ld, n_rows);
}

}  // namespace hetgpu
