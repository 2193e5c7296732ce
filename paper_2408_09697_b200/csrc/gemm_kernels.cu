// SIMT fp32 tile kernels for the small dense contractions of the hot path:
// the fused gather-mean-project of every layer (hgnn.cpp:173-203), the
// backward weight gradient dW += mean^T . dpre (matrix.hpp:49-61) and the
// mean gradient dmean = dpre . W^T / deg (matrix.hpp:64-78, hgnn.cpp:344-353).
// One 64x64 output tile per CTA, 256 threads with a 4x4 register tile each,
// K staged through shared memory in 32-deep slabs. Several independent
// problems share one launch (tile ids are linearised over the problems).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "adam.cuh"
#include "gemm.cuh"

#ifndef HG_GATHER_WAVES
#define HG_GATHER_WAVES 24  // CTAs per SM of the gather grids (8 resident: three waves)
#endif

namespace hetgpu {

namespace {

constexpr int kT = 256;   // threads
constexpr int kTile = 64; // output tile (rows and cols)
constexpr int kKS = 32;   // K slab
constexpr int kLd = kTile + 4;

struct Acc {
  float v[4][4];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) v[i][j] = 0.f;
  }
};

// acc += As[k][ty*4..+4] (x) Bs[k][tx*4..+4] over k < kn
__device__ __forceinline__ void slab_fma(const float* As, const float* Bs, int kn, int ty, int tx, Acc& acc) {
#pragma unroll 8
  for (int k = 0; k < kn; ++k) {
    const float4 a = *reinterpret_cast<const float4*>(As + k * kLd + ty * 4);
    const float4 b = *reinterpret_cast<const float4*>(Bs + k * kLd + tx * 4);
    const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc.v[i][j] = fmaf(av[i], bv[j], acc.v[i][j]);
  }
}

__device__ __forceinline__ int find_problem(const int* tile_base, int np, int tile) {
  int p = 0;
  while (p + 1 < np && tile >= tile_base[p + 1]) ++p;
  return p;
}

// ---- dpre staging helpers (ReLU mask fused) -------------------------------------------------
__device__ __forceinline__ float4 load_dpre4(const DpreView& d, int row, int col) {
  const std::size_t at = static_cast<std::size_t>(row * d.stride + d.offset) * d.ld + col;
  float4 v = *reinterpret_cast<const float4*>(d.g + at);
  if (d.h) {  // dpre = dH * [H > 0] (hgnn.cpp:326-328); H in the group's own row space
    const float4 h = *reinterpret_cast<const float4*>(d.h + static_cast<std::size_t>(row) * d.ld + col);
    if (h.x <= 0.f) v.x = 0.f;
    if (h.y <= 0.f) v.y = 0.f;
    if (h.z <= 0.f) v.z = 0.f;
    if (h.w <= 0.f) v.w = 0.f;
  }
  return v;
}

// ---- backward: weight gradient partials --------------------------------------------------
// problem p: partial[chunk][i][j] = sum_{r in chunk} mean[r][i] * dpre[r][j]
__global__ void __launch_bounds__(kT) k_wgrad_tiles(WGradBatch b) {
  pdl_enter();
  __shared__ __align__(16) float As[kKS * kLd];
  __shared__ __align__(16) float Bs[kKS * kLd];
  const int p = find_problem(b.tile_base, b.np, blockIdx.x);
  const WGradProblem& P = b.p[p];
  const int t = blockIdx.x - b.tile_base[p];
  const int mt = (P.din + kTile - 1) / kTile, nt = (P.d.cols + kTile - 1) / kTile;
  const int chunk = t / (mt * nt), mi = (t / nt) % mt, ni = t % nt;
  const int n = *P.n_rows;
  const int r0 = chunk * kWChunkRows;
  if (r0 >= n) return;
  const int r1 = min(n, r0 + kWChunkRows);
  const int i0 = mi * kTile, j0 = ni * kTile;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  Acc acc;
  acc.zero();
  for (int k0 = r0; k0 < r1; k0 += kKS) {
    const int kn = min(kKS, r1 - k0);
    __syncthreads();
    for (int x = tid; x < kKS * kTile / 4; x += kT) {
      const int k = x / (kTile / 4), q = (x % (kTile / 4)) * 4;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), bb = a;
      if (k < kn) {
        if (i0 + q < P.din)
          a = *reinterpret_cast<const float4*>(P.mean + static_cast<std::size_t>(k0 + k) * P.ld_mean + i0 + q);
        if (j0 + q < P.d.cols) bb = load_dpre4(P.d, k0 + k, j0 + q);
      }
      *reinterpret_cast<float4*>(As + k * kLd + q) = a;
      *reinterpret_cast<float4*>(Bs + k * kLd + q) = bb;
    }
    __syncthreads();
    slab_fma(As, Bs, kn, ty, tx, acc);
  }
  float* out = P.partial + static_cast<std::size_t>(chunk) * P.din * P.d.cols;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = i0 + ty * 4 + i;
    if (row >= P.din) break;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = j0 + tx * 4 + j;
      if (c < P.d.cols) out[static_cast<std::size_t>(row) * P.d.cols + c] = acc.v[i][j];
    }
  }
}

// ordered sum of the chunk partials into dW (deterministic): one thread per
// output element of every problem, chunks summed in order, 8 loads in flight
__global__ void __launch_bounds__(256) k_wgrad_reduce(WGradBatch b, int total_out) {
  pdl_enter();
  __shared__ AdamStep ks;
  if (b.step) {
    if (threadIdx.x == 0) ks = adam_step_of(b.hp, static_cast<double>(*b.step));
    __syncthreads();
  }
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < total_out; x += gridDim.x * blockDim.x) {
    int p = 0, base = 0;
    while (p + 1 < b.np && x >= base + b.p[p].din * b.p[p].d.cols) {
      base += b.p[p].din * b.p[p].d.cols;
      ++p;
    }
    const WGradProblem& P = b.p[p];
    const int total = P.din * P.d.cols;
    const int o = x - base;
    const int chunks = (*P.n_rows + kWChunkRows - 1) / kWChunkRows;
    const float* src = P.partial + o;
    float s = 0.f;
    int c = 0;
    for (; c + 8 <= chunks; c += 8) {
      float v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = src[static_cast<std::size_t>(c + q) * total];
#pragma unroll
      for (int q = 0; q < 8; ++q) s += v[q];
    }
    for (; c < chunks; ++c) s += src[static_cast<std::size_t>(c) * total];
    // each slot's gradient is produced by exactly one problem: overwrite (no memset)
    const std::size_t at = static_cast<std::size_t>(o / P.d.cols) * P.ld_dw + o % P.d.cols;
    P.dw[at] = s;
    if (P.w) {  // adam_update_model for this element (hgnn.cpp:379-390)
      float w = P.w[at], m = P.m[at], v = P.v[at];
      adam1(w, m, v, s, ks, b.err);
      P.w[at] = w;
      P.m[at] = m;
      P.v[at] = v;
    }
  }
}

// ---- backward: mean gradient ---------------------------------------------------------------------
// dmean[r][c] = (sum_j dpre[r][j] * W[c][j]) / deg(r)
__global__ void __launch_bounds__(kT) k_dmean_tiles(DMeanBatch b) {
  pdl_enter();
  __shared__ __align__(16) float As[kKS * kLd];
  __shared__ __align__(16) float Bs[kKS * kLd];
  const int p = find_problem(b.tile_base, b.np, blockIdx.x);
  const DMeanProblem& P = b.p[p];
  const int t = blockIdx.x - b.tile_base[p];
  const int nt = (P.din + kTile - 1) / kTile;
  const int rb = t / nt, cb = t % nt;
  const int n = *P.n_rows;
  const int row0 = rb * kTile, col0 = cb * kTile;
  if (row0 >= n) return;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  Acc acc;
  acc.zero();
  const int K = P.d.cols;
  for (int k0 = 0; k0 < K; k0 += kKS) {
    const int kn = min(kKS, K - k0);
    __syncthreads();
    // As[k][m] = dpre[row0+m][k0+k]; Bs[k][c] = W[col0+c][k0+k] (both transposed on the way in)
    for (int x = tid; x < kTile * kKS / 4; x += kT) {
      const int m = x / (kKS / 4), kq = (x % (kKS / 4)) * 4;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), w = a;
      if (row0 + m < n && k0 + kq < K) a = load_dpre4(P.d, row0 + m, k0 + kq);
      if (col0 + m < P.din && k0 + kq < K)
        w = *reinterpret_cast<const float4*>(P.w + static_cast<std::size_t>(col0 + m) * P.ld_w + k0 + kq);
      As[(kq + 0) * kLd + m] = a.x;
      As[(kq + 1) * kLd + m] = a.y;
      As[(kq + 2) * kLd + m] = a.z;
      As[(kq + 3) * kLd + m] = a.w;
      Bs[(kq + 0) * kLd + m] = w.x;
      Bs[(kq + 1) * kLd + m] = w.y;
      Bs[(kq + 2) * kLd + m] = w.z;
      Bs[(kq + 3) * kLd + m] = w.w;
    }
    __syncthreads();
    slab_fma(As, Bs, kn, ty, tx, acc);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = row0 + ty * 4 + i;
    if (row >= n) break;
    const std::uint32_t deg = P.indptr[row + 1] - P.indptr[row];
    const float inv = deg ? 1.0f / static_cast<float>(deg) : 0.0f;
    const int c = col0 + tx * 4;
    if (c < P.din) {
      float4 o = make_float4(acc.v[i][0] * inv, acc.v[i][1] * inv, acc.v[i][2] * inv, acc.v[i][3] * inv);
      *reinterpret_cast<float4*>(P.dmean + static_cast<std::size_t>(row) * P.ld_dmean + c) = o;
    }
  }
}

// ---- gather-mean: 16 lanes x float4 per (row, 64-column chunk); a warp carries
// two such items, kGatherBatch edges in flight per lane ----------------------------------------
#ifndef HG_GATHER_BATCH
#define HG_GATHER_BATCH 5
#endif
constexpr int kGatherBatch = HG_GATHER_BATCH;  // neighbour rows in flight per lane
#ifndef HG_GATHER_BATCH_WIDE
#define HG_GATHER_BATCH_WIDE 5  // half tables in HBM
#endif
#ifndef HG_GATHER_BATCH_SMALL
#define HG_GATHER_BATCH_SMALL 13  // small launches: fanout 25 in two round trips
#endif
// 4 consecutive fp32 features (columns c..c+3) of row `key` (one 16-byte load); a
// cached host table reads the HBM copy when the row is cached
#ifndef HG_GATHER_L2HINT
#define HG_GATHER_L2HINT 1  // measured: aggregate 50.7 -> 49.4 us/step (the backward gather gets slower: not used there)
#endif
// a feature-row float4 that no other lane reads again: read-only path, no L1 allocation,
// L2 fetch in 256-byte blocks (a half-warp reads 256 contiguous bytes of the row)
__device__ __forceinline__ float4 ld_row_stream(const float* p) {
#if HG_GATHER_L2HINT
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
#else
  return __ldg(reinterpret_cast<const float4*>(p));
#endif
}

__device__ __forceinline__ float4 load_row4(const MeanBlock& B, std::uint32_t key, int c) {
  const float* base = B.h;
  std::size_t row = key;
  if (B.slot) {
    const int sl = __ldg(B.slot + key);
    if (sl >= 0) {
      base = B.cache;
      row = static_cast<std::size_t>(sl);
    }
  }
  return __ldg(reinterpret_cast<const float4*>(base + row * B.ld_h + c));
}

#ifndef HG_WIDE_NOALLOC
#define HG_WIDE_NOALLOC 0
#endif
#ifndef HG_FADD2_WIDE
#define HG_FADD2_WIDE 1
#endif
#ifndef HG_FADD2_F32
#define HG_FADD2_F32 0
#endif
// 8 consecutive features of a half-precision row (one 16-byte load)
template <bool CACHED>
__device__ __forceinline__ uint4 load_row8(const MeanBlock& B, std::uint32_t key, int c) {
  const void* base = B.h;
  std::size_t row = key;
  if (CACHED && B.slot) {
    const int sl = __ldg(B.slot + key);
    if (sl >= 0) {
      base = B.cache;
      row = static_cast<std::size_t>(sl);
    }
  }
  // (the L2 256-byte hint of the fp32 rows measured slower here: 394 -> 410 us/step on C5)
  const std::uint16_t* p = static_cast<const std::uint16_t*>(base) + row * B.ld_h + c;
#if HG_WIDE_NOALLOC
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
#else
  return __ldg(reinterpret_cast<const uint4*>(p));
#endif
}

// 8 half features (one raw 16-byte row chunk) added into s (features 0-3) and s2 (4-7)
__device__ __forceinline__ void add_row8(const uint4& raw, int h_dtype, float4& s, float4& s2) {
  float2 f[4];
  const std::uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
  for (int j = 0; j < 4; ++j)
    f[j] = h_dtype == kF16 ? __half22float2(*reinterpret_cast<const __half2*>(&w[j]))
                           : __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[j]));
#if HG_FADD2_WIDE
  // packed fp32 adds (round to nearest per lane: the same sums as the scalar adds)
  float2 a = __fadd2_rn(make_float2(s.x, s.y), f[0]), b = __fadd2_rn(make_float2(s.z, s.w), f[1]);
  float2 c = __fadd2_rn(make_float2(s2.x, s2.y), f[2]), d = __fadd2_rn(make_float2(s2.z, s2.w), f[3]);
  s = make_float4(a.x, a.y, b.x, b.y);
  s2 = make_float4(c.x, c.y, d.x, d.y);
#else
  s.x += f[0].x;
  s.y += f[0].y;
  s.z += f[1].x;
  s.w += f[1].y;
  s2.x += f[2].x;
  s2.y += f[2].y;
  s2.z += f[3].x;
  s2.w += f[3].y;
#endif
}

__device__ __forceinline__ void add4(float4& s, const float4& v) {
#if HG_FADD2_F32
  const float2 a = __fadd2_rn(make_float2(s.x, s.y), make_float2(v.x, v.y));
  const float2 b = __fadd2_rn(make_float2(s.z, s.w), make_float2(v.z, v.w));
  s = make_float4(a.x, a.y, b.x, b.y);
#else
  s.x += v.x;
  s.y += v.y;
  s.z += v.z;
  s.w += v.w;
#endif
}
__device__ __forceinline__ float4 scale4(float4 s, float k) { return make_float4(s.x * k, s.y * k, s.z * k, s.w * k); }

// a kernel-parameter value held in a register for the whole item: without this the
// compiler re-reads the block's fields from the parameter bank (an LDC indexed by the
// block number, issued through the ADU) for every neighbour
template <typename T>
__device__ __forceinline__ T* pin_ptr(T* p) {
  std::uint64_t r;
  asm volatile("mov.b64 %0, %1;" : "=l"(r) : "l"(reinterpret_cast<std::uint64_t>(p)));
  return reinterpret_cast<T*>(r);
}
__device__ __forceinline__ std::uint32_t pin_u32(std::uint32_t x) {
  std::uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}

// columns per half-warp item: 16 lanes x 4 fp32 features, or 16 lanes x 8 half features
__host__ __device__ inline int gather_chunk(int h_dtype) { return h_dtype == kF32 ? 64 : 128; }

// WIDE: the batch holds a half-precision table (8-feature lanes); the fp32-only
// instantiation keeps the original register budget (one float4 per neighbour)
// CACHED: a host-resident table with an HBM cache is in the batch (per-row slot lookup).
// fp32-only batches (WIDE = false) run the 64-column items with one float4 per neighbour.
// NB: neighbour rows in flight per lane (kGatherBatch; launches too small to fill the GPU
// — the top layer's 1024 rows — take more per trip so their few round trips finish sooner)
#ifndef HG_GATHER_WIDE_MINB
#define HG_GATHER_WIDE_MINB 5
#endif
template <bool WIDE, bool CACHED, int NB>
__global__ void __launch_bounds__(256, WIDE ? HG_GATHER_WIDE_MINB : NB > kGatherBatch ? 4 : 8) k_gather_mean(MeanBatch m) {
  pdl_enter();
  const int hl = threadIdx.x & 15;
  const int halves = gridDim.x * (blockDim.x >> 4);
  int b = 0;  // WIDE: items only grow, the block search resumes where the last item's ended
  for (int item = blockIdx.x * (blockDim.x >> 4) + (threadIdx.x >> 4); item < m.item_base[m.nb]; item += halves) {
    if constexpr (!WIDE) b = 0;  // (the fp32 instantiation keeps its measured per-item search)
    while (b + 1 < m.nb && item >= m.item_base[b + 1]) ++b;
    const MeanBlock& B = m.b[b];
    const int n = *B.n_rows;
    const int local = item - m.item_base[b];
    if constexpr (!WIDE) {
      const int nch = (B.din + 63) / 64;
      const int i = local / nch, c = (local % nch) * 64 + 4 * hl;
      if (c >= B.ld_mean) continue;
      if (i >= n) {
        // zero tail up to the next 32-row boundary: the tensor-core weight gradient
        // streams whole 32-row K chunks of the tape
        if (i < ((n + 31) & ~31))
          *reinterpret_cast<float4*>(B.mean + static_cast<std::size_t>(i) * B.ld_mean + c) = make_float4(0.f, 0.f, 0.f, 0.f);
        continue;
      }
      const std::uint32_t lo = B.indptr[i], hi = B.indptr[i + 1];
      const float* base = B.h + c;  // (pinning the block fields here measured slower: 49.4 -> 54.6 us/step on C2)
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
      // batches of NB neighbours (the last one predicated): one key round trip and
      // one row round trip per batch, summed in edge order
      for (std::uint32_t e = lo; e < hi; e += NB) {
        const std::uint32_t cnt = min(static_cast<std::uint32_t>(NB), hi - e);
        std::uint32_t kk[NB];
#pragma unroll
        for (int q = 0; q < NB; ++q) kk[q] = q < cnt ? __ldg(B.keys + e + q) : 0u;
        float4 v[NB];
#pragma unroll
        for (int q = 0; q < NB; ++q) {
          if (CACHED)
            v[q] = q < cnt ? load_row4(B, kk[q], c) : make_float4(0.f, 0.f, 0.f, 0.f);
          else
            v[q] = q < cnt ? ld_row_stream(base + static_cast<std::size_t>(kk[q]) * B.ld_h)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < NB; ++q) add4(s, v[q]);
      }
      if (hi > lo) s = scale4(s, 1.0f / static_cast<float>(hi - lo));
      *reinterpret_cast<float4*>(B.mean + static_cast<std::size_t>(i) * B.ld_mean + c) = s;
    } else {
      const bool wide = B.h_dtype != kF32;  // 8 features per lane
      const int chunk = gather_chunk(B.h_dtype);
      const int nch = (B.din + chunk - 1) / chunk;
      const int i = local / nch, c = (local % nch) * chunk + (wide ? 8 : 4) * hl;
      if (c >= B.ld_mean) continue;
      const bool second = wide && c + 4 < B.ld_mean;  // the lane's second float4 of output
      float* orow = B.mean + static_cast<std::size_t>(i) * B.ld_mean + c;
      if (i >= n) {
        if (i < ((n + 31) & ~31)) {
          *reinterpret_cast<float4*>(orow) = make_float4(0.f, 0.f, 0.f, 0.f);
          if (second) *reinterpret_cast<float4*>(orow + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        continue;
      }
      const std::uint32_t lo = B.indptr[i], hi = B.indptr[i + 1];
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f), s2 = s;
      const std::uint32_t* keys = pin_ptr(B.keys);
      const int dt = static_cast<int>(pin_u32(static_cast<std::uint32_t>(B.h_dtype)));
      const std::size_t rowb = static_cast<std::size_t>(pin_u32(static_cast<std::uint32_t>(B.ld_h))) * (wide ? 2 : 4);
      const char* hb = pin_ptr(reinterpret_cast<const char*>(B.h) + static_cast<std::size_t>(c) * (wide ? 2 : 4));
      for (std::uint32_t e = lo; e < hi; e += NB) {
        const std::uint32_t cnt = min(static_cast<std::uint32_t>(NB), hi - e);
        std::uint32_t kk[NB];
#pragma unroll
        for (int q = 0; q < NB; ++q) kk[q] = q < cnt ? __ldg(keys + e + q) : 0u;
        if (!CACHED) {
          // HBM tables: one raw 16-byte chunk per neighbour (4 fp32 or 8 half features),
          // converted after the round trip: the register budget holds
          // HG_GATHER_WIDE_MINB CTAs per SM
          uint4 v[NB];
#pragma unroll
          for (int q = 0; q < NB; ++q)
            v[q] = q < cnt ? __ldg(reinterpret_cast<const uint4*>(hb + kk[q] * rowb)) : make_uint4(0u, 0u, 0u, 0u);
          if (wide) {
#pragma unroll
            for (int q = 0; q < NB; ++q) add_row8(v[q], dt, s, s2);
          } else {
#pragma unroll
            for (int q = 0; q < NB; ++q)
              add4(s, make_float4(__uint_as_float(v[q].x), __uint_as_float(v[q].y), __uint_as_float(v[q].z),
                                  __uint_as_float(v[q].w)));
          }
        } else if (!wide) {
          float4 v[NB];
#pragma unroll
          for (int q = 0; q < NB; ++q) v[q] = q < cnt ? load_row4(B, kk[q], c) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int q = 0; q < NB; ++q) add4(s, v[q]);
        } else {
          uint4 v[NB];
#pragma unroll
          for (int q = 0; q < NB; ++q) v[q] = q < cnt ? load_row8<CACHED>(B, kk[q], c) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
          for (int q = 0; q < NB; ++q) add_row8(v[q], B.h_dtype, s, s2);
        }
      }
      const float inv = hi > lo ? 1.0f / static_cast<float>(hi - lo) : 0.f;
      *reinterpret_cast<float4*>(orow) = scale4(s, inv);
      if (second) *reinterpret_cast<float4*>(orow + 4) = scale4(s2, inv);
    }
  }
}

// ---- half-precision tables in HBM: one warp per destination row -----------------------------
// Lane l holds the 16-byte column slices p * 512 + 16 l (p < PM passes: 768 halves = 3, 1024 = 4)
// of NB neighbour rows at a time, so a row is read whole by one warp (one key load per edge
// instead of one per 128-column item) and the per-item bookkeeping is paid once per row.
// Sums per column in edge order, as k_gather_mean: bit-identical results.
#ifndef HG_ROWS_NB
#define HG_ROWS_NB 2
#endif
#ifndef HG_ROWS_MINB
#define HG_ROWS_MINB 3
#endif
template <int NB, int PM>
__global__ void __launch_bounds__(256, HG_ROWS_MINB) k_gather_rows_half(MeanBatch m) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  int b = 0;
  for (int item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); item < m.item_base[m.nb]; item += warps) {
    while (b + 1 < m.nb && item >= m.item_base[b + 1]) ++b;
    const MeanBlock& B = m.b[b];
    const int n = *B.n_rows;
    const int i = item - m.item_base[b];
    const int ldm = B.ld_mean;
    float* orow = B.mean + static_cast<std::size_t>(i) * ldm;
    if (i >= n) {
      if (i < ((n + 31) & ~31))
        for (int c = 4 * lane; c < ldm; c += 128) *reinterpret_cast<float4*>(orow + c) = make_float4(0.f, 0.f, 0.f, 0.f);
      continue;
    }
    const std::uint32_t lo = B.indptr[i], hi = B.indptr[i + 1];
    const std::uint32_t* keys = pin_ptr(B.keys);
    const int dt = static_cast<int>(pin_u32(static_cast<std::uint32_t>(B.h_dtype)));
    const std::uint32_t ldh = pin_u32(static_cast<std::uint32_t>(B.ld_h));
    const std::size_t rowb = static_cast<std::size_t>(ldh) * 2;
    const char* hb = pin_ptr(reinterpret_cast<const char*>(B.h) + 16 * lane);
    float4 s[PM], s2[PM];
#pragma unroll
    for (int p = 0; p < PM; ++p) s[p] = s2[p] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (std::uint32_t e = lo; e < hi; e += NB) {
      const std::uint32_t cnt = min(static_cast<std::uint32_t>(NB), hi - e);
      std::uint32_t kk[NB];
#pragma unroll
      for (int q = 0; q < NB; ++q) kk[q] = q < cnt ? __ldg(keys + e + q) : 0u;
      uint4 v[NB][PM];
#pragma unroll
      for (int q = 0; q < NB; ++q)
#pragma unroll
        for (int p = 0; p < PM; ++p)
          v[q][p] = q < cnt && static_cast<std::uint32_t>(p * 256 + 8 * lane) < ldh
                        ? __ldg(reinterpret_cast<const uint4*>(hb + kk[q] * rowb + p * 512))
                        : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
      for (int q = 0; q < NB; ++q)
#pragma unroll
        for (int p = 0; p < PM; ++p) add_row8(v[q][p], dt, s[p], s2[p]);
    }
    const float inv = hi > lo ? 1.0f / static_cast<float>(hi - lo) : 0.f;
#pragma unroll
    for (int p = 0; p < PM; ++p) {
      const int c = p * 256 + 8 * lane;
      if (c < ldm) *reinterpret_cast<float4*>(orow + c) = scale4(s[p], inv);
      if (c + 4 < ldm) *reinterpret_cast<float4*>(orow + c + 4) = scale4(s2[p], inv);
    }
  }
}

// ---- fp32 tables / inner-layer rows: one half-warp per destination row --------------------
// (HG_GATHER_ROWS_F32=0: the 64-column half-warp items instead): lane l holds the float4 slices 256 p + 16 l (bytes) of NB
// neighbour rows; keys once per row; edge-order sums per column as k_gather_mean.
#ifndef HG_GATHER_ROWS_F32
#define HG_GATHER_ROWS_F32 1
#endif
#ifndef HG_ROWSF_NB
#define HG_ROWSF_NB 3
#endif
#ifndef HG_ROWSF_MINB
#define HG_ROWSF_MINB 5
#endif
template <int NB, int PM>
__global__ void __launch_bounds__(256, HG_ROWSF_MINB) k_gather_rows_f32(MeanBatch m) {
  pdl_enter();
  const int hl = threadIdx.x & 15;
  const int halves = gridDim.x * (blockDim.x >> 4);
  int b = 0;
  for (int item = blockIdx.x * (blockDim.x >> 4) + (threadIdx.x >> 4); item < m.item_base[m.nb]; item += halves) {
    while (b + 1 < m.nb && item >= m.item_base[b + 1]) ++b;
    const MeanBlock& B = m.b[b];
    const int n = *B.n_rows;
    const int i = item - m.item_base[b];
    const int ldm = B.ld_mean;
    float* orow = B.mean + static_cast<std::size_t>(i) * ldm;
    if (i >= n) {
      if (i < ((n + 31) & ~31))
        for (int c = 4 * hl; c < ldm; c += 64) *reinterpret_cast<float4*>(orow + c) = make_float4(0.f, 0.f, 0.f, 0.f);
      continue;
    }
    const std::uint32_t lo = B.indptr[i], hi = B.indptr[i + 1];
    const int ldh = B.ld_h;
    const float* base = B.h + 4 * hl;
    float4 s[PM];
#pragma unroll
    for (int p = 0; p < PM; ++p) s[p] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (std::uint32_t e = lo; e < hi; e += NB) {
      const std::uint32_t cnt = min(static_cast<std::uint32_t>(NB), hi - e);
      std::uint32_t kk[NB];
#pragma unroll
      for (int q = 0; q < NB; ++q) kk[q] = q < cnt ? __ldg(B.keys + e + q) : 0u;
      float4 v[NB][PM];
#pragma unroll
      for (int q = 0; q < NB; ++q)
#pragma unroll
        for (int p = 0; p < PM; ++p)
          v[q][p] = q < cnt && p * 64 + 4 * hl < ldm
                        ? ld_row_stream(base + static_cast<std::size_t>(kk[q]) * ldh + p * 64)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int q = 0; q < NB; ++q)
#pragma unroll
        for (int p = 0; p < PM; ++p) add4(s[p], v[q][p]);
    }
#pragma unroll
    for (int p = 0; p < PM; ++p) {
      const int c = p * 64 + 4 * hl;
      if (c < ldm) *reinterpret_cast<float4*>(orow + c) = hi > lo ? scale4(s[p], 1.0f / static_cast<float>(hi - lo)) : s[p];
    }
  }
}

// ---- projection: out = sum_r mean_r . W_r (agg_all over relations), ReLU ------------------
__global__ void __launch_bounds__(kT) k_project_tiles(ProjBatch pb) {
  pdl_enter();
  __shared__ __align__(16) float As[kKS * kLd];
  __shared__ __align__(16) float Bs[kKS * kLd];
  const int gi = find_problem(pb.tile_base, pb.ng, blockIdx.x);
  const ProjGroup& g = pb.g[gi];
  const int t = blockIdx.x - pb.tile_base[gi];
  const int ncb = (g.dout + kTile - 1) / kTile;
  const int rb = t / ncb, cb = t % ncb;
  const int n = *g.n_rows;
  const int row0 = rb * kTile, col0 = cb * kTile;
  if (row0 >= n) return;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  Acc acc;
  acc.zero();
  for (int q = 0; q < g.nrel; ++q) {
    const ProjRel& r = g.r[q];
    for (int k0 = 0; k0 < r.din; k0 += kKS) {
      const int kn = min(kKS, r.din - k0);
      __syncthreads();
      for (int x = tid; x < kTile * kKS / 4; x += kT) {
        const int m = x / (kKS / 4), kq = (x % (kKS / 4)) * 4;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row0 + m < n && kq < kn)
          a = *reinterpret_cast<const float4*>(r.mean + static_cast<std::size_t>(row0 + m) *
                                                             (r.row_stride ? r.row_stride : r.ld_mean) + k0 + kq);
        As[(kq + 0) * kLd + m] = a.x;
        As[(kq + 1) * kLd + m] = a.y;
        As[(kq + 2) * kLd + m] = a.z;
        As[(kq + 3) * kLd + m] = a.w;
      }
      for (int x = tid; x < kKS * kTile / 4; x += kT) {
        const int k = x / (kTile / 4), nq = (x % (kTile / 4)) * 4;
        float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k < kn && col0 + nq < g.dout)
          w = __ldg(reinterpret_cast<const float4*>(r.w + static_cast<std::size_t>(k0 + k) * r.ld_w + col0 + nq));
        *reinterpret_cast<float4*>(Bs + k * kLd + nq) = w;
      }
      __syncthreads();
      slab_fma(As, Bs, kn, ty, tx, acc);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = row0 + ty * 4 + i;
    if (row >= n) break;
    float* orow = g.out + static_cast<std::size_t>(row * g.out_stride + g.out_offset) * g.ld_out;
    const int c = col0 + tx * 4;
    if (c < g.dout) {
      float4 o = make_float4(acc.v[i][0], acc.v[i][1], acc.v[i][2], acc.v[i][3]);
      if (g.relu) {
        o.x = fmaxf(o.x, 0.f);
        o.y = fmaxf(o.y, 0.f);
        o.z = fmaxf(o.z, 0.f);
        o.w = fmaxf(o.w, 0.f);
      }
      *reinterpret_cast<float4*>(orow + c) = o;
    }
  }
}

}  // namespace

#ifndef HG_GATHER_ROWS
#define HG_GATHER_ROWS 1
#endif
void gather_mean(MeanBatch& m, cudaStream_t st) {
  if (m.nb == 0) return;
#if HG_GATHER_ROWS
  {
    // half-precision HBM blocks go to the warp-per-row kernel, the rest stay below
    bool any_half = false, any_cached = false;
    int pm = 0;
    for (int b = 0; b < m.nb; ++b) {
      any_cached = any_cached || m.b[b].slot != nullptr;
      if (m.b[b].h_dtype != kF32) {
        any_half = true;
        pm = std::max(pm, static_cast<int>(ceil_div(static_cast<std::uint64_t>(m.b[b].ld_h), 256)));
      }
    }
    if (any_half && !any_cached && pm <= 4) {
      MeanBatch hv{}, rest{};
      int rows = 0;
      for (int b = 0; b < m.nb; ++b) {
        if (m.b[b].h_dtype != kF32) {
          hv.item_base[hv.nb] = rows;
          rows += m.b[b].rows_cap;
          hv.b[hv.nb++] = m.b[b];
        } else {
          rest.b[rest.nb++] = m.b[b];
        }
      }
      hv.item_base[hv.nb] = rows;
      const unsigned grid = static_cast<unsigned>(
          std::max<std::uint64_t>(1, std::min<std::uint64_t>(ceil_div(rows, 8), HG_GATHER_WAVES * num_sms())));
      if (pm <= 2)
        launch_pdl(k_gather_rows_half<HG_ROWS_NB, 2>, grid, 256, 0, st, hv);
      else if (pm == 3)
        launch_pdl(k_gather_rows_half<HG_ROWS_NB, 3>, grid, 256, 0, st, hv);
      else
        launch_pdl(k_gather_rows_half<HG_ROWS_NB, 4>, grid, 256, 0, st, hv);
      if (rest.nb) gather_mean(rest, st);
      return;
    }
  }
#endif
#if HG_GATHER_ROWS_F32
  {
    bool plain = true;
    int pm = 0;
    for (int b = 0; b < m.nb; ++b) {
      plain = plain && m.b[b].slot == nullptr && m.b[b].h_dtype == kF32;
      pm = std::max(pm, static_cast<int>(ceil_div(static_cast<std::uint64_t>(m.b[b].ld_mean), 64)));
    }
    int rows = 0;
    for (int b = 0; b < m.nb; ++b) rows += m.b[b].rows_cap;
    if (plain && pm <= 2 && rows > 8 * 16 * num_sms()) {
      rows = 0;
      for (int b = 0; b < m.nb; ++b) {
        m.item_base[b] = rows;
        rows += m.b[b].rows_cap;
      }
      m.item_base[m.nb] = rows;
      const unsigned grid = static_cast<unsigned>(
          std::max<std::uint64_t>(1, std::min<std::uint64_t>(ceil_div(rows, 16), HG_GATHER_WAVES * num_sms())));
      if (pm <= 1)
        launch_pdl(k_gather_rows_f32<HG_ROWSF_NB, 1>, grid, 256, 0, st, m);
      else
        launch_pdl(k_gather_rows_f32<HG_ROWSF_NB, 2>, grid, 256, 0, st, m);
      return;
    }
  }
#endif
  int items = 0;
  for (int b = 0; b < m.nb; ++b) {
    m.item_base[b] = items;
    items += m.b[b].rows_cap * static_cast<int>(ceil_div(m.b[b].din, gather_chunk(m.b[b].h_dtype)));
  }
  m.item_base[m.nb] = items;
  const unsigned grid = static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(ceil_div(items, 16), HG_GATHER_WAVES * num_sms())));
  bool wide = false, cached = false;
  for (int b = 0; b < m.nb; ++b) {
    wide = wide || m.b[b].h_dtype != kF32;
    cached = cached || m.b[b].slot != nullptr;
  }
  const bool small = items <= 8 * 16 * num_sms();  // fewer half-warp items than 8 warps per SM
  if (wide && cached)
    launch_pdl(k_gather_mean<true, true, kGatherBatch>, grid, 256, 0, st, m);  // half tables in host memory
  else if (wide)
    launch_pdl(k_gather_mean<true, false, HG_GATHER_BATCH_WIDE>, grid, 256, 0, st, m);  // half tables in HBM
  else if (cached)
    launch_pdl(k_gather_mean<false, true, kGatherBatch>, grid, 256, 0, st, m);
  else if (small)
    launch_pdl(k_gather_mean<false, false, HG_GATHER_BATCH_SMALL>, grid, 256, 0, st, m);
  else
    launch_pdl(k_gather_mean<false, false, kGatherBatch>, grid, 256, 0, st, m);
}

void project_tiles(ProjBatch& p, cudaStream_t st) {
  if (p.ng == 0) return;
  int tiles = 0;
  for (int g = 0; g < p.ng; ++g) {
    p.tile_base[g] = tiles;
    tiles += static_cast<int>(ceil_div(std::max(1, p.g[g].rows_cap), kTile) * ceil_div(p.g[g].dout, kTile));
  }
  p.tile_base[p.ng] = tiles;
  launch_pdl(k_project_tiles, std::max(1, tiles), kT, 0, st, p);
}

void wgrad_tiles(WGradBatch& b, cudaStream_t st) {
  if (b.np == 0) return;
  int tiles = 0;
  for (int p = 0; p < b.np; ++p) {
    const WGradProblem& P = b.p[p];
    b.tile_base[p] = tiles;
    tiles += static_cast<int>(ceil_div(std::max(1, P.rows_cap), kWChunkRows) * ceil_div(P.din, kTile) *
                              ceil_div(P.d.cols, kTile));
  }
  launch_pdl(k_wgrad_tiles, std::max(1, tiles), kT, 0, st, b);
  if (!b.defer_reduce) wgrad_reduce(b, st);
}

void wgrad_reduce(WGradBatch& b, cudaStream_t st) {
  int total_out = 0;
  for (int p = 0; p < b.np; ++p) total_out += b.p[p].din * b.p[p].d.cols;
  if (total_out > 0) launch_pdl(k_wgrad_reduce, static_cast<unsigned>(ceil_div(total_out, 256)), 256, 0, st, b, total_out);
}

void dmean_tiles(DMeanBatch& b, cudaStream_t st) {
  if (b.np == 0) return;
  int tiles = 0;
  for (int p = 0; p < b.np; ++p) {
    const DMeanProblem& P = b.p[p];
    b.tile_base[p] = tiles;
    tiles += static_cast<int>(ceil_div(std::max(1, P.rows_cap), kTile) * ceil_div(P.din, kTile));
  }
  launch_pdl(k_dmean_tiles, std::max(1, tiles), kT, 0, st, b);
}

}  // namespace hetgpu
