// Floating-point work of the hot path (fp32 storage, fp32 accumulate):
// relation-first mean aggregation fused with the per-relation projection and
// the AGG_all sum over relations (hgnn.cpp:173-203, 215-279), the softmax
// cross-entropy (hgnn.cpp:281-307), the backward pass (hgnn.cpp:309-362) with a
// deterministic transposed gather instead of the scatter, and Adam
// (hgnn.cpp:364-410). This file is the portable SIMT path: any dims, any
// shape. (The tcgen05 projection lives in umma_kernels.cu.)
#include <cfloat>

#include "adam.cuh"
#include "kernels.cuh"

#ifndef HG_FRONT_WAVES
#define HG_FRONT_WAVES 4  // x-extent (CTAs per SM) of the per-block relabel / transpose grids
#endif
#ifndef HG_RSUM_WAVES
#define HG_RSUM_WAVES 8  // CTAs per SM of the replica sum + Adam grid (8 measured best at p=4)
#endif
#ifndef HG_CSC_WAVES
#define HG_CSC_WAVES 8  // CTAs per SM of the backward-gather grid (8: one resident wave, measured best)
#endif
#ifndef HG_GATHER_WAVES
#define HG_GATHER_WAVES 24  // CTAs per SM of the gather grids (8 resident: three waves)
#endif

namespace hetgpu {

namespace {
constexpr int kThreads = 256;
#ifndef HG_CE_REG
#define HG_CE_REG 1  // cross entropy: a row in registers (one read) instead of three passes
#endif
#if HG_CE_REG
constexpr int kCeRegs = 16;  // logits per lane held in registers (C <= 512)
#endif
}  // namespace

// ---- cross entropy ---------------------------------------------------------------------

namespace {

__global__ void __launch_bounds__(kThreads) k_cross_entropy(LossArgs a) {
  pdl_enter();
  const int n = *a.n_rows;
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (kThreads / 32);
  const float invb = 1.0f / static_cast<float>(a.sc->batch_len);
  for (int i = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); i < n; i += warps) {
    const float* z = a.logits + static_cast<std::size_t>(i) * a.ld;
    float* dz = a.dlogits + static_cast<std::size_t>(i) * a.ld;
    const float m = a.mult[i];
    const std::int32_t y = a.labels[a.row_ids[i]];
    if (m == 0.0f) {
      for (int c = lane; c < a.C; c += 32) {
        dz[c] = 0.f;
      }
      if (lane == 0) a.row_loss[i] = 0.0;
      continue;
    }
    if (y < 0 || y >= a.C) {  // never reached: the host validates labels before enqueueing
      for (int c = lane; c < a.C; c += 32) {
        dz[c] = 0.f;
      }
      if (lane == 0) {
        a.row_loss[i] = 0.0;
        atomicOr(a.err, 2u);
      }
      continue;
    }
    // fp32 log-sum-exp (the reference's f64 agrees to ~1e-7 relative)
    const float scale = m * invb;
#if HG_CE_REG
    if (a.C <= 32 * kCeRegs) {  // the row read once into registers (C <= 512)
      float zv[kCeRegs];
      float zmax = -FLT_MAX;
#pragma unroll
      for (int u = 0; u < kCeRegs; ++u) {
        const int c = lane + 32 * u;
        zv[u] = c < a.C ? z[c] : -FLT_MAX;
        zmax = fmaxf(zmax, zv[u]);
      }
      for (int o = 16; o > 0; o >>= 1) zmax = fmaxf(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
      float sum = 0.f;
#pragma unroll
      for (int u = 0; u < kCeRegs; ++u) {
        zv[u] = expf(zv[u] - zmax);  // 0 for the padding lanes
        sum += zv[u];
      }
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const float inv = 1.0f / sum;
#pragma unroll
      for (int u = 0; u < kCeRegs; ++u) {
        const int c = lane + 32 * u;
        if (c < a.C) dz[c] = (zv[u] * inv - (c == y ? 1.0f : 0.0f)) * scale;
      }
      if (lane == 0) a.row_loss[i] = static_cast<double>(zmax + logf(sum) - z[y]) * static_cast<double>(scale);
      continue;
    }
#endif
    float zmax = -FLT_MAX;
    for (int c = lane; c < a.C; c += 32) zmax = fmaxf(zmax, z[c]);
    for (int o = 16; o > 0; o >>= 1) zmax = fmaxf(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
    float sum = 0.f;
    for (int c = lane; c < a.C; c += 32) sum += expf(z[c] - zmax);
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float lse = zmax + logf(sum);
    for (int c = lane; c < a.C; c += 32) {
      const float g = (expf(z[c] - lse) - (c == y ? 1.0f : 0.0f)) * scale;
      dz[c] = g;
    }
    if (lane == 0) a.row_loss[i] = static_cast<double>(lse - z[y]) * static_cast<double>(scale);
  }
  // the last CTA to finish sums the rows in a fixed order (deterministic) and
  // moves the learnable tables' Adam steps
  __shared__ bool last;
  __shared__ double part[kThreads];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(a.done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += kThreads) s += __ldcg(a.row_loss + i);
  part[threadIdx.x] = s;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *a.loss_out = part[0];
    *a.done = 0u;
  }
  if (threadIdx.x < a.bumps.count && *a.bumps.n[threadIdx.x] > 0) ++*a.bumps.step[threadIdx.x];
}

}  // namespace

void cross_entropy(const LossArgs& a, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::max<std::uint64_t>(
      1, std::min<std::uint64_t>(ceil_div(a.rows_cap, kThreads / 32), 4 * num_sms())));
  launch_pdl(k_cross_entropy, grid, kThreads, 0, st, a);
}

// ---- transposed gather for the backward scatter ------------------------------------------------

namespace {

// entries hold the packed (block, destination row) of every sampled edge
// (block index in the top 4 bits): the backward gather reads dmean rows directly
constexpr int kRowBits = 28;
__global__ void k_csc_fill(CscHop h) {
  pdl_enter();
  const int bi = blockIdx.y;
  const CscEdges& b = h.b[bi];
  const CscType& t = h.t[b.type];
  const std::uint32_t total = b.indptr[*b.n_rows];
  for (std::uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const std::uint32_t c = b.col[e];
    const std::uint32_t pos = atomicAdd(t.cursor + c, 1u);
    t.entries[t.offs[c] - 1 - pos] = (static_cast<std::uint32_t>(bi) << kRowBits) | (h.edge_ids ? e : b.erow[e]);
  }
}

// make every segment ascending in (block, row): deterministic summation order.
// A lane owns a segment; short ones (<= kShortSeg) it insertion-sorts alone, longer
// ones (hub sources of power-law graphs) the whole warp sorts together: a bitonic
// network in shared memory up to kWarpSort entries, beyond that sorted runs of
// kWarpSort merged pairwise through the type's scratch array (O(n log^2 n) instead of
// the O(n^2) of one insertion sort).
constexpr std::uint32_t kShortSeg = 32;
constexpr int kWarpSort = 1024;
constexpr int kSortThreads = 256;

__device__ void warp_bitonic(std::uint32_t* a, int n, int lane) {
  int P = 1;
  while (P < n) P <<= 1;
  for (int i = n + lane; i < P; i += 32) a[i] = 0xFFFFFFFFu;
  __syncwarp();
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < P; i += 32) {
        const int l = i ^ j;
        if (l > i) {
          const std::uint32_t x = a[i], y = a[l];
          if ((x > y) == ((i & k) == 0)) {
            a[i] = y;
            a[l] = x;
          }
        }
      }
      __syncwarp();
    }
}

// the warp sorts seg[0, n) in place (tmp: n words of scratch)
__device__ void warp_sort_segment(std::uint32_t* seg, std::uint32_t* tmp, std::uint32_t n, std::uint32_t* sm, int lane) {
  for (std::uint32_t r0 = 0; r0 < n; r0 += kWarpSort) {  // sorted runs
    const int m = static_cast<int>(min(static_cast<std::uint32_t>(kWarpSort), n - r0));
    for (int i = lane; i < m; i += 32) sm[i] = seg[r0 + i];
    __syncwarp();
    warp_bitonic(sm, m, lane);
    for (int i = lane; i < m; i += 32) seg[r0 + i] = sm[i];
    __syncwarp();
  }
  std::uint32_t* src = seg;
  std::uint32_t* dst = tmp;
  for (std::uint32_t w = kWarpSort; w < n; w <<= 1) {  // pairwise merges by rank
    for (std::uint32_t i = lane; i < n; i += 32) {
      const std::uint32_t a0 = (i / (2 * w)) * (2 * w), b0 = min(a0 + w, n), b1 = min(a0 + 2 * w, n);
      const std::uint32_t x = src[i];
      std::uint32_t lo, hi, pos;
      if (i < b0) {  // rank in the right run: elements < x
        lo = b0;
        hi = b1;
        while (lo < hi) {
          const std::uint32_t mid = (lo + hi) >> 1;
          if (src[mid] < x) lo = mid + 1; else hi = mid;
        }
        pos = a0 + (i - a0) + (lo - b0);
      } else {  // rank in the left run: elements <= x
        lo = a0;
        hi = b0;
        while (lo < hi) {
          const std::uint32_t mid = (lo + hi) >> 1;
          if (src[mid] <= x) lo = mid + 1; else hi = mid;
        }
        pos = a0 + (i - b0) + (lo - a0);
      }
      dst[pos] = x;
    }
    __syncwarp();
    std::uint32_t* t = src;
    src = dst;
    dst = t;
  }
  if (src != seg) {
    for (std::uint32_t i = lane; i < n; i += 32) seg[i] = src[i];
    __syncwarp();
  }
}

__global__ void __launch_bounds__(kSortThreads) k_csc_sort(CscHop h) {
  pdl_enter();
  __shared__ std::uint32_t sm[kSortThreads / 32][kWarpSort];
  const CscType& t = h.t[blockIdx.y];
  const int n = *t.n_src;
  const int lane = threadIdx.x & 31;
  std::uint32_t* wsm = sm[threadIdx.x >> 5];
  const int stride = gridDim.x * blockDim.x;
  // whole warps iterate together (the long segments need every lane)
  for (int base = blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n; base += stride) {
    const int c = base + lane;
    std::uint32_t lo = 0, hi = 0;
    if (c < n) {
      lo = c ? t.offs[c - 1] : 0u;
      hi = t.offs[c];
    }
    const bool is_long = hi - lo > kShortSeg;
    // the warp's sources are consecutive, so their segments are one contiguous span:
    // when it fits the warp's shared buffer, stage it with coalesced loads, sort every
    // lane's segment there and store it back (no dependent global round trips)
    const std::uint32_t wlo = base ? t.offs[base - 1] : 0u;
    const std::uint32_t whi = t.offs[min(base + 31, n - 1)];
    if (!__any_sync(0xffffffffu, is_long) && whi - wlo <= static_cast<std::uint32_t>(kWarpSort)) {
      for (std::uint32_t x = wlo + lane; x < whi; x += 32) wsm[x - wlo] = t.entries[x];
      __syncwarp();
      std::uint32_t* seg = wsm + (hi > lo ? lo - wlo : 0u);
      for (std::uint32_t x = 1; x < hi - lo; ++x) {
        const std::uint32_t v = seg[x];
        std::uint32_t y = x;
        while (y > 0 && seg[y - 1] > v) {
          seg[y] = seg[y - 1];
          --y;
        }
        seg[y] = v;
      }
      __syncwarp();
      for (std::uint32_t x = wlo + lane; x < whi; x += 32) t.entries[x] = wsm[x - wlo];
      __syncwarp();
      continue;
    }
    if (!is_long) {
      for (std::uint32_t x = lo + 1; x < hi; ++x) {
        const std::uint32_t v = t.entries[x];
        std::uint32_t y = x;
        while (y > lo && t.entries[y - 1] > v) {
          t.entries[y] = t.entries[y - 1];
          --y;
        }
        t.entries[y] = v;
      }
    }
    unsigned todo = __ballot_sync(0xffffffffu, is_long);
    while (todo) {
      const int src_lane = __ffs(todo) - 1;
      todo &= todo - 1;
      const std::uint32_t slo = __shfl_sync(0xffffffffu, lo, src_lane);
      const std::uint32_t shi = __shfl_sync(0xffffffffu, hi, src_lane);
      warp_sort_segment(t.entries + slo, t.tmp + slo, shi - slo, wsm, lane);
    }
  }
}

#ifndef HG_CSC_BATCH
#define HG_CSC_BATCH 2
#endif
constexpr int kCscBatch = HG_CSC_BATCH;  // dmean rows in flight per lane

// one half-warp per (source row, 64-column chunk): ordered sum of the dmean rows
// of its sampled edges; learnable leaves apply Adam to their table row directly
__global__ void __launch_bounds__(256) k_csc_gather(CscHop h, AdamHyper hp, std::uint32_t* err) {
  pdl_enter();
  __shared__ AdamStep ks[kMaxSegs];
  if (threadIdx.x < h.nt) {
    const CscType& t = h.t[threadIdx.x];
    ks[threadIdx.x] = adam_step_of(hp, t.step ? static_cast<double>(*t.step) : 1.0);
  }
  __syncthreads();
  const int hl = threadIdx.x & 15;
  const int halves = gridDim.x * (blockDim.x >> 4);
  for (int ty = 0; ty < h.nt; ++ty) {
    const CscType& t = h.t[ty];
    const int n = *t.n_src;
    const int nch = (t.din + 63) / 64;
    for (int item = blockIdx.x * (blockDim.x >> 4) + (threadIdx.x >> 4); item < n * nch; item += halves) {
      const int c = item / nch;
      const int f = (item % nch) * 64 + 4 * hl;
      if (f >= t.ld_dh) continue;
      const std::uint32_t lo = c ? t.offs[c - 1] : 0u, hi = t.offs[c];
      // loads that do not depend on the sum go out first: the ReLU mask row, and the
      // learnable row's w / m / v (their DRAM round trip overlaps the gather's)
      float4 hm4 = make_float4(1.f, 1.f, 1.f, 1.f), w0, m0, v0;
      std::size_t at_w = 0;
      if (t.relu_h) hm4 = *reinterpret_cast<const float4*>(t.relu_h + static_cast<std::size_t>(c) * t.ld_h + f);
      if (t.w) {
        at_w = static_cast<std::size_t>(t.ids[c]) * t.ld_w + f;
        w0 = *reinterpret_cast<const float4*>(t.w + at_w);
        m0 = *reinterpret_cast<const float4*>(t.m + at_w);
        v0 = *reinterpret_cast<const float4*>(t.v + at_w);
      }
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
      // up to kCscBatch edges in flight: packed entries, then dmean rows
      for (std::uint32_t x0 = lo; x0 < hi; x0 += kCscBatch) {
        const int cnt = min(static_cast<std::uint32_t>(kCscBatch), hi - x0);
        const float* rowp[kCscBatch];
#pragma unroll
        for (int q = 0; q < kCscBatch; ++q) {
          rowp[q] = nullptr;
          if (q < cnt) {
            const std::uint32_t key = __ldg(t.entries + x0 + q);  // packed (block, row)
            const CscEdges& b = h.b[key >> kRowBits];
            rowp[q] = b.dmean + static_cast<std::size_t>(key & ((1u << kRowBits) - 1)) * b.ld_dmean + f;
          }
        }
        float4 v[kCscBatch];
#pragma unroll
        for (int q = 0; q < kCscBatch; ++q)
          v[q] = q < cnt ? *reinterpret_cast<const float4*>(rowp[q]) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int q = 0; q < kCscBatch; ++q) {
          s.x += v[q].x;
          s.y += v[q].y;
          s.z += v[q].z;
          s.w += v[q].w;
        }
      }
      if (t.relu_h) {
        if (hm4.x <= 0.f) s.x = 0.f;
        if (hm4.y <= 0.f) s.y = 0.f;
        if (hm4.z <= 0.f) s.z = 0.f;
        if (hm4.w <= 0.f) s.w = 0.f;
      }
      if (t.dh) *reinterpret_cast<float4*>(t.dh + static_cast<std::size_t>(c) * t.ld_dh + f) = s;
      if (t.w) {
        adam4(w0, m0, v0, s, ks[ty], err);
        *reinterpret_cast<float4*>(t.w + at_w) = w0;
        *reinterpret_cast<float4*>(t.m + at_w) = m0;
        *reinterpret_cast<float4*>(t.v + at_w) = v0;
      }
    }
  }
}

}  // namespace

void csc_prepare(const CscHop& h, LbScratch& lb, cudaStream_t st) {
  if (h.nt == 0) return;
  ScanArgs sa{};
  sa.nseg = h.nt;
  for (int i = 0; i < h.nt; ++i) sa.s[i] = {h.t[i].offs, h.t[i].n_src, h.t[i].src_cap};
  scan_inclusive(sa, lb, st);
  int cap = 1, scap = 1;
  for (int i = 0; i < h.nb; ++i) cap = std::max(cap, h.b[i].cap);
  for (int i = 0; i < h.nt; ++i) scap = std::max(scap, h.t[i].src_cap);
  dim3 grid(static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(cap, 256), HG_FRONT_WAVES * num_sms())), h.nb);
  launch_pdl(k_csc_fill, grid, 256, 0, st, h);
  dim3 g2(static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(scap, 256), HG_FRONT_WAVES * num_sms())), h.nt);
  launch_pdl(k_csc_sort, g2, 256, 0, st, h);
}

void csc_gather(const CscHop& h, AdamHyper hp, std::uint32_t* err, cudaStream_t st) {
  if (h.nt == 0) return;
  int items = 0;
  for (int i = 0; i < h.nt; ++i) items += h.t[i].src_cap * static_cast<int>(ceil_div(h.t[i].din, 64));
  const unsigned grid = static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(ceil_div(items, 16), HG_CSC_WAVES * num_sms())));
  launch_pdl(k_csc_gather, grid, 256, 0, st, h, hp, err);
}

// ---- Adam ---------------------------------------------------------------------------------------

namespace {

// every model slot in one launch: flat [rows x ld] arrays (padding is zero
// in w, m, v and g, so updating it is a no-op)
__global__ void __launch_bounds__(256) k_adam_model(AdamModelBatch b, const std::int64_t* step, AdamHyper hp,
                                                    std::uint32_t* err) {
  pdl_enter();
  __shared__ AdamStep ks;
  if (threadIdx.x == 0) ks = adam_step_of(hp, static_cast<double>(*step));
  __syncthreads();
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < b.total4; x += gridDim.x * blockDim.x) {
    int s = 0;
    while (s + 1 < b.n && x >= b.base4[s + 1]) ++s;
    const int off = (x - b.base4[s]) * 4;
    float4 w = *reinterpret_cast<float4*>(b.w[s] + off);
    float4 m = *reinterpret_cast<float4*>(b.m[s] + off);
    float4 v = *reinterpret_cast<float4*>(b.v[s] + off);
    const float4 g = *reinterpret_cast<const float4*>(b.g[s] + off);
    adam4(w, m, v, g, ks, err);
    *reinterpret_cast<float4*>(b.w[s] + off) = w;
    *reinterpret_cast<float4*>(b.m[s] + off) = m;
    *reinterpret_cast<float4*>(b.v[s] + off) = v;
  }
}

// per table: step += 1 iff it has gradient rows this batch (hgnn.cpp:392-394)
__global__ void k_bump_steps(AdamRowsBatch b) {
  pdl_enter();
  const int t = threadIdx.x;
  if (t < b.n && *b.t[t].n_rows > 0) ++*b.t[t].step;
}

// sparse learnable rows of every table in one launch: one float4 per thread
__global__ void __launch_bounds__(256) k_adam_rows(AdamRowsBatch b, AdamHyper hp, std::uint32_t* err) {
  pdl_enter();
  __shared__ AdamStep ks[kMaxSegs];
  if (threadIdx.x < b.n) ks[threadIdx.x] = adam_step_of(hp, static_cast<double>(*b.t[threadIdx.x].step));
  __syncthreads();
  // per table, only its live rows (capacities can be far larger than the union)
  for (int s = 0; s < b.n; ++s) {
    const AdamRowsTable& T = b.t[s];
    const int per_row = T.ld / 4;
    const int total = *T.n_rows * per_row;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += gridDim.x * blockDim.x) {
    const int i = x / per_row, c = (x % per_row) * 4;
    const std::size_t at = static_cast<std::size_t>(T.ids[i]) * T.ld + c;
    float4 w = *reinterpret_cast<float4*>(T.w + at);
    float4 m = *reinterpret_cast<float4*>(T.m + at);
    float4 v = *reinterpret_cast<float4*>(T.v + at);
    const float4 g = *reinterpret_cast<const float4*>(T.g + static_cast<std::size_t>(i) * T.ld_g + c);
    adam4(w, m, v, g, ks[s], err);
    *reinterpret_cast<float4*>(T.w + at) = w;
    *reinterpret_cast<float4*>(T.m + at) = m;
    *reinterpret_cast<float4*>(T.v + at) = v;
    }
  }
}

__global__ void k_zero_rows(float* p, int ld, const int* n_rows) {
  pdl_enter();
  const std::size_t total = static_cast<std::size_t>(*n_rows) * ld;
  for (std::size_t x = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<std::size_t>(gridDim.x) * blockDim.x)
    p[x] = 0.f;
}

}  // namespace

namespace {
struct BumpArgs {
  std::int64_t* step[kMaxSegs];
  const int* n[kMaxSegs];
  int count;
};
__global__ void k_bump_list(BumpArgs a) {
  pdl_enter();
  const int t = threadIdx.x;
  if (t < a.count && *a.n[t] > 0) ++*a.step[t];
}
// half-warp per (union row of this shard, 64-column chunk): replicas' rows
// summed in replica order (hgnn.cpp:83-113 accumulate), then Adam on the table
// row (hgnn.cpp:392-410). The shard owns the row's m / v; its new w is stored
// into every replica's copy of the table (NVLink stores to the peers).
template <int R>  // replicas in the group (register footprint: R float4 partials)
__global__ void __launch_bounds__(256) k_rsum_adam(ReplicaMerge m, ReplicaAdam a, AdamHyper hp,
                                                   std::uint32_t* err) {
  pdl_enter();
  __shared__ AdamStep ks;
  if (threadIdx.x == 0) ks = adam_step_of(hp, static_cast<double>(*a.step));
  __syncthreads();
  const int hl = threadIdx.x & 15;
  const int n = *m.u.count;
  const int nch = (m.din + 63) / 64;
  const int halves = gridDim.x * (blockDim.x >> 4);
  for (int item = blockIdx.x * (blockDim.x >> 4) + (threadIdx.x >> 4); item < n * nch; item += halves) {
    const int u = item / nch;
    const int f = (item % nch) * 64 + 4 * hl;
    if (f >= m.ld) continue;
    // independent loads first: the replicas' row slots and the union id, then the
    // replicas' gradient rows (peers over NVLink) and the table row state
    int rows[R];
#pragma unroll
    for (int r = 0; r < R; ++r) rows[r] = r < m.n_rep ? m.slot[static_cast<std::size_t>(r) * m.u.cap + u] : -1;
    const std::size_t at = static_cast<std::size_t>(m.u.list[u]) * a.ld_w + f;
    float4 part[R];
#pragma unroll
    for (int r = 0; r < R; ++r)
      part[r] = rows[r] >= 0 ? *reinterpret_cast<const float4*>(m.dh[r] + static_cast<std::size_t>(rows[r]) * m.ld + f)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 w = *reinterpret_cast<const float4*>(a.w + at);
    float4 mm = *reinterpret_cast<const float4*>(a.m + at);
    float4 v = *reinterpret_cast<const float4*>(a.v + at);
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int r = 0; r < R; ++r) {  // replica order
      s.x += part[r].x;
      s.y += part[r].y;
      s.z += part[r].z;
      s.w += part[r].w;
    }
    if (m.ug) *reinterpret_cast<float4*>(m.ug + static_cast<std::size_t>(u) * m.ld + f) = s;
    adam4(w, mm, v, s, ks, err);
    *reinterpret_cast<float4*>(a.m + at) = mm;
    *reinterpret_cast<float4*>(a.v + at) = v;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (r < a.n_rep) *reinterpret_cast<float4*>(a.peer_w[r] + at) = w;
  }
  if (a.n_rep > 1) __threadfence_system();  // peers read their tables after the replica barrier
}

}  // namespace

void replica_sum_adam(const ReplicaMerge& m, const ReplicaAdam& a, AdamHyper hp, std::uint32_t* err,
                      cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(
      std::max<std::uint64_t>(1, std::min<std::uint64_t>(ceil_div(m.u.cap * ceil_div(m.din, 64), 16), HG_RSUM_WAVES * num_sms())));
  switch (m.n_rep) {
    case 1: launch_pdl(k_rsum_adam<1>, grid, 256, 0, st, m, a, hp, err); break;
    case 2: launch_pdl(k_rsum_adam<2>, grid, 256, 0, st, m, a, hp, err); break;
    case 3: launch_pdl(k_rsum_adam<3>, grid, 256, 0, st, m, a, hp, err); break;
    case 4: launch_pdl(k_rsum_adam<4>, grid, 256, 0, st, m, a, hp, err); break;
    default: launch_pdl(k_rsum_adam<kMaxRep>, grid, 256, 0, st, m, a, hp, err); break;
  }
}

void bump_steps(const std::int64_t* const* steps, const int* const* counts, int n, cudaStream_t st) {
  if (n == 0) return;
  BumpArgs a{};
  for (int i = 0; i < n && i < kMaxSegs; ++i) {
    a.step[i] = const_cast<std::int64_t*>(steps[i]);
    a.n[i] = counts[i];
  }
  a.count = n;
  launch_pdl(k_bump_list, 1, 32, 0, st, a);
}

void adam_model(AdamModelBatch& b, const std::int64_t* step, AdamHyper hp, std::uint32_t* err, cudaStream_t st) {
  if (b.n == 0) return;
  const unsigned grid = static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(
                                                                            ceil_div(b.total4, 256), 4 * num_sms())));
  launch_pdl(k_adam_model, grid, 256, 0, st, b, step, hp, err);
}

void adam_rows(AdamRowsBatch& b, AdamHyper hp, std::uint32_t* err, cudaStream_t st) {
  if (b.n == 0) return;
  launch_pdl(k_bump_steps, 1, 32, 0, st, b);
  const unsigned grid = static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(
                                                                            ceil_div(b.total4, 256), 8 * num_sms())));
  launch_pdl(k_adam_rows, grid, 256, 0, st, b, hp, err);
}

void zero_rows(float* p, int ld, const int* n_rows, int rows_cap, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::max<std::uint64_t>(
      1, std::min<std::uint64_t>(ceil_div(static_cast<std::uint64_t>(rows_cap) * ld, 256), 4 * num_sms())));
  launch_pdl(k_zero_rows, grid, 256, 0, st, p, ld, n_rows);
}

}  // namespace hetgpu
