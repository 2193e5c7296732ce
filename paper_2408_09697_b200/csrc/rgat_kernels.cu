// RGAT kernels (definitions in rgat.cuh). One warp per destination row (forward,
// edge gradients) or per source row (the transposed backward gather); a lane holds
// the row's columns lane, lane + 32, ... in registers. Every sum runs in a fixed
// order (edges ascending, relations ascending, lanes by a fixed butterfly), so the
// results are bit-reproducible.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cfloat>

#include "common.cuh"
#include "rgat.cuh"

namespace hetgpu {

namespace {

constexpr unsigned kFull = 0xffffffffu;
// NU: column registers per lane (row width <= 32 NU), a template parameter so the
// 64-column layers keep their footprint small
constexpr int kRowBitsAtt = 28;       // CSC entries: block << 28 | edge

__device__ __forceinline__ float lrelu(float x) { return x > 0.f ? x : kAttSlope * x; }
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// item -> (group, row) over the groups' row capacities
__device__ __forceinline__ bool group_row(const AttBatch& b, int item, int& g, int& i) {
  g = 0;
  i = item;
  while (g < b.ng && i >= b.g[g].rows_cap) {
    i -= b.g[g].rows_cap;
    ++g;
  }
  return g < b.ng;
}

template <int kU>
__global__ void __launch_bounds__(256) k_att_forward(AttBatch b, int total) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); item < total; item += warps) {
    int g, i;
    if (!group_row(b, item, g, i)) break;
    const AttGroup& G = b.g[g];
    if (i >= *G.n_rows) continue;
    const int H = G.heads, F = G.cols / H, nu = (G.ld + 31) / 32;
    float acc[kU];
    int hc[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      acc[u] = 0.f;
      const int c = lane + 32 * u;
      hc[u] = c < G.cols ? c / F : 0;
    }
    for (int q = 0; q < G.nrel; ++q) {
      const AttRel& R = G.r[q];
      const std::uint32_t lo = R.indptr[i], hi = R.indptr[i + 1];
      if (lo == hi) continue;
      // pass 1: per head, online max / sum over this lane's edges, merged over lanes
      float m[kAttMaxHeads], s[kAttMaxHeads];
#pragma unroll
      for (int h = 0; h < kAttMaxHeads; ++h) {
        m[h] = -FLT_MAX;
        s[h] = 0.f;
      }
      for (std::uint32_t e = lo + lane; e < hi; e += 32) {
        const std::uint32_t j = R.col[e];
#pragma unroll
        for (int h = 0; h < kAttMaxHeads; ++h) {
          if (h >= H) break;
          const float x = lrelu(R.t[static_cast<std::size_t>(j) * H + h]);
          if (x > m[h]) {
            s[h] = s[h] * __expf(m[h] - x) + 1.f;
            m[h] = x;
          } else {
            s[h] += __expf(x - m[h]);
          }
        }
      }
      float lse[kAttMaxHeads];
#pragma unroll
      for (int h = 0; h < kAttMaxHeads; ++h) {
        if (h >= H) break;
        const float M = warp_max(m[h]);
        const float S = warp_sum(s[h] > 0.f ? s[h] * __expf(m[h] - M) : 0.f);
        lse[h] = M + __logf(S);
        if (lane == h) R.lse[static_cast<std::size_t>(i) * H + h] = lse[h];
      }
      // pass 2: 32 edges at a time; lane q owns edge q's weights, the warp sums rows
      for (std::uint32_t base = lo; base < hi; base += 32) {
        const int cnt = static_cast<int>(min(32u, hi - base));
        std::uint32_t my_j = 0;
        float al[kAttMaxHeads];
        if (lane < cnt) {
          my_j = R.col[base + lane];
#pragma unroll
          for (int h = 0; h < kAttMaxHeads; ++h) {
            if (h >= H) break;
            al[h] = __expf(lrelu(R.t[static_cast<std::size_t>(my_j) * H + h]) - lse[h]);
            R.alpha[static_cast<std::size_t>(base + lane) * H + h] = al[h];
          }
        }
        for (int q0 = 0; q0 < cnt; q0 += 4) {
          float zv[4][kU];
          float a4[4][kAttMaxHeads];
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const int qq = min(q0 + w, cnt - 1);
            const std::uint32_t j = __shfl_sync(kFull, my_j, qq);
#pragma unroll
            for (int h = 0; h < kAttMaxHeads; ++h)
              if (h < H) a4[w][h] = __shfl_sync(kFull, al[h], qq);
            const float* zr = R.z + static_cast<std::size_t>(j) * G.ld;
#pragma unroll
            for (int u = 0; u < kU; ++u) zv[w][u] = (u < nu && lane + 32 * u < G.ld) ? zr[lane + 32 * u] : 0.f;
          }
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            if (q0 + w >= cnt) break;
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              float a = a4[w][0];
#pragma unroll
              for (int h = 1; h < kAttMaxHeads; ++h)
                if (h < H && hc[u] == h) a = a4[w][h];
              acc[u] += a * zv[w][u];
            }
          }
        }
      }
    }
    float* o = G.out + static_cast<std::size_t>(i) * G.ld;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int c = lane + 32 * u;
      if (u < nu && c < G.ld) o[c] = (G.relu && acc[u] < 0.f) ? 0.f : acc[u];
    }
  }
}

template <int kU>
__global__ void __launch_bounds__(256) k_att_edge_grad(AttBatch b, int total) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); item < total; item += warps) {
    int g, i;
    if (!group_row(b, item, g, i)) break;
    const AttGroup& G = b.g[g];
    if (i >= *G.n_rows) continue;
    const int H = G.heads, F = G.cols / H, nu = (G.ld + 31) / 32;
    float dv[kU];
    int hc[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int c = lane + 32 * u;
      hc[u] = c < G.cols ? c / F : -1;
      dv[u] = 0.f;
      if (u < nu && c < G.cols) {
        const std::size_t at = static_cast<std::size_t>(i) * G.ld + c;
        dv[u] = G.dout[at];
        if (G.relu_h && G.relu_h[at] <= 0.f) dv[u] = 0.f;
      }
    }
    for (int q = 0; q < G.nrel; ++q) {
      const AttRel& R = G.r[q];
      const std::uint32_t lo = R.indptr[i], hi = R.indptr[i + 1];
      if (lo == hi) continue;
      // pass A: d alpha of every edge (a warp-wide dot per head), kept in dt;
      // c_h = sum_e alpha_e^h d alpha_e^h
      float csum[kAttMaxHeads];
#pragma unroll
      for (int h = 0; h < kAttMaxHeads; ++h) csum[h] = 0.f;
      for (std::uint32_t base = lo; base < hi; base += 32) {
        const int cnt = static_cast<int>(min(32u, hi - base));
        const std::uint32_t my_j = lane < cnt ? R.col[base + lane] : 0u;
        float my_da[kAttMaxHeads];
#pragma unroll
        for (int h = 0; h < kAttMaxHeads; ++h) my_da[h] = 0.f;
        for (int qq = 0; qq < cnt; ++qq) {
          const std::uint32_t j = __shfl_sync(kFull, my_j, qq);
          const float* zr = R.z + static_cast<std::size_t>(j) * G.ld;
          float p[kAttMaxHeads];
#pragma unroll
          for (int h = 0; h < kAttMaxHeads; ++h) p[h] = 0.f;
#pragma unroll
          for (int u = 0; u < kU; ++u)
            if (u < nu && hc[u] >= 0) {
              const float x = dv[u] * zr[lane + 32 * u];
#pragma unroll
              for (int h = 0; h < kAttMaxHeads; ++h)
                if (hc[u] == h) p[h] += x;
            }
#pragma unroll
          for (int h = 0; h < kAttMaxHeads; ++h) {
            if (h >= H) break;
            const float d = warp_sum(p[h]);
            if (lane == qq) my_da[h] = d;
          }
        }
        if (lane < cnt) {
#pragma unroll
          for (int h = 0; h < kAttMaxHeads; ++h) {
            if (h >= H) break;
            const std::size_t at = static_cast<std::size_t>(base + lane) * H + h;
            R.dt[at] = my_da[h];
            csum[h] += R.alpha[at] * my_da[h];
          }
        }
      }
#pragma unroll
      for (int h = 0; h < kAttMaxHeads; ++h)
        if (h < H) csum[h] = warp_sum(csum[h]);
      __syncwarp();
      // pass B: dt = alpha (d alpha - c) LeakyReLU'(t)
      for (std::uint32_t e = lo + lane; e < hi; e += 32) {
        const std::uint32_t j = R.col[e];
#pragma unroll
        for (int h = 0; h < kAttMaxHeads; ++h) {
          if (h >= H) break;
          const std::size_t at = static_cast<std::size_t>(e) * H + h;
          const float x = R.t[static_cast<std::size_t>(j) * H + h];
          R.dt[at] = R.alpha[at] * (R.dt[at] - csum[h]) * (x > 0.f ? 1.f : kAttSlope);
        }
      }
      __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(256) k_att_scores(AttScoreBatch b, int total) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); item < total; item += warps) {
    int q = 0, j = item;
    while (q < b.n && j >= b.j[q].rows_cap) {
      j -= b.j[q].rows_cap;
      ++q;
    }
    if (q >= b.n) break;
    const AttScoreJob& J = b.j[q];
    if (j >= *J.n_rows) continue;
    const int F = J.cols / J.heads;
    const float* zr = J.z + static_cast<std::size_t>(j) * J.ld;
    for (int h = 0; h < J.heads; ++h) {
      float p = 0.f;
      for (int c = h * F + lane; c < (h + 1) * F; c += 32) p += J.a[c] * zr[c];
      p = warp_sum(p);
      if (lane == 0) J.t[static_cast<std::size_t>(j) * J.heads + h] = p;
    }
  }
}

template <int kU>
__device__ __forceinline__ void flush_block(const AttScatterBlock& B, int j, const float* acc, const float* ts,
                                            int lane) {
  const int H = B.heads, F = B.cols / H, nu = (B.ld + 31) / 32;
  float* o = B.dz + static_cast<std::size_t>(j) * B.ld;
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const int c = lane + 32 * u;
    if (u < nu && c < B.ld) {
      float v = 0.f;
      if (c < B.cols) {
        const int h = c / F;
        float th = ts[0];
#pragma unroll
        for (int x = 1; x < kAttMaxHeads; ++x)
          if (x == h) th = ts[x];
        v = acc[u] + th * B.a[c];
      }
      o[c] = v;
    }
  }
  if (lane < H) {
    float th = ts[0];
#pragma unroll
    for (int x = 1; x < kAttMaxHeads; ++x)
      if (x == lane) th = ts[x];
    B.tsum[static_cast<std::size_t>(j) * H + lane] = th;
  }
}

template <int kU>
__global__ void __launch_bounds__(256) k_att_scatter(AttScatter s, int total) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  const float zero[kAttMaxHeads] = {};
  float zacc[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) zacc[u] = 0.f;
  for (int item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); item < total; item += warps) {
    int t = 0, j = item;
    while (t < s.nt && j >= ((s.src_cap[t] + 31) & ~31)) {
      j -= (s.src_cap[t] + 31) & ~31;
      ++t;
    }
    if (t >= s.nt) break;
    const int n = *s.n_src[t];
    if (j >= n) {  // zero rows up to the next multiple of 32 (weight-gradient K chunk)
      if (j < ((n + 31) & ~31))
        for (int bi = 0; bi < s.nb; ++bi)
          if (s.b[bi].type == t) flush_block<kU>(s.b[bi], j, zacc, zero, lane);
      continue;
    }
    const std::uint32_t lo = j ? s.offs[t][j - 1] : 0u, hi = s.offs[t][j];
    int cur = -1;  // block being accumulated
    float acc[kU], ts[kAttMaxHeads];
    auto open = [&](int upto) {  // zero rows for this type's blocks in (cur, upto)
      for (int bi = cur + 1; bi < upto; ++bi)
        if (s.b[bi].type == t) flush_block<kU>(s.b[bi], j, zacc, zero, lane);
    };
    for (std::uint32_t base = lo; base < hi; base += 32) {
      const int cnt = static_cast<int>(min(32u, hi - base));
      std::uint32_t my_key = 0, my_row = 0;
      float my_al[kAttMaxHeads], my_dt[kAttMaxHeads];
      if (lane < cnt) {
        my_key = s.entries[t][base + lane];
        const AttScatterBlock& B = s.b[my_key >> kRowBitsAtt];
        const std::uint32_t e = my_key & ((1u << kRowBitsAtt) - 1);
        my_row = B.erow[e];
#pragma unroll
        for (int h = 0; h < kAttMaxHeads; ++h) {
          my_al[h] = h < B.heads ? B.alpha[static_cast<std::size_t>(e) * B.heads + h] : 0.f;
          my_dt[h] = h < B.heads ? B.dt[static_cast<std::size_t>(e) * B.heads + h] : 0.f;
        }
      }
      for (int qq = 0; qq < cnt; ++qq) {
        const std::uint32_t key = __shfl_sync(kFull, my_key, qq);
        const std::uint32_t row = __shfl_sync(kFull, my_row, qq);
        const int bi = static_cast<int>(key >> kRowBitsAtt);
        if (bi != cur) {
          if (cur >= 0) flush_block<kU>(s.b[cur], j, acc, ts, lane);
          open(bi);
          cur = bi;
#pragma unroll
          for (int u = 0; u < kU; ++u) acc[u] = 0.f;
#pragma unroll
          for (int h = 0; h < kAttMaxHeads; ++h) ts[h] = 0.f;
        }
        const AttScatterBlock& B = s.b[bi];
        const int H = B.heads, F = B.cols / H, nu = (B.ld + 31) / 32;
        float al[kAttMaxHeads];
#pragma unroll
        for (int h = 0; h < kAttMaxHeads; ++h) {
          al[h] = __shfl_sync(kFull, my_al[h], qq);
          ts[h] += __shfl_sync(kFull, my_dt[h], qq);
        }
        const float* dr = B.dout + static_cast<std::size_t>(row) * B.ld_dout;
        const float* mr = B.relu_h ? B.relu_h + static_cast<std::size_t>(row) * B.ld_dout : nullptr;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int c = lane + 32 * u;
          if (u < nu && c < B.cols) {
            float d = dr[c];
            if (mr && mr[c] <= 0.f) d = 0.f;
            const int h = c / F;
            float a = al[0];
#pragma unroll
            for (int x = 1; x < kAttMaxHeads; ++x)
              if (x == h) a = al[x];
            acc[u] += a * d;
          }
        }
      }
    }
    if (cur >= 0) flush_block<kU>(s.b[cur], j, acc, ts, lane);
    open(s.nb);
  }
}

__global__ void __launch_bounds__(128) k_att_da_partial(AttDaBatch b) {
  pdl_enter();
  const AttDaJob& J = b.j[blockIdx.y];
  const int n = *J.n_rows;
  const int r0 = blockIdx.x * kAttDaChunk;
  if (r0 >= n) return;
  const int r1 = min(n, r0 + kAttDaChunk);
  const int F = J.cols / J.heads;
  for (int c = threadIdx.x; c < J.ld; c += blockDim.x) {
    float p = 0.f;
    if (c < J.cols) {
      const int h = c / F;
      for (int r = r0; r < r1; ++r)
        p += J.tsum[static_cast<std::size_t>(r) * J.heads + h] * J.z[static_cast<std::size_t>(r) * J.ld + c];
    }
    J.partial[static_cast<std::size_t>(blockIdx.x) * J.ld + c] = p;
  }
}

__global__ void __launch_bounds__(128) k_att_da_reduce(AttDaBatch b) {
  pdl_enter();
  const AttDaJob& J = b.j[blockIdx.x];
  const int chunks = static_cast<int>(ceil_div(*J.n_rows, kAttDaChunk));
  for (int c = threadIdx.x; c < J.ld; c += blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < chunks; ++k) s += J.partial[static_cast<std::size_t>(k) * J.ld + c];
    J.da[c] = s;
  }
}

__global__ void __launch_bounds__(256) k_leaf_gather(LeafGatherBatch b) {
  pdl_enter();
  const LeafGatherJob& J = b.j[blockIdx.y];
  const std::size_t total = static_cast<std::size_t>(*J.n) * J.ld_out;
  for (std::size_t x = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    const std::size_t i = x / J.ld_out;
    const int c = static_cast<int>(x % J.ld_out);
    float v = 0.f;
    if (c < J.dim) {
      const std::size_t at = static_cast<std::size_t>(J.ids[i]) * J.ld_t + c;
      if (J.dtype == kF32)
        v = static_cast<const float*>(J.table)[at];
      else if (J.dtype == kF16)
        v = __half2float(static_cast<const __half*>(J.table)[at]);
      else
        v = __bfloat162float(static_cast<const __nv_bfloat16*>(J.table)[at]);
    }
    J.out[x] = v;
  }
}

__global__ void __launch_bounds__(256) k_transpose_slots(TransposeBatch b) {
  pdl_enter();
  const TransposeJob& J = b.j[blockIdx.y];
  const int total = J.din * J.dout;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += gridDim.x * blockDim.x) {
    const int i = x / J.dout, c = x % J.dout;
    J.wt[static_cast<std::size_t>(c) * J.ld_wt + i] = J.w[static_cast<std::size_t>(i) * J.ld_w + c];
  }
}

int nu_for(int ld) { return ld <= 64 ? 2 : ld <= 128 ? 4 : ld <= 256 ? 8 : 16; }

unsigned warp_grid(std::uint64_t items) {
  return static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(ceil_div(items, 8), 16 * num_sms())));
}

}  // namespace

void att_forward(const AttBatch& b, cudaStream_t st) {
  int total = 0;
  for (int g = 0; g < b.ng; ++g) {
    if (b.g[g].ld > kAttMaxCols || b.g[g].heads > kAttMaxHeads || b.g[g].heads < 1 || b.g[g].cols % b.g[g].heads)
      throw std::invalid_argument("attention layer shape not supported (cols <= 512, heads <= 8 dividing cols)");
    total += b.g[g].rows_cap;
  }
  if (total == 0) return;
  int ld = 1;
  for (int g = 0; g < b.ng; ++g) ld = std::max(ld, b.g[g].ld);
  switch (nu_for(ld)) {
    case 2: launch_pdl(k_att_forward<2>, warp_grid(total), 256, 0, st, b, total); break;
    case 4: launch_pdl(k_att_forward<4>, warp_grid(total), 256, 0, st, b, total); break;
    case 8: launch_pdl(k_att_forward<8>, warp_grid(total), 256, 0, st, b, total); break;
    default: launch_pdl(k_att_forward<16>, warp_grid(total), 256, 0, st, b, total); break;
  }
}

void att_edge_grad(const AttBatch& b, cudaStream_t st) {
  int total = 0;
  for (int g = 0; g < b.ng; ++g) total += b.g[g].rows_cap;
  if (total == 0) return;
  int ld = 1;
  for (int g = 0; g < b.ng; ++g) ld = std::max(ld, b.g[g].ld);
  switch (nu_for(ld)) {
    case 2: launch_pdl(k_att_edge_grad<2>, warp_grid(total), 256, 0, st, b, total); break;
    case 4: launch_pdl(k_att_edge_grad<4>, warp_grid(total), 256, 0, st, b, total); break;
    case 8: launch_pdl(k_att_edge_grad<8>, warp_grid(total), 256, 0, st, b, total); break;
    default: launch_pdl(k_att_edge_grad<16>, warp_grid(total), 256, 0, st, b, total); break;
  }
}

void att_scores(const AttScoreBatch& b, cudaStream_t st) {
  int total = 0;
  for (int q = 0; q < b.n; ++q) total += b.j[q].rows_cap;
  if (total == 0) return;
  launch_pdl(k_att_scores, warp_grid(total), 256, 0, st, b, total);
}

void att_scatter(const AttScatter& s, cudaStream_t st) {
  int total = 0;
  for (int t = 0; t < s.nt; ++t) total += (s.src_cap[t] + 31) & ~31;
  if (total == 0) return;
  int ld = 1;
  for (int q = 0; q < s.nb; ++q) ld = std::max(ld, s.b[q].ld);
  switch (nu_for(ld)) {
    case 2: launch_pdl(k_att_scatter<2>, warp_grid(total), 256, 0, st, s, total); break;
    case 4: launch_pdl(k_att_scatter<4>, warp_grid(total), 256, 0, st, s, total); break;
    case 8: launch_pdl(k_att_scatter<8>, warp_grid(total), 256, 0, st, s, total); break;
    default: launch_pdl(k_att_scatter<16>, warp_grid(total), 256, 0, st, s, total); break;
  }
}

void att_da(const AttDaBatch& b, cudaStream_t st) {
  if (b.n == 0) return;
  int chunks = 1;
  for (int q = 0; q < b.n; ++q) chunks = std::max(chunks, static_cast<int>(ceil_div(std::max(1, b.j[q].rows_cap), kAttDaChunk)));
  launch_pdl(k_att_da_partial, dim3(chunks, b.n), 128, 0, st, b);
  launch_pdl(k_att_da_reduce, dim3(b.n), 128, 0, st, b);
}

void leaf_gather(const LeafGatherBatch& b, cudaStream_t st) {
  if (b.n == 0) return;
  std::uint64_t most = 1;
  for (int q = 0; q < b.n; ++q) most = std::max<std::uint64_t>(most, static_cast<std::uint64_t>(b.j[q].cap) * b.j[q].ld_out);
  const unsigned gx = static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(most, 256), 8 * num_sms()));
  launch_pdl(k_leaf_gather, dim3(gx, b.n), 256, 0, st, b);
}

void transpose_slots(const TransposeBatch& b, cudaStream_t st) {
  if (b.n == 0) return;
  int most = 1;
  for (int q = 0; q < b.n; ++q) most = std::max(most, b.j[q].din * b.j[q].dout);
  launch_pdl(k_transpose_slots, dim3(static_cast<unsigned>(ceil_div(most, 256)), b.n), 256, 0, st, b);
}

}  // namespace hetgpu
