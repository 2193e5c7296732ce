// RGAT kernels (definitions in rgat.cuh). One half-warp per destination row (forward,
// edge gradients) or per source row (the transposed backward gather); lane l holds
// the float4 columns 4l + 64u of the row in registers. Every sum runs in a fixed
// order (edges ascending, relations ascending, lanes by a fixed butterfly), so the
// results are bit-reproducible.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cfloat>

#include "common.cuh"
#include "rgat.cuh"

namespace hetgpu {

namespace {

constexpr int kRowBitsAtt = 28;       // CSC entries: block << 28 | edge

__device__ __forceinline__ float lrelu(float x) { return x > 0.f ? x : kAttSlope * x; }

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

// Half-warp layout: 16 lanes own a row; lane hl holds the float4 columns 4 hl + 64 u.
// Heads are F = cols / H columns wide (F % 4 == 0 or H == 1), so a float4 lies in one head.
__device__ __forceinline__ float hsum(float v, unsigned m) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(m, v, o, 16);
  return v;
}
__device__ __forceinline__ float hmax(float v, unsigned m) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(m, v, o, 16));
  return v;
}
__device__ __forceinline__ float dot4(const float4 a, const float4 b) {
  return a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w;
}
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float pick(const float* v, int h) {  // v[h] without local memory
  float r = v[0];
#pragma unroll
  for (int x = 1; x < kAttMaxHeads; ++x)
    if (x == h) r = v[x];
  return r;
}

template <int NU4>
__global__ void __launch_bounds__(256) k_att_forward(AttBatch b, int total) {
  pdl_enter();
  constexpr int EIF = NU4 <= 2 ? 4 : 2;  // edges in flight
  const int lane = threadIdx.x & 31, hl = lane & 15;
  const unsigned hm = 0xFFFFu << (lane & 16);
  const int halves = gridDim.x * (blockDim.x >> 4);
  for (int item = blockIdx.x * (blockDim.x >> 4) + (threadIdx.x >> 4); item < total; item += halves) {
    int g, i;
    if (!group_row(b, item, g, i)) break;
    const AttGroup& G = b.g[g];
    if (i >= *G.n_rows) continue;
    const int H = G.heads, F = G.cols / H, nu4 = (G.ld + 63) / 64;
    int hu[NU4];
    float4 acc[NU4];
#pragma unroll
    for (int u = 0; u < NU4; ++u) {
      const int c = 4 * hl + 64 * u;
      hu[u] = c < G.cols ? c / F : 0;
      acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int q = 0; q < G.nrel; ++q) {
      const AttRel& R = G.r[q];
      const std::uint32_t lo = R.indptr[i], hi = R.indptr[i + 1];
      if (lo == hi) continue;
      // pass 1: per head, online max / sum over this lane's edges, merged over the half-warp
      float m[kAttMaxHeads], s[kAttMaxHeads];
#pragma unroll
      for (int h = 0; h < kAttMaxHeads; ++h) {
        m[h] = -FLT_MAX;
        s[h] = 0.f;
      }
      for (std::uint32_t e = lo + hl; e < hi; e += 16) {
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
        lse[h] = 0.f;
        if (h >= H) continue;
        const float M = hmax(m[h], hm);
        const float S = hsum(s[h] > 0.f ? s[h] * __expf(m[h] - M) : 0.f, hm);
        lse[h] = M + __logf(S);
        if (hl == h) R.lse[static_cast<std::size_t>(i) * H + h] = lse[h];
      }
      // pass 2: 16 edges at a time; lane q owns edge q's weights, the half-warp sums rows
      for (std::uint32_t base = lo; base < hi; base += 16) {
        const int cnt = static_cast<int>(min(16u, hi - base));
        std::uint32_t my_j = 0;
        float al[kAttMaxHeads];
#pragma unroll
        for (int h = 0; h < kAttMaxHeads; ++h) al[h] = 0.f;
        if (hl < cnt) {
          my_j = R.col[base + hl];
#pragma unroll
          for (int h = 0; h < kAttMaxHeads; ++h) {
            if (h >= H) break;
            al[h] = __expf(lrelu(R.t[static_cast<std::size_t>(my_j) * H + h]) - lse[h]);
            R.alpha[static_cast<std::size_t>(base + hl) * H + h] = al[h];
          }
        }
        for (int q0 = 0; q0 < cnt; q0 += EIF) {
          float4 zv[EIF][NU4];
          float aw[EIF][NU4];
#pragma unroll
          for (int w = 0; w < EIF; ++w) {
            const int qq = min(q0 + w, cnt - 1);
            const std::uint32_t j = __shfl_sync(hm, my_j, qq, 16);
            float ah[kAttMaxHeads];
#pragma unroll
            for (int h = 0; h < kAttMaxHeads; ++h) ah[h] = h < H ? __shfl_sync(hm, al[h], qq, 16) : 0.f;
            const float* zr = R.z + static_cast<std::size_t>(j) * G.ld;
#pragma unroll
            for (int u = 0; u < NU4; ++u) {
              const int c = 4 * hl + 64 * u;
              zv[w][u] = (u < nu4 && c < G.ld) ? ld4(zr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
              aw[w][u] = pick(ah, hu[u]);
            }
          }
#pragma unroll
          for (int w = 0; w < EIF; ++w) {
            if (q0 + w >= cnt) break;
#pragma unroll
            for (int u = 0; u < NU4; ++u) {
              acc[u].x += aw[w][u] * zv[w][u].x;
              acc[u].y += aw[w][u] * zv[w][u].y;
              acc[u].z += aw[w][u] * zv[w][u].z;
              acc[u].w += aw[w][u] * zv[w][u].w;
            }
          }
        }
      }
    }
    float* o = G.out + static_cast<std::size_t>(i) * G.ld;
#pragma unroll
    for (int u = 0; u < NU4; ++u) {
      const int c = 4 * hl + 64 * u;
      if (u < nu4 && c < G.ld) {
        float4 v = acc[u];
        if (G.relu) {
          v.x = fmaxf(v.x, 0.f);
          v.y = fmaxf(v.y, 0.f);
          v.z = fmaxf(v.z, 0.f);
          v.w = fmaxf(v.w, 0.f);
        }
        *reinterpret_cast<float4*>(o + c) = v;
      }
    }
  }
}

template <int NU4>
__global__ void __launch_bounds__(256) k_att_edge_grad(AttBatch b, int total) {
  pdl_enter();
  constexpr int EIF = NU4 <= 2 ? 4 : 2;
  const int lane = threadIdx.x & 31, hl = lane & 15;
  const unsigned hm = 0xFFFFu << (lane & 16);
  const int halves = gridDim.x * (blockDim.x >> 4);
  for (int item = blockIdx.x * (blockDim.x >> 4) + (threadIdx.x >> 4); item < total; item += halves) {
    int g, i;
    if (!group_row(b, item, g, i)) break;
    const AttGroup& G = b.g[g];
    if (i >= *G.n_rows) continue;
    const int H = G.heads, F = G.cols / H, nu4 = (G.ld + 63) / 64;
    // one float4 per lane and heads of 4..64 columns: a head is an aligned group of F/4 lanes
    const int gsz = F / 4;
    const bool seg = NU4 == 1 && H > 1 && F % 4 == 0 && gsz <= 16 && (gsz & (gsz - 1)) == 0;
    int hu[NU4];
    float4 dv[NU4];
#pragma unroll
    for (int u = 0; u < NU4; ++u) {
      const int c = 4 * hl + 64 * u;
      hu[u] = c < G.cols ? c / F : -1;
      dv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (u < nu4 && c < G.ld) {
        const std::size_t at = static_cast<std::size_t>(i) * G.ld + c;
        dv[u] = ld4(G.dout + at);
        if (G.relu_h) {
          const float4 hv = ld4(G.relu_h + at);
          if (hv.x <= 0.f) dv[u].x = 0.f;
          if (hv.y <= 0.f) dv[u].y = 0.f;
          if (hv.z <= 0.f) dv[u].z = 0.f;
          if (hv.w <= 0.f) dv[u].w = 0.f;
        }
      }
    }
    for (int q = 0; q < G.nrel; ++q) {
      const AttRel& R = G.r[q];
      const std::uint32_t lo = R.indptr[i], hi = R.indptr[i + 1];
      if (lo == hi) continue;
      // pass A: d alpha of every edge (a dot per head over the half-warp), kept in dt;
      // c_h = sum_e alpha_e^h d alpha_e^h
      float csum[kAttMaxHeads];
#pragma unroll
      for (int h = 0; h < kAttMaxHeads; ++h) csum[h] = 0.f;
      for (std::uint32_t base = lo; base < hi; base += 16) {
        const int cnt = static_cast<int>(min(16u, hi - base));
        const std::uint32_t my_j = hl < cnt ? R.col[base + hl] : 0u;
        float my_da[kAttMaxHeads];
#pragma unroll
        for (int h = 0; h < kAttMaxHeads; ++h) my_da[h] = 0.f;
        for (int q0 = 0; q0 < cnt; q0 += EIF) {
          float4 zv[EIF][NU4];
#pragma unroll
          for (int w = 0; w < EIF; ++w) {
            const int qq = min(q0 + w, cnt - 1);
            const std::uint32_t j = __shfl_sync(hm, my_j, qq, 16);
            const float* zr = R.z + static_cast<std::size_t>(j) * G.ld;
#pragma unroll
            for (int u = 0; u < NU4; ++u) {
              const int c = 4 * hl + 64 * u;
              zv[w][u] = (u < nu4 && c < G.ld) ? ld4(zr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
#pragma unroll
          for (int w = 0; w < EIF; ++w) {
            if (q0 + w >= cnt) break;
            if (seg) {
              float p = dot4(dv[0], zv[w][0]);
              for (int o = gsz >> 1; o > 0; o >>= 1) p += __shfl_xor_sync(hm, p, o, 16);
#pragma unroll
              for (int h = 0; h < kAttMaxHeads; ++h) {
                if (h >= H) break;
                const float d = __shfl_sync(hm, p, h * gsz, 16);
                if (hl == q0 + w) my_da[h] = d;
              }
            } else {
#pragma unroll
              for (int h = 0; h < kAttMaxHeads; ++h) {
                if (h >= H) break;
                float p = 0.f;
#pragma unroll
                for (int u = 0; u < NU4; ++u)
                  if (hu[u] == h) p += dot4(dv[u], zv[w][u]);
                p = hsum(p, hm);
                if (hl == q0 + w) my_da[h] = p;
              }
            }
          }
        }
        if (hl < cnt) {
#pragma unroll
          for (int h = 0; h < kAttMaxHeads; ++h) {
            if (h >= H) break;
            const std::size_t at = static_cast<std::size_t>(base + hl) * H + h;
            R.dt[at] = my_da[h];
            csum[h] += R.alpha[at] * my_da[h];
          }
        }
      }
#pragma unroll
      for (int h = 0; h < kAttMaxHeads; ++h)
        if (h < H) csum[h] = hsum(csum[h], hm);
      __syncwarp(hm);
      // pass B: dt = alpha (d alpha - c) LeakyReLU'(t)
      for (std::uint32_t e = lo + hl; e < hi; e += 16) {
        const std::uint32_t j = R.col[e];
#pragma unroll
        for (int h = 0; h < kAttMaxHeads; ++h) {
          if (h >= H) break;
          const std::size_t at = static_cast<std::size_t>(e) * H + h;
          const float x = R.t[static_cast<std::size_t>(j) * H + h];
          R.dt[at] = R.alpha[at] * (R.dt[at] - csum[h]) * (x > 0.f ? 1.f : kAttSlope);
        }
      }
      __syncwarp(hm);
    }
  }
}

// one thread per (source row, head): t = a^(h) . z^(h)
__global__ void __launch_bounds__(256) k_att_scores(AttScoreBatch b) {
  pdl_enter();
  const AttScoreJob& J = b.j[blockIdx.y];
  const int H = J.heads, F = J.cols / H;
  const std::int64_t total = static_cast<std::int64_t>(*J.n_rows) * H;
  for (std::int64_t x = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t row = x / H;
    const int h = static_cast<int>(x % H);
    const float* zr = J.z + row * J.ld + h * F;
    const float* a = J.a + h * F;
    float p = 0.f;
    if (F % 4 == 0) {
      for (int c = 0; c < F; c += 4) p += dot4(ld4(zr + c), ld4(a + c));
    } else {
      for (int c = 0; c < F; ++c) p += zr[c] * a[c];
    }
    J.t[x] = p;
  }
}

template <int NU4>
__device__ __forceinline__ void flush_block(const AttScatterBlock& B, int j, const float4* acc, const float* ts,
                                            int hl) {
  const int H = B.heads, F = B.cols / H, nu4 = (B.ld + 63) / 64;
  float* o = B.dz + static_cast<std::size_t>(j) * B.ld;
#pragma unroll
  for (int u = 0; u < NU4; ++u) {
    const int c = 4 * hl + 64 * u;
    if (u < nu4 && c < B.ld) {
      const float th = c < B.cols ? pick(ts, c / F) : 0.f;
      const float4 a = ld4(B.a + c);
      float4 v = acc[u];
      v.x += th * a.x;
      v.y += th * a.y;
      v.z += th * a.z;
      v.w += th * a.w;
      *reinterpret_cast<float4*>(o + c) = v;
    }
  }
  if (hl < H) B.tsum[static_cast<std::size_t>(j) * H + hl] = pick(ts, hl);
}

template <int NU4>
__global__ void __launch_bounds__(256) k_att_scatter(AttScatter s, int total) {
  pdl_enter();
  const int lane = threadIdx.x & 31, hl = lane & 15;
  const unsigned hm = 0xFFFFu << (lane & 16);
  const int halves = gridDim.x * (blockDim.x >> 4);
  const float zero[kAttMaxHeads] = {};
  float4 zacc[NU4];
#pragma unroll
  for (int u = 0; u < NU4; ++u) zacc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int item = blockIdx.x * (blockDim.x >> 4) + (threadIdx.x >> 4); item < total; item += halves) {
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
          if (s.b[bi].type == t) flush_block<NU4>(s.b[bi], j, zacc, zero, hl);
      continue;
    }
    const std::uint32_t lo = j ? s.offs[t][j - 1] : 0u, hi = s.offs[t][j];
    int cur = -1;  // block being accumulated
    float4 acc[NU4];
    float ts[kAttMaxHeads];
#pragma unroll
    for (int u = 0; u < NU4; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int h = 0; h < kAttMaxHeads; ++h) ts[h] = 0.f;
    for (std::uint32_t base = lo; base < hi; base += 16) {
      const int cnt = static_cast<int>(min(16u, hi - base));
      std::uint32_t my_key = 0, my_row = 0;
      float my_al[kAttMaxHeads], my_dt[kAttMaxHeads];
#pragma unroll
      for (int h = 0; h < kAttMaxHeads; ++h) my_al[h] = my_dt[h] = 0.f;
      if (hl < cnt) {
        my_key = s.entries[t][base + hl];
        const AttScatterBlock& B = s.b[my_key >> kRowBitsAtt];
        const std::uint32_t e = my_key & ((1u << kRowBitsAtt) - 1);
        my_row = B.erow[e];
#pragma unroll
        for (int h = 0; h < kAttMaxHeads; ++h)
          if (h < B.heads) {
            my_al[h] = B.alpha[static_cast<std::size_t>(e) * B.heads + h];
            my_dt[h] = B.dt[static_cast<std::size_t>(e) * B.heads + h];
          }
      }
      for (int qq = 0; qq < cnt; ++qq) {
        const std::uint32_t key = __shfl_sync(hm, my_key, qq, 16);
        const std::uint32_t row = __shfl_sync(hm, my_row, qq, 16);
        const int bi = static_cast<int>(key >> kRowBitsAtt);
        if (bi != cur) {
          if (cur >= 0) flush_block<NU4>(s.b[cur], j, acc, ts, hl);
          for (int x = cur + 1; x < bi; ++x)
            if (s.b[x].type == t) flush_block<NU4>(s.b[x], j, zacc, zero, hl);
          cur = bi;
#pragma unroll
          for (int u = 0; u < NU4; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int h = 0; h < kAttMaxHeads; ++h) ts[h] = 0.f;
        }
        const AttScatterBlock& B = s.b[bi];
        const int H = B.heads, F = B.cols / H, nu4 = (B.ld + 63) / 64;
        float al[kAttMaxHeads];
#pragma unroll
        for (int h = 0; h < kAttMaxHeads; ++h) {
          al[h] = __shfl_sync(hm, my_al[h], qq, 16);
          ts[h] += __shfl_sync(hm, my_dt[h], qq, 16);
        }
        const float* dr = B.dout + static_cast<std::size_t>(row) * B.ld_dout;
        const float* mr = B.relu_h ? B.relu_h + static_cast<std::size_t>(row) * B.ld_dout : nullptr;
        float4 d4[NU4];
#pragma unroll
        for (int u = 0; u < NU4; ++u) {
          const int c = 4 * hl + 64 * u;
          d4[u] = (u < nu4 && c < B.ld) ? ld4(dr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < NU4; ++u) {
          const int c = 4 * hl + 64 * u;
          if (u < nu4 && c < B.cols) {
            float4 d = d4[u];
            if (mr) {
              const float4 hv = ld4(mr + c);
              if (hv.x <= 0.f) d.x = 0.f;
              if (hv.y <= 0.f) d.y = 0.f;
              if (hv.z <= 0.f) d.z = 0.f;
              if (hv.w <= 0.f) d.w = 0.f;
            }
            const float a = pick(al, c / F);
            acc[u].x += a * d.x;
            acc[u].y += a * d.y;
            acc[u].z += a * d.z;
            acc[u].w += a * d.w;
          }
        }
      }
    }
    if (cur >= 0) flush_block<NU4>(s.b[cur], j, acc, ts, hl);
    for (int x = cur + 1; x < s.nb; ++x)
      if (s.b[x].type == t) flush_block<NU4>(s.b[x], j, zacc, zero, hl);
  }
}

// da partials: CTA = one chunk of kAttDaChunk rows of one job; 16 row groups x 16 float4
// columns (16 independent rows in flight per thread), combined in a fixed order
__global__ void __launch_bounds__(256) k_att_da_partial(AttDaBatch b) {
  pdl_enter();
  __shared__ float4 part[16][kAttMaxCols / 4];
  const AttDaJob& J = b.j[blockIdx.y];
  const int n = *J.n_rows;
  const int r0 = blockIdx.x * kAttDaChunk;
  if (r0 >= n) return;
  const int F = J.cols / J.heads, nf4 = J.ld / 4;
  const int cf = threadIdx.x & 15, rg = threadIdx.x >> 4;
  for (int f = cf; f < nf4; f += 16) {
    const int c = 4 * f;
    const int h = c < J.cols ? c / F : 0;
    float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
    for (int k = 0; k < kAttDaChunk / 16; ++k) {
      const int r = r0 + rg + 16 * k;
      if (r < n) {
        const float ts = J.tsum[static_cast<std::size_t>(r) * J.heads + h];
        const float4 z = ld4(J.z + static_cast<std::size_t>(r) * J.ld + c);
        p.x += ts * z.x;
        p.y += ts * z.y;
        p.z += ts * z.z;
        p.w += ts * z.w;
      }
    }
    part[rg][f] = p;
  }
  __syncthreads();
  for (int f = threadIdx.x; f < nf4; f += blockDim.x) {
    float4 s = part[0][f];
    for (int g = 1; g < 16; ++g) {
      s.x += part[g][f].x;
      s.y += part[g][f].y;
      s.z += part[g][f].z;
      s.w += part[g][f].w;
    }
    *reinterpret_cast<float4*>(J.partial + static_cast<std::size_t>(blockIdx.x) * J.ld + 4 * f) = s;
  }
}

__global__ void __launch_bounds__(256) k_att_da_reduce(AttDaBatch b) {
  pdl_enter();
  __shared__ float4 part[16][kAttMaxCols / 4];
  const AttDaJob& J = b.j[blockIdx.x];
  const int chunks = static_cast<int>(ceil_div(*J.n_rows, kAttDaChunk));
  const int nf4 = J.ld / 4;
  const int cf = threadIdx.x & 15, rg = threadIdx.x >> 4;
  for (int f = cf; f < nf4; f += 16) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = rg; k < chunks; k += 16) {
      const float4 v = ld4(J.partial + static_cast<std::size_t>(k) * J.ld + 4 * f);
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
    part[rg][f] = s;
  }
  __syncthreads();
  for (int f = threadIdx.x; f < nf4; f += blockDim.x) {
    float4 s = part[0][f];
    for (int g = 1; g < 16; ++g) {
      s.x += part[g][f].x;
      s.y += part[g][f].y;
      s.z += part[g][f].z;
      s.w += part[g][f].w;
    }
    *reinterpret_cast<float4*>(J.da + 4 * f) = s;
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

int nu4_for(int ld) { return ld <= 64 ? 1 : ld <= 128 ? 2 : ld <= 256 ? 4 : 8; }

unsigned half_grid(std::uint64_t items) {
  return static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(ceil_div(items, 16), 16 * num_sms())));
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
  switch (nu4_for(ld)) {
    case 1: launch_pdl(k_att_forward<1>, half_grid(total), 256, 0, st, b, total); break;
    case 2: launch_pdl(k_att_forward<2>, half_grid(total), 256, 0, st, b, total); break;
    case 4: launch_pdl(k_att_forward<4>, half_grid(total), 256, 0, st, b, total); break;
    default: launch_pdl(k_att_forward<8>, half_grid(total), 256, 0, st, b, total); break;
  }
}

void att_edge_grad(const AttBatch& b, cudaStream_t st) {
  int total = 0;
  for (int g = 0; g < b.ng; ++g) total += b.g[g].rows_cap;
  if (total == 0) return;
  int ld = 1;
  for (int g = 0; g < b.ng; ++g) ld = std::max(ld, b.g[g].ld);
  switch (nu4_for(ld)) {
    case 1: launch_pdl(k_att_edge_grad<1>, half_grid(total), 256, 0, st, b, total); break;
    case 2: launch_pdl(k_att_edge_grad<2>, half_grid(total), 256, 0, st, b, total); break;
    case 4: launch_pdl(k_att_edge_grad<4>, half_grid(total), 256, 0, st, b, total); break;
    default: launch_pdl(k_att_edge_grad<8>, half_grid(total), 256, 0, st, b, total); break;
  }
}

void att_scores(const AttScoreBatch& b, cudaStream_t st) {
  if (b.n == 0) return;
  std::uint64_t most = 1;
  for (int q = 0; q < b.n; ++q) most = std::max<std::uint64_t>(most, static_cast<std::uint64_t>(b.j[q].rows_cap) * b.j[q].heads);
  const unsigned gx = static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(most, 256), 8 * num_sms()));
  launch_pdl(k_att_scores, dim3(gx, b.n), 256, 0, st, b);
}

void att_scatter(const AttScatter& s, cudaStream_t st) {
  int total = 0;
  for (int t = 0; t < s.nt; ++t) total += (s.src_cap[t] + 31) & ~31;
  if (total == 0) return;
  int ld = 1;
  for (int q = 0; q < s.nb; ++q) ld = std::max(ld, s.b[q].ld);
  switch (nu4_for(ld)) {
    case 1: launch_pdl(k_att_scatter<1>, half_grid(total), 256, 0, st, s, total); break;
    case 2: launch_pdl(k_att_scatter<2>, half_grid(total), 256, 0, st, s, total); break;
    case 4: launch_pdl(k_att_scatter<4>, half_grid(total), 256, 0, st, s, total); break;
    default: launch_pdl(k_att_scatter<8>, half_grid(total), 256, 0, st, s, total); break;
  }
}

void att_da(const AttDaBatch& b, cudaStream_t st) {
  if (b.n == 0) return;
  int chunks = 1;
  for (int q = 0; q < b.n; ++q) chunks = std::max(chunks, static_cast<int>(ceil_div(std::max(1, b.j[q].rows_cap), kAttDaChunk)));
  launch_pdl(k_att_da_partial, dim3(chunks, b.n), 256, 0, st, b);
  launch_pdl(k_att_da_reduce, dim3(b.n), 256, 0, st, b);
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
