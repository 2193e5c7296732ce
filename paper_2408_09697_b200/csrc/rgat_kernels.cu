// RGAT kernels (definitions in rgat.cuh). One half-warp per destination row (the
// aggregate-first forward and edge gradients) or a 16/32-lane group per source row (the
// transposed backward gather); lane l holds the float4 columns 4l + 4 GL u of the row in
// registers. Every sum runs in a fixed order (edges ascending, relations ascending, lanes
// by a fixed butterfly, partials by index), so the results are bit-reproducible.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cfloat>

#include "common.cuh"
#include "rgat.cuh"

namespace hetgpu {

namespace {

constexpr int kRowBitsAtt = 28;       // CSC entries: block << 28 | edge

__device__ __forceinline__ float lrelu(float x) { return x > 0.f ? x : kAttSlope * x; }

// Half-warp layout: 16 lanes own a row; lane hl holds the float4 columns 4 hl + 64 u.
// Heads are F = cols / H columns wide (F % 4 == 0 or H == 1), so a float4 lies in one head.
__device__ __forceinline__ float hsum(float v, unsigned m) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(m, v, o, 16);
  return v;
}
template <int G>
__device__ __forceinline__ float gsum(float v, unsigned m) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(m, v, o, G);
  return v;
}
template <int G>
__device__ __forceinline__ unsigned group_mask(int lane) {
  return G == 32 ? 0xffffffffu : (0xFFFFu << (lane & 16));
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

template <int GL, int NU4>
__device__ __forceinline__ void flush_block(const AttScatterBlock& B, int j, const float4* acc, const float* ts,
                                            int hl) {
  const int H = B.heads, F = B.cols / H, nu4 = (B.ld + 4 * GL - 1) / (4 * GL);
  float* o = B.dz + static_cast<std::size_t>(j) * B.ld;
#pragma unroll
  for (int u = 0; u < NU4; ++u) {
    const int c = 4 * hl + 4 * GL * u;
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

template <int GL, int NU4>
__global__ void __launch_bounds__(256) k_att_scatter(AttScatter s, int total) {
  pdl_enter();
  const int lane = threadIdx.x & 31, hl = lane & (GL - 1);
  const unsigned hm = group_mask<GL>(lane);
  const int halves = gridDim.x * (blockDim.x / GL);
  const float zero[kAttMaxHeads] = {};
  float4 zacc[NU4];
#pragma unroll
  for (int u = 0; u < NU4; ++u) zacc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int item = blockIdx.x * (blockDim.x / GL) + (threadIdx.x / GL); item < total; item += halves) {
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
          if (s.b[bi].type == t) flush_block<GL, NU4>(s.b[bi], j, zacc, zero, hl);
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
    for (std::uint32_t base = lo; base < hi; base += GL) {
      const int cnt = static_cast<int>(min(static_cast<std::uint32_t>(GL), hi - base));
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
        const std::uint32_t key = __shfl_sync(hm, my_key, qq, GL);
        const std::uint32_t row = __shfl_sync(hm, my_row, qq, GL);
        const int bi = static_cast<int>(key >> kRowBitsAtt);
        if (bi != cur) {
          if (cur >= 0) flush_block<GL, NU4>(s.b[cur], j, acc, ts, hl);
          for (int x = cur + 1; x < bi; ++x)
            if (s.b[x].type == t) flush_block<GL, NU4>(s.b[x], j, zacc, zero, hl);
          cur = bi;
#pragma unroll
          for (int u = 0; u < NU4; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int h = 0; h < kAttMaxHeads; ++h) ts[h] = 0.f;
        }
        const AttScatterBlock& B = s.b[bi];
        const int H = B.heads, F = B.cols / H, nu4 = (B.ld + 4 * GL - 1) / (4 * GL);
        float al[kAttMaxHeads];
#pragma unroll
        for (int h = 0; h < kAttMaxHeads; ++h) {
          al[h] = __shfl_sync(hm, my_al[h], qq, GL);
          ts[h] += __shfl_sync(hm, my_dt[h], qq, GL);
        }
        const std::size_t drow = static_cast<std::size_t>(row) * B.row_stride + B.row_offset;
        const float* dr = B.dout + drow * B.ld_dout;
        const float* mr = B.relu_h ? B.relu_h + drow * B.ld_dout : nullptr;
        float4 d4[NU4];
#pragma unroll
        for (int u = 0; u < NU4; ++u) {
          const int c = 4 * hl + 4 * GL * u;
          d4[u] = (u < nu4 && c < B.ld) ? ld4(dr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < NU4; ++u) {
          const int c = 4 * hl + 4 * GL * u;
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
    if (cur >= 0) flush_block<GL, NU4>(s.b[cur], j, acc, ts, hl);
    for (int x = cur + 1; x < s.nb; ++x)
      if (s.b[x].type == t) flush_block<GL, NU4>(s.b[x], j, zacc, zero, hl);
  }
}

// ---- layer 1, aggregate first (rgat.cuh) ------------------------------------------------
__device__ __forceinline__ float4 load_x4(const void* table, int dtype, std::size_t at) {
  if (dtype == kF32) return ld4(static_cast<const float*>(table) + at);
  const uint2 r = *reinterpret_cast<const uint2*>(static_cast<const unsigned short*>(table) + at);
  float2 lo, hi;
  if (dtype == kF16) {
    lo = __half22float2(*reinterpret_cast<const __half2*>(&r.x));
    hi = __half22float2(*reinterpret_cast<const __half2*>(&r.y));
  } else {
    lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.x));
    hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.y));
  }
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}
__device__ __forceinline__ int round32i(int x) { return (x + 31) & ~31; }

#ifndef HG_ATT_MINB
#define HG_ATT_MINB 3  // forward: 3 CTAs per SM (80 registers) measured 198 -> 187 us/step on C3
#endif
template <int H, int NU4>
__global__ void __launch_bounds__(256, HG_ATT_MINB) k_att_leaf_forward(AttLeafBatch b, int total) {
  pdl_enter();
  const int lane = threadIdx.x & 31, hl = lane & 15;
  const unsigned hm = 0xFFFFu << (lane & 16);
  const int halves = gridDim.x * (blockDim.x >> 4);
  for (int item = blockIdx.x * (blockDim.x >> 4) + (threadIdx.x >> 4); item < total; item += halves) {
    int q = 0, i = item;
    while (q < b.n && i >= round32i(b.j[q].rows_cap)) {
      i -= round32i(b.j[q].rows_cap);
      ++q;
    }
    if (q >= b.n) break;
    const AttLeafJob& J = b.j[q];
    const int n = *J.n_rows;
    const int ldg = H * J.din_p;
    float* arow = J.agg + static_cast<std::size_t>(i) * ldg;
    if (i >= n) {  // zero rows up to the next multiple of 32 (weight-gradient K chunks)
      if (i < round32i(n))
        for (int c = 4 * hl; c < ldg; c += 64) *reinterpret_cast<float4*>(arow + c) = make_float4(0.f, 0.f, 0.f, 0.f);
      continue;
    }
    float4 qv[H][NU4], acc[H][NU4];
    float m[H], s[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      m[h] = -FLT_MAX;
      s[h] = 0.f;
#pragma unroll
      for (int u = 0; u < NU4; ++u) {
        const int c = 4 * hl + 64 * u;
        qv[h][u] = c < J.din_p ? ld4(J.q + h * J.din_p + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        acc[h][u] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    const std::uint32_t lo = J.indptr[i], hi = J.indptr[i + 1];
    auto step = [&](std::uint32_t e, const float4* x) {
#pragma unroll
      for (int h = 0; h < H; ++h) {
        float p = 0.f;
#pragma unroll
        for (int u = 0; u < NU4; ++u) p += dot4(qv[h][u], x[u]);
        const float t = hsum(p, hm);
        if (hl == h) J.te[static_cast<std::size_t>(e) * H + h] = t;
        const float xl = lrelu(t);
        if (xl > m[h]) {  // uniform over the half-warp (t is)
          const float sc = __expf(m[h] - xl);
          s[h] = s[h] * sc + 1.f;
          m[h] = xl;
#pragma unroll
          for (int u = 0; u < NU4; ++u) {
            acc[h][u].x = acc[h][u].x * sc + x[u].x;
            acc[h][u].y = acc[h][u].y * sc + x[u].y;
            acc[h][u].z = acc[h][u].z * sc + x[u].z;
            acc[h][u].w = acc[h][u].w * sc + x[u].w;
          }
        } else {
          const float w = __expf(xl - m[h]);
          s[h] += w;
#pragma unroll
          for (int u = 0; u < NU4; ++u) {
            acc[h][u].x += w * x[u].x;
            acc[h][u].y += w * x[u].y;
            acc[h][u].z += w * x[u].z;
            acc[h][u].w += w * x[u].w;
          }
        }
      }
    };
    // keys of 16 edges at a time, rows of two edges in flight
    for (std::uint32_t base = lo; base < hi; base += 16) {
      const int cnt = static_cast<int>(min(16u, hi - base));
      const std::uint32_t my_key = hl < cnt ? J.keys[base + hl] : 0u;
      for (int qq = 0; qq < cnt; qq += 2) {
        const std::size_t r0 = static_cast<std::size_t>(__shfl_sync(hm, my_key, qq, 16)) * J.ld_t;
        const std::size_t r1 = static_cast<std::size_t>(__shfl_sync(hm, my_key, min(qq + 1, cnt - 1), 16)) * J.ld_t;
        float4 x0[NU4], x1[NU4];
#pragma unroll
        for (int u = 0; u < NU4; ++u) {
          const int c = 4 * hl + 64 * u;
          const bool in = c < J.din_p;
          x0[u] = in ? load_x4(J.table, J.dtype, r0 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
          x1[u] = in ? load_x4(J.table, J.dtype, r1 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        step(base + qq, x0);
        if (qq + 1 < cnt) step(base + qq + 1, x1);
      }
    }
    float lse[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      lse[h] = lo < hi ? m[h] + __logf(s[h]) : 0.f;
      if (hl == h) J.lse[static_cast<std::size_t>(i) * H + h] = lse[h];
      const float inv = lo < hi ? 1.f / s[h] : 0.f;
#pragma unroll
      for (int u = 0; u < NU4; ++u) {
        const int c = 4 * hl + 64 * u;
        if (c < J.din_p)
          *reinterpret_cast<float4*>(arow + h * J.din_p + c) =
              make_float4(acc[h][u].x * inv, acc[h][u].y * inv, acc[h][u].z * inv, acc[h][u].w * inv);
      }
    }
    __syncwarp(hm);  // te of this row's edges (written by this half-warp) -> alpha
    for (std::uint32_t e = lo + hl; e < hi; e += 16)
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const std::size_t at = static_cast<std::size_t>(e) * H + h;
        J.alpha[at] = __expf(lrelu(J.te[at]) - lse[h]);
      }
  }
}

template <int H, int NU4>
__global__ void __launch_bounds__(256) k_att_leaf_grad(AttLeafBatch b) {
  pdl_enter();
  const int lane = threadIdx.x & 31, hl = lane & 15;
  const unsigned hm = 0xFFFFu << (lane & 16);
  const int halves = gridDim.x * (blockDim.x >> 4);
  const int me = blockIdx.x * (blockDim.x >> 4) + (threadIdx.x >> 4);
  for (int q = 0; q < b.n; ++q) {
    const AttLeafJob& J = b.j[q];
    const int n = *J.n_rows;
    const int ldg = H * J.din_p;
    float4 dq[H][NU4];
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
      for (int u = 0; u < NU4; ++u) dq[h][u] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = me; i < n; i += halves) {
      const std::uint32_t lo = J.indptr[i], hi = J.indptr[i + 1];
      if (lo == hi) continue;
      float4 dg[H][NU4];
      float cs[H], ls[H];
#pragma unroll
      for (int h = 0; h < H; ++h) {
        float p = 0.f;
#pragma unroll
        for (int u = 0; u < NU4; ++u) {
          const int c = 4 * hl + 64 * u;
          const std::size_t at = static_cast<std::size_t>(i) * ldg + h * J.din_p + c;
          dg[h][u] = c < J.din_p ? ld4(J.dagg + at) : make_float4(0.f, 0.f, 0.f, 0.f);
          if (c < J.din_p) p += dot4(dg[h][u], ld4(J.agg + at));
        }
        cs[h] = hsum(p, hm);  // c_h = dagg^h . agg^h = sum_e alpha d alpha
        ls[h] = J.lse[static_cast<std::size_t>(i) * H + h];
      }
      auto step = [&](std::uint32_t e, const float4* x, const float* te) {
#pragma unroll
        for (int h = 0; h < H; ++h) {
          float p = 0.f;
#pragma unroll
          for (int u = 0; u < NU4; ++u) p += dot4(dg[h][u], x[u]);
          const float da = hsum(p, hm);
          const float t = te[h];
          const float al = __expf(lrelu(t) - ls[h]);
          const float d = al * (da - cs[h]) * (t > 0.f ? 1.f : kAttSlope);
          if (hl == h) J.dt[static_cast<std::size_t>(e) * H + h] = d;
#pragma unroll
          for (int u = 0; u < NU4; ++u) {
            dq[h][u].x += d * x[u].x;
            dq[h][u].y += d * x[u].y;
            dq[h][u].z += d * x[u].z;
            dq[h][u].w += d * x[u].w;
          }
        }
      };
      for (std::uint32_t base = lo; base < hi; base += 16) {
        const int cnt = static_cast<int>(min(16u, hi - base));
        std::uint32_t my_key = 0;
        float my_te[H];
#pragma unroll
        for (int h = 0; h < H; ++h) my_te[h] = 0.f;
        if (hl < cnt) {
          my_key = J.keys[base + hl];
#pragma unroll
          for (int h = 0; h < H; ++h) my_te[h] = J.te[static_cast<std::size_t>(base + hl) * H + h];
        }
        for (int qq = 0; qq < cnt; qq += 2) {
          const int q1 = min(qq + 1, cnt - 1);
          const std::size_t r0 = static_cast<std::size_t>(__shfl_sync(hm, my_key, qq, 16)) * J.ld_t;
          const std::size_t r1 = static_cast<std::size_t>(__shfl_sync(hm, my_key, q1, 16)) * J.ld_t;
          float t0[H], t1[H];
#pragma unroll
          for (int h = 0; h < H; ++h) {
            t0[h] = __shfl_sync(hm, my_te[h], qq, 16);
            t1[h] = __shfl_sync(hm, my_te[h], q1, 16);
          }
          float4 x0[NU4], x1[NU4];
#pragma unroll
          for (int u = 0; u < NU4; ++u) {
            const int c = 4 * hl + 64 * u;
            const bool in = c < J.din_p;
            x0[u] = in ? load_x4(J.table, J.dtype, r0 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
            x1[u] = in ? load_x4(J.table, J.dtype, r1 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
          step(base + qq, x0, t0);
          if (qq + 1 < cnt) step(base + qq + 1, x1, t1);
        }
      }
    }
    float* part = J.dq_part + static_cast<std::size_t>(me) * ldg;
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
      for (int u = 0; u < NU4; ++u) {
        const int c = 4 * hl + 64 * u;
        if (c < J.din_p) *reinterpret_cast<float4*>(part + h * J.din_p + c) = dq[h][u];
      }
  }
}

__global__ void __launch_bounds__(256) k_att_leaf_prep(AttLeafParams ps) {
  pdl_enter();
  const AttLeafParam& P = ps.p[blockIdx.y];
  const int F = P.dout / P.heads, ldg = P.heads * P.din_p;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < ldg * P.ld_w; x += gridDim.x * blockDim.x) {
    const int row = x / P.ld_w, c = x % P.ld_w;  // row = h din_p + i
    const int h = row / P.din_p, i = row % P.din_p;
    const float v = (i < P.din && c < P.dout && c / F == h) ? P.w[static_cast<std::size_t>(i) * P.ld_w + c] : 0.f;
    P.wbd[x] = v;
    if (c < P.dout) P.wbdt[static_cast<std::size_t>(c) * ldg + row] = v;
    if (c == 0) {  // q[h][i] = W^(h)[i] . a^(h)
      float qv = 0.f;
      if (i < P.din)
        for (int cc = h * F; cc < (h + 1) * F; ++cc) qv += P.w[static_cast<std::size_t>(i) * P.ld_w + cc] * P.a[cc];
      P.q[row] = qv;
    }
  }
}

constexpr int kLeafMaxG = 4096;  // H din_p held in shared memory by the finish kernel
constexpr int kLeafDqGroups = 32;  // stage 1 of the dq reduction: groups of half-warp partials

// stage 1: CTA (64-column chunk, group, block) sums its group's partials in a fixed order
// into dq[group] (P.dq holds kLeafDqGroups + 1 rows: the groups, then the total)
__global__ void __launch_bounds__(256) k_att_leaf_dq(AttLeafParams ps, int halves) {
  pdl_enter();
  __shared__ float part[4][64];
  const AttLeafParam& P = ps.p[blockIdx.z];
  const int ldg = P.heads * P.din_p;
  const int c = blockIdx.x * 64 + (threadIdx.x & 63), rg = threadIdx.x >> 6;
  const int per = (halves + kLeafDqGroups - 1) / kLeafDqGroups;
  const int k0 = blockIdx.y * per, k1 = min(halves, k0 + per);
  float acc = 0.f;
  if (c < ldg)
#pragma unroll 4
    for (int k = k0 + rg; k < k1; k += 4) acc += P.dq_part[static_cast<std::size_t>(k) * ldg + c];
  part[rg][threadIdx.x & 63] = acc;
  __syncthreads();
  if (rg == 0 && c < ldg)
    P.dq[static_cast<std::size_t>(blockIdx.y) * ldg + c] =
        ((part[0][threadIdx.x] + part[1][threadIdx.x]) + part[2][threadIdx.x]) + part[3][threadIdx.x];
}

// stage 2 (one CTA per block): dq = ordered sum of the groups, dW = diagonal blocks of
// dW_bd + dq a^T, da = W^T dq
__global__ void __launch_bounds__(256) k_att_leaf_finish(AttLeafParams ps) {
  pdl_enter();
  __shared__ float dq[kLeafMaxG];
  const AttLeafParam& P = ps.p[blockIdx.x];
  const int F = P.dout / P.heads, ldg = P.heads * P.din_p;
  for (int r = threadIdx.x; r < ldg; r += blockDim.x) {
    float s = 0.f;
#pragma unroll 8
    for (int g = 0; g < kLeafDqGroups; ++g) s += P.dq[static_cast<std::size_t>(g) * ldg + r];
    dq[r] = s;
    P.dq[static_cast<std::size_t>(kLeafDqGroups) * ldg + r] = s;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < P.din * P.dout; x += blockDim.x) {
    const int i = x / P.dout, c = x % P.dout, h = c / F;
    const std::size_t at = static_cast<std::size_t>(i) * P.ld_w + c;
    P.dw[at] = P.dwfull[static_cast<std::size_t>(h * P.din_p + i) * P.ld_w + c] + dq[h * P.din_p + i] * P.a[c];
  }
  const int lane = threadIdx.x & 31;
  for (int c = threadIdx.x >> 5; c < P.dout; c += blockDim.x >> 5) {  // a warp per column
    const int h = c / F;
    float s = 0.f;
    for (int i = lane; i < P.din; i += 32) s += P.w[static_cast<std::size_t>(i) * P.ld_w + c] * dq[h * P.din_p + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) P.da[c] = s;
  }
}

__global__ void __launch_bounds__(256) k_relu_mask(float* x, const float* h, int ld, const int* n) {
  pdl_enter();
  const std::size_t total = static_cast<std::size_t>(*n) * ld;
  for (std::size_t k = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; k < total;
       k += static_cast<std::size_t>(gridDim.x) * blockDim.x)
    if (h[k] <= 0.f) x[k] = 0.f;
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

unsigned warp_grid(std::uint64_t items) {
  return static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(ceil_div(items, 8), 16 * num_sms())));
}

unsigned half_grid(std::uint64_t items) {
  return static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(ceil_div(items, 16), 16 * num_sms())));
}

}  // namespace

void att_scatter(const AttScatter& s, cudaStream_t st) {
  int total = 0;
  for (int t = 0; t < s.nt; ++t) total += (s.src_cap[t] + 31) & ~31;
  if (total == 0) return;
  int ld = 1;
  for (int q = 0; q < s.nb; ++q) ld = std::max(ld, s.b[q].ld);
  const unsigned grid16 = half_grid(total), grid32 = warp_grid(total);
  if (ld <= 64)
    launch_pdl(k_att_scatter<16, 1>, grid16, 256, 0, st, s, total);
  else if (ld <= 128)
    launch_pdl(k_att_scatter<16, 2>, grid16, 256, 0, st, s, total);
  else if (ld <= 256)
    launch_pdl(k_att_scatter<32, 2>, grid32, 256, 0, st, s, total);
  else
    launch_pdl(k_att_scatter<32, 4>, grid32, 256, 0, st, s, total);
}

void transpose_slots(const TransposeBatch& b, cudaStream_t st) {
  if (b.n == 0) return;
  int most = 1;
  for (int q = 0; q < b.n; ++q) most = std::max(most, b.j[q].din * b.j[q].dout);
  launch_pdl(k_transpose_slots, dim3(static_cast<unsigned>(ceil_div(most, 256)), b.n), 256, 0, st, b);
}

int att_leaf_halves() { return 2 * num_sms() * 16; }

namespace {
template <int H>
void leaf_fwd_h(const AttLeafBatch& b, int nu4, int total, cudaStream_t st) {
  const unsigned grid = half_grid(total);
  switch (nu4) {
    case 1: launch_pdl(k_att_leaf_forward<H, 1>, grid, 256, 0, st, b, total); break;
    case 2: launch_pdl(k_att_leaf_forward<H, 2>, grid, 256, 0, st, b, total); break;
    default: launch_pdl(k_att_leaf_forward<H, 4>, grid, 256, 0, st, b, total); break;
  }
}
template <int H>
void leaf_grad_h(const AttLeafBatch& b, int nu4, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(att_leaf_halves() / 16);
  switch (nu4) {
    case 1: launch_pdl(k_att_leaf_grad<H, 1>, grid, 256, 0, st, b); break;
    case 2: launch_pdl(k_att_leaf_grad<H, 2>, grid, 256, 0, st, b); break;
    default: launch_pdl(k_att_leaf_grad<H, 4>, grid, 256, 0, st, b); break;
  }
}
int leaf_shape(const AttLeafBatch& b, int& H) {
  int din = 4;
  H = b.j[0].heads;
  for (int q = 0; q < b.n; ++q) {
    if (b.j[q].heads != H) throw std::invalid_argument("attention jobs of one launch must share the head count");
    din = std::max(din, b.j[q].din_p);
  }
  if (din > 256) throw std::invalid_argument("aggregate-first attention supports layer-0 rows up to 256 columns");
  return din <= 64 ? 1 : din <= 128 ? 2 : 4;
}
}  // namespace

void att_leaf_forward(const AttLeafBatch& b, cudaStream_t st) {
  if (b.n == 0) return;
  int H = 1;
  const int nu4 = leaf_shape(b, H);
  int total = 0;
  for (int q = 0; q < b.n; ++q) total += (b.j[q].rows_cap + 31) & ~31;
  switch (H) {
    case 1: leaf_fwd_h<1>(b, nu4, total, st); break;
    case 2: leaf_fwd_h<2>(b, nu4, total, st); break;
    case 4: leaf_fwd_h<4>(b, nu4, total, st); break;
    case 8: leaf_fwd_h<8>(b, nu4, total, st); break;
    default: throw std::invalid_argument("attention heads must be 1, 2, 4 or 8");
  }
}

void att_leaf_grad(const AttLeafBatch& b, cudaStream_t st) {
  if (b.n == 0) return;
  int H = 1;
  const int nu4 = leaf_shape(b, H);
  switch (H) {
    case 1: leaf_grad_h<1>(b, nu4, st); break;
    case 2: leaf_grad_h<2>(b, nu4, st); break;
    case 4: leaf_grad_h<4>(b, nu4, st); break;
    case 8: leaf_grad_h<8>(b, nu4, st); break;
    default: throw std::invalid_argument("attention heads must be 1, 2, 4 or 8");
  }
}

void att_leaf_prep(const AttLeafParams& p, cudaStream_t st) {
  if (p.n == 0) return;
  int most = 1;
  for (int q = 0; q < p.n; ++q) most = std::max(most, p.p[q].heads * p.p[q].din_p * p.p[q].ld_w);
  launch_pdl(k_att_leaf_prep, dim3(static_cast<unsigned>(ceil_div(most, 256)), p.n), 256, 0, st, p);
}

void att_leaf_finish(const AttLeafParams& p, cudaStream_t st) {
  if (p.n == 0) return;
  int ldg = 1;
  for (int q = 0; q < p.n; ++q) {
    if (p.p[q].heads * p.p[q].din_p > kLeafMaxG) throw std::invalid_argument("attention layer-0 block too wide");
    ldg = std::max(ldg, p.p[q].heads * p.p[q].din_p);
  }
  launch_pdl(k_att_leaf_dq, dim3(static_cast<unsigned>(ceil_div(ldg, 64)), kLeafDqGroups, p.n), 256, 0, st, p,
             att_leaf_halves());
  launch_pdl(k_att_leaf_finish, dim3(p.n), 256, 0, st, p);
}

int att_leaf_dq_rows() { return kLeafDqGroups + 1; }

void relu_mask(float* x, const float* h, int ld, const int* n, int rows_cap, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::max<std::uint64_t>(
      1, std::min<std::uint64_t>(ceil_div(static_cast<std::uint64_t>(rows_cap) * ld, 256), 4 * num_sms())));
  launch_pdl(k_relu_mask, grid, 256, 0, st, x, h, ld, n);
}

}  // namespace hetgpu
