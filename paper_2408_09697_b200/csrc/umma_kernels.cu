// The dense contractions of the hot path on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulators in TMEM), replacing the reference's
// naive f64 loops:
//   projection   out   = sum_r mean_r . W_r  (+ReLU)     matmul + agg_all, hgnn.cpp:189-203, 267-272
//   mean grad    dmean = (dpre . W^T) / deg              matmul_nt, matrix.hpp:64-78; hgnn.cpp:337-353
//   weight grad  dW   += mean^T . dpre  (split-K)        matmul_tn_acc, matrix.hpp:49-61; hgnn.cpp:334
// Parity: operands are split x = hi + lo in tf32 and hi.hi + hi.lo + lo.hi is
// accumulated in fp32 (3xTF32), which keeps fp32-level accuracy (the north
// star's 1e-3 tolerance is for fp32 accumulate).
//
// One CTA = 128 threads = one 128-row output tile x NT columns. Per 32-wide K
// chunk every thread loads its float4s from global memory (coalesced), splits
// them and stores hi/lo into 128B-swizzled K-major tiles; thread 0 issues the
// 4 k-steps x 3 MMAs and commits them to the stage's mbarrier. Two smem stages:
// the global loads of chunk c+1 are in flight while the tensor core runs chunk
// c. The epilogue reads TMEM with tcgen05.ld (warp w owns TMEM lanes 32w..32w+31,
// i.e. tile rows) and applies the fused ReLU / 1/deg scaling / row remap.
#include "gemm.cuh"
#include "umma.cuh"

namespace hetgpu {

namespace {

constexpr int kUT = 256;             // threads per CTA (8 warps: 2 per TMEM lane quadrant)
constexpr int kAV = 128 * 32 / 4 / kUT;  // A float4 per thread per chunk
constexpr int kATile = 128 * 128;    // bytes of one 128 x 32 fp32 operand tile

template <int NT>
struct UStage {
  static constexpr int kB = NT * 128;
  static constexpr int kBytes = 2 * kATile + 2 * kB;  // A hi, A lo, B hi, B lo
  static constexpr int kSmem = 2 * kBytes + 1024 + 64;  // two stages + alignment + barriers
  static constexpr int kTmemCols = NT <= 32 ? 32 : NT <= 64 ? 64 : NT <= 128 ? 128 : 256;
  static constexpr std::uint32_t kSboA = 128 / 32 * umma::kMnLbo;  // MN-major A: 4-row K-group stride
  static constexpr std::uint32_t kSboB = NT / 32 * umma::kMnLbo;   // MN-major B: 4-row K-group stride
};
// operand majors per mode: projection B = W[k][n] and the weight gradient's
// A = mean[row][c], B = dpre[row][j] are row-contiguous -> MN-major tiles
template <int MODE> struct Majors;

__device__ __forceinline__ float4 f4zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }

// K-contiguous float4 (4 consecutive k of row r) -> hi/lo tiles
__device__ __forceinline__ void st_kc(std::uint8_t* hi, std::uint8_t* lo, int r, int kq, float4 v) {
  float4 h, l;
  umma::split_tf32(v.x, h.x, l.x);
  umma::split_tf32(v.y, h.y, l.y);
  umma::split_tf32(v.z, h.z, l.z);
  umma::split_tf32(v.w, h.w, l.w);
  const std::uint32_t off = umma::sw128_chunk(r, kq >> 2);
  *reinterpret_cast<float4*>(hi + off) = h;
  *reinterpret_cast<float4*>(lo + off) = l;
}
// M/N-contiguous float4 (elements m..m+3 at one k) -> MN-major hi/lo tiles
__device__ __forceinline__ void st_mn(std::uint8_t* hi, std::uint8_t* lo, int m, int k, std::uint32_t sbo, float4 v) {
  float4 h, l;
  umma::split_tf32(v.x, h.x, l.x);
  umma::split_tf32(v.y, h.y, l.y);
  umma::split_tf32(v.z, h.z, l.z);
  umma::split_tf32(v.w, h.w, l.w);
  const std::uint32_t off = umma::sw128b32_mn(m, k, sbo);
  *reinterpret_cast<float4*>(hi + off) = h;
  *reinterpret_cast<float4*>(lo + off) = l;
}

__device__ __forceinline__ float4 load_dpre(const DpreView& d, int row, int col) {
  const std::size_t at = static_cast<std::size_t>(row * d.stride + d.offset) * d.ld + col;
  float4 v = *reinterpret_cast<const float4*>(d.g + at);
  if (d.h) {  // dpre = dH * [H > 0] (hgnn.cpp:326-328)
    const float4 h = *reinterpret_cast<const float4*>(d.h + static_cast<std::size_t>(row) * d.ld + col);
    if (h.x <= 0.f) v.x = 0.f;
    if (h.y <= 0.f) v.y = 0.f;
    if (h.z <= 0.f) v.z = 0.f;
    if (h.w <= 0.f) v.w = 0.f;
  }
  return v;
}

__device__ __forceinline__ int find_tile(const int* base, int n, int tile) {
  int p = 0;
  while (p + 1 < n && tile >= base[p + 1]) ++p;
  return p;
}

enum Mode { kProject = 0, kDMean = 1, kWGrad = 2 };
template <> struct Majors<kProject> { static constexpr int a = 0, b = 1; };
template <> struct Majors<kDMean> { static constexpr int a = 0, b = 0; };
template <> struct Majors<kWGrad> { static constexpr int a = 1, b = 1; };

template <typename Batch>
struct UmmaArgs {
  Batch b;
  int tile_base[kMaxProblems + 1];
  int n_tiles[kMaxProblems];  // column tiles per problem
  int m_tiles[kMaxProblems];  // wgrad: din tiles per problem
  int np;
};

// Per-CTA description of the tile being computed, filled by the mode.
struct TileCtx {
  int mode;
  int p;          // problem / group index
  int row0;       // first output row (project/dmean) or first K row (wgrad)
  int m0, n0;     // wgrad: first din row; all: first output column
  int nch;        // K chunks
  int n_live;     // live rows
};

template <int NT, int MODE, typename Batch>
__global__ void __launch_bounds__(kUT) k_umma(UmmaArgs<Batch> args) {
  extern __shared__ std::uint8_t smem_raw[];
  std::uint8_t* smem = reinterpret_cast<std::uint8_t*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                        ~static_cast<std::uintptr_t>(1023));
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem + 2 * UStage<NT>::kBytes);
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- tile lookup ----------------------------------------------------------------------
  const int p = find_tile(args.tile_base, args.np, blockIdx.x);
  const int t = blockIdx.x - args.tile_base[p];
  const int ntl = args.n_tiles[p];
  TileCtx c{};
  c.mode = MODE;
  c.p = p;
  if constexpr (MODE == kProject) {
    const ProjGroup& g = args.b.g[p];
    c.n_live = *g.n_rows;
    c.row0 = (t / ntl) * 128;
    c.n0 = (t % ntl) * NT;
    int nch = 0;
    for (int q = 0; q < g.nrel; ++q) nch += (g.r[q].din + 31) / 32;
    c.nch = nch;
  } else if constexpr (MODE == kDMean) {
    const DMeanProblem& P = args.b.p[p];
    c.n_live = *P.n_rows;
    c.row0 = (t / ntl) * 128;
    c.n0 = (t % ntl) * NT;
    c.nch = (P.d.cols + 31) / 32;
  } else {
    const WGradProblem& P = args.b.p[p];
    c.n_live = *P.n_rows;
    const int mt = args.m_tiles[p];
    const int chunk = t / (mt * ntl);
    c.m0 = ((t / ntl) % mt) * 128;
    c.n0 = (t % ntl) * NT;
    c.row0 = chunk * kWChunkRows;
    c.nch = (min(kWChunkRows, c.n_live - c.row0) + 31) / 32;
  }
  if (MODE != kWGrad && c.row0 >= c.n_live) return;
  if (MODE == kWGrad && c.row0 >= c.n_live) return;

  // ---- setup: barriers, TMEM ---------------------------------------------------------------
  if (tid == 0) {
    umma::mbar_init(umma::smem_u32(&bars[0]), 1);
    umma::mbar_init(umma::smem_u32(&bars[1]), 1);
    umma::fence_mbar_init();
  }
  if (warp == 0) umma::tmem_alloc(umma::smem_u32(tmem_slot), UStage<NT>::kTmemCols);
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const std::uint32_t tmem = *tmem_slot;

  // ---- operand loaders ------------------------------------------------------------------------
  constexpr int kBV = NT * 32 / 4 / kUT;  // B float4 per thread per chunk
  float4 ra[kAV], rb[kBV];
  auto load = [&](int ch) {
    if constexpr (MODE == kProject) {
      const ProjGroup& g = args.b.g[p];
      int q = 0, k0 = ch * 32;
      while (q + 1 < g.nrel && k0 >= ((g.r[q].din + 31) / 32) * 32) {
        k0 -= ((g.r[q].din + 31) / 32) * 32;
        ++q;
      }
      const ProjRel& r = g.r[q];
#pragma unroll
      for (int i = 0; i < kAV; ++i) {  // A: mean rows, K-contiguous
        const int m = (tid >> 3) + (kUT / 8) * i, k = k0 + (tid & 7) * 4, row = c.row0 + m;
        ra[i] = (row < c.n_live && k < r.ld_mean)
                    ? __ldg(reinterpret_cast<const float4*>(r.mean + static_cast<std::size_t>(row) * r.ld_mean + k))
                    : f4zero();
      }
#pragma unroll
      for (int i = 0; i < kBV; ++i) {  // B[n][k] = W[k][n]: N-contiguous
        const int f = tid + kUT * i, k = f / (NT / 4), n = c.n0 + (f % (NT / 4)) * 4, kk = k0 + k;
        rb[i] = (kk < r.din && n < r.ld_w)
                    ? __ldg(reinterpret_cast<const float4*>(r.w + static_cast<std::size_t>(kk) * r.ld_w + n))
                    : f4zero();
      }
    } else if constexpr (MODE == kDMean) {
      const DMeanProblem& P = args.b.p[p];
      const int cols4 = (P.d.cols + 3) & ~3;
#pragma unroll
      for (int i = 0; i < kAV; ++i) {  // A: dpre rows (ReLU mask, row remap), K-contiguous
        const int m = (tid >> 3) + (kUT / 8) * i, k = ch * 32 + (tid & 7) * 4, row = c.row0 + m;
        ra[i] = (row < c.n_live && k < cols4) ? load_dpre(P.d, row, k) : f4zero();
      }
#pragma unroll
      for (int i = 0; i < kBV; ++i) {  // B[n=c][k=j] = W[c][j]: K-contiguous
        const int n = c.n0 + (tid >> 3) + (kUT / 8) * i, k = ch * 32 + (tid & 7) * 4;
        rb[i] = (n < P.din && k < P.ld_w)
                    ? __ldg(reinterpret_cast<const float4*>(P.w + static_cast<std::size_t>(n) * P.ld_w + k))
                    : f4zero();
      }
    } else {
      const WGradProblem& P = args.b.p[p];
      const int cols4 = (P.d.cols + 3) & ~3;
#pragma unroll
      for (int i = 0; i < kAV; ++i) {  // A[m=c][k=row] = mean[row][c]: M-contiguous
        const int k = (tid >> 5) + (kUT / 32) * i, m = c.m0 + (tid & 31) * 4, row = c.row0 + ch * 32 + k;
        ra[i] = (row < c.n_live && m < P.ld_mean)
                    ? *reinterpret_cast<const float4*>(P.mean + static_cast<std::size_t>(row) * P.ld_mean + m)
                    : f4zero();
      }
#pragma unroll
      for (int i = 0; i < kBV; ++i) {  // B[n=j][k=row] = dpre[row][j]: N-contiguous
        const int f = tid + kUT * i, k = f / (NT / 4), n = c.n0 + (f % (NT / 4)) * 4, row = c.row0 + ch * 32 + k;
        rb[i] = (row < c.n_live && n < cols4) ? load_dpre(P.d, row, n) : f4zero();
      }
    }
  };
  auto store = [&](std::uint8_t* st) {
    std::uint8_t *ahi = st, *alo = st + kATile, *bhi = st + 2 * kATile, *blo = bhi + UStage<NT>::kB;
    if constexpr (Majors<MODE>::a) {
#pragma unroll
      for (int i = 0; i < kAV; ++i) st_mn(ahi, alo, (tid & 31) * 4, (tid >> 5) + (kUT / 32) * i, UStage<NT>::kSboA, ra[i]);
    } else {
#pragma unroll
      for (int i = 0; i < kAV; ++i) st_kc(ahi, alo, (tid >> 3) + (kUT / 8) * i, (tid & 7) * 4, ra[i]);
    }
    if constexpr (Majors<MODE>::b) {
#pragma unroll
      for (int i = 0; i < kBV; ++i) {
        const int f = tid + kUT * i;
        st_mn(bhi, blo, (f % (NT / 4)) * 4, f / (NT / 4), UStage<NT>::kSboB, rb[i]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < kBV; ++i) st_kc(bhi, blo, (tid >> 3) + (kUT / 8) * i, (tid & 7) * 4, rb[i]);
    }
  };

  // ---- main loop: two stages, MMAs of chunk c overlap the loads of chunk c+1 -------------------
  constexpr std::uint32_t kIdesc = umma::idesc_tf32(128, NT, Majors<MODE>::a, Majors<MODE>::b);
  auto desc_a = [&](std::uint32_t base, int kk) {
    return Majors<MODE>::a ? umma::desc_mn_sw128_32b(base + 2 * kk * UStage<NT>::kSboA, UStage<NT>::kSboA)
                           : umma::desc_k_sw128(base + 32u * kk);
  };
  auto desc_b = [&](std::uint32_t base, int kk) {
    return Majors<MODE>::b ? umma::desc_mn_sw128_32b(base + 2 * kk * UStage<NT>::kSboB, UStage<NT>::kSboB)
                           : umma::desc_k_sw128(base + 32u * kk);
  };
  std::uint32_t phase[2] = {0u, 0u};
  load(0);
  for (int ch = 0; ch < c.nch; ++ch) {
    const int s = ch & 1;
    std::uint8_t* st = smem + s * UStage<NT>::kBytes;
    if (ch >= 2) {
      umma::mbar_wait(umma::smem_u32(&bars[s]), phase[s]);
      phase[s] ^= 1u;
    }
    store(st);
    if (ch + 1 < c.nch) load(ch + 1);
    umma::fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      umma::fence_after_sync();
      const std::uint32_t a_hi = umma::smem_u32(st), a_lo = a_hi + kATile;
      const std::uint32_t b_hi = a_hi + 2 * kATile, b_lo = b_hi + UStage<NT>::kB;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {  // 8 tf32 of K per MMA
        umma::mma_tf32(tmem, desc_a(a_hi, kk), desc_b(b_hi, kk), kIdesc, (ch > 0 || kk > 0) ? 1u : 0u);
        umma::mma_tf32(tmem, desc_a(a_hi, kk), desc_b(b_lo, kk), kIdesc, 1u);
        umma::mma_tf32(tmem, desc_a(a_lo, kk), desc_b(b_hi, kk), kIdesc, 1u);
      }
      umma::commit(umma::smem_u32(&bars[s]));
    }
  }
  {
    const int s = (c.nch - 1) & 1;
    umma::mbar_wait(umma::smem_u32(&bars[s]), phase[s]);
  }
  umma::fence_after_sync();

  // ---- epilogue: TMEM -> registers -> global ------------------------------------------------------
  // warp w reads TMEM lane quadrant (w % 4) = tile rows 32(w%4)..+31, columns
  // [(w / 4) * NT / 2, ...) : the two warps of a quadrant split the columns
  constexpr int kHalves = kUT / 128;
  const int quad = warp & 3, half = warp >> 2;
  const int m = quad * 32 + lane;  // tile row owned by this thread
  const std::uint32_t trow = tmem + (static_cast<std::uint32_t>(quad * 32) << 16);
#pragma unroll 1
  for (int c0 = half * (NT / kHalves); c0 < (half + 1) * (NT / kHalves); c0 += 16) {
    float v[16];
    umma::tmem_ld16(trow + c0, v);
    if constexpr (MODE == kProject) {
      const ProjGroup& g = args.b.g[p];
      const int row = c.row0 + m;
      if (row < c.n_live) {
        float* orow = g.out + static_cast<std::size_t>(row * g.out_stride + g.out_offset) * g.ld_out;
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          const int col = c.n0 + c0 + j;
          if (col < g.ld_out) {
            float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            if (g.relu) {
              o.x = fmaxf(o.x, 0.f);
              o.y = fmaxf(o.y, 0.f);
              o.z = fmaxf(o.z, 0.f);
              o.w = fmaxf(o.w, 0.f);
            }
            *reinterpret_cast<float4*>(orow + col) = o;
          }
        }
      }
    } else if constexpr (MODE == kDMean) {
      const DMeanProblem& P = args.b.p[p];
      const int row = c.row0 + m;
      if (row < c.n_live) {
        const std::uint32_t deg = P.indptr[row + 1] - P.indptr[row];
        const float inv = deg ? 1.0f / static_cast<float>(deg) : 0.0f;
        float* orow = P.dmean + static_cast<std::size_t>(row) * P.ld_dmean;
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          const int col = c.n0 + c0 + j;
          if (col < P.ld_dmean)
            *reinterpret_cast<float4*>(orow + col) =
                make_float4(v[j] * inv, v[j + 1] * inv, v[j + 2] * inv, v[j + 3] * inv);
        }
      }
    } else {
      const WGradProblem& P = args.b.p[p];
      const int row = c.m0 + m;  // din index
      if (row < P.din) {
        const int chunk = c.row0 / kWChunkRows;
        float* out = P.partial + (static_cast<std::size_t>(chunk) * P.din + row) * P.d.cols;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int col = c.n0 + c0 + j;
          if (col < P.d.cols) out[col] = v[j];
        }
      }
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, UStage<NT>::kTmemCols);
}

template <int NT, int MODE, typename Batch>
void launch(UmmaArgs<Batch>& a, int tiles, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    HG_CUDA(cudaFuncSetAttribute(k_umma<NT, MODE, Batch>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 UStage<NT>::kSmem));
    attr = true;
  }
  k_umma<NT, MODE, Batch><<<tiles, kUT, UStage<NT>::kSmem, st>>>(a);
}

// column tile width for an output of `cols` columns (multiples of 32 for the
// MN-major atoms); wider outputs take several 128-wide tiles (349 classes -> 3)
int pick_nt(int cols) {
  if (cols <= 32) return 32;
  if (cols <= 64) return 64;
  return 128;
}

template <int MODE, typename Batch>
void dispatch(UmmaArgs<Batch>& a, int nt, int tiles, cudaStream_t st) {
  if (tiles <= 0) return;
  switch (nt) {
    case 32: launch<32, MODE>(a, tiles, st); break;
    case 64: launch<64, MODE>(a, tiles, st); break;
    default: launch<128, MODE>(a, tiles, st); break;
  }
}

}  // namespace

// All problems of one launch share one column-tile width (the widest needed).
void project_umma(ProjBatch& pb, cudaStream_t st) {
  if (pb.ng == 0) return;
  UmmaArgs<ProjBatch> a{};
  a.b = pb;
  a.np = pb.ng;
  int nt = 32;
  for (int g = 0; g < pb.ng; ++g) nt = std::max(nt, pick_nt(pb.g[g].ld_out));
  int tiles = 0;
  for (int g = 0; g < pb.ng; ++g) {
    a.tile_base[g] = tiles;
    a.n_tiles[g] = static_cast<int>(ceil_div(pb.g[g].ld_out, nt));
    tiles += static_cast<int>(ceil_div(std::max(1, pb.g[g].rows_cap), 128)) * a.n_tiles[g];
  }
  a.tile_base[pb.ng] = tiles;
  dispatch<kProject>(a, nt, tiles, st);
}

void dmean_umma(DMeanBatch& b, cudaStream_t st) {
  if (b.np == 0) return;
  UmmaArgs<DMeanBatch> a{};
  a.b = b;
  a.np = b.np;
  int nt = 32;
  for (int q = 0; q < b.np; ++q) nt = std::max(nt, pick_nt(b.p[q].ld_dmean));
  int tiles = 0;
  for (int q = 0; q < b.np; ++q) {
    a.tile_base[q] = tiles;
    a.n_tiles[q] = static_cast<int>(ceil_div(b.p[q].ld_dmean, nt));
    tiles += static_cast<int>(ceil_div(std::max(1, b.p[q].rows_cap), 128)) * a.n_tiles[q];
  }
  a.tile_base[b.np] = tiles;
  dispatch<kDMean>(a, nt, tiles, st);
}

void wgrad_umma(WGradBatch& b, cudaStream_t st) {
  if (b.np == 0) return;
  UmmaArgs<WGradBatch> a{};
  a.b = b;
  a.np = b.np;
  int nt = 32;
  for (int q = 0; q < b.np; ++q) nt = std::max(nt, pick_nt(b.p[q].d.cols));
  int tiles = 0;
  for (int q = 0; q < b.np; ++q) {
    const WGradProblem& P = b.p[q];
    a.tile_base[q] = tiles;
    a.n_tiles[q] = static_cast<int>(ceil_div(P.d.cols, nt));
    a.m_tiles[q] = static_cast<int>(ceil_div(P.din, 128));
    tiles += static_cast<int>(ceil_div(std::max(1, P.rows_cap), kWChunkRows)) * a.m_tiles[q] * a.n_tiles[q];
  }
  a.tile_base[b.np] = tiles;
  dispatch<kWGrad>(a, nt, tiles, st);
  wgrad_reduce(b, st);
}

}  // namespace hetgpu
