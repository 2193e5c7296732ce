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
// One CTA = 256 threads = one 128-row output tile x NT columns. Operands are
// staged per 32-wide K chunk in a 4-deep ring: every thread cp.async-copies its
// 16-byte pieces of raw fp32 straight into the canonical UMMA layout (K-major
// 128B-swizzled, or MN-major SW128_32B for row-contiguous sources that the
// tensor core reads transposed), zero-filling rows / columns outside the live
// extent; chunks are prefetched 2 ahead. The raw tile is the "hi" operand (the
// tensor core reads the top 19 bits), one elementwise pass writes lo = x -
// trunc(x), and thread 0 issues 4 k-steps x 3 MMAs and commits them to the
// stage's mbarrier. The epilogue reads TMEM with tcgen05.ld (warps w and w+4 own
// TMEM lane quadrant w%4) and applies the fused ReLU / 1/deg scaling / row remap.
#include "gemm.cuh"
#include "umma.cuh"

namespace hetgpu {

namespace {

constexpr int kUT = 256;             // threads per CTA (8 warps: 2 per TMEM lane quadrant)
constexpr int kATile = 128 * 128;    // bytes of one 128 x 32 fp32 operand tile

constexpr int kRing = 4;   // raw (hi) operand stages
constexpr int kAhead = 2;  // chunks prefetched ahead of the one being multiplied

template <int NT>
struct UStage {
  static constexpr int kB = NT * 128;
  static constexpr int kHi = kATile + kB;              // one raw stage: A, B
  static constexpr int kLo = kATile + kB;              // one lo stage: A, B
  static constexpr int kSmem = kRing * kHi + 2 * kLo + 1024 + 128;  // + alignment + barriers
  static constexpr int kTmemCols = NT <= 32 ? 32 : NT <= 64 ? 64 : NT <= 128 ? 128 : 256;
  static constexpr std::uint32_t kSboA = 128 / 32 * umma::kMnLbo;  // MN-major A: 4-row K-group stride
  static constexpr std::uint32_t kSboB = NT / 32 * umma::kMnLbo;   // MN-major B: 4-row K-group stride
};
// operand majors per mode: projection B = W[k][n] and the weight gradient's
// A = mean[row][c], B = dpre[row][j] are row-contiguous -> MN-major tiles
template <int MODE> struct Majors;


// 16-byte async copy global -> shared; src_bytes = 0 zero-fills (outside the live extent)
__device__ __forceinline__ void cp16(std::uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_ahead() {
  asm volatile("cp.async.wait_group %0;" ::"n"(kAhead) : "memory");
}
// dpre rows (row remap for replica shards); the ReLU mask was applied upstream
__device__ __forceinline__ const float* dpre_ptr(const DpreView& d, int row, int col) {
  return d.g + static_cast<std::size_t>(row * d.stride + d.offset) * d.ld + col;
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
  std::uint8_t* hi_ring = smem;                                  // kRing x (A, B)
  std::uint8_t* lo_ring = smem + kRing * UStage<NT>::kHi;        // 2 x (A, B)
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(lo_ring + 2 * UStage<NT>::kLo);  // per hi stage
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + kRing);
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
    for (int i = 0; i < kRing; ++i) umma::mbar_init(umma::smem_u32(&bars[i]), 1);
    umma::fence_mbar_init();
  }
  if (warp == 0) umma::tmem_alloc(umma::smem_u32(tmem_slot), UStage<NT>::kTmemCols);
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const std::uint32_t tmem = *tmem_slot;

  // ---- staging: cp.async of chunk ch's raw fp32 into hi stage `slot` ----------------------------
  constexpr int kAV = 128 * 32 / 4 / kUT;  // A 16-byte pieces per thread per chunk
  constexpr int kBV = NT * 32 / 4 / kUT;   // B 16-byte pieces per thread per chunk
  auto issue = [&](int ch, int slot) {
    std::uint8_t* st = hi_ring + slot * UStage<NT>::kHi;
    const std::uint32_t a_s = umma::smem_u32(st), b_s = a_s + kATile;
    if constexpr (MODE == kProject) {
      const ProjGroup& g = args.b.g[p];
      int q = 0, k0 = ch * 32;
      while (q + 1 < g.nrel && k0 >= ((g.r[q].din + 31) / 32) * 32) {
        k0 -= ((g.r[q].din + 31) / 32) * 32;
        ++q;
      }
      const ProjRel& r = g.r[q];
#pragma unroll
      for (int i = 0; i < kAV; ++i) {  // A = mean rows, K-major
        const int m = (tid >> 3) + (kUT / 8) * i, kq = (tid & 7) * 4, k = k0 + kq, row = c.row0 + m;
        const bool ok = row < c.n_live && k < r.ld_mean;
        cp16(a_s + umma::sw128_chunk(m, kq >> 2), ok ? r.mean + static_cast<std::size_t>(row) * r.ld_mean + k : r.mean, ok);
      }
#pragma unroll
      for (int i = 0; i < kBV; ++i) {  // B[n][k] = W[k][n], MN-major
        const int f = tid + kUT * i, k = f / (NT / 4), nq = (f % (NT / 4)) * 4, kk = k0 + k, n = c.n0 + nq;
        const bool ok = kk < r.din && n < r.ld_w;
        cp16(b_s + umma::sw128b32_mn(nq, k, UStage<NT>::kSboB), ok ? r.w + static_cast<std::size_t>(kk) * r.ld_w + n : r.w, ok);
      }
    } else if constexpr (MODE == kDMean) {
      const DMeanProblem& P = args.b.p[p];
      const int cols4 = (P.d.cols + 3) & ~3;
#pragma unroll
      for (int i = 0; i < kAV; ++i) {  // A = dpre rows, K-major
        const int m = (tid >> 3) + (kUT / 8) * i, kq = (tid & 7) * 4, k = ch * 32 + kq, row = c.row0 + m;
        const bool ok = row < c.n_live && k < cols4;
        cp16(a_s + umma::sw128_chunk(m, kq >> 2), ok ? dpre_ptr(P.d, row, k) : P.d.g, ok);
      }
#pragma unroll
      for (int i = 0; i < kBV; ++i) {  // B[n=c][k=j] = W[c][j], K-major
        const int nl = (tid >> 3) + (kUT / 8) * i, kq = (tid & 7) * 4, n = c.n0 + nl, k = ch * 32 + kq;
        const bool ok = n < P.din && k < P.ld_w;
        cp16(b_s + umma::sw128_chunk(nl, kq >> 2), ok ? P.w + static_cast<std::size_t>(n) * P.ld_w + k : P.w, ok);
      }
    } else {
      const WGradProblem& P = args.b.p[p];
      const int cols4 = (P.d.cols + 3) & ~3;
#pragma unroll
      for (int i = 0; i < kAV; ++i) {  // A[m=c][k=row] = mean[row][c], MN-major
        const int k = (tid >> 5) + (kUT / 32) * i, mq = (tid & 31) * 4, m = c.m0 + mq, row = c.row0 + ch * 32 + k;
        const bool ok = row < c.n_live && m < P.ld_mean;
        cp16(a_s + umma::sw128b32_mn(mq, k, UStage<NT>::kSboA),
             ok ? P.mean + static_cast<std::size_t>(row) * P.ld_mean + m : P.mean, ok);
      }
#pragma unroll
      for (int i = 0; i < kBV; ++i) {  // B[n=j][k=row] = dpre[row][j], MN-major
        const int f = tid + kUT * i, k = f / (NT / 4), nq = (f % (NT / 4)) * 4, n = c.n0 + nq,
                  row = c.row0 + ch * 32 + k;
        const bool ok = row < c.n_live && n < cols4;
        cp16(b_s + umma::sw128b32_mn(nq, k, UStage<NT>::kSboB), ok ? dpre_ptr(P.d, row, n) : P.d.g, ok);
      }
    }
  };
  // lo = x - trunc_tf32(x) over the raw stage (elementwise: layout-agnostic)
  auto make_lo = [&](int hslot, int lslot) {
    const float4* src = reinterpret_cast<const float4*>(hi_ring + hslot * UStage<NT>::kHi);
    float4* dst = reinterpret_cast<float4*>(lo_ring + lslot * UStage<NT>::kLo);
#pragma unroll
    for (int i = 0; i < (UStage<NT>::kHi / 16) / kUT; ++i) {
      const float4 x = src[tid + kUT * i];
      float4 h, l;
      umma::split_tf32(x.x, h.x, l.x);
      umma::split_tf32(x.y, h.y, l.y);
      umma::split_tf32(x.z, h.z, l.z);
      umma::split_tf32(x.w, h.w, l.w);
      dst[tid + kUT * i] = l;
    }
  };

  // ---- main loop ---------------------------------------------------------------------------------
  constexpr std::uint32_t kIdesc = umma::idesc_tf32(128, NT, Majors<MODE>::a, Majors<MODE>::b);
  auto desc_a = [&](std::uint32_t base, int kk) {
    return Majors<MODE>::a ? umma::desc_mn_sw128_32b(base + 2 * kk * UStage<NT>::kSboA, UStage<NT>::kSboA)
                           : umma::desc_k_sw128(base + 32u * kk);
  };
  auto desc_b = [&](std::uint32_t base, int kk) {
    return Majors<MODE>::b ? umma::desc_mn_sw128_32b(base + 2 * kk * UStage<NT>::kSboB, UStage<NT>::kSboB)
                           : umma::desc_k_sw128(base + 32u * kk);
  };
  for (int j = 0; j < kAhead; ++j) {
    if (j < c.nch) issue(j, j);
    cp_commit();
  }
  for (int ch = 0; ch < c.nch; ++ch) {
    // MMAs of chunk ch-2 read hi stage (ch+2)%4 and lo stage ch%2: both free after them
    if (ch >= 2) umma::mbar_wait(umma::smem_u32(&bars[(ch - 2) % kRing]), ((ch - 2) / kRing) & 1);
    if (ch + kAhead < c.nch) issue(ch + kAhead, (ch + kAhead) % kRing);
    cp_commit();
    cp_wait_ahead();  // this thread's pieces of chunk ch have landed
    __syncthreads();  // ... and everybody else's
    make_lo(ch % kRing, ch & 1);
    umma::fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      umma::fence_after_sync();
      const std::uint32_t a_hi = umma::smem_u32(hi_ring + (ch % kRing) * UStage<NT>::kHi), b_hi = a_hi + kATile;
      const std::uint32_t a_lo = umma::smem_u32(lo_ring + (ch & 1) * UStage<NT>::kLo), b_lo = a_lo + kATile;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {  // 8 tf32 of K per MMA
        umma::mma_tf32(tmem, desc_a(a_hi, kk), desc_b(b_hi, kk), kIdesc, (ch > 0 || kk > 0) ? 1u : 0u);
        umma::mma_tf32(tmem, desc_a(a_hi, kk), desc_b(b_lo, kk), kIdesc, 1u);
        umma::mma_tf32(tmem, desc_a(a_lo, kk), desc_b(b_hi, kk), kIdesc, 1u);
      }
      umma::commit(umma::smem_u32(&bars[ch % kRing]));
    }
  }
  umma::mbar_wait(umma::smem_u32(&bars[(c.nch - 1) % kRing]), ((c.nch - 1) / kRing) & 1);
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
  for (int q = 0; q < b.np; ++q)
    if (b.p[q].d.h) throw std::invalid_argument("tcgen05 mean gradient expects an already masked dpre");
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
  for (int q = 0; q < b.np; ++q)
    if (b.p[q].d.h) throw std::invalid_argument("tcgen05 weight gradient expects an already masked dpre");
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
