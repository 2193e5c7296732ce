// The dense contractions of the hot path on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulators in TMEM, operands by TMA), replacing
// the reference's naive f64 loops:
//   projection   out   = sum_r mean_r . W_r  (+ReLU)     matmul + agg_all, hgnn.cpp:189-203, 267-272
//   mean grad    dmean = (dpre . W^T) / deg              matmul_nt, matrix.hpp:64-78; hgnn.cpp:337-353
//   weight grad  dW   += mean^T . dpre  (split-K)        matmul_tn_acc, matrix.hpp:49-61; hgnn.cpp:334
// Parity: every operand x is split as hi = x (the tensor core reads its top 19
// bits) plus lo = x - trunc_tf32(x); the sum hi.hi + hi.lo + lo.hi accumulated in
// fp32 (3xTF32) keeps fp32-level accuracy (the north star's 1e-3 tolerance is for
// fp32 accumulate). Only x travels from HBM: lo is formed in shared memory.
//
// One CTA = 128 threads = one 128-row output tile x NT columns, warp-specialised:
// warp 0 (one lane) streams 32-wide K chunks of A and B through a kStages-deep
// shared-memory ring with 2-D TMA loads (K-major tiles with the 128-byte swizzle;
// row-contiguous operands the tensor core reads transposed as MN-major SW128_32B
// tiles); warps 2-3 turn each landed tile into its tf32 residual next to it (an
// elementwise pass, so the swizzled layout carries over) and hand the stage on
// through a second barrier; warp 1 (one lane) issues 4 k-steps x 3 MMAs per chunk
// and commits them to the stage's "empty" barrier; all four warps then drain TMEM
// with tcgen05.ld (warp w owns TMEM lanes 32w..32w+31) and apply the fused ReLU /
// 1/deg scaling / row remap. Rows and columns outside a tensor's extent are
// zero-filled by TMA; rows beyond the live count inside the extent are either
// never stored (projection, mean gradient) or zero in the tape (weight gradient).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "gemm.cuh"
#include "umma.cuh"

namespace hetgpu {

namespace {

#ifndef HG_UMMA_ACC
#define HG_UMMA_ACC 4
#endif
#ifndef HG_UMMA_WARPS
#define HG_UMMA_WARPS 8
#endif
constexpr int kUT = HG_UMMA_WARPS * 32;  // threads per CTA: 4 or 8 warps (one or two per TMEM lane quadrant)
constexpr int kConvWarps = HG_UMMA_WARPS - 2;  // warps 2.. form the tf32 residuals
constexpr int kATile = 128 * 128;  // bytes of one 128 x 32 fp32 operand tile
constexpr int kMaxMaps = 2 * kProjGroups * kProjRels;  // [A, B] per (group, relation); 128

template <int NT>
#ifndef HG_PROJ_NT
#define HG_PROJ_NT 64  // widest projection tile
#endif
#ifndef HG_USTAGES128
#define HG_USTAGES128 3  // pipeline stages of the 128-column tiles
#endif
#ifndef HG_USTAGES
#define HG_USTAGES 2  // pipeline stages of the <=64-column tiles (2 measured best: two CTAs per SM)
#endif
struct UStage {
  static constexpr int kB = NT * 128;
  static constexpr int kBytes = 2 * kATile + 2 * kB;  // A, A lo, B, B lo
  static constexpr int kTxBytes = kATile + kB;         // what TMA brings in per stage
  static constexpr int kStages = NT <= 64 ? HG_USTAGES : HG_USTAGES128;
  static constexpr int kSmem = kStages * kBytes + 1024 + 128;
  // kAcc independent TMEM accumulators take the K chunks round robin and are summed in
  // fp32 by the epilogue: the tensor core's accumulation error grows with the length of
  // one accumulation chain (measured: 9e-7 at K = 32, 1e-5 at K = 1024 against fp32)
  static constexpr int kAcc = NT <= 64 ? HG_UMMA_ACC : (HG_UMMA_ACC > 2 ? 2 : HG_UMMA_ACC);
  static constexpr int kAccCols = NT <= 32 ? 32 : NT <= 64 ? 64 : NT <= 128 ? 128 : 256;
  static constexpr int kTmemCols = kAcc * kAccCols;
};

enum Mode { kProject = 0, kDMean = 1, kWGrad = 2 };
// operand majors: projection B = W[k][n] and the weight gradient's A = mean[row][c],
// B = dpre[row][j] are row-contiguous -> MN-major tiles the tensor core transposes
template <int MODE> struct Majors;
template <> struct Majors<kProject> { static constexpr int a = 0, b = 1; };
template <> struct Majors<kDMean> { static constexpr int a = 0, b = 0; };
template <> struct Majors<kWGrad> { static constexpr int a = 1, b = 1; };

template <typename Batch>
struct alignas(64) UmmaArgs {
  CUtensorMap maps[kMaxMaps];  // [A, B] per (problem[, relation])
  Batch b;
  int tile_base[kMaxProblems + 1];
  int n_tiles[kMaxProblems];  // column tiles per problem
  int m_tiles[kMaxProblems];  // weight gradient: din tiles per problem
  int np;
};
__host__ __device__ constexpr int map_index(int mode, int p, int r, int which) {
  return mode == kProject ? (p * kProjRels + r) * 2 + which : p * 2 + which;
}

__device__ __forceinline__ int find_tile(const int* base, int n, int tile) {
  int p = 0;
  while (p + 1 < n && tile >= base[p + 1]) ++p;
  return p;
}

template <int NT, int MODE, typename Batch>
__global__ void __launch_bounds__(kUT) k_umma(const __grid_constant__ UmmaArgs<Batch> args) {
  constexpr int S = UStage<NT>::kStages;
  extern __shared__ std::uint8_t smem_raw[];
  std::uint8_t* smem = reinterpret_cast<std::uint8_t*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                        ~static_cast<std::uintptr_t>(1023));
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + S * UStage<NT>::kBytes);
  std::uint64_t* conv = full + S;  // the stage's tf32 residuals are in place
  std::uint64_t* empty = conv + S;
  std::uint64_t* done = empty + S;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(done + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int p = find_tile(args.tile_base, args.np, blockIdx.x);
  const int t = blockIdx.x - args.tile_base[p];
  const int ntl = args.n_tiles[p];

  // ---- setup, overlapping the predecessor's drain (PDL): barriers, TMEM, the
  // tensor-map descriptors this CTA will use --------------------------------------------------
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      umma::mbar_init(umma::smem_u32(&full[i]), 1);
      umma::mbar_init(umma::smem_u32(&conv[i]), kConvWarps);  // one arrival per converter warp
      umma::mbar_init(umma::smem_u32(&empty[i]), 1);
    }
    umma::mbar_init(umma::smem_u32(done), 1);
    umma::fence_mbar_init();
    int nmaps = 2;
    if constexpr (MODE == kProject) nmaps = 2 * args.b.g[p].nrel;
    for (int i = 0; i < nmaps; ++i) umma::tma_prefetch_desc(&args.maps[map_index(MODE, p, 0, 0) + i]);
  }
  if (warp == 0) umma::tmem_alloc(umma::smem_u32(tmem_slot), UStage<NT>::kTmemCols);
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const std::uint32_t tmem = *tmem_slot;
  pdl_enter();  // everything below reads what earlier kernels wrote

  // ---- tile of this CTA -----------------------------------------------------------------
  int row0 = 0, m0 = 0, n0 = 0, nch = 0, n_live = 0;
  if constexpr (MODE == kProject) {
    const ProjGroup& g = args.b.g[p];
    n_live = *g.n_rows;
    row0 = (t / ntl) * 128;
    n0 = (t % ntl) * NT;
    for (int q = 0; q < g.nrel; ++q) nch += (g.r[q].din + 31) / 32;
  } else if constexpr (MODE == kDMean) {
    const DMeanProblem& P = args.b.p[p];
    n_live = *P.n_rows;
    row0 = (t / ntl) * 128;
    n0 = (t % ntl) * NT;
    nch = (P.d.cols + 31) / 32;
  } else {
    const WGradProblem& P = args.b.p[p];
    n_live = *P.n_rows;
    const int mt = args.m_tiles[p];
    m0 = ((t / ntl) % mt) * 128;
    n0 = (t % ntl) * NT;
    row0 = (t / (mt * ntl)) * kWChunkRows;
    if (row0 < n_live) nch = (min(kWChunkRows, n_live - row0) + 31) / 32;
  }
  if (row0 >= n_live) {  // an idle tile (capacity beyond the live rows)
    if (warp == 0) umma::tmem_dealloc(tmem, UStage<NT>::kTmemCols);
    return;
  }

  if (warp == 0 && lane == 0) {
    // ===== TMA producer =====
    for (int ch = 0; ch < nch; ++ch) {
      const int s = ch % S;
      if (ch >= S) umma::mbar_wait(umma::smem_u32(&empty[s]), ((ch / S) - 1) & 1);
      const std::uint32_t bar = umma::smem_u32(&full[s]);
      umma::mbar_expect_tx(bar, UStage<NT>::kTxBytes);
      const std::uint32_t a_hi = umma::smem_u32(smem + s * UStage<NT>::kBytes);
      const std::uint32_t b_hi = a_hi + 2 * kATile;
      if constexpr (MODE == kProject) {
        const ProjGroup& g = args.b.g[p];
        int q = 0, k0 = ch * 32;
        while (q + 1 < g.nrel && k0 >= ((g.r[q].din + 31) / 32) * 32) {
          k0 -= ((g.r[q].din + 31) / 32) * 32;
          ++q;
        }
        const CUtensorMap* M = &args.maps[map_index(MODE, p, q, 0)];
        umma::tma_load_2d(a_hi, M + 0, k0, row0, bar);  // A = mean rows, K-major
        for (int j = 0; j < NT / 32; ++j)                // B = W[k][n] boxes of 32 n x 32 k
          umma::tma_load_2d(b_hi + j * 4096, M + 1, n0 + 32 * j, k0, bar);
      } else if constexpr (MODE == kDMean) {
        const CUtensorMap* M = &args.maps[map_index(MODE, p, 0, 0)];
        umma::tma_load_2d(a_hi, M + 0, ch * 32, row0, bar);  // A = dpre rows, K-major
        umma::tma_load_2d(b_hi, M + 1, ch * 32, n0, bar);    // B = W rows c, K-major
      } else {
        const CUtensorMap* M = &args.maps[map_index(MODE, p, 0, 0)];
        const int r = row0 + ch * 32;
        for (int j = 0; j < 4; ++j)  // A = mean[row][c]: boxes of 32 c x 32 rows
          umma::tma_load_2d(a_hi + j * 4096, M + 0, m0 + 32 * j, r, bar);
        for (int j = 0; j < NT / 32; ++j)  // B = dpre[row][j]: boxes of 32 j x 32 rows
          umma::tma_load_2d(b_hi + j * 4096, M + 1, n0 + 32 * j, r, bar);
      }
    }
  } else if (warp >= 2) {
    // ===== tf32 split: lo = x - trunc_tf32(x) of the tiles that just landed, written
    // beside them (elementwise, so the swizzled layout carries over) =====
    constexpr int kCT = kConvWarps * 32;
    const int ct = tid - 64;
    for (int ch = 0; ch < nch; ++ch) {
      const int s = ch % S;
      umma::mbar_wait(umma::smem_u32(&full[s]), (ch / S) & 1);
      const float4* a = reinterpret_cast<const float4*>(smem + s * UStage<NT>::kBytes);
      float4* a_lo = const_cast<float4*>(a) + kATile / 16;
#pragma unroll 4
      for (int i = ct; i < kATile / 16; i += kCT) a_lo[i] = tf32_lo4(a[i]);
      const float4* b = a + 2 * kATile / 16;
      float4* b_lo = const_cast<float4*>(b) + UStage<NT>::kB / 16;
#pragma unroll 4
      for (int i = ct; i < UStage<NT>::kB / 16; i += kCT) b_lo[i] = tf32_lo4(b[i]);
      umma::fence_async_smem();  // generic-proxy writes -> visible to the tensor core
      __syncwarp();
      if (lane == 0) umma::mbar_arrive(umma::smem_u32(&conv[s]));
    }
  } else if (warp == 1 && lane == 0) {
    // ===== MMA issuer =====
    constexpr std::uint32_t kIdesc = umma::idesc_tf32(128, NT, Majors<MODE>::a, Majors<MODE>::b);
    auto dsc = [](bool mn, std::uint32_t base, int kk) {
      return mn ? umma::desc_mn_tma(base + 1024u * kk) : umma::desc_k_sw128(base + 32u * kk);
    };
    for (int ch = 0; ch < nch; ++ch) {
      const int s = ch % S;
      const std::uint32_t a_hi = umma::smem_u32(smem + s * UStage<NT>::kBytes), a_lo = a_hi + kATile;
      const std::uint32_t b_hi = a_hi + 2 * kATile, b_lo = b_hi + UStage<NT>::kB;
      // chunk ch accumulates into TMEM accumulator ch % kAcc (its first chunk starts it)
      constexpr int kA = UStage<NT>::kAcc;
      const std::uint32_t acc = tmem + static_cast<std::uint32_t>((ch % kA) * UStage<NT>::kAccCols);
      const bool first = ch < kA;
      // hi.hi as soon as the tiles land (overlaps the residual pass) ...
      umma::mbar_wait(umma::smem_u32(&full[s]), (ch / S) & 1);
      umma::fence_after_sync();
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)  // 8 tf32 of K per MMA
        umma::mma_tf32(acc, dsc(Majors<MODE>::a, a_hi, kk), dsc(Majors<MODE>::b, b_hi, kk), kIdesc,
                       (!first || kk > 0) ? 1u : 0u);
      // ... then the two residual products
      umma::mbar_wait(umma::smem_u32(&conv[s]), (ch / S) & 1);
      umma::fence_after_sync();
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const std::uint64_t ah = dsc(Majors<MODE>::a, a_hi, kk), al = dsc(Majors<MODE>::a, a_lo, kk);
        const std::uint64_t bh = dsc(Majors<MODE>::b, b_hi, kk), bl = dsc(Majors<MODE>::b, b_lo, kk);
        umma::mma_tf32(acc, ah, bl, kIdesc, 1u);
        umma::mma_tf32(acc, al, bh, kIdesc, 1u);
      }
      umma::commit(umma::smem_u32(&empty[s]));  // frees the stage once these MMAs are done
    }
    umma::commit(umma::smem_u32(done));  // accumulator complete
  }
  __syncwarp();
  umma::mbar_wait(umma::smem_u32(done), 0);
  umma::fence_after_sync();

  // ---- epilogue: TMEM -> registers -> global ---------------------------------------------------
  // warp w reads TMEM lane quadrant w % 4 (its tile rows) and column half w / 4
  const int quad = warp & 3;
  const int m = quad * 32 + lane;  // tile row owned by this thread
  const std::uint32_t trow = tmem + (static_cast<std::uint32_t>(quad * 32) << 16);
  constexpr int kEpiWarps = HG_UMMA_WARPS < 8 ? HG_UMMA_WARPS : 8;  // warps draining TMEM
  constexpr int kColsPerWarp = NT / (kEpiWarps / 4);
  const int c_begin = warp < kEpiWarps ? (warp >> 2) * kColsPerWarp : NT;
#pragma unroll 1
  for (int c0 = c_begin; c0 < c_begin + kColsPerWarp && c0 < NT; c0 += 16) {
    float v[16];
    umma::tmem_ld16(trow + c0, v);
    // the other accumulators (only those that received a chunk), summed in fp32
    for (int a = 1; a < UStage<NT>::kAcc && a < nch; ++a) {
      float u[16];
      umma::tmem_ld16(trow + static_cast<std::uint32_t>(a * UStage<NT>::kAccCols) + c0, u);
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] += u[j];
    }
    if constexpr (MODE == kProject) {
      const ProjGroup& g = args.b.g[p];
      const int row = row0 + m;
      if (row < n_live) {
        float* orow = g.out + static_cast<std::size_t>(row * g.out_stride + g.out_offset) * g.ld_out;
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          const int col = n0 + c0 + j;
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
      const int row = row0 + m;
      if (row < n_live) {
        const std::uint32_t deg = P.indptr[row + 1] - P.indptr[row];
        const float inv = deg ? 1.0f / static_cast<float>(deg) : 0.0f;
        float* orow = P.dmean + static_cast<std::size_t>(row) * P.ld_dmean;
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          const int col = n0 + c0 + j;
          if (col < P.ld_dmean)
            *reinterpret_cast<float4*>(orow + col) =
                make_float4(v[j] * inv, v[j + 1] * inv, v[j + 2] * inv, v[j + 3] * inv);
        }
      }
    } else {
      const WGradProblem& P = args.b.p[p];
      const int row = m0 + m;  // din index
      if (row < P.din) {
        const int chunk = row0 / kWChunkRows;
        float* out = P.partial + (static_cast<std::size_t>(chunk) * P.din + row) * P.d.cols;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int col = n0 + c0 + j;
          if (col < P.d.cols) out[col] = v[j];
        }
      }
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, UStage<NT>::kTmemCols);
}

// ---- host side: tensor maps ----------------------------------------------------------------------

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    HG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// fp32 row-major [rows x cols] with `row_stride` elements between rows, read in
// boxes of 32 columns x box_rows rows
void encode(CUtensorMap* m, const float* base, std::uint64_t cols, std::uint64_t rows, std::uint64_t row_stride,
            std::uint32_t box_rows, bool mn_major) {
  if (!base) throw std::invalid_argument("tensor-core operand without a buffer");
  const cuuint64_t dims[2] = {cols, std::max<std::uint64_t>(1, rows)};
  const cuuint64_t strides[1] = {row_stride * 4};
  const cuuint32_t box[2] = {32, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
}

template <int NT, int MODE, typename Batch>
void launch(UmmaArgs<Batch>& a, int tiles, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    HG_CUDA(cudaFuncSetAttribute(k_umma<NT, MODE, Batch>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 UStage<NT>::kSmem));
    attr = true;
  }
  launch_pdl(k_umma<NT, MODE, Batch>, tiles, kUT, UStage<NT>::kSmem, st, a);
}

// column tile width (multiples of 32 for the MN-major boxes); wider outputs take
// several 128-wide tiles (349 classes -> 3)
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
// The tensor maps are encoded on the host per launch and travel in the kernel
// parameters (a captured CUDA graph keeps them).
void project_umma(ProjBatch& pb, cudaStream_t st) {
  if (pb.ng == 0) return;
  static thread_local UmmaArgs<ProjBatch> a;
  a = UmmaArgs<ProjBatch>{};
  a.b = pb;
  a.np = pb.ng;
  int nt = 32;
  for (int g = 0; g < pb.ng; ++g) nt = std::max(nt, pick_nt(pb.g[g].ld_out));
  // at most 64 columns per tile: the top layer (C = 349) then runs 48 CTAs
  // instead of 24, which shortens its latency-bound launch (measured +2%); outputs of
  // 512+ columns (RGAT's per-head aggregates) keep 128-wide tiles (half the CTAs)
  int widest = 0;
  for (int g = 0; g < pb.ng; ++g) widest = std::max(widest, pb.g[g].ld_out);
  if (widest < 512) nt = std::min(nt, HG_PROJ_NT);
  int tiles = 0;
  for (int g = 0; g < pb.ng; ++g) {
    const ProjGroup& G = pb.g[g];
    a.tile_base[g] = tiles;
    a.n_tiles[g] = static_cast<int>(ceil_div(G.ld_out, nt));
    tiles += static_cast<int>(ceil_div(std::max(1, G.rows_cap), 128)) * a.n_tiles[g];
    for (int r = 0; r < G.nrel; ++r) {
      const ProjRel& R = G.r[r];
      CUtensorMap* M = &a.maps[map_index(kProject, g, r, 0)];
      encode(M + 0, R.mean, R.ld_mean, G.rows_cap, R.row_stride ? R.row_stride : R.ld_mean, 128, false);
      encode(M + 1, R.w, R.ld_w, R.din, R.ld_w, 32, true);
    }
  }
  a.tile_base[pb.ng] = tiles;
  dispatch<kProject>(a, nt, tiles, st);
}

void dmean_umma(DMeanBatch& b, cudaStream_t st) {
  if (b.np == 0) return;
  static thread_local UmmaArgs<DMeanBatch> a;
  a = UmmaArgs<DMeanBatch>{};
  a.b = b;
  a.np = b.np;
  int nt = 32;
  for (int q = 0; q < b.np; ++q) nt = std::max(nt, pick_nt(b.p[q].ld_dmean));
  int tiles = 0;
  for (int q = 0; q < b.np; ++q) {
    const DMeanProblem& P = b.p[q];
    if (P.d.h) throw std::invalid_argument("tcgen05 mean gradient expects an already masked dpre");
    a.tile_base[q] = tiles;
    a.n_tiles[q] = static_cast<int>(ceil_div(P.ld_dmean, nt));
    tiles += static_cast<int>(ceil_div(std::max(1, P.rows_cap), 128)) * a.n_tiles[q];
    CUtensorMap* M = &a.maps[map_index(kDMean, q, 0, 0)];
    const std::size_t off = static_cast<std::size_t>(P.d.offset) * P.d.ld;
    const std::uint64_t rstride = static_cast<std::uint64_t>(P.d.stride) * P.d.ld;
    encode(M + 0, P.d.g + off, P.d.ld, P.rows_cap, rstride, 128, false);
    encode(M + 1, P.w, P.ld_w, P.din, P.ld_w, nt, false);
  }
  a.tile_base[b.np] = tiles;
  dispatch<kDMean>(a, nt, tiles, st);
}

void wgrad_umma(WGradBatch& b, cudaStream_t st) {
  if (b.np == 0) return;
  static thread_local UmmaArgs<WGradBatch> a;
  a = UmmaArgs<WGradBatch>{};
  a.b = b;
  a.np = b.np;
  int nt = 32;
  for (int q = 0; q < b.np; ++q) nt = std::max(nt, pick_nt(b.p[q].d.cols));
  int tiles = 0;
  for (int q = 0; q < b.np; ++q) {
    const WGradProblem& P = b.p[q];
    if (P.d.h) throw std::invalid_argument("tcgen05 weight gradient expects an already masked dpre");
    a.tile_base[q] = tiles;
    a.n_tiles[q] = static_cast<int>(ceil_div(P.d.cols, nt));
    a.m_tiles[q] = static_cast<int>(ceil_div(P.din, 128));
    tiles += static_cast<int>(ceil_div(std::max(1, P.rows_cap), kWChunkRows)) * a.m_tiles[q] * a.n_tiles[q];
    CUtensorMap* M = &a.maps[map_index(kWGrad, q, 0, 0)];
    const std::size_t off = static_cast<std::size_t>(P.d.offset) * P.d.ld;
    const std::uint64_t rstride = static_cast<std::uint64_t>(P.d.stride) * P.d.ld;
    encode(M + 0, P.mean, P.ld_mean, P.rows_cap, P.ld_mean, 32, true);
    encode(M + 1, P.d.g + off, P.d.ld, P.rows_cap, rstride, 32, true);
  }
  a.tile_base[b.np] = tiles;
  dispatch<kWGrad>(a, nt, tiles, st);
  if (!b.defer_reduce) wgrad_reduce(b, st);
}

}  // namespace hetgpu
