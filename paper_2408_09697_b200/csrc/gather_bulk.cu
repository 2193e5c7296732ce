// Layer-input gather-mean through bulk copies (hgnn.cpp:223-242 gather, raf.cpp:178-194
// mean; same sums as k_gather_mean, bit for bit): every neighbour row is one
// cp.async.bulk global -> shared of the whole row, so a row costs one request, the
// copy engine keeps HG_BULK_SLOTS rows in flight per warp independently of the
// register budget, and the row is read from HBM contiguously.
//
// A warp owns a contiguous slice of destination rows of one block, hence one
// contiguous edge range [E0, E1) of its CSR; it streams those edges through a ring of
// HG_BULK_SLOTS row slots in shared memory (slot j % S, mbarrier phase (j / S) & 1):
// the edge j + S is issued as soon as edge j's row has been summed. Keys come 32 at a
// time (lane l holds key E0 + 32 w + l and issues that edge's copy); row ends come 32
// at a time from indptr. Each lane sums 16-byte column chunks (p * 32 + lane) of every
// row in edge order, as the register gather does, and writes the mean row.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "gemm.cuh"
#include "umma.cuh"

#ifndef HG_BULK_SLOTS
#define HG_BULK_SLOTS 16
#endif
#ifndef HG_BULK_WARPS
#define HG_BULK_WARPS 4
#endif

namespace hetgpu {

namespace {

constexpr int kSlots = HG_BULK_SLOTS;  // rows in flight per warp (divides 32)
constexpr int kWarps = HG_BULK_WARPS;  // warps per CTA
constexpr int kMaxRowBytes = 4096;     // 16-byte chunks per lane: <= 8 fp32 or 4 half chunks
static_assert(32 % kSlots == 0, "a lane issues the copies of the edges it holds keys for");

__device__ __forceinline__ void bulk_row(std::uint32_t dst, const void* src, std::uint32_t bytes, std::uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// acc += the 16-byte chunk of one row
template <bool HALF>
__device__ __forceinline__ void add_chunk(float* acc, const uint4& raw, int dtype) {
  if constexpr (HALF) {
    const std::uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = dtype == kF16 ? __half22float2(*reinterpret_cast<const __half2*>(&w[j]))
                                     : __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[j]));
      acc[2 * j] += f.x;
      acc[2 * j + 1] += f.y;
    }
  } else {
    acc[0] += __uint_as_float(raw.x);
    acc[1] += __uint_as_float(raw.y);
    acc[2] += __uint_as_float(raw.z);
    acc[3] += __uint_as_float(raw.w);
  }
}

// one block segment [r0, r1) of a warp: HALF = 8 features per chunk (P <= 4), else 4 (P <= 8)
template <bool HALF>
__device__ __forceinline__ void segment(const MeanBlock& B, int r0, int r1, std::uint32_t ring, std::uint32_t bars,
                                        std::uint32_t row_bytes, std::uint32_t& uses, int lane) {
  constexpr int PMAX = HALF ? 4 : 8;
  constexpr int F = HALF ? 8 : 4;
  const int P = static_cast<int>((row_bytes + 511) / 512);
  const std::uint32_t E0 = __ldg(B.indptr + r0), E1 = __ldg(B.indptr + r1);
  const char* table = reinterpret_cast<const char*>(B.h);
  std::uint32_t key = 0;
  // producer: edge j of the segment (uniform j); the lane holding its key issues the copy
  auto issue = [&](std::uint32_t j) {
    if ((j & 31u) == 0) key = E0 + j + lane < E1 ? __ldg(B.keys + E0 + j + lane) : 0u;
    if (lane == static_cast<int>(j & 31u)) {
      const std::uint32_t u = uses + j, s = u % kSlots;
      umma::fence_async_smem();  // the slot's previous row was read through the generic proxy
      umma::mbar_expect_tx(bars + 8 * s, row_bytes);
      bulk_row(ring + s * row_bytes, table + static_cast<std::size_t>(key) * row_bytes, row_bytes, bars + 8 * s);
    }
  };
  const std::uint32_t n = E1 - E0;
  for (std::uint32_t j = 0; j < min(n, static_cast<std::uint32_t>(kSlots)); ++j) issue(j);
  // row ends, 32 rows per load
  int rbase = r0;
  std::uint32_t ends = rbase + lane < r1 ? __ldg(B.indptr + rbase + 1 + lane) : 0u;
  int r = r0;
  std::uint32_t rend = __shfl_sync(0xffffffffu, ends, 0);
  float acc[PMAX * F];
#pragma unroll
  for (int k = 0; k < PMAX * F; ++k) acc[k] = 0.f;
  auto finish_row = [&](std::uint32_t lo) {
    const std::uint32_t deg = rend - lo;
    const float inv = deg ? 1.0f / static_cast<float>(deg) : 0.f;
    float* orow = B.mean + static_cast<std::size_t>(r) * B.ld_mean;
#pragma unroll
    for (int p = 0; p < PMAX; ++p) {
      const int c = (p * 32 + lane) * F;
#pragma unroll
      for (int q = 0; q < F; q += 4)
        if (p < P && c + q < B.ld_mean)
          *reinterpret_cast<float4*>(orow + c + q) = make_float4(acc[p * F + q] * inv, acc[p * F + q + 1] * inv,
                                                                 acc[p * F + q + 2] * inv, acc[p * F + q + 3] * inv);
    }
#pragma unroll
    for (int k = 0; k < PMAX * F; ++k) acc[k] = 0.f;
    ++r;
    if (r < r1) {
      if (r - rbase == 32) {
        rbase = r;
        ends = rbase + lane < r1 ? __ldg(B.indptr + rbase + 1 + lane) : 0u;
      }
      rend = __shfl_sync(0xffffffffu, ends, r - rbase);
    }
  };
  std::uint32_t rlo = E0;
  for (std::uint32_t j = 0; j < n; ++j) {
    const std::uint32_t e = E0 + j;
    while (e == rend) {  // rows that end here (empty rows included)
      finish_row(rlo);
      rlo = e;
    }
    const std::uint32_t u = uses + j, s = u % kSlots;
    umma::mbar_wait(bars + 8 * s, (u / kSlots) & 1u);
#pragma unroll
    for (int p = 0; p < PMAX; ++p) {
      if (p < P && static_cast<std::uint32_t>(p * 32 + lane) * 16u < row_bytes) {
        uint4 raw;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(raw.x), "=r"(raw.y), "=r"(raw.z), "=r"(raw.w)
                     : "r"(ring + s * row_bytes + (p * 32 + lane) * 16));
        add_chunk<HALF>(acc + p * F, raw, B.h_dtype);
      }
    }
    __syncwarp();
    if (j + kSlots < n) issue(j + kSlots);
  }
  while (r < r1) {  // the last rows (and trailing empty ones)
    finish_row(rlo);
    rlo = E1;
  }
  uses += n;
}

__global__ void __launch_bounds__(kWarps * 32) k_gather_bulk(MeanBatch m, std::uint32_t slot_bytes) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t bars = umma::smem_u32(smem) + warp * kSlots * 8;
  const std::uint32_t ring = umma::smem_u32(smem) + kWarps * kSlots * 8 + warp * kSlots * slot_bytes;
  if (lane == 0) {
    for (int s = 0; s < kSlots; ++s) umma::mbar_init(bars + 8 * s, 1);
    umma::fence_mbar_init();
  }
  __syncwarp();
  pdl_enter();
  // live rows of every block, split evenly over the grid's warps
  int total = 0;
  for (int b = 0; b < m.nb; ++b) total += *m.b[b].n_rows;
  const int nw = gridDim.x * kWarps, w = blockIdx.x * kWarps + warp;
  const int g0 = static_cast<int>(static_cast<long long>(total) * w / nw);
  const int g1 = static_cast<int>(static_cast<long long>(total) * (w + 1) / nw);
  std::uint32_t uses = 0;
  int base = 0;
  for (int b = 0; b < m.nb && base < g1; ++b) {
    const MeanBlock& B = m.b[b];
    const int n = *B.n_rows;
    const int r0 = max(g0 - base, 0), r1 = min(g1 - base, n);
    if (r0 < r1) {
      const std::uint32_t rb = static_cast<std::uint32_t>(B.ld_h) * (B.h_dtype == kF32 ? 4u : 2u);
      if (B.h_dtype == kF32)
        segment<false>(B, r0, r1, ring, bars, rb, uses, lane);
      else
        segment<true>(B, r0, r1, ring, bars, rb, uses, lane);
    }
    base += n;
  }
  // zero tails up to the next 32-row boundary (the weight gradient's K chunks)
  for (int b = 0; b < m.nb; ++b) {
    const MeanBlock& B = m.b[b];
    const int n = *B.n_rows, pad = ((n + 31) & ~31) - n;
    const int per = B.ld_mean / 4;
    for (int x = w * 32 + lane; x < pad * per; x += nw * 32)
      *reinterpret_cast<float4*>(B.mean + static_cast<std::size_t>(n + x / per) * B.ld_mean + 4 * (x % per)) =
          make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

}  // namespace

bool gather_mean_bulk(MeanBatch& m, cudaStream_t st) {
  static const bool on = [] {
    const char* e = std::getenv("HG_GATHER_BULK");
    return e != nullptr && e[0] == '1';
  }();
  if (!on || m.nb == 0) return false;
  std::uint32_t slot = 0;
  long long cap = 0;
  for (int b = 0; b < m.nb; ++b) {
    const MeanBlock& B = m.b[b];
    if (B.slot != nullptr || B.ld_mean % 4 != 0) return false;  // host tables keep the slot-map gather
    const std::uint32_t rb = static_cast<std::uint32_t>(B.ld_h) * (B.h_dtype == kF32 ? 4u : 2u);
    if (rb % 16 != 0 || rb > static_cast<std::uint32_t>(kMaxRowBytes)) return false;
    if (B.ld_mean > B.ld_h) return false;
    slot = std::max(slot, rb);
    cap += B.rows_cap;
  }
  const std::size_t smem = static_cast<std::size_t>(kWarps) * kSlots * (8 + slot);
  static int max_smem = 0;
  if (!max_smem) {
    HG_CUDA(cudaFuncSetAttribute(k_gather_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    max_smem = 227 * 1024;
  }
  if (smem > static_cast<std::size_t>(max_smem)) return false;
  const int per_sm = std::max(1, std::min(32 / kWarps, static_cast<int>((228 * 1024) / (smem + 1024))));
  const unsigned grid = static_cast<unsigned>(
      std::max<long long>(1, std::min<long long>(static_cast<long long>(per_sm) * num_sms(), ceil_div(cap, 8 * kWarps))));
  launch_pdl(k_gather_bulk, grid, kWarps * 32, smem, st, m, slot);
  return true;
}

}  // namespace hetgpu
