// tcgen05 (5th-gen tensor core) building blocks for sm_100a, written as inline
// PTX: TMEM allocation, shared-memory matrix descriptors (K-major, 128-byte
// swizzle), the kind::tf32 MMA, commit-to-mbarrier and the TMEM -> register
// epilogue load. Descriptor bit layouts follow the sm100 UMMA formats
// (SmemDescriptor / InstrDescriptor).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace hetgpu {
namespace umma {

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier ----------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(std::uint32_t bar, std::uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint32_t bar, std::uint32_t parity) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t"
      "}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(std::uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// ---- fences --------------------------------------------------------------------------------
// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// ---- TMEM allocation (one full warp) -------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(std::uint32_t slot_smem, std::uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot_smem), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(std::uint32_t taddr, std::uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// ---- descriptors -------------------------------------------------------------------------------
// K-major operand tile, rows of 128 bytes (32 fp32/tf32 elements of K), 128-byte
// swizzle: 16-byte chunk c of row r lives at chunk (c ^ (r & 7)); 8-row groups
// are 1024 bytes apart (SBO). The tile base must be 1024-byte aligned.
__device__ __forceinline__ std::uint64_t desc_k_sw128(std::uint32_t saddr) {
  std::uint64_t d = 0;
  d |= static_cast<std::uint64_t>((saddr & 0x3FFFFu) >> 4);  // start address  [0,14)
  d |= static_cast<std::uint64_t>(1) << 16;                   // LBO (unused for swizzled K-major)
  d |= static_cast<std::uint64_t>(1024 >> 4) << 32;           // SBO = 1024 B   [32,46)
  d |= static_cast<std::uint64_t>(1) << 46;                   // descriptor version (sm100)
  d |= static_cast<std::uint64_t>(2) << 61;                   // SWIZZLE_128B
  return d;
}
// MN-major tf32 operand tile (the only MN-major layout tcgen05 accepts for
// 32-bit types: SWIZZLE_128B_BASE32B): 32 consecutive M (or N) elements form a
// 128-byte row, 4 K-rows form a 512-byte atom in which 32-byte chunk c of row r
// lives at chunk (c ^ r). Atoms along M/N are LBO = 512 bytes apart, 4-row K
// groups SBO bytes apart; one MMA (K = 8) spans two K groups. The tensor core
// reads the transpose directly, so row-contiguous sources are stored with
// 16-byte vector stores (no bank conflicts).
constexpr std::uint32_t kMnLbo = 512;
__device__ __forceinline__ std::uint64_t desc_mn_sw128_32b(std::uint32_t saddr, std::uint32_t sbo) {
  std::uint64_t d = 0;
  d |= static_cast<std::uint64_t>((saddr & 0x3FFFFu) >> 4);  // start address
  d |= static_cast<std::uint64_t>(kMnLbo >> 4) << 16;         // LBO: next 32-element M/N atom
  d |= static_cast<std::uint64_t>(sbo >> 4) << 32;            // SBO: next 4-row K group
  d |= static_cast<std::uint64_t>(1) << 46;                   // descriptor version (sm100)
  d |= static_cast<std::uint64_t>(1) << 61;                   // SWIZZLE_128B_BASE32B
  return d;
}
// The same MN-major layout as written by TMA boxes of 32 (M/N) x 32 (K) fp32
// with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B: each box is 32 K-rows of 128 bytes
// (4-row groups SBO = 512 bytes apart), consecutive M/N atoms LBO = 4096 apart.
__device__ __forceinline__ std::uint64_t desc_mn_tma(std::uint32_t saddr) {
  std::uint64_t d = 0;
  d |= static_cast<std::uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<std::uint64_t>(4096 >> 4) << 16;  // LBO: next 32-element M/N box
  d |= static_cast<std::uint64_t>(512 >> 4) << 32;   // SBO: next 4-row K group
  d |= static_cast<std::uint64_t>(1) << 46;
  d |= static_cast<std::uint64_t>(1) << 61;          // SWIZZLE_128B_BASE32B
  return d;
}

// ---- TMA ----------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_expect_tx(std::uint32_t bar, std::uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// 2-D tiled bulk tensor copy global -> shared, completion counted on `bar`
__device__ __forceinline__ void tma_load_2d(std::uint32_t dst, const void* tmap, int c0, int c1, std::uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(tmap), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

// byte offset of elements (m..m+3, k) (m % 4 == 0) in such a tile
__device__ __forceinline__ std::uint32_t sw128b32_mn(int m, int k, std::uint32_t sbo) {
  return static_cast<std::uint32_t>((k >> 2) * sbo + (m >> 5) * kMnLbo + (k & 3) * 128 +
                                    ((((m & 31) >> 3) ^ (k & 3)) << 5) + ((m & 7) << 2));
}
// byte offset of the 16-byte chunk `c` (0..7) of row `r` in such a tile
__device__ __forceinline__ std::uint32_t sw128_chunk(int r, int c) {
  return static_cast<std::uint32_t>((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}

// instruction descriptor: D f32, A/B tf32, M x N; a_mn / b_mn select MN-major operands
__host__ __device__ constexpr std::uint32_t idesc_tf32(int M, int N, int a_mn = 0, int b_mn = 0) {
  return (1u << 4)                                       // D format f32
         | (2u << 7)                                     // A format tf32
         | (2u << 10)                                    // B format tf32
         | (static_cast<std::uint32_t>(a_mn) << 15)      // A major
         | (static_cast<std::uint32_t>(b_mn) << 16)      // B major
         | (static_cast<std::uint32_t>(N >> 3) << 17)    // N / 8
         | (static_cast<std::uint32_t>(M >> 4) << 24);   // M / 16
}

// D[tmem] (+)= A[smem] . B[smem]^T, issued by one thread
__device__ __forceinline__ void mma_tf32(std::uint32_t d_tmem, std::uint64_t a, std::uint64_t b, std::uint32_t idesc,
                                         std::uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on `bar` once every previously issued tcgen05 op of this thread completed
__device__ __forceinline__ void commit(std::uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// 32 lanes x 16 consecutive fp32 columns: thread t of the warp gets lane (base lane + t)
__device__ __forceinline__ void tmem_ld16(std::uint32_t taddr, float (&v)[16]) {
  std::uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 3xTF32 split: x = hi + lo with hi = x truncated to tf32 (the tensor core reads
// the top 19 bits of each 32-bit container) and lo = x - hi exactly in fp32.
// hi.hi + hi.lo + lo.hi recovers ~fp32 accuracy (error ~2^-21 relative).
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = x - hi;
}

}  // namespace umma
}  // namespace hetgpu
