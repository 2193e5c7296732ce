// Integer/byte work of the hot path: per-relation fanout sampling with the
// reference's exact RNG, segmented scans, and the bitmap frontier that
// replaces the reference's per-hop sort+unique (sampling.cpp:82-89) and its
// per-edge binary searches (hgnn.cpp:166-171). All HBM-bound; grids are sized
// in multiples of the SM count or from capacities and read live counts.
#include <algorithm>

#include "kernels.cuh"

namespace hetgpu {

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  HG_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) HG_CUDA(cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev));
  return cache[dev];
}

namespace {

#ifndef HG_SAMPLE_RNG_FIRST
#define HG_SAMPLE_RNG_FIRST 0
#endif
#ifndef HG_SAMPLE_UNROLL
#define HG_SAMPLE_UNROLL 4  // sampled edges in flight per lane in the sampler's gather
#endif
#ifndef HG_SCAN_THREADS
#define HG_SCAN_THREADS 512
#endif
constexpr int kScanThreads = HG_SCAN_THREADS;
constexpr int kScanPer = kScanTile / kScanThreads;  // 8 elements per thread

__device__ __forceinline__ std::uint32_t warp_incl_scan(std::uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const std::uint32_t n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// block-wide inclusive scan of one value per thread; returns inclusive value,
// *total receives the block total
template <int NT>
__device__ __forceinline__ std::uint32_t block_incl_scan(std::uint32_t v, std::uint32_t* total) {
  __shared__ std::uint32_t warp_tot[NT / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  std::uint32_t x = warp_incl_scan(v);
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    std::uint32_t t = lane < NT / 32 ? warp_tot[lane] : 0u;
    t = warp_incl_scan(t);
    if (lane < NT / 32) warp_tot[lane] = t;
  }
  __syncthreads();
  if (wid > 0) x += warp_tot[wid - 1];
  if (total) *total = warp_tot[NT / 32 - 1];
  __syncthreads();
  return x;
}

// Decoupled look-back (single-pass prefix): tiles take dynamic ticket ids in
// launch order, publish their aggregate, then walk back until a tile that has
// published its inclusive prefix. Flag and value share one 64-bit word.
constexpr unsigned long long kLbAgg = 1ull << 32, kLbPre = 2ull << 32;

__device__ __forceinline__ unsigned long long lb_load(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

// warp 0 only (all 32 lanes): exclusive prefix of tile t inside its segment
// state array. The warp inspects 32 predecessors at once: the nearest one with
// an inclusive prefix ends the walk, aggregates in between are summed; a
// predecessor that has published nothing yet makes the warp re-read.
__device__ __forceinline__ std::uint32_t lb_prefix(unsigned long long* st, int t, std::uint32_t agg) {
  const int lane = threadIdx.x & 31;
  if (t == 0) {
    if (lane == 0) atomicExch(st, kLbPre | agg);
    return 0;
  }
  if (lane == 0) atomicExch(st + t, kLbAgg | agg);
  std::uint32_t excl = 0;
  int hi = t - 1;  // window [hi-31, hi]
  while (true) {
    const int j = hi - lane;
    const unsigned long long v = j >= 0 ? lb_load(st + j) : kLbPre;  // virtual prefix 0 before tile 0
    const unsigned long long flag = v >> 32;
    const unsigned waiting = __ballot_sync(0xffffffffu, flag == 0);
    const unsigned prefix = __ballot_sync(0xffffffffu, flag == 2);
    // lanes up to the nearest prefix (lowest lane with flag 2) must all be ready
    const int stop = prefix ? __ffs(prefix) - 1 : 31;
    const unsigned needed = stop == 31 ? 0xffffffffu : ((1u << (stop + 1)) - 1u);
    if (waiting & needed) continue;  // spin on the same window
    std::uint32_t part = lane <= stop ? static_cast<std::uint32_t>(v) : 0u;
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    excl += part;
    if (prefix) break;
    hi -= 32;
  }
  if (lane == 0) atomicExch(st + t, kLbPre | (excl + agg));
  return excl;
}

// ticket -> (segment, tile) over per-segment tile counts (tile_base prefix)
__device__ __forceinline__ int seg_of(const int* base, int nseg, int ticket) {
  int s = 0;
  while (s + 1 < nseg && ticket >= base[s + 1]) ++s;
  return s;
}

struct LbLayout {
  int base[kMaxSegs + 1];  // per segment: first ticket / first state slot
  int nseg;
  int item[kMaxSegs];      // sampler: the block each segment (in ticket order) stands for
};

__global__ void __launch_bounds__(kScanThreads) k_scan_lb(ScanArgs a, LbLayout L, unsigned long long* state,
                                                          int* ticket) {
  pdl_enter();
  __shared__ int s_tile;
  __shared__ std::uint32_t s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
  __syncthreads();
  const int tk = s_tile;
  if (tk >= L.base[L.nseg]) return;
  const int sg = seg_of(L.base, L.nseg, tk);
  const int t = tk - L.base[sg];
  const ScanSeg& S = a.s[sg];
  const int n = *S.n;
  const int first = t * kScanTile + threadIdx.x * kScanPer;
  if (t * kScanTile >= n) return;  // beyond the live data: nobody waits on it
  std::uint32_t v[kScanPer];
  std::uint32_t local = 0;
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) {
    const int idx = first + j;
    v[j] = idx < n ? S.data[idx] : 0u;
    local += v[j];
  }
  std::uint32_t tot;
  const std::uint32_t incl = block_incl_scan<kScanThreads>(local, &tot);
  if (threadIdx.x < 32) {
    const std::uint32_t p = lb_prefix(state + L.base[sg], t, tot);
    if (threadIdx.x == 0) s_prefix = p;
  }
  __syncthreads();
  std::uint32_t run = s_prefix + incl - local;
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) {
    const int idx = first + j;
    run += v[j];
    if (idx < n) S.data[idx] = run;
  }
}

}  // namespace

void scan_inclusive(const ScanArgs& a, LbScratch& lb, cudaStream_t st) {
  if (a.nseg == 0) return;
  LbLayout L{};
  L.nseg = a.nseg;
  int tiles = 0;
  for (int i = 0; i < a.nseg; ++i) {
    L.base[i] = tiles;
    tiles += static_cast<int>(ceil_div(std::max(1, a.s[i].cap), kScanTile));
  }
  L.base[a.nseg] = tiles;
  lb.reset(tiles, st);
  launch_pdl(k_scan_lb, tiles, kScanThreads, 0, st, a, L, lb.state, lb.ticket);
}

// ---- sampling -------------------------------------------------------------------------

namespace {

constexpr int kSampleThreads = kSampleTileRows;
constexpr int kSlowThreads = 4096;  // concurrent slow-path rows (global scratch)

// Same draws with the dependency chain cut short. The mt19937_64 outputs
// j < fanout need only x[j], x[j+1] and x[j+156] of the seeding recurrence
// (first twist), so after the 156-step seeding two independent step chains
// produce all outputs; each output's Lemire offset depends only on it and on
// deg - i (assuming no rejection: a product below the range, probability
// ~deg/2^64, sends the row to the exact slow path). The partial Fisher-Yates
// is then resolved per draw without sequential swaps: the value at position p
// before swap i is p unless an earlier swap k < i moved position k onto p
// (j_k == p, the latest such k), in which case it is the value position k held
// before swap k (sampling.cpp:28-37). jcol: this lane's column of MAXF words.
template <int MAXF>
__device__ __forceinline__ bool draw_positions_fast(std::uint64_t seed, std::uint64_t deg, int fanout,
                                                    std::uint32_t* out) {
  std::uint64_t xa = seed, xa1 = Mt64::step(seed, 1), xb = xa1;
#pragma unroll 4
  for (std::uint32_t i = 2; i <= 156; ++i) xb = Mt64::step(xb, i);
  bool exact = true;
  std::uint32_t jr[MAXF];  // j_q = q + offset_q, in registers (the loops below are unrolled)
#pragma unroll
  for (int q = 0; q < MAXF; ++q) {
    jr[q] = 0xFFFFFFFFu;
    if (q < fanout) {
      const std::uint64_t t = Mt64::temper(Mt64::twist(xa, xa1, xb));
      const std::uint64_t range = deg - static_cast<std::uint64_t>(q);
      exact &= t * range >= range;  // otherwise Lemire may reject: replay exactly
      jr[q] = static_cast<std::uint32_t>(q + __umul64hi(t, range));
      xa = xa1;
      xa1 = Mt64::step(xa1, static_cast<std::uint32_t>(q) + 2u);
      xb = Mt64::step(xb, static_cast<std::uint32_t>(q) + 157u);
    }
  }
  if (!exact) return false;
#pragma unroll
  for (int i = 0; i < MAXF; ++i) {
    if (i < fanout) {
      std::uint32_t p = jr[i];
      int found = -1;  // latest earlier swap that moved a position onto p
#pragma unroll
      for (int q = 0; q < i; ++q)
        if (jr[q] == p) found = q;
      while (found >= 0) {  // rare: follow the chain of displaced positions
        const int k = found;
        p = static_cast<std::uint32_t>(k);
        found = -1;
#pragma unroll
        for (int q = 0; q < MAXF; ++q)
          if (q < k && jr[q] == p) found = q;
      }
      out[i] = p;  // position in the CSR row; the warp gathers the ids afterwards
    }
  }
  return true;
}

// generic (memory-backed map) variant for the slow path
template <typename Eng>
__device__ bool draw_row(Eng& eng, std::uint64_t deg, int fanout, const std::uint32_t* nbr,
                         std::uint32_t* out, std::uint32_t* mpos, std::uint32_t* mval) {
  int nmap = 0;
  for (int i = 0; i < fanout; ++i) {
    std::uint64_t off;
    if (!lemire(eng, deg - static_cast<std::uint64_t>(i), off)) return false;
    const std::uint32_t jpos = static_cast<std::uint32_t>(i + off);
    std::uint32_t vi = static_cast<std::uint32_t>(i), vj = jpos;
    int slot_j = -1;
    for (int q = 0; q < nmap; ++q) {
      const std::uint32_t pq = mpos[q];
      if (pq == static_cast<std::uint32_t>(i)) vi = mval[q];
      if (pq == jpos) {
        vj = mval[q];
        slot_j = q;
      }
    }
    if (jpos != static_cast<std::uint32_t>(i)) {
      if (slot_j < 0) {
        slot_j = nmap++;
        mpos[slot_j] = jpos;
      }
      mval[slot_j] = vi;
    }
    out[i] = nbr[vj];
  }
  return true;
}

// One CTA = one tile of 256 rows of one block. Counts -> CTA scan -> look-back
// for the tile's offset -> block offsets written -> copy-all rows (warp-
// cooperative, coalesced) and RNG rows (one lane each, map in registers).
template <int MAXF>
__global__ void __launch_bounds__(kSampleThreads) k_sample_fused(SampleHop h, LbLayout L, const StepScalars* sc,
                                                                 unsigned long long* state, int* ticket,
                                                                 std::uint32_t* slow, int* n_slow) {
  pdl_enter();
  __shared__ int s_tile;
  __shared__ std::uint32_t s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
  __syncthreads();
  const int tk = s_tile;
  if (tk >= L.base[L.nseg]) return;
  const int sg = seg_of(L.base, L.nseg, tk);
  const int t = tk - L.base[sg];
  const int bi = L.item[sg];
  const SampleBlock& b = h.b[bi];
  const int n = *b.n_rows;
  const int base = t * kSampleThreads;
  if (base >= n) return;
  unsigned long long t0 = 0;
  if (h.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  const int i = base + threadIdx.x;
  const bool live = i < n;
  const std::uint64_t fo = static_cast<std::uint64_t>(h.fanout);
  std::uint32_t d = 0, cnt = 0;
  std::uint64_t lo = 0, deg = 0;
  if (live) {
    d = b.dst_list[i];
    lo = b.csr_ptr[d];
    deg = b.csr_ptr[d + 1] - lo;
    cnt = static_cast<std::uint32_t>(deg < fo ? deg : fo);
  }
  std::uint32_t tot;
  const std::uint32_t incl = block_incl_scan<kSampleThreads>(cnt, &tot);
  if (threadIdx.x < 32) {
    const std::uint32_t p = lb_prefix(state + L.base[sg], t, tot);
    if (threadIdx.x == 0) s_prefix = p;
  }
  __syncthreads();
  const std::uint32_t o = s_prefix + incl - cnt;
  if (live) b.indptr[i + 1] = o + cnt;
  if (i == 0) b.indptr[0] = 0;
  unsigned long long t1 = 0;
  if (h.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));

  // Phase 1 — RNG rows (deg > fanout): one lane per row runs the exact
  // mt19937_64 + Lemire + partial Fisher-Yates and records the drawn CSR
  // positions in its output slots. Rows that overflow the streaming engine (or
  // the shared-memory map) go to the slow list and are skipped below.
  bool rng_ok = false;
  if (live && deg > fo) {
    if (h.fanout <= MAXF) {
      const std::uint64_t rel_key = (static_cast<std::uint64_t>(h.hop) << 32) | static_cast<std::uint64_t>(b.rel);
      rng_ok = draw_positions_fast<MAXF>(dmix_seed(sc->rng_seed, dmix_seed(rel_key, d)), deg, h.fanout,
                                         b.src_ids + o);
    }
    if (!rng_ok) {
      const int q = atomicAdd(n_slow, 1);
      slow[2 * q] = static_cast<std::uint32_t>(bi);
      slow[2 * q + 1] = static_cast<std::uint32_t>(i);
    }
  }
  __syncwarp();
  if (h.trace) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t2, smid;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
      asm volatile("mov.u32 %0, %%smid;" : "=r"(*reinterpret_cast<unsigned*>(&smid)));
      unsigned long long* r = h.trace + static_cast<std::size_t>(tk) * 8;
      r[0] = t0;
      r[1] = t1;
      r[2] = t2;
      r[4] = static_cast<unsigned long long>(bi);
      r[5] = smid & 0xffffffffull;
    }
  }

  // Phase 2 — warp-flattened gather: the warp's 32 consecutive rows own one
  // contiguous output range, so lane l takes edges q = l, l+32, ... (row found
  // by a shuffle binary search over the warp's inclusive counts). Copy-all rows
  // (sampling.cpp:22-25) read the CSR slice in order; RNG rows read the drawn
  // positions back. kUnroll edges per lane are resolved first and their loads
  // issued together, so a lane keeps several independent DRAM reads in flight.
  const int lane = threadIdx.x & 31;
  const unsigned take_mask = __ballot_sync(0xffffffffu, live && (deg <= fo || rng_ok));
  const unsigned rng_mask = __ballot_sync(0xffffffffu, rng_ok);
  std::uint32_t wincl = cnt;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const std::uint32_t y = __shfl_up_sync(0xffffffffu, wincl, off);
    if (lane >= off) wincl += y;
  }
  const std::uint32_t wtotal = __shfl_sync(0xffffffffu, wincl, 31);
  const std::uint32_t o0 = __shfl_sync(0xffffffffu, o, 0);
  const std::uint32_t row_base = static_cast<std::uint32_t>(base + (threadIdx.x & ~31));
  constexpr int kUnroll = HG_SAMPLE_UNROLL;
  for (std::uint32_t q0 = 0; q0 < wtotal; q0 += 32 * kUnroll) {  // warp-uniform trip count
    std::uint32_t at[kUnroll], pos[kUnroll];
    std::uint64_t rlo[kUnroll];
    int rr[kUnroll];
    bool ok[kUnroll], rng[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const std::uint32_t q = q0 + 32 * u + lane;
      int r = 0;  // smallest lane r with wincl[r] > q
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const std::uint32_t v = __shfl_sync(0xffffffffu, wincl, r + step - 1);
        if (v <= q) r += step;
      }
      r = min(r, 31);
      const std::uint32_t rincl = __shfl_sync(0xffffffffu, wincl, r);
      const std::uint32_t rcnt = __shfl_sync(0xffffffffu, cnt, r);
      rlo[u] = __shfl_sync(0xffffffffu, lo, r);
      rr[u] = r;
      at[u] = o0 + q;
      ok[u] = q < wtotal && ((take_mask >> r) & 1u);
      rng[u] = (rng_mask >> r) & 1u;
      pos[u] = q - (rincl - rcnt);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (ok[u] && rng[u]) pos[u] = b.src_ids[at[u]];
    std::uint32_t val[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (ok[u]) val[u] = __ldg(b.csr_src + rlo[u] + pos[u]);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const std::uint32_t q = q0 + 32 * u + lane;
      if (q < wtotal) b.erow[o0 + q] = row_base + static_cast<std::uint32_t>(rr[u]);
      if (ok[u]) b.src_ids[at[u]] = val[u];
    }
    // frontier mark fused here (the ids are in registers): one atomicOr per edge
    if (b.mark_bits) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (ok[u]) atomicOr(b.mark_bits + (val[u] >> 5), 1u << (val[u] & 31));
    }
  }
  if (h.trace) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t3;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t3));
      h.trace[static_cast<std::size_t>(tk) * 8 + 3] = t3;
    }
  }
}

__global__ void __launch_bounds__(128) k_sample_slow(SampleHop h, const StepScalars* sc,
                                                     const std::uint32_t* slow, const int* n_slow,
                                                     std::uint64_t* scratch) {
  pdl_enter();
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  std::uint64_t* x = scratch + static_cast<std::size_t>(tid) * (312 + h.fanout);
  std::uint32_t* mpos = reinterpret_cast<std::uint32_t*>(x + 312);
  std::uint32_t* mval = mpos + h.fanout;
  const int total = *n_slow;
  for (int q = tid; q < total; q += gridDim.x * blockDim.x) {
    const SampleBlock& b = h.b[slow[2 * q]];
    const std::uint32_t i = slow[2 * q + 1];
    const std::uint32_t d = b.dst_list[i];
    const std::uint64_t lo = b.csr_ptr[d];
    const std::uint64_t deg = b.csr_ptr[d + 1] - lo;
    const std::uint64_t rel_key = (static_cast<std::uint64_t>(h.hop) << 32) | static_cast<std::uint64_t>(b.rel);
    MtFull eng{x, 0};
    eng.seed(dmix_seed(sc->rng_seed, dmix_seed(rel_key, d)));
    std::uint32_t* out = b.src_ids + b.indptr[i];
    draw_row(eng, deg, h.fanout, b.csr_src + lo, out, mpos, mval);
    if (b.mark_bits)
      for (int e = 0; e < h.fanout; ++e) atomicOr(b.mark_bits + (out[e] >> 5), 1u << (out[e] & 31));
  }
}

// one row of sample_neighbors (sampling.cpp:17-39) on the full-state engine
__global__ void k_sample_row(const std::uint32_t* nbr, std::uint64_t deg, int fanout, std::uint64_t seed,
                             std::uint32_t* out, std::uint64_t* scratch) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  MtFull eng{scratch, 0};
  eng.seed(seed);
  std::uint32_t* mpos = reinterpret_cast<std::uint32_t*>(scratch + 312);
  draw_row(eng, deg, fanout, nbr, out, mpos, mpos + fanout);
}

}  // namespace

void sample_row(const std::uint32_t* d_nbr, std::uint64_t deg, int fanout, std::uint64_t seed, std::uint32_t* d_out,
                std::uint64_t* d_scratch, cudaStream_t st) {
  k_sample_row<<<1, 32, 0, st>>>(d_nbr, deg, fanout, seed, d_out, d_scratch);
  HG_CUDA(cudaGetLastError());
}

std::size_t sample_scratch_words(int fanout) {
  return static_cast<std::size_t>(kSlowThreads) * (312 + static_cast<std::size_t>(fanout));
}

void sample_hop(const SampleHop& h, const StepScalars* sc, std::uint32_t* slow, int* n_slow,
                std::uint64_t* scratch, LbScratch& lb, cudaStream_t st) {
  if (h.nblk == 0) return;
  LbLayout L{};
  L.nseg = h.nblk;
  // tickets go out in launch order, block by block. HG_SAMPLE_RNG_FIRST gives the
  // blocks with the most RNG rows (the 156-step seeding chains) the first tiles instead:
  // measured slower on C2 (sampling 63 -> 70 us/step), so off by default
  for (int i = 0; i < h.nblk; ++i) L.item[i] = i;
#if HG_SAMPLE_RNG_FIRST
  std::stable_sort(L.item, L.item + h.nblk,
                   [&](int a, int b) { return h.b[a].rng_frac * h.b[a].rows_cap > h.b[b].rng_frac * h.b[b].rows_cap; });
#endif
  int tiles = 0;
  for (int i = 0; i < h.nblk; ++i) {
    L.base[i] = tiles;
    tiles += static_cast<int>(ceil_div(std::max(1, h.b[L.item[i]].rows_cap), kSampleThreads));
  }
  L.base[h.nblk] = tiles;
  lb.reset(tiles, st);
  HG_CUDA(cudaMemsetAsync(n_slow, 0, sizeof(int), st));
  if (h.fanout <= 16)
    launch_pdl(k_sample_fused<16>, tiles, kSampleThreads, 0, st, h, L, sc, lb.state, lb.ticket, slow, n_slow);
  else
    launch_pdl(k_sample_fused<32>, tiles, kSampleThreads, 0, st, h, L, sc, lb.state, lb.ticket, slow, n_slow);
  launch_pdl(k_sample_slow, kSlowThreads / 128, 128, 0, st, h, sc, slow, n_slow, scratch);
}

// ---- frontier ---------------------------------------------------------------------------

namespace {

#ifndef HG_FRONT_WAVES
#define HG_FRONT_WAVES 4  // x-extent (CTAs per SM) of the per-block relabel / transpose grids
#endif
constexpr int kFrontThreads = 256;

__global__ void __launch_bounds__(kFrontThreads) k_mark_batch(const std::uint32_t* ids,
                                                              const StepScalars* sc,
                                                              std::uint32_t* bits) {
  pdl_enter();
  const int n = sc->batch_len;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const std::uint32_t id = ids[e];
    atomicOr(bits + (id >> 5), 1u << (id & 31));
  }
}

constexpr int kWordsPerThread = 1;  // short per-thread emission loops; more tiles in flight
constexpr int kWordsPerTile = kFrontThreads * kWordsPerThread;
static_assert(kWordsPerTile == kCompactWordsPerTile, "look-back scratch sizing");

// popcount of 1024 words per tile -> CTA scan -> look-back -> inclusive word
// prefix (the rank structure) and the sorted ids of the set bits
__global__ void __launch_bounds__(kFrontThreads) k_compact(FrontierArgs f, LbLayout L, unsigned long long* state,
                                                           int* ticket) {
  pdl_enter();
  __shared__ int s_tile;
  __shared__ std::uint32_t s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
  __syncthreads();
  const int tk = s_tile;
  if (tk >= L.base[L.nseg]) return;
  const int ti = seg_of(L.base, L.nseg, tk);
  const int t = tk - L.base[ti];
  const BitmapType& T = f.t[ti];
  const int w0 = t * kWordsPerTile + threadIdx.x * kWordsPerThread;
  std::uint32_t bits[kWordsPerThread];
  std::uint32_t local = 0;
#pragma unroll
  for (int j = 0; j < kWordsPerThread; ++j) {
    bits[j] = w0 + j < T.words ? T.bits[w0 + j] : 0u;
    local += __popc(bits[j]);
  }
  std::uint32_t tot;
  const std::uint32_t incl = block_incl_scan<kFrontThreads>(local, &tot);
  if (threadIdx.x < 32) {
    const std::uint32_t p = lb_prefix(state + L.base[ti], t, tot);
    if (threadIdx.x == 0) s_prefix = p;
  }
  __syncthreads();
  std::uint32_t at = s_prefix + incl - local;
#pragma unroll
  for (int j = 0; j < kWordsPerThread; ++j) {
    const int w = w0 + j;
    if (w >= T.words) break;
    std::uint32_t b = bits[j];
    const std::uint32_t start = at;
    while (b) {
      const int q = __ffs(b) - 1;
      b &= b - 1;
      T.list[at++] = static_cast<std::uint32_t>(w) * 32u + static_cast<std::uint32_t>(q);
    }
    T.wscan[w] = at;  // inclusive prefix through word w
    (void)start;
    if (w == T.words - 1) *T.count = static_cast<int>(at);
  }
}

__device__ __forceinline__ std::uint32_t bitmap_rank(const BitmapType& t, std::uint32_t id) {
  const std::uint32_t w = id >> 5;
  const std::uint32_t bits = t.bits[w];
  const std::uint32_t below = bits & ((1u << (id & 31)) - 1u);
  return t.wscan[w] - __popc(bits) + __popc(below);
}

__global__ void __launch_bounds__(kFrontThreads) k_relabel(RelabelArgs r, FrontierArgs f) {
  pdl_enter();
  const RelabelBlock& b = r.b[blockIdx.y];
  const std::uint32_t total = b.indptr[*b.n_rows];
  const BitmapType& t = f.t[b.slot];
  for (std::uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const std::uint32_t c = bitmap_rank(t, b.ids[e]);
    b.col[e] = c;
    if (b.csc_count) atomicAdd(b.csc_count + c, 1u);
  }
}

__global__ void __launch_bounds__(kFrontThreads) k_batch_mult(const std::uint32_t* ids, const StepScalars* sc,
                                                              BitmapType t, float* mult) {
  pdl_enter();
  const int n = sc->batch_len;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x)
    atomicAdd(mult + bitmap_rank(t, ids[e]), 1.0f);
}

}  // namespace

void frontier_mark_batch(const std::uint32_t* ids, const StepScalars* sc, int cap, const BitmapType& t,
                         cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(cap, kFrontThreads), num_sms()));
  launch_pdl(k_mark_batch, grid, kFrontThreads, 0, st, ids, sc, t.bits);
}

void frontier_compact(const FrontierArgs& f, LbScratch& lb, cudaStream_t st) {
  if (f.ntypes == 0) return;
  LbLayout L{};
  L.nseg = f.ntypes;
  int tiles = 0;
  for (int i = 0; i < f.ntypes; ++i) {
    L.base[i] = tiles;
    tiles += static_cast<int>(ceil_div(std::max(1, f.t[i].words), kWordsPerTile));
  }
  L.base[f.ntypes] = tiles;
  lb.reset(tiles, st);
  launch_pdl(k_compact, tiles, kFrontThreads, 0, st, f, L, lb.state, lb.ticket);
}

void frontier_relabel(const RelabelArgs& r, const FrontierArgs& f, cudaStream_t st) {
  if (r.nblk == 0) return;
  int cap = 1;
  for (int i = 0; i < r.nblk; ++i) cap = max(cap, r.b[i].cap);
  dim3 grid(static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(cap, kFrontThreads), HG_FRONT_WAVES * num_sms())), r.nblk);
  launch_pdl(k_relabel, grid, kFrontThreads, 0, st, r, f);
}

void batch_multiplicity(const std::uint32_t* ids, const StepScalars* sc, int cap, const BitmapType& t,
                        float* mult, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(cap, kFrontThreads), num_sms()));
  launch_pdl(k_batch_mult, grid, kFrontThreads, 0, st, ids, sc, t, mult);
}

// ---- replica gradient merge -------------------------------------------------------------------

namespace {

__global__ void k_rmark(ReplicaMerge m) {
  pdl_enter();
  const int r = blockIdx.y;
  const int n = *m.count[r];
  const std::uint32_t* ids = m.ids[r];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const std::uint32_t id = ids[i];
    atomicOr(m.u.bits + (id >> 5), 1u << (id & 31));
  }
}

// bits of word w whose id is in shard s of n (id % n == s)
__device__ __forceinline__ std::uint32_t shard_mask(std::uint32_t w, int s, int n) {
  if (n == 1) return 0xFFFFFFFFu;
  std::uint32_t mask = 0;
  const int o = static_cast<int>((static_cast<std::uint64_t>(w) * 32u) % static_cast<std::uint64_t>(n));
  int first = s - o;  // first bit j with (o + j) % n == s
  if (first < 0) first += n;
  for (int j = first; j < 32; j += n) mask |= 1u << j;
  return mask;
}

__global__ void k_rslot(ReplicaMerge m) {
  pdl_enter();
  const int r = blockIdx.y;
  const int n = *m.count[r];
  const std::uint32_t* ids = m.ids[r];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const std::uint32_t id = ids[i];
    if (static_cast<int>(id % static_cast<std::uint32_t>(m.nshard)) != m.shard) continue;
    const std::uint32_t w = id >> 5;
    const std::uint32_t bits = m.u.bits[w] & shard_mask(w, m.shard, m.nshard);
    const std::uint32_t rank = m.u.wscan[w] - __popc(bits) + __popc(bits & ((1u << (id & 31)) - 1u));
    m.slot[static_cast<std::size_t>(r) * m.u.cap + rank] = i;
  }
}

// union compaction restricted to this shard's ids (rank structure over the
// shard's bits) plus the size of the whole union
__global__ void __launch_bounds__(kFrontThreads) k_shard_compact(ReplicaMerge m, LbLayout L,
                                                                 unsigned long long* state, int* ticket) {
  pdl_enter();
  __shared__ int s_tile;
  __shared__ std::uint32_t s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
  __syncthreads();
  const int t = s_tile;
  if (t >= L.base[L.nseg]) return;
  const BitmapType& T = m.u;
  const int w = t * kFrontThreads + threadIdx.x;
  const std::uint32_t all = w < T.words ? T.bits[w] : 0u;
  const std::uint32_t mine = all & shard_mask(static_cast<std::uint32_t>(w), m.shard, m.nshard);
  const std::uint32_t local = __popc(mine);
  std::uint32_t tot;
  const std::uint32_t incl = block_incl_scan<kFrontThreads>(local, &tot);
  if (threadIdx.x < 32) {
    const std::uint32_t p = lb_prefix(state, t, tot);
    if (threadIdx.x == 0) s_prefix = p;
  }
  // whole-union size: warp-aggregated popcounts
  int c = __popc(all);
  for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(m.total, c);
  __syncthreads();
  if (w >= T.words) return;
  std::uint32_t at = s_prefix + incl - local;
  std::uint32_t b = mine;
  while (b) {
    const int q = __ffs(b) - 1;
    b &= b - 1;
    for (int r = 0; r < m.n_rep; ++r) m.slot[static_cast<std::size_t>(r) * T.cap + at] = -1;  // k_rslot fills
    T.list[at++] = static_cast<std::uint32_t>(w) * 32u + static_cast<std::uint32_t>(q);
  }
  T.wscan[w] = at;
  if (w == T.words - 1) *T.count = static_cast<int>(at);
}

}  // namespace

void replica_union(const ReplicaMerge& m, LbScratch& lb, cudaStream_t st) {
  HG_CUDA(cudaMemsetAsync(m.u.bits, 0, static_cast<std::size_t>(m.u.words) * 4, st));
  HG_CUDA(cudaMemsetAsync(m.total, 0, sizeof(int), st));
  const dim3 grid(static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(m.u.cap, 256), 2 * num_sms())), m.n_rep);
  launch_pdl(k_rmark, grid, 256, 0, st, m);
  LbLayout L{};
  L.nseg = 1;
  L.base[0] = 0;
  L.base[1] = static_cast<int>(ceil_div(std::max(1, m.u.words), kFrontThreads));
  lb.reset(L.base[1], st);
  launch_pdl(k_shard_compact, L.base[1], kFrontThreads, 0, st, m, L, lb.state, lb.ticket);
}
void replica_slots(const ReplicaMerge& m, cudaStream_t st) {
  // slots of this shard's union rows were reset to -1 by the compaction
  const dim3 grid(static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(m.u.cap, 256), 2 * num_sms())), m.n_rep);
  launch_pdl(k_rslot, grid, 256, 0, st, m);
}
// ---- cache / hotness counters -------------------------------------------------------------

namespace {

__global__ void k_cache_count(const std::uint32_t* ids, const int* n, const std::uint32_t* cached,
                              unsigned long long* hm) {
  pdl_enter();
  const int total = *n;
  unsigned long long hit = 0, miss = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const std::uint32_t id = ids[i];
    if ((cached[id >> 5] >> (id & 31)) & 1u)
      ++hit;
    else
      ++miss;
  }
  // warp-aggregated counters (integer: order independent)
  for (int o = 16; o > 0; o >>= 1) {
    hit += __shfl_down_sync(0xffffffffu, hit, o);
    miss += __shfl_down_sync(0xffffffffu, miss, o);
  }
  if ((threadIdx.x & 31) == 0 && (hit | miss)) {
    atomicAdd(hm, hit);
    atomicAdd(hm + 1, miss);
  }
}

// u64 visit counts, as the reference's HotnessTable (cache.hpp:38-41)
__global__ void k_hot_add(const std::uint32_t* ids, const std::uint32_t* indptr, const int* n_rows,
                          unsigned long long* counts) {
  pdl_enter();
  const std::uint32_t total = indptr[*n_rows];
  for (std::uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x)
    atomicAdd(counts + ids[e], 1ull);
}

__global__ void k_hot_add_list(const std::uint32_t* ids, const int* n, unsigned long long* counts) {
  pdl_enter();
  const int total = *n;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x)
    atomicAdd(counts + ids[e], 1ull);
}

}  // namespace

void cache_count(const std::uint32_t* ids, const int* n, int cap, const std::uint32_t* cached_bits,
                 unsigned long long* hm, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(cap, 256), 2 * num_sms()));
  launch_pdl(k_cache_count, std::max(grid, 1u), 256, 0, st, ids, n, cached_bits, hm);
}

namespace {
__global__ void k_union_mark(const std::uint32_t* ids, const int* n, std::uint8_t* map) {
  pdl_enter();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < *n; i += gridDim.x * blockDim.x) map[ids[i]] = 1;
}
__global__ void k_union_count(const std::uint8_t* map, std::uint64_t n, const std::uint32_t* cached,
                              unsigned long long* hm) {
  pdl_enter();
  unsigned long long hit = 0, miss = 0;
  for (std::uint64_t v = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; v < n;
       v += static_cast<std::uint64_t>(gridDim.x) * blockDim.x)
    if (map[v]) {
      if ((cached[v >> 5] >> (v & 31)) & 1u)
        ++hit;
      else
        ++miss;
    }
  for (int o = 16; o > 0; o >>= 1) {
    hit += __shfl_down_sync(0xffffffffu, hit, o);
    miss += __shfl_down_sync(0xffffffffu, miss, o);
  }
  if ((threadIdx.x & 31) == 0 && (hit | miss)) {
    atomicAdd(hm, hit);
    atomicAdd(hm + 1, miss);
  }
}
}  // namespace

void union_mark(const std::uint32_t* ids, const int* n, int cap, std::uint8_t* map, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(std::max(1, cap), 256), 2 * num_sms()));
  launch_pdl(k_union_mark, std::max(grid, 1u), 256, 0, st, ids, n, map);
}

void union_count(const std::uint8_t* map, std::uint64_t n, const std::uint32_t* cached_bits, unsigned long long* hm,
                 cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(std::max<std::uint64_t>(1, n), 256),
                                                                      4 * num_sms()));
  launch_pdl(k_union_count, std::max(grid, 1u), 256, 0, st, map, n, cached_bits, hm);
}

void hotness_add(const std::uint32_t* ids, const std::uint32_t* indptr, const int* n_rows, int cap,
                 unsigned long long* counts, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(cap, 256), 4 * num_sms()));
  launch_pdl(k_hot_add, std::max(grid, 1u), 256, 0, st, ids, indptr, n_rows, counts);
}

void hotness_add_list(const std::uint32_t* ids, const int* n, int cap, unsigned long long* counts, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(cap, 256), 2 * num_sms()));
  launch_pdl(k_hot_add_list, std::max(grid, 1u), 256, 0, st, ids, n, counts);
}

// ---- replica barrier ----------------------------------------------------------------------------

namespace {
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__global__ void k_replica_barrier(ReplicaBarrier b) {
  pdl_enter();  // every read of the peers' arenas by the merge kernels has completed
  if (threadIdx.x != 0) return;
  const unsigned e = *b.epoch + 1u;
  *b.epoch = e;
  for (int r = 0; r < b.n; ++r) st_release_sys(b.peer_flags[r] + b.pos, e);
  for (int r = 0; r < b.n; ++r)
    while (static_cast<int>(ld_acquire_sys(b.my_flags + r) - e) < 0) __nanosleep(100);
}
}  // namespace

void replica_barrier(const ReplicaBarrier& b, cudaStream_t st) {
  if (b.n <= 1) return;
  launch_pdl(k_replica_barrier, 1, 32, 0, st, b);
}

}  // namespace hetgpu
