// Integer/byte work of the hot path: per-relation fanout sampling with the
// reference's exact RNG, segmented scans, and the bitmap frontier that
// replaces the reference's per-hop sort+unique (sampling.cpp:82-89) and its
// per-edge binary searches (hgnn.cpp:166-171). All HBM-bound; grids are sized
// in multiples of the SM count or from capacities and read live counts.
#include "kernels.cuh"

namespace hetgpu {

namespace {

constexpr int kScanThreads = 512;
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

__global__ void __launch_bounds__(kScanThreads) scan_tile_sums(ScanArgs a, std::uint32_t* partials,
                                                               int tiles_stride) {
  const ScanSeg& s = a.s[blockIdx.y];
  const int n = *s.n;
  const int base = blockIdx.x * kScanTile;
  if (base >= n) return;
  std::uint32_t sum = 0;
  for (int i = threadIdx.x; i < kScanTile; i += kScanThreads) {
    const int idx = base + i;
    if (idx < n) sum += s.data[idx];
  }
  std::uint32_t tot;
  block_incl_scan<kScanThreads>(sum, &tot);
  if (threadIdx.x == 0) partials[blockIdx.y * tiles_stride + blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads) scan_partials(ScanArgs a, std::uint32_t* partials,
                                                              int tiles_stride) {
  const ScanSeg& s = a.s[blockIdx.x];
  const int n = *s.n;
  const int tiles = (n + kScanTile - 1) / kScanTile;
  std::uint32_t carry = 0;
  std::uint32_t* p = partials + blockIdx.x * tiles_stride;
  for (int b = 0; b < tiles; b += kScanThreads) {
    const int i = b + threadIdx.x;
    const std::uint32_t v = i < tiles ? p[i] : 0u;
    std::uint32_t tot;
    const std::uint32_t incl = block_incl_scan<kScanThreads>(v, &tot);
    if (i < tiles) p[i] = carry + incl - v;  // exclusive tile prefix
    carry += tot;
  }
}

__global__ void __launch_bounds__(kScanThreads) scan_apply(ScanArgs a, const std::uint32_t* partials,
                                                           int tiles_stride) {
  const ScanSeg& s = a.s[blockIdx.y];
  const int n = *s.n;
  const int base = blockIdx.x * kScanTile;
  if (base >= n) return;
  // each thread owns kScanPer consecutive elements
  const int first = base + threadIdx.x * kScanPer;
  std::uint32_t v[kScanPer];
  std::uint32_t local = 0;
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) {
    const int idx = first + j;
    v[j] = idx < n ? s.data[idx] : 0u;
    local += v[j];
  }
  std::uint32_t incl = block_incl_scan<kScanThreads>(local, nullptr);
  std::uint32_t run = partials[blockIdx.y * tiles_stride + blockIdx.x] + incl - local;
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) {
    const int idx = first + j;
    run += v[j];
    if (idx < n) s.data[idx] = run;
  }
}

}  // namespace

void scan_inclusive(const ScanArgs& a, std::uint32_t* partials, cudaStream_t st) {
  if (a.nseg == 0) return;
  int max_cap = 1;
  for (int i = 0; i < a.nseg; ++i) max_cap = max(max_cap, a.s[i].cap);
  const int tiles = static_cast<int>(ceil_div(max_cap, kScanTile));
  dim3 grid(tiles, a.nseg);
  scan_tile_sums<<<grid, kScanThreads, 0, st>>>(a, partials, tiles);
  scan_partials<<<a.nseg, kScanThreads, 0, st>>>(a, partials, tiles);
  scan_apply<<<grid, kScanThreads, 0, st>>>(a, partials, tiles);
}

// ---- sampling -------------------------------------------------------------------------

namespace {

constexpr int kSampleThreads = 256;
constexpr int kMapCap = 64;       // displaced-position map held in local memory
constexpr int kSlowThreads = 4096;  // concurrent slow-path rows (global scratch)

__global__ void __launch_bounds__(kSampleThreads) k_sample_count(SampleHop h) {
  const SampleBlock& b = h.b[blockIdx.y];
  const int n = *b.n_rows;
  const std::uint64_t fo = static_cast<std::uint64_t>(h.fanout);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const std::uint32_t d = b.dst_list[i];
    const std::uint64_t deg = b.csr_ptr[d + 1] - b.csr_ptr[d];
    b.indptr[i + 1] = static_cast<std::uint32_t>(deg < fo ? deg : fo);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) b.indptr[0] = 0;
}

// Partial Fisher-Yates over [0, deg) with a sparse map of displaced positions
// (sampling.cpp:29-37 keeps a dense O(deg) index array). Position p holds p
// unless overridden; position i is final once drawn, so only the j side needs
// remembering. Returns false if a streaming engine ran dry (caller replays).
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

__global__ void __launch_bounds__(kSampleThreads) k_sample_draw(SampleHop h, const StepScalars* sc,
                                                                std::uint32_t* slow, int* n_slow) {
  const SampleBlock& b = h.b[blockIdx.y];
  const int n = *b.n_rows;
  const std::uint64_t fo = static_cast<std::uint64_t>(h.fanout);
  const std::uint64_t rng_seed = sc->rng_seed;
  const std::uint64_t rel_key = (static_cast<std::uint64_t>(h.hop) << 32) | static_cast<std::uint64_t>(b.rel);
  const int lane = threadIdx.x & 31;
  const int stride = gridDim.x * blockDim.x;
  for (int base = blockIdx.x * blockDim.x; base < n; base += stride) {
    const int i = base + threadIdx.x;
    const bool live = i < n;
    std::uint32_t d = 0, o = 0, cnt = 0;
    std::uint64_t lo = 0, deg = 0;
    if (live) {
      d = b.dst_list[i];
      lo = b.csr_ptr[d];
      deg = b.csr_ptr[d + 1] - lo;
      o = b.indptr[i];
      cnt = b.indptr[i + 1] - o;
    }
    // warp-cooperative, coalesced writes: the row index of every edge, and the
    // copy-all rows (deg <= fanout) in CSR order (sampling.cpp:22-25)
    unsigned live_mask = __ballot_sync(0xffffffffu, live);
    const unsigned copy_mask = __ballot_sync(0xffffffffu, live && deg <= fo);
    while (live_mask) {
      const int sl = __ffs(live_mask) - 1;
      live_mask &= live_mask - 1;
      const std::uint64_t rlo = __shfl_sync(0xffffffffu, lo, sl);
      const std::uint32_t ro = __shfl_sync(0xffffffffu, o, sl);
      const std::uint32_t rc = __shfl_sync(0xffffffffu, cnt, sl);
      const std::uint32_t row = static_cast<std::uint32_t>(base + (threadIdx.x & ~31) + sl);
      const bool copy = (copy_mask >> sl) & 1u;
      for (std::uint32_t e = lane; e < rc; e += 32) {
        b.erow[ro + e] = row;
        if (copy) b.src_ids[ro + e] = b.csr_src[rlo + e];
      }
    }
    if (live && deg > fo) {
      bool done = false;
      if (h.fanout <= kMapCap) {
        std::uint32_t mpos[kMapCap], mval[kMapCap];
        MtStream eng;
        eng.seed(dmix_seed(rng_seed, dmix_seed(rel_key, d)));
        done = draw_row(eng, deg, h.fanout, b.csr_src + lo, b.src_ids + o, mpos, mval);
      }
      if (!done) {
        // more than 156 engine outputs (Lemire rejections) or a fanout above
        // the local map: replay on the full-state engine in a second pass
        const int q = atomicAdd(n_slow, 1);
        slow[2 * q] = blockIdx.y;
        slow[2 * q + 1] = static_cast<std::uint32_t>(i);
      }
    }
  }
}

__global__ void __launch_bounds__(128) k_sample_slow(SampleHop h, const StepScalars* sc,
                                                     const std::uint32_t* slow, const int* n_slow,
                                                     std::uint64_t* scratch) {
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
    draw_row(eng, deg, h.fanout, b.csr_src + lo, b.src_ids + b.indptr[i], mpos, mval);
  }
}

}  // namespace

void sample_count(const SampleHop& h, cudaStream_t st) {
  if (h.nblk == 0) return;
  int cap = 1;
  for (int i = 0; i < h.nblk; ++i) cap = max(cap, h.b[i].rows_cap);
  dim3 grid(static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(cap, kSampleThreads), 4 * kNumSMs)), h.nblk);
  k_sample_count<<<grid, kSampleThreads, 0, st>>>(h);
}

std::size_t sample_scratch_words(int fanout) {
  return static_cast<std::size_t>(kSlowThreads) * (312 + static_cast<std::size_t>(fanout));
}

void sample_draw(const SampleHop& h, const StepScalars* sc, std::uint32_t* slow, int* n_slow,
                 std::uint64_t* scratch, cudaStream_t st) {
  if (h.nblk == 0) return;
  int cap = 1;
  for (int i = 0; i < h.nblk; ++i) cap = max(cap, h.b[i].rows_cap);
  HG_CUDA(cudaMemsetAsync(n_slow, 0, sizeof(int), st));
  dim3 grid(static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(cap, kSampleThreads), 4 * kNumSMs)), h.nblk);
  k_sample_draw<<<grid, kSampleThreads, 0, st>>>(h, sc, slow, n_slow);
  k_sample_slow<<<kSlowThreads / 128, 128, 0, st>>>(h, sc, slow, n_slow, scratch);
}

// ---- frontier ---------------------------------------------------------------------------

namespace {

constexpr int kFrontThreads = 256;

__global__ void __launch_bounds__(kFrontThreads) k_mark(MarkArgs m, FrontierArgs f) {
  const MarkSource& s = m.s[blockIdx.y];
  const std::uint32_t total = s.indptr[*s.n_rows];
  std::uint32_t* bits = f.t[s.slot].bits;
  for (std::uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const std::uint32_t id = s.ids[e];
    atomicOr(bits + (id >> 5), 1u << (id & 31));
  }
}

__global__ void __launch_bounds__(kFrontThreads) k_mark_batch(const std::uint32_t* ids,
                                                              const StepScalars* sc,
                                                              std::uint32_t* bits) {
  const int n = sc->batch_len;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const std::uint32_t id = ids[e];
    atomicOr(bits + (id >> 5), 1u << (id & 31));
  }
}

__global__ void __launch_bounds__(kFrontThreads) k_popc(FrontierArgs f) {
  const BitmapType& t = f.t[blockIdx.y];
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < t.words; w += gridDim.x * blockDim.x)
    t.wscan[w] = __popc(t.bits[w]);
}

__global__ void __launch_bounds__(kFrontThreads) k_emit(FrontierArgs f) {
  const BitmapType& t = f.t[blockIdx.y];
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < t.words; w += gridDim.x * blockDim.x) {
    std::uint32_t bits = t.bits[w];
    const std::uint32_t incl = t.wscan[w];
    std::uint32_t at = incl - __popc(bits);
    while (bits) {
      const int j = __ffs(bits) - 1;
      bits &= bits - 1;
      t.list[at++] = static_cast<std::uint32_t>(w) * 32u + static_cast<std::uint32_t>(j);
    }
    if (w == t.words - 1) *t.count = static_cast<int>(incl);
  }
}

__device__ __forceinline__ std::uint32_t bitmap_rank(const BitmapType& t, std::uint32_t id) {
  const std::uint32_t w = id >> 5;
  const std::uint32_t bits = t.bits[w];
  const std::uint32_t below = bits & ((1u << (id & 31)) - 1u);
  return t.wscan[w] - __popc(bits) + __popc(below);
}

__global__ void __launch_bounds__(kFrontThreads) k_relabel(RelabelArgs r, FrontierArgs f) {
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
  const int n = sc->batch_len;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x)
    atomicAdd(mult + bitmap_rank(t, ids[e]), 1.0f);
}

}  // namespace

void frontier_mark(const MarkArgs& m, const FrontierArgs& f, cudaStream_t st) {
  if (m.nsrc == 0) return;
  int cap = 1;
  for (int i = 0; i < m.nsrc; ++i) cap = max(cap, m.s[i].cap);
  dim3 grid(static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(cap, kFrontThreads), 4 * kNumSMs)), m.nsrc);
  k_mark<<<grid, kFrontThreads, 0, st>>>(m, f);
}

void frontier_mark_batch(const std::uint32_t* ids, const StepScalars* sc, int cap, const BitmapType& t,
                         cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(cap, kFrontThreads), kNumSMs));
  k_mark_batch<<<grid, kFrontThreads, 0, st>>>(ids, sc, t.bits);
}

void frontier_compact(const FrontierArgs& f, const int* words_dev, std::uint32_t* partials, cudaStream_t st) {
  if (f.ntypes == 0) return;
  int maxw = 1;
  for (int i = 0; i < f.ntypes; ++i) maxw = max(maxw, f.t[i].words);
  dim3 grid(static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(maxw, kFrontThreads), 8 * kNumSMs)), f.ntypes);
  k_popc<<<grid, kFrontThreads, 0, st>>>(f);
  ScanArgs sa{};
  sa.nseg = f.ntypes;
  for (int i = 0; i < f.ntypes; ++i) sa.s[i] = {f.t[i].wscan, words_dev + i, f.t[i].words};
  scan_inclusive(sa, partials, st);
  k_emit<<<grid, kFrontThreads, 0, st>>>(f);
}

void frontier_relabel(const RelabelArgs& r, const FrontierArgs& f, cudaStream_t st) {
  if (r.nblk == 0) return;
  int cap = 1;
  for (int i = 0; i < r.nblk; ++i) cap = max(cap, r.b[i].cap);
  dim3 grid(static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(cap, kFrontThreads), 4 * kNumSMs)), r.nblk);
  k_relabel<<<grid, kFrontThreads, 0, st>>>(r, f);
}

void batch_multiplicity(const std::uint32_t* ids, const StepScalars* sc, int cap, const BitmapType& t,
                        float* mult, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(cap, kFrontThreads), kNumSMs));
  k_batch_mult<<<grid, kFrontThreads, 0, st>>>(ids, sc, t, mult);
}

// ---- cache / hotness counters -------------------------------------------------------------

namespace {

__global__ void k_cache_count(const std::uint32_t* ids, const int* n, const std::uint32_t* cached,
                              unsigned long long* hm) {
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

__global__ void k_hot_add(const std::uint32_t* ids, const std::uint32_t* indptr, const int* n_rows,
                          std::uint32_t* counts) {
  const std::uint32_t total = indptr[*n_rows];
  for (std::uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x)
    atomicAdd(counts + ids[e], 1u);
}

__global__ void k_hot_add_list(const std::uint32_t* ids, const int* n, std::uint32_t* counts) {
  const int total = *n;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x)
    atomicAdd(counts + ids[e], 1u);
}

}  // namespace

void cache_count(const std::uint32_t* ids, const int* n, int cap, const std::uint32_t* cached_bits,
                 unsigned long long* hm, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(cap, 256), 2 * kNumSMs));
  k_cache_count<<<std::max(grid, 1u), 256, 0, st>>>(ids, n, cached_bits, hm);
}

void hotness_add(const std::uint32_t* ids, const std::uint32_t* indptr, const int* n_rows, int cap,
                 std::uint32_t* counts, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(cap, 256), 4 * kNumSMs));
  k_hot_add<<<std::max(grid, 1u), 256, 0, st>>>(ids, indptr, n_rows, counts);
}

void hotness_add_list(const std::uint32_t* ids, const int* n, int cap, std::uint32_t* counts, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(cap, 256), 2 * kNumSMs));
  k_hot_add_list<<<std::max(grid, 1u), 256, 0, st>>>(ids, n, counts);
}

}  // namespace hetgpu
