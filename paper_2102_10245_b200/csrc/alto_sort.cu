// alto_sort.cu — K2 hand-written stable LSD radix sort on linearized keys
// (+ payload), K3 duplicate detection.
//
// Replaces np.lexsort over the index words with last word primary and the
// co-permutation of values (format.py:79-82, :94-97).  Because keys occupy
// only bits [0, total_bits), exactly ceil(total_bits/9) 9-bit digit passes
// are run by the one-sweep path (ceil(total_bits/8) 8-bit passes by the
// three-kernel fallback for m >= 2^30).
//
// One pass = three stream-ordered kernels:
//   1. radix_hist   : per-tile digit histogram -> counts[digit * ntiles + tile]
//   2. exclusive scan of counts (digit-major, so the scan yields the global
//      destination of (digit, tile) directly)
//   3. radix_scatter: stable in-tile ranking.  Each warp owns a contiguous
//      256-key slice of the 2048-key tile, visited in index order
//      (round j, lane l); __match_any_sync groups equal digits, the group's
//      lower lanes give the rank, per-warp running digit counters carry the
//      rank across rounds, and a per-digit exclusive scan over warps orders
//      the warps.  The tile is first scattered, stably, into shared memory
//      in digit order; it is then written out with consecutive threads on
//      consecutive tile positions, so each digit's run of the tile lands in
//      consecutive global addresses (scan[digit, tile] + position in run):
//      coalesced stores instead of one scattered store per key.
#include <climits>

#include "alto_common.cuh"

namespace alto {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;   // 2048 keys
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kWarpSlice = kSortTile / kSortWarps;     // 256 keys per warp
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanChunk = kScanThreads * kScanItems;  // 4096 counters

template <int W>
__device__ __forceinline__ unsigned digit_of(const Key<W>& k, int shift) {
  // select the word without dynamic indexing (which would place the key in local memory)
  uint64_t w = k.w[0];
  if constexpr (W == 2) w = shift >= 64 ? k.w[1] : k.w[0];
  return static_cast<unsigned>(w >> (shift & 63)) & 0xffu;
}

template <int W>
__global__ void __launch_bounds__(kSortThreads) radix_hist(const uint64_t* __restrict__ keys, long long m,
                                                           int shift, unsigned* __restrict__ counts,
                                                           long long ntiles) {
  __shared__ unsigned s_hist[kSortWarps][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kSortWarps * 256; i += blockDim.x) (&s_hist[0][0])[i] = 0;
  __syncthreads();
  const long long tile = blockIdx.x;
  const long long base = tile * kSortTile + static_cast<long long>(warp) * kWarpSlice;
#pragma unroll 4
  for (int j = 0; j < kSortItems; ++j) {
    const long long i = base + j * 32 + lane;
    if (i < m) {
      const Key<W> k = load_key<W>(keys, i);
      atomicAdd(&s_hist[warp][digit_of<W>(k, shift)], 1u);
    }
  }
  __syncthreads();
  const int d = threadIdx.x;  // 256 threads = 256 digits
  unsigned sum = 0;
#pragma unroll
  for (int w = 0; w < kSortWarps; ++w) sum += s_hist[w][d];
  counts[static_cast<long long>(d) * ntiles + tile] = sum;
}

// --- exclusive scan of unsigned counters (3 phases) -----------------------

__device__ __forceinline__ unsigned block_exclusive_scan(unsigned v, unsigned* s_tmp, unsigned* total) {
  // s_tmp: >= 32 entries
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_tmp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    unsigned w = lane < nw ? s_tmp[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) s_tmp[lane] = w;
  }
  __syncthreads();
  const unsigned warp_prefix = warp > 0 ? s_tmp[warp - 1] : 0u;
  if (total) *total = s_tmp[(blockDim.x >> 5) - 1];
  __syncthreads();
  return warp_prefix + x - v;
}

__global__ void __launch_bounds__(kScanThreads) scan_reduce(const unsigned* __restrict__ in, long long n,
                                                            unsigned* __restrict__ partial) {
  __shared__ unsigned s_tmp[32];
  const long long base = static_cast<long long>(blockIdx.x) * kScanChunk;
  unsigned sum = 0;
  for (int j = 0; j < kScanItems; ++j) {
    const long long i = base + static_cast<long long>(j) * kScanThreads + threadIdx.x;
    if (i < n) sum += in[i];
  }
  unsigned total;
  block_exclusive_scan(sum, s_tmp, &total);
  if (threadIdx.x == 0) partial[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) scan_partials(unsigned* __restrict__ partial, long long n) {
  __shared__ unsigned s_tmp[32];
  unsigned carry = 0;
  for (long long base = 0; base < n; base += blockDim.x) {
    const long long i = base + threadIdx.x;
    const unsigned v = i < n ? partial[i] : 0u;
    unsigned total;
    const unsigned ex = block_exclusive_scan(v, s_tmp, &total);
    if (i < n) partial[i] = carry + ex;
    carry += total;
  }
}

__global__ void __launch_bounds__(kScanThreads) scan_down(unsigned* __restrict__ data, long long n,
                                                          const unsigned* __restrict__ partial) {
  __shared__ unsigned s_tmp[32];
  const long long base = static_cast<long long>(blockIdx.x) * kScanChunk;
  // thread t owns kScanItems consecutive counters (blocked arrangement)
  const long long first = base + static_cast<long long>(threadIdx.x) * kScanItems;
  unsigned v[kScanItems];
  unsigned sum = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    v[j] = (first + j < n) ? data[first + j] : 0u;
    sum += v[j];
  }
  unsigned run = block_exclusive_scan(sum, s_tmp, nullptr) + partial[blockIdx.x];
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    if (first + j < n) data[first + j] = run;
    run += v[j];
  }
}

// --- stable scatter ------------------------------------------------------------

template <int W, int P>
__global__ void __launch_bounds__(kSortThreads) radix_scatter(const uint64_t* __restrict__ keys_in,
                                                              const void* __restrict__ pay_in,
                                                              uint64_t* __restrict__ keys_out,
                                                              void* __restrict__ pay_out, long long m, int shift,
                                                              const unsigned* __restrict__ offsets,
                                                              long long ntiles) {
  __shared__ unsigned s_warp[kSortWarps][256];
  __shared__ unsigned s_base[256];
  __shared__ unsigned s_dstart[256];
  __shared__ unsigned s_scan[32];
  extern __shared__ __align__(16) unsigned char s_dyn[];  // digit-sorted tile: keys, then payload
  uint64_t* s_keys = reinterpret_cast<uint64_t*>(s_dyn);
  unsigned* s_pay32 = reinterpret_cast<unsigned*>(s_dyn + static_cast<size_t>(kSortTile) * W * 8);
  uint64_t* s_pay64 = reinterpret_cast<uint64_t*>(s_dyn + static_cast<size_t>(kSortTile) * W * 8);
  (void)s_pay32;
  (void)s_pay64;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kSortWarps * 256; i += blockDim.x) (&s_warp[0][0])[i] = 0;
  const long long tile = blockIdx.x;
  s_base[threadIdx.x] = offsets[static_cast<long long>(threadIdx.x) * ntiles + tile];
  __syncthreads();

  const long long base = tile * kSortTile + static_cast<long long>(warp) * kWarpSlice;
  const unsigned lt_mask = (1u << lane) - 1u;
  // Ranking pass: only the key word holding the digit is read; each item
  // keeps (rank << 8 | digit) in one register (ranks < 2048), so the kernel
  // stays small enough for several CTAs per SM; keys and payload are re-read
  // (L2 hits) in the placement pass below.
  const int dw = shift >> 6;
  unsigned rd[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const long long i = base + j * 32 + lane;
    const bool valid = i < m;
    unsigned d = 0x100u + lane;  // invalid lanes: singleton groups
    if (valid) d = static_cast<unsigned>(__ldg(keys_in + i * W + dw) >> (shift & 63)) & 0xffu;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned r = __popc(peers & lt_mask);
    unsigned prior = 0;
    if (valid) prior = s_warp[warp][d];
    __syncwarp();
    if (valid && r == 0) s_warp[warp][d] = prior + __popc(peers);
    __syncwarp();
    rd[j] = ((prior + r) << 8) | (d & 0xffu);
  }
  __syncthreads();
  {
    // per-digit exclusive scan over warps (stable order of warps), and the
    // tile-local exclusive scan over digits (start of digit d's run in the tile)
    const int d = threadIdx.x;
    unsigned run = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      const unsigned c = s_warp[w][d];
      s_warp[w][d] = run;
      run += c;
    }
    unsigned total;
    s_dstart[d] = block_exclusive_scan(run, s_scan, &total);
  }
  __syncthreads();
  // 1) stable local scatter into shared memory (digit-sorted tile)
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const long long i = base + j * 32 + lane;
    if (i < m) {
      const unsigned d = rd[j] & 0xffu;
      const unsigned lp = s_dstart[d] + s_warp[warp][d] + (rd[j] >> 8);
      const Key<W> k = load_key<W>(keys_in, i);
      if constexpr (W == 1) {
        s_keys[lp] = k.w[0];
      } else {
        s_keys[2 * lp] = k.w[0];
        s_keys[2 * lp + 1] = k.w[1];
      }
      if constexpr (P == 4) s_pay32[lp] = static_cast<const unsigned*>(pay_in)[i];
      if constexpr (P == 8) s_pay64[lp] = static_cast<const uint64_t*>(pay_in)[i];
    }
  }
  __syncthreads();
  // 2) coalesced write-out: consecutive tile positions of one digit go to
  //    consecutive global positions
  const int cnt = static_cast<int>(min(static_cast<long long>(kSortTile), m - tile * kSortTile));
  for (int lp = threadIdx.x; lp < cnt; lp += kSortThreads) {
    Key<W> key;
    if constexpr (W == 1) {
      key.w[0] = s_keys[lp];
    } else {
      key.w[0] = s_keys[2 * lp];
      key.w[1] = s_keys[2 * lp + 1];
    }
    const unsigned d = digit_of<W>(key, shift);
    const long long dst = static_cast<long long>(s_base[d]) + (lp - s_dstart[d]);
    store_key<W>(keys_out, dst, key);
    if constexpr (P == 4) static_cast<unsigned*>(pay_out)[dst] = s_pay32[lp];
    if constexpr (P == 8) static_cast<uint64_t*>(pay_out)[dst] = s_pay64[lp];
  }
}

// --- one-sweep passes (decoupled look-back) ------------------------------------
// Used when m < 2^30: one histogram kernel for every pass up front
// (onesweep_hist + onesweep_scan: global digit bases), then per pass a single
// kernel that reads each key/payload once and writes it once.  Digits are 9
// bits wide (512 bins = one per thread of the 512-thread CTA: cfg5's 71 key
// bits take 8 passes instead of 9, and an even pass count ends in the caller's
// buffer).  A CTA claims the next 4096-key tile in order (atomic counter),
// ranks it like radix_scatter, publishes its per-digit counts at once (flag
// AGGREGATE), stages the tile digit-sorted in shared memory, then looks back
// over earlier tiles until it finds an inclusive prefix (flag PREFIX) —
// their aggregates were published before their own staging, so the walk
// rarely spins — publishes its own prefix and writes the tile out in
// coalesced runs.  Tiles are claimed in order, so every tile a CTA waits on
// belongs to a CTA that is already running.
constexpr int kMaxPasses = 16;
constexpr int kOnesweepThreads = 512;  // one-sweep CTA: 4096-key tiles
constexpr int kOneBits = 9;            // one-sweep digit width: 512 bins, one per thread of the CTA
constexpr int kOneBins = 1 << kOneBits;
static_assert(kOneBins == kOnesweepThreads, "thread d of a one-sweep CTA owns digit d");
constexpr unsigned kFlagAgg = 1u << 30, kFlagPrefix = 2u << 30, kValMask = (1u << 30) - 1u;

// kOneBits-wide digit at bit `shift` (may straddle the two key words)
template <int W>
__device__ __forceinline__ unsigned digit9(const Key<W>& k, int shift) {
  if constexpr (W == 1) {
    return static_cast<unsigned>(k.w[0] >> shift) & (kOneBins - 1);
  } else {
    const int sh = shift & 63;
    uint64_t v = (shift >= 64 ? k.w[1] : k.w[0]) >> sh;
    if (shift < 64 && sh > 64 - kOneBits) v |= k.w[1] << (64 - sh);
    return static_cast<unsigned>(v) & (kOneBins - 1);
  }
}

template <int W>
__global__ void __launch_bounds__(kSortThreads) onesweep_hist(const uint64_t* __restrict__ keys, long long m,
                                                              int passes, unsigned* __restrict__ ghist) {
  __shared__ unsigned s_h[kMaxPasses * kOneBins];
  for (int i = threadIdx.x; i < passes * kOneBins; i += blockDim.x) s_h[i] = 0;
  __syncthreads();
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m; i += stride) {
    const Key<W> k = load_key<W>(keys, i);
    for (int p = 0; p < passes; ++p) atomicAdd(&s_h[p * kOneBins + digit9<W>(k, kOneBits * p)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kOneBins; i += blockDim.x)
    if (s_h[i]) atomicAdd(ghist + i, s_h[i]);
}

__global__ void __launch_bounds__(kOneBins) onesweep_scan(unsigned* __restrict__ ghist) {
  __shared__ unsigned s_tmp[32];
  unsigned* h = ghist + static_cast<long long>(blockIdx.x) * kOneBins;
  const unsigned v = h[threadIdx.x];
  unsigned total;
  const unsigned ex = block_exclusive_scan(v, s_tmp, &total);
  h[threadIdx.x] = ex;
}

__device__ __forceinline__ unsigned ld_status(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_status(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// OT = kOneBins threads per CTA, tile = OT * kSortItems keys; thread d owns digit d.
template <int W, int P, int OT>
__global__ void __launch_bounds__(OT, 1024 / OT) onesweep_pass(const uint64_t* __restrict__ keys_in,
                                                              const void* __restrict__ pay_in,
                                                              uint64_t* __restrict__ keys_out,
                                                              void* __restrict__ pay_out, long long m, int shift,
                                                              const unsigned* __restrict__ gbase,
                                                              unsigned* __restrict__ status,
                                                              unsigned* __restrict__ tile_ctr) {
  static_assert(OT == kOneBins, "one digit per thread");
  constexpr int NW = OT / 32, TILE = OT * kSortItems, SLICE = TILE / NW;
  static_assert(SLICE <= 65535 && TILE <= 65535, "16-bit per-warp digit counters");
  __shared__ unsigned short s_warp[NW][kOneBins];  // per-warp digit counts, then exclusive scan over warps
  __shared__ unsigned s_base[kOneBins];
  __shared__ unsigned short s_dstart[kOneBins];
  __shared__ unsigned s_scan[32];
  __shared__ unsigned s_tile;
  extern __shared__ __align__(16) unsigned char s_dyn[];  // digit-sorted tile: keys, then payload
  uint64_t* s_keys = reinterpret_cast<uint64_t*>(s_dyn);
  unsigned* s_pay32 = reinterpret_cast<unsigned*>(s_dyn + static_cast<size_t>(TILE) * W * 8);
  uint64_t* s_pay64 = reinterpret_cast<uint64_t*>(s_dyn + static_cast<size_t>(TILE) * W * 8);
  (void)s_pay32;
  (void)s_pay64;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  for (int i = threadIdx.x; i < NW * kOneBins / 2; i += blockDim.x) reinterpret_cast<unsigned*>(&s_warp[0][0])[i] = 0;
  __syncthreads();
  const long long tile = s_tile;
  const long long base = tile * TILE + static_cast<long long>(warp) * SLICE;
  const unsigned lt_mask = (1u << lane) - 1u;
  uint64_t k0[kSortItems], k1[kSortItems];  // key words (k1 unused for W = 1)
  uint64_t pv[kSortItems];
  unsigned rd[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const long long i = base + j * 32 + lane;
    const bool valid = i < m;
    unsigned d = kOneBins + lane;  // invalid lanes: singleton groups
    k0[j] = 0;
    k1[j] = 0;
    pv[j] = 0;
    if (valid) {
      const Key<W> kk = load_key<W>(keys_in, i);
      k0[j] = kk.w[0];
      if constexpr (W == 2) k1[j] = kk.w[1];
      if constexpr (P == 4) pv[j] = static_cast<const unsigned*>(pay_in)[i];
      if constexpr (P == 8) pv[j] = static_cast<const uint64_t*>(pay_in)[i];
      d = digit9<W>(kk, shift);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned r = __popc(peers & lt_mask);
    unsigned prior = 0;
    if (valid) prior = s_warp[warp][d];
    __syncwarp();
    if (valid && r == 0) s_warp[warp][d] = static_cast<unsigned short>(prior + __popc(peers));
    __syncwarp();
    rd[j] = ((prior + r) << kOneBits) | (d & (kOneBins - 1));
  }
  __syncthreads();
  // per-digit exclusive scan over warps (stable order of warps); thread d owns
  // digit d and publishes the tile's count for it at once (AGGREGATE), so the
  // later tiles' look-back does not wait for this tile's scatter
  const int d = threadIdx.x;
  unsigned run = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const unsigned c = s_warp[w][d];
    s_warp[w][d] = static_cast<unsigned short>(run);
    run += c;
  }
  unsigned* st = status + tile * kOneBins + d;
  st_status(st, (tile == 0 ? kFlagPrefix : kFlagAgg) | run);
  {
    // tile-local exclusive scan over digits
    unsigned total;
    const unsigned ds = block_exclusive_scan(run, s_scan, &total);
    s_dstart[d] = static_cast<unsigned short>(ds);
  }
  __syncthreads();
  // stage the tile digit-sorted in shared memory (independent of the look-back)
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const long long i = base + j * 32 + lane;
    if (i < m) {
      const unsigned dd = rd[j] & (kOneBins - 1);
      const unsigned lp = s_dstart[dd] + s_warp[warp][dd] + (rd[j] >> kOneBits);
      if constexpr (W == 1) {
        s_keys[lp] = k0[j];
      } else {
        s_keys[2 * lp] = k0[j];
        s_keys[2 * lp + 1] = k1[j];
      }
      if constexpr (P == 4) s_pay32[lp] = static_cast<unsigned>(pv[j]);
      if constexpr (P == 8) s_pay64[lp] = pv[j];
    }
  }
  {
    // decoupled look-back over the earlier tiles for digit d (their
    // aggregates were published before their scatter, so this rarely spins)
    unsigned excl = 0;
    if (tile > 0) {
      const unsigned* q = st - kOneBins;
      while (true) {
        unsigned v;
        do {
          v = ld_status(q);
        } while ((v & ~kValMask) == 0u);
        excl += v & kValMask;
        if ((v & ~kValMask) == kFlagPrefix) break;
        q -= kOneBins;
      }
      st_status(st, kFlagPrefix | (excl + run));
    }
    s_base[d] = gbase[d] + excl;
  }
  __syncthreads();
  const int cnt = static_cast<int>(min(static_cast<long long>(TILE), m - tile * TILE));
  for (int lp = threadIdx.x; lp < cnt; lp += OT) {
    Key<W> key;
    if constexpr (W == 1) {
      key.w[0] = s_keys[lp];
    } else {
      key.w[0] = s_keys[2 * lp];
      key.w[1] = s_keys[2 * lp + 1];
    }
    const unsigned dd = digit9<W>(key, shift);
    const long long dst = static_cast<long long>(s_base[dd]) + (lp - s_dstart[dd]);
    store_key<W>(keys_out, dst, key);
    if constexpr (P == 4) static_cast<unsigned*>(pay_out)[dst] = s_pay32[lp];
    if constexpr (P == 8) static_cast<uint64_t*>(pay_out)[dst] = s_pay64[lp];
  }
}

// --- K3 duplicates -----------------------------------------------------------

template <int W>
__global__ void find_dup_kernel(const uint64_t* __restrict__ keys, long long m, long long* __restrict__ first) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = 1 + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m; i += stride) {
    const Key<W> a = load_key<W>(keys, i - 1);
    const Key<W> b = load_key<W>(keys, i);
    bool eq = true;
#pragma unroll
    for (int w = 0; w < W; ++w) eq &= (a.w[w] == b.w[w]);
    if (eq) atomicMin(reinterpret_cast<unsigned long long*>(first), static_cast<unsigned long long>(i));
  }
}
__global__ void dup_init(long long* p) { *p = LLONG_MAX; }
__global__ void dup_fini(long long* p) {
  if (*p == LLONG_MAX) *p = -1;
}

struct SortWs {
  uint64_t* keys_alt;
  void* pay_alt;
  unsigned* counts;   // per (digit, tile) counts; one-sweep: per (tile, digit) status words
  unsigned* partial;
  unsigned* ghist;    // one-sweep: kMaxPasses x kOneBins digit bases + kMaxPasses tile counters
  size_t bytes;
};

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static SortWs carve(void* base, long long m, int W, int P) {
  SortWs w{};
  const long long ntiles = (m + kSortTile - 1) / kSortTile;
  const long long ncounts = 256 * ntiles + 256;  // one-sweep: kOneBins status words per 4096-key tile
  const long long nparts = (ncounts + kScanChunk - 1) / kScanChunk;
  size_t off = 0;
  char* b = static_cast<char*>(base);
  w.keys_alt = reinterpret_cast<uint64_t*>(b ? b + off : nullptr);
  off += align256(static_cast<size_t>(m) * W * 8);
  w.pay_alt = b ? b + off : nullptr;
  off += align256(static_cast<size_t>(m) * P);
  w.counts = reinterpret_cast<unsigned*>(b ? b + off : nullptr);
  off += align256(static_cast<size_t>(ncounts) * 4);
  w.partial = reinterpret_cast<unsigned*>(b ? b + off : nullptr);
  off += align256(static_cast<size_t>(nparts + 1) * 4);
  w.ghist = reinterpret_cast<unsigned*>(b ? b + off : nullptr);
  off += align256(static_cast<size_t>(kMaxPasses) * (kOneBins + 1) * 4);
  w.bytes = off;
  return w;
}

template <int W, int P>
static int sort_impl(uint64_t* keys, void* pay, long long m, int total_bits, const SortWs& ws, cudaStream_t s) {
  const long long ntiles = (m + kSortTile - 1) / kSortTile;
  const long long ncounts = 256 * ntiles + 256;  // one-sweep: kOneBins status words per 4096-key tile
  const long long nparts = (ncounts + kScanChunk - 1) / kScanChunk;
  const int passes = (total_bits + 7) / 8;
  const size_t smem = static_cast<size_t>(kSortTile) * (W * 8 + P);
  static bool attr_set = false;
  if (!attr_set) {
    ALTO_CUDA_TRY(cudaFuncSetAttribute(radix_scatter<W, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
    attr_set = true;
  }
  uint64_t* kin = keys;
  uint64_t* kout = ws.keys_alt;
  void* pin = pay;
  void* pout = ws.pay_alt;
  const int opasses = (total_bits + kOneBits - 1) / kOneBits;
  if (m < (1ll << 30) && opasses <= kMaxPasses) {
    constexpr int OT = kOnesweepThreads;
    const long long otiles = (m + OT * kSortItems - 1) / (OT * kSortItems);
    const size_t osmem = static_cast<size_t>(OT) * kSortItems * (W * 8 + P);
    static bool os_attr = false;
    if (!os_attr) {
      ALTO_CUDA_TRY(cudaFuncSetAttribute(onesweep_pass<W, P, OT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(osmem)));
      os_attr = true;
    }
    unsigned* ctr = ws.ghist + kMaxPasses * kOneBins;
    ALTO_CUDA_TRY(cudaMemsetAsync(ws.ghist, 0, static_cast<size_t>(kMaxPasses) * (kOneBins + 1) * 4, s));
    onesweep_hist<W><<<grid_for(m, kSortThreads, kSMs * 4), kSortThreads, 0, s>>>(kin, m, opasses, ws.ghist);
    onesweep_scan<<<opasses, kOneBins, 0, s>>>(ws.ghist);
    for (int p = 0; p < opasses; ++p) {
      ALTO_CUDA_TRY(cudaMemsetAsync(ws.counts, 0, static_cast<size_t>(otiles) * kOneBins * 4, s));
      onesweep_pass<W, P, OT><<<static_cast<unsigned>(otiles), OT, osmem, s>>>(
          kin, pin, kout, pout, m, kOneBits * p, ws.ghist + p * kOneBins, ws.counts, ctr + p);
      std::swap(kin, kout);
      std::swap(pin, pout);
    }
  } else {
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    radix_hist<W><<<static_cast<unsigned>(ntiles), kSortThreads, 0, s>>>(kin, m, shift, ws.counts, ntiles);
    scan_reduce<<<static_cast<unsigned>(nparts), kScanThreads, 0, s>>>(ws.counts, ncounts, ws.partial);
    scan_partials<<<1, 1024, 0, s>>>(ws.partial, nparts);
    scan_down<<<static_cast<unsigned>(nparts), kScanThreads, 0, s>>>(ws.counts, ncounts, ws.partial);
    radix_scatter<W, P><<<static_cast<unsigned>(ntiles), kSortThreads, smem, s>>>(kin, pin, kout, pout, m, shift,
                                                                                 ws.counts, ntiles);
    std::swap(kin, kout);
    std::swap(pin, pout);
  }
  }
  ALTO_LAUNCH_CHECK("alto_sort_pairs");
  if (kin != keys) {
    ALTO_CUDA_TRY(cudaMemcpyAsync(keys, kin, static_cast<size_t>(m) * W * 8, cudaMemcpyDeviceToDevice, s));
    if (P > 0)
      ALTO_CUDA_TRY(cudaMemcpyAsync(pay, pin, static_cast<size_t>(m) * P, cudaMemcpyDeviceToDevice, s));
  }
  return ALTO_OK;
}

}  // namespace alto

using namespace alto;

extern "C" {

size_t alto_sort_workspace_bytes(int64_t m, int32_t n_words, int32_t payload_bytes) {
  if (m < 0) m = 0;
  return carve(nullptr, m, n_words, payload_bytes).bytes;
}

int alto_sort_pairs(uint64_t* keys, void* payload, int64_t m, int32_t n_words, int32_t payload_bytes,
                    int32_t total_bits, void* workspace, size_t workspace_bytes, void* stream) {
  ALTO_REQUIRE(n_words == 1 || n_words == 2, "n_words must be 1 or 2");
  ALTO_REQUIRE(payload_bytes == 0 || payload_bytes == 4 || payload_bytes == 8, "payload_bytes must be 0, 4 or 8");
  ALTO_REQUIRE(total_bits >= 0 && total_bits <= 64 * n_words, "total_bits out of range");
  ALTO_REQUIRE(m >= 0 && m < (1ll << 32) - 1, "sort supports fewer than 2^32 elements");
  if (m <= 1 || total_bits == 0) return ALTO_OK;
  const SortWs ws = carve(workspace, m, n_words, payload_bytes);
  ALTO_REQUIRE(workspace != nullptr && workspace_bytes >= ws.bytes, "sort workspace too small");
  cudaStream_t s = as_stream(stream);
  if (n_words == 1) {
    if (payload_bytes == 0) return sort_impl<1, 0>(keys, payload, m, total_bits, ws, s);
    if (payload_bytes == 4) return sort_impl<1, 4>(keys, payload, m, total_bits, ws, s);
    return sort_impl<1, 8>(keys, payload, m, total_bits, ws, s);
  }
  if (payload_bytes == 0) return sort_impl<2, 0>(keys, payload, m, total_bits, ws, s);
  if (payload_bytes == 4) return sort_impl<2, 4>(keys, payload, m, total_bits, ws, s);
  return sort_impl<2, 8>(keys, payload, m, total_bits, ws, s);
}

int alto_find_duplicate(const uint64_t* keys, int64_t m, int32_t n_words, int64_t* d_first, void* stream) {
  ALTO_REQUIRE(n_words == 1 || n_words == 2, "n_words must be 1 or 2");
  cudaStream_t s = as_stream(stream);
  auto* f = reinterpret_cast<long long*>(d_first);
  dup_init<<<1, 1, 0, s>>>(f);
  if (m > 1) {
    const int grid = grid_for(m, 256);
    if (n_words == 1)
      find_dup_kernel<1><<<grid, 256, 0, s>>>(keys, m, f);
    else
      find_dup_kernel<2><<<grid, 256, 0, s>>>(keys, m, f);
  }
  dup_fini<<<1, 1, 0, s>>>(f);
  ALTO_LAUNCH_CHECK("alto_find_duplicate");
  return ALTO_OK;
}

}  // extern "C"
