// alto_coo.cu — COO ingestion on the device: coalesce.
//
// Reference semantics (pkg/src/altotensor/coo.py:97-114): rows sorted
// lexicographically with mode 0 as the primary key (stable), duplicate
// coordinates summed with np.bincount, i.e. sequentially in that stable
// order starting from 0.0.  Here:
//   1. lex_pack_kernel: one mixed-radix key per row (mode 0 in the most
//      significant bits, b_n = bits_for(I_n) bits per mode, <= 128 bits),
//      payload = row index;
//   2. K2 (alto_sort_pairs): stable LSD radix sort of (key, index) — the
//      stable lexicographic order;
//   3. head flags (row differs from its predecessor) and an exclusive scan
//      give each distinct coordinate its output slot;
//   4. seg_sum_kernel: a thread per distinct coordinate adds the values of
//      its run in sorted (= original) order in float64 from 0.0 — the same
//      additions as bincount, so the sums are bitwise equal — and unpacks
//      the coordinates.
#include "alto_common.cuh"

namespace alto {

struct LexLayout {
  int order;
  int n_words;
  int shift[ALTO_MAX_ORDER];  // bit offset of mode n in the key (mode 0 highest)
  int bits[ALTO_MAX_ORDER];
};

template <int W>
__global__ void lex_pack_kernel(const __grid_constant__ LexLayout L, const long long* __restrict__ coords,
                                long long m, uint64_t* __restrict__ keys, unsigned* __restrict__ idx) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m; i += stride) {
    uint64_t w[2] = {0ull, 0ull};
    for (int n = 0; n < L.order; ++n) {
      const uint64_t c = static_cast<uint64_t>(coords[i * L.order + n]);
      const int s = L.shift[n];
      if (s < 64) {
        w[0] |= c << s;
        if (s > 0 && L.bits[n] + s > 64) w[1] |= c >> (64 - s);
      } else {
        w[1] |= c << (s - 64);
      }
    }
    keys[i * W] = w[0];
    if (W == 2) keys[i * W + 1] = w[1];
    idx[i] = static_cast<unsigned>(i);
  }
}

template <int W>
__global__ void head_kernel(const uint64_t* __restrict__ keys, long long m, unsigned* __restrict__ head) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m; i += stride) {
    bool h = i == 0;
    if (!h) {
      h = keys[i * W] != keys[(i - 1) * W];
      if (W == 2) h = h || keys[i * W + 1] != keys[(i - 1) * W + 1];
    }
    head[i] = h ? 1u : 0u;
  }
}

constexpr int kScanBlock = 1024;

// exclusive scan of 0/1 flags: per-block sums, a one-block scan of those, then
// block-local scans with the block offset
__global__ void __launch_bounds__(kScanBlock) flag_block_sums(const unsigned* __restrict__ f, long long m,
                                                              long long* __restrict__ bsum) {
  __shared__ unsigned s[kScanBlock / 32];
  const long long i = blockIdx.x * static_cast<long long>(kScanBlock) + threadIdx.x;
  unsigned v = i < m ? f[i] : 0u;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned t = s[threadIdx.x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) bsum[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kScanBlock) scan_block_sums(long long* __restrict__ bsum, long long nb,
                                                              long long* __restrict__ total) {
  __shared__ long long s[kScanBlock];
  long long carry = 0;
  for (long long base = 0; base < nb; base += kScanBlock) {
    const long long i = base + threadIdx.x;
    const long long v = i < nb ? bsum[i] : 0;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < kScanBlock; o <<= 1) {
      const long long t = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
      __syncthreads();
      s[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < nb) bsum[i] = carry + s[threadIdx.x] - v;  // exclusive
    carry += s[kScanBlock - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// Slot of every distinct row: block-local exclusive scan of the head flags
// plus the block offset; records the run start of each slot and gathers the
// values into sorted order (sv[j] = values[idx[j]]).
__global__ void __launch_bounds__(kScanBlock) seg_slots_kernel(const unsigned* __restrict__ idx,
                                                               const double* __restrict__ vals,
                                                               const unsigned* __restrict__ head,
                                                               const long long* __restrict__ boff, long long m,
                                                               long long* __restrict__ start,
                                                               double* __restrict__ sv) {
  __shared__ unsigned s[kScanBlock / 32];
  const long long i = blockIdx.x * static_cast<long long>(kScanBlock) + threadIdx.x;
  const unsigned h = i < m ? head[i] : 0u;
  if (i < m) sv[i] = vals[idx[i]];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned x = h;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s[warp] = x;
  __syncthreads();
  if (warp == 0) {
    unsigned t = s[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    s[lane] = t;
  }
  __syncthreads();
  if (h) start[boff[blockIdx.x] + (warp > 0 ? s[warp - 1] : 0u) + x - 1] = i;
}

// A thread per distinct row: the run's values summed in sorted (= original)
// order from 0.0 — the additions of np.bincount — loads batched 8 ahead.
template <int W>
__global__ void seg_sum_kernel(const uint64_t* __restrict__ keys, const double* __restrict__ sv,
                               const long long* __restrict__ start, const long long* __restrict__ count,
                               long long m, const __grid_constant__ LexLayout L, long long* __restrict__ out_coords,
                               double* __restrict__ out_vals) {
  const long long k = *count;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long slot = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; slot < k; slot += stride) {
    const long long a = start[slot], b = slot + 1 < k ? start[slot + 1] : m;
    double sum = 0.0;
    long long j = a;
    for (; j + 8 <= b; j += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = sv[j + u];
#pragma unroll
      for (int u = 0; u < 8; ++u) sum += v[u];
    }
    for (; j < b; ++j) sum += sv[j];
    out_vals[slot] = sum;
    const uint64_t w[2] = {keys[a * W], W == 2 ? keys[a * W + 1] : 0ull};
    for (int n = 0; n < L.order; ++n) {
      const int sh = L.shift[n], bn = L.bits[n];
      uint64_t c;
      if (sh >= 64) {
        c = w[1] >> (sh - 64);
      } else {
        c = w[0] >> sh;
        if (sh > 0) c |= w[1] << (64 - sh);
      }
      if (bn < 64) c &= (1ull << bn) - 1ull;
      out_coords[slot * L.order + n] = static_cast<long long>(c);
    }
  }
}

}  // namespace alto

using namespace alto;

namespace {

struct CoWs {
  uint64_t* keys;
  unsigned* idx;
  unsigned* head;
  long long* start;
  double* sv;
  long long* bsum;
  void* sort_ws;
  size_t sort_bytes;
  size_t bytes;
};

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

CoWs carve_co(void* base, long long m, int W) {
  CoWs w{};
  char* p = static_cast<char*>(base);
  size_t off = 0;
  w.keys = reinterpret_cast<uint64_t*>(p + off);
  off += align256(static_cast<size_t>(m) * 8 * W);
  w.idx = reinterpret_cast<unsigned*>(p + off);
  off += align256(static_cast<size_t>(m) * 4);
  w.head = reinterpret_cast<unsigned*>(p + off);
  off += align256(static_cast<size_t>(m) * 4);
  w.start = reinterpret_cast<long long*>(p + off);
  off += align256(static_cast<size_t>(m + 1) * 8);
  w.sv = reinterpret_cast<double*>(p + off);
  off += align256(static_cast<size_t>(m) * 8);
  const long long nb = (m + kScanBlock - 1) / kScanBlock;
  w.bsum = reinterpret_cast<long long*>(p + off);
  off += align256(static_cast<size_t>(nb + 1) * 8);
  w.sort_ws = p + off;
  w.sort_bytes = alto_sort_workspace_bytes(m, W, 4);
  off += w.sort_bytes;
  w.bytes = off;
  return w;
}

}  // namespace

extern "C" {

size_t alto_coalesce_workspace_bytes(int64_t m, int32_t n_words) {
  if (m < 0) m = 0;
  return carve_co(nullptr, m, n_words == 2 ? 2 : 1).bytes;
}

int alto_coalesce(const int64_t* coords, const double* values, int64_t m, int32_t order, const int32_t* bits,
                  int64_t* out_coords, double* out_values, int64_t* d_count, void* ws, size_t ws_bytes,
                  void* stream) {
  ALTO_REQUIRE(order >= 1 && order <= ALTO_MAX_ORDER, "order out of range");
  ALTO_REQUIRE(bits != nullptr, "bits missing");
  ALTO_REQUIRE(m >= 0 && m < (1ll << 32) - 1, "coalesce supports fewer than 2^32 rows");
  LexLayout L{};
  L.order = order;
  int total = 0;
  for (int n = order - 1; n >= 0; --n) {
    ALTO_REQUIRE(bits[n] >= 0 && bits[n] <= 63, "mode bits out of range");
    L.shift[n] = total;
    L.bits[n] = bits[n];
    total += bits[n];
  }
  ALTO_REQUIRE(total <= 128, "coordinates need more than 128 key bits");
  const int W = total > 64 ? 2 : 1;
  L.n_words = W;
  cudaStream_t s = as_stream(stream);
  ALTO_CUDA_TRY(cudaMemsetAsync(d_count, 0, sizeof(int64_t), s));
  if (m == 0) return ALTO_OK;
  ALTO_REQUIRE(ws && ws_bytes >= alto_coalesce_workspace_bytes(m, W), "coalesce workspace too small");
  const CoWs w = carve_co(ws, m, W);
  const int grid = grid_for(m, 256, kSMs * 8);
  if (W == 1)
    lex_pack_kernel<1><<<grid, 256, 0, s>>>(L, reinterpret_cast<const long long*>(coords), m, w.keys, w.idx);
  else
    lex_pack_kernel<2><<<grid, 256, 0, s>>>(L, reinterpret_cast<const long long*>(coords), m, w.keys, w.idx);
  ALTO_LAUNCH_CHECK("alto_coalesce/pack");
  const int st = alto_sort_pairs(w.keys, w.idx, m, W, 4, total, w.sort_ws, w.sort_bytes, stream);
  if (st) return st;
  if (W == 1)
    head_kernel<1><<<grid, 256, 0, s>>>(w.keys, m, w.head);
  else
    head_kernel<2><<<grid, 256, 0, s>>>(w.keys, m, w.head);
  const long long nb = (m + kScanBlock - 1) / kScanBlock;
  flag_block_sums<<<static_cast<unsigned>(nb), kScanBlock, 0, s>>>(w.head, m, w.bsum);
  scan_block_sums<<<1, kScanBlock, 0, s>>>(w.bsum, nb, reinterpret_cast<long long*>(d_count));
  seg_slots_kernel<<<static_cast<unsigned>(nb), kScanBlock, 0, s>>>(w.idx, values, w.head, w.bsum, m, w.start,
                                                                    w.sv);
  const auto* cnt = reinterpret_cast<const long long*>(d_count);
  if (W == 1)
    seg_sum_kernel<1><<<grid, 256, 0, s>>>(w.keys, w.sv, w.start, cnt, m, L, reinterpret_cast<long long*>(out_coords),
                                           out_values);
  else
    seg_sum_kernel<2><<<grid, 256, 0, s>>>(w.keys, w.sv, w.start, cnt, m, L, reinterpret_cast<long long*>(out_coords),
                                           out_values);
  ALTO_LAUNCH_CHECK("alto_coalesce");
  return ALTO_OK;
}

}  // extern "C"
