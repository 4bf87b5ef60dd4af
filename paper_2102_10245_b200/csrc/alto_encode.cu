// alto_encode.cu — layout tables, K1 linearize, K4 delinearize, error plumbing.
//
// Replaces layout.py:148-182 (per-bit NumPy passes) with one table-driven
// pass per element.  See alto_common.cuh for the table scheme.
#include <algorithm>
#include <climits>
#include <cstring>
#include <string>
#include <vector>

#include "alto_common.cuh"

namespace alto {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

int cuda_status(cudaError_t e, const char* where) {
  g_err = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
  return ALTO_ECUDA;
}

DevLayout make_dev_layout(const alto_layout* lay) {
  DevLayout d;
  std::memset(&d, 0, sizeof(d));
  d.order = lay->order;
  d.n_words = lay->n_words;
  d.total_bits = lay->total_bits;
  int off = 0, entry = 0;
  for (int n = 0; n < lay->order; ++n) {
    d.bits[n] = lay->bits[n];
    d.dims[n] = lay->dims[n];
    d.pack_off[n] = off;
    off += lay->bits[n];
    d.enc_off[n] = entry;
    d.enc_bytes[n] = (lay->bits[n] + 7) / 8;
    entry += d.enc_bytes[n] * 256;
  }
  d.dec_off = entry;
  d.dec_bytes = (lay->total_bits + 7) / 8;
  entry += d.dec_bytes * 256;
  d.n_entries = entry;
  return d;
}

static int check_layout(const alto_layout* lay) {
  if (lay == nullptr) { set_error("layout is NULL"); return ALTO_EINVAL; }
  if (lay->order < 1 || lay->order > ALTO_MAX_ORDER) {
    set_error("layout order must be in [1, 8]");
    return ALTO_EUNSUPPORTED;
  }
  if (lay->n_words != 1 && lay->n_words != 2) { set_error("n_words must be 1 or 2"); return ALTO_EINVAL; }
  int total = 0;
  for (int n = 0; n < lay->order; ++n) {
    if (lay->bits[n] < 0 || lay->bits[n] > 63) { set_error("mode bits out of range"); return ALTO_EINVAL; }
    total += lay->bits[n];
  }
  if (total != lay->total_bits || total > 64 * lay->n_words) {
    set_error("layout total_bits inconsistent with bits/width");
    return ALTO_EINVAL;
  }
  return ALTO_OK;
}

// --- K1 linearize ---------------------------------------------------------

template <int W>
__global__ void linearize_kernel(const __grid_constant__ DevLayout L, const uint64_t* __restrict__ tab,
                                 const long long* __restrict__ coords, long long m,
                                 uint64_t* __restrict__ keys, long long* __restrict__ bad) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m; i += stride) {
    Key<W> k;
#pragma unroll
    for (int w = 0; w < W; ++w) k.w[w] = 0;
    bool ok = true;
    for (int n = 0; n < L.order; ++n) {
      const long long c = __ldg(coords + i * L.order + n);
      ok &= (c >= 0) & (c < L.dims[n]);
      const unsigned long long uc = static_cast<unsigned long long>(c);
      for (int b = 0; b < L.enc_bytes[n]; ++b) {
        const unsigned byte = static_cast<unsigned>(uc >> (8 * b)) & 0xffu;
        const uint64_t* e = tab + static_cast<long long>(L.enc_off[n] + b * 256 + byte) * W;
#pragma unroll
        for (int w = 0; w < W; ++w) k.w[w] |= __ldg(e + w);
      }
    }
    if (!ok) atomicMin(reinterpret_cast<unsigned long long*>(bad), static_cast<unsigned long long>(i));
    store_key<W>(keys, i, k);
  }
}

__global__ void sentinel_to_minus_one(long long* p) {
  if (*p == LLONG_MAX) *p = -1;
}
__global__ void set_sentinel(long long* p) { *p = LLONG_MAX; }

// --- K4 delinearize -------------------------------------------------------

template <int W>
__global__ void delinearize_kernel(const __grid_constant__ DevLayout L, const uint64_t* __restrict__ tab,
                                   const uint64_t* __restrict__ keys, long long m, int mode,
                                   long long* __restrict__ out) {
  extern __shared__ uint64_t s_dec[];
  copy_to_smem(s_dec, tab + static_cast<long long>(L.dec_off) * W, L.dec_bytes * 256 * W);
  __syncthreads();
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m; i += stride) {
    const Key<W> k = load_key<W>(keys, i);
    const Key<W> p = decode_packed<W>(s_dec, L.dec_bytes, k);
    if (mode >= 0) {
      out[i] = packed_field<W>(p, L.pack_off[mode], L.bits[mode]);
    } else {
      for (int n = 0; n < L.order; ++n) out[i * L.order + n] = packed_field<W>(p, L.pack_off[n], L.bits[n]);
    }
  }
}

// Elements per row of one mode (the hot-row plans need only these counts).  The
// warp's 32 consecutive ALTO elements mostly share a few rows: equal rows are
// grouped with match.any and one lane adds the group's size — into a small
// direct-mapped table of the CTA in shared memory (row -> count; a colliding
// row evicts the resident one to global memory), so the Zipf-head rows, which
// every warp sees, reach their global counters once per CTA instead of once
// per warp instruction (same-address atomics serialise in one L2 slice).
constexpr int kCountSlots = 1024;

template <int W>
__global__ void row_count_kernel(const __grid_constant__ DevLayout L, const uint64_t* __restrict__ tab,
                                 const uint64_t* __restrict__ keys, long long m, int mode,
                                 unsigned* __restrict__ counts) {
  extern __shared__ uint64_t s_dec[];
  __shared__ unsigned long long s_slot[kCountSlots];  // (row + 1) << 32 | count; 0 = empty
  copy_to_smem(s_dec, tab + static_cast<long long>(L.dec_off) * W, L.dec_bytes * 256 * W);
  for (int i = threadIdx.x; i < kCountSlots; i += blockDim.x) s_slot[i] = 0ull;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  // a CTA walks a contiguous chunk (consecutive ALTO elements share rows)
  const long long per = (m + gridDim.x - 1) / gridDim.x;
  const long long lo = blockIdx.x * per, hi = min(m, lo + per);
  const long long n_round = lo + (hi - lo + blockDim.x - 1) / blockDim.x * blockDim.x;  // whole warps stay together
  for (long long i = lo + threadIdx.x; i < n_round; i += blockDim.x) {
    const bool ok = i < hi;
    unsigned long long row = 0xffffffff00000000ull | static_cast<unsigned>(lane);  // idle lanes: singletons
    if (ok) {
      const Key<W> p = decode_packed<W>(s_dec, L.dec_bytes, load_key<W>(keys, i));
      row = static_cast<unsigned long long>(packed_field<W>(p, L.pack_off[mode], L.bits[mode]));
    }
    const unsigned peers = __match_any_sync(0xffffffffu, row);
    if (ok && (peers & ((1u << lane) - 1u)) == 0u) {
      const unsigned add = static_cast<unsigned>(__popc(peers));
      unsigned long long* slot = s_slot + (static_cast<unsigned>(row) & (kCountSlots - 1));
      const unsigned long long tag = (row + 1ull) << 32;
      unsigned long long cur = *slot;
      while (true) {
        if ((cur >> 32) == (tag >> 32)) {  // resident: add (count < 2^32 per CTA chunk)
          const unsigned long long seen = atomicCAS(slot, cur, cur + add);
          if (seen == cur) break;
          cur = seen;
        } else {  // empty or another row: take the slot, flush what was there
          const unsigned long long seen = atomicCAS(slot, cur, tag | add);
          if (seen == cur) {
            if (cur) atomicAdd(counts + ((cur >> 32) - 1ull), static_cast<unsigned>(cur));
            break;
          }
          cur = seen;
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kCountSlots; i += blockDim.x) {
    const unsigned long long cur = s_slot[i];
    if (cur) atomicAdd(counts + ((cur >> 32) - 1ull), static_cast<unsigned>(cur));
  }
}

// Per-mode maximum coordinate (container validation: a corrupt file must not
// drive out-of-range factor/output rows).  Warp max, then one atomicMax per
// warp and mode.
template <int W>
__global__ void coord_max_kernel(const __grid_constant__ DevLayout L, const uint64_t* __restrict__ tab,
                                 const uint64_t* __restrict__ keys, long long m,
                                 unsigned long long* __restrict__ out) {
  extern __shared__ uint64_t s_dec[];
  copy_to_smem(s_dec, tab + static_cast<long long>(L.dec_off) * W, L.dec_bytes * 256 * W);
  __syncthreads();
  unsigned long long mx[ALTO_MAX_ORDER];
  for (int n = 0; n < ALTO_MAX_ORDER; ++n) mx[n] = 0ull;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m; i += stride) {
    const Key<W> p = decode_packed<W>(s_dec, L.dec_bytes, load_key<W>(keys, i));
    for (int n = 0; n < L.order; ++n) {
      const unsigned long long c = static_cast<unsigned long long>(packed_field<W>(p, L.pack_off[n], L.bits[n]));
      mx[n] = c > mx[n] ? c : mx[n];
    }
  }
  for (int n = 0; n < L.order; ++n) {
    unsigned long long v = mx[n];
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long u = __shfl_down_sync(0xffffffffu, v, o);
      v = u > v ? u : v;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(out + n, v);
  }
}

}  // namespace alto

using namespace alto;

extern "C" {

int alto_coord_max(const alto_layout* lay, const void* d_tables, const uint64_t* keys, int64_t m,
                   uint64_t* out_max, void* stream) {
  int st = check_layout(lay);
  if (st != ALTO_OK) return st;
  cudaStream_t s = as_stream(stream);
  ALTO_CUDA_TRY(cudaMemsetAsync(out_max, 0, sizeof(uint64_t) * lay->order, s));
  if (m <= 0) return ALTO_OK;
  const DevLayout d = make_dev_layout(lay);
  const int block = 256;
  const int grid = grid_for(m, block, kSMs * 4);
  const size_t smem = static_cast<size_t>(d.dec_bytes) * 256 * d.n_words * sizeof(uint64_t);
  const auto* tab = static_cast<const uint64_t*>(d_tables);
  auto* o = reinterpret_cast<unsigned long long*>(out_max);
  if (d.n_words == 1) {
    ALTO_CUDA_TRY(cudaFuncSetAttribute(coord_max_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    coord_max_kernel<1><<<grid, block, smem, s>>>(d, tab, keys, m, o);
  } else {
    ALTO_CUDA_TRY(cudaFuncSetAttribute(coord_max_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    coord_max_kernel<2><<<grid, block, smem, s>>>(d, tab, keys, m, o);
  }
  ALTO_LAUNCH_CHECK("alto_coord_max");
  return ALTO_OK;
}

const char* alto_last_error(void) { return g_err.c_str(); }
int alto_version(void) { return 1; }

size_t alto_tables_bytes(const alto_layout* lay) {
  if (check_layout(lay) != ALTO_OK) return 0;
  const DevLayout d = make_dev_layout(lay);
  return static_cast<size_t>(d.n_entries) * lay->n_words * sizeof(uint64_t);
}

int alto_build_tables(const alto_layout* lay, void* d_tables, void* stream) {
  int st = check_layout(lay);
  if (st != ALTO_OK) return st;
  const DevLayout d = make_dev_layout(lay);
  const int W = lay->n_words;
  std::vector<uint64_t> host(static_cast<size_t>(d.n_entries) * W, 0ull);
  // Encode: ENC[n][k][b] deposits byte k of a mode-n coordinate.
  for (int n = 0; n < d.order; ++n) {
    for (int k = 0; k < d.enc_bytes[n]; ++k) {
      for (int b = 0; b < 256; ++b) {
        uint64_t* e = &host[static_cast<size_t>(d.enc_off[n] + k * 256 + b) * W];
        for (int t = 0; t < 8; ++t) {
          const int g = 8 * k + t;
          if (g >= d.bits[n] || !((b >> t) & 1)) continue;
          const int p = lay->pos[n][g];
          e[p >> 6] |= 1ull << (p & 63);
        }
      }
    }
  }
  // Decode: owner of every key bit below total_bits.
  std::vector<int> owner_mode(ALTO_MAX_BITS, -1), owner_g(ALTO_MAX_BITS, -1);
  for (int n = 0; n < d.order; ++n)
    for (int g = 0; g < d.bits[n]; ++g) {
      const int p = lay->pos[n][g];
      if (p < 0 || p >= d.total_bits || owner_mode[p] != -1) {
        set_error("layout positions are not a bijection onto [0, total_bits)");
        return ALTO_EINVAL;
      }
      owner_mode[p] = n;
      owner_g[p] = g;
    }
  for (int j = 0; j < d.dec_bytes; ++j) {
    for (int b = 0; b < 256; ++b) {
      uint64_t* e = &host[static_cast<size_t>(d.dec_off + j * 256 + b) * W];
      for (int t = 0; t < 8; ++t) {
        const int q = 8 * j + t;
        if (q >= d.total_bits || !((b >> t) & 1)) continue;
        const int pb = d.pack_off[owner_mode[q]] + owner_g[q];
        e[pb >> 6] |= 1ull << (pb & 63);
      }
    }
  }
  ALTO_CUDA_TRY(cudaMemcpyAsync(d_tables, host.data(), host.size() * sizeof(uint64_t),
                                cudaMemcpyHostToDevice, as_stream(stream)));
  ALTO_CUDA_TRY(cudaStreamSynchronize(as_stream(stream)));
  return ALTO_OK;
}

int alto_linearize(const alto_layout* lay, const void* d_tables, const int64_t* coords, int64_t m,
                   uint64_t* keys, int64_t* d_bad, void* stream) {
  int st = check_layout(lay);
  if (st != ALTO_OK) return st;
  ALTO_REQUIRE(m >= 0, "nnz must be nonnegative");
  const DevLayout d = make_dev_layout(lay);
  cudaStream_t s = as_stream(stream);
  auto* bad = reinterpret_cast<long long*>(d_bad);
  set_sentinel<<<1, 1, 0, s>>>(bad);
  if (m > 0) {
    const int block = 256;
    const int grid = grid_for(m, block);
    const auto* tab = static_cast<const uint64_t*>(d_tables);
    const auto* c = reinterpret_cast<const long long*>(coords);
    if (d.n_words == 1)
      linearize_kernel<1><<<grid, block, 0, s>>>(d, tab, c, m, keys, bad);
    else
      linearize_kernel<2><<<grid, block, 0, s>>>(d, tab, c, m, keys, bad);
  }
  sentinel_to_minus_one<<<1, 1, 0, s>>>(bad);
  ALTO_LAUNCH_CHECK("alto_linearize");
  return ALTO_OK;
}

int alto_delinearize(const alto_layout* lay, const void* d_tables, const uint64_t* keys, int64_t m,
                     int32_t mode, int64_t* out, void* stream) {
  int st = check_layout(lay);
  if (st != ALTO_OK) return st;
  ALTO_REQUIRE(mode >= -1 && mode < lay->order, "mode out of range");
  if (m <= 0) return ALTO_OK;
  const DevLayout d = make_dev_layout(lay);
  cudaStream_t s = as_stream(stream);
  const int block = 256;
  const int grid = grid_for(m, block, kSMs * 8);
  const size_t smem = static_cast<size_t>(d.dec_bytes) * 256 * d.n_words * sizeof(uint64_t);
  const auto* tab = static_cast<const uint64_t*>(d_tables);
  auto* o = reinterpret_cast<long long*>(out);
  if (d.n_words == 1) {
    ALTO_CUDA_TRY(cudaFuncSetAttribute(delinearize_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    delinearize_kernel<1><<<grid, block, smem, s>>>(d, tab, keys, m, mode, o);
  } else {
    ALTO_CUDA_TRY(cudaFuncSetAttribute(delinearize_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    delinearize_kernel<2><<<grid, block, smem, s>>>(d, tab, keys, m, mode, o);
  }
  ALTO_LAUNCH_CHECK("alto_delinearize");
  return ALTO_OK;
}

int alto_row_counts(const alto_layout* lay, const void* d_tables, const uint64_t* keys, int64_t m, int32_t mode,
                    uint32_t* counts, void* stream) {
  const int st = check_layout(lay);
  if (st) return st;
  ALTO_REQUIRE(mode >= 0 && mode < lay->order, "mode out of range");
  ALTO_REQUIRE(m >= 0 && m < (1ll << 32), "row counts support fewer than 2^32 elements");
  if (m == 0) return ALTO_OK;
  ALTO_REQUIRE(d_tables && keys && counts, "null argument");
  const DevLayout d = make_dev_layout(lay);
  cudaStream_t s = as_stream(stream);
  const int block = 256;
  const int grid = grid_for(m, block, kSMs * 8);
  const size_t smem = static_cast<size_t>(d.dec_bytes) * 256 * d.n_words * sizeof(uint64_t);
  const auto* tab = static_cast<const uint64_t*>(d_tables);
  if (d.n_words == 1) {
    ALTO_CUDA_TRY(cudaFuncSetAttribute(row_count_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    row_count_kernel<1><<<grid, block, smem, s>>>(d, tab, keys, m, mode, counts);
  } else {
    ALTO_CUDA_TRY(cudaFuncSetAttribute(row_count_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    row_count_kernel<2><<<grid, block, smem, s>>>(d, tab, keys, m, mode, counts);
  }
  ALTO_LAUNCH_CHECK("alto_row_counts");
  return ALTO_OK;
}

}  // extern "C"
