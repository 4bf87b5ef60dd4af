// alto_partition.cu — K5 partition intervals/spans, K6 boundary flags,
// read/clear flags, and per-tile mode intervals for the MTTKRP plan.
//
// The reference de-linearizes the whole tensor on the host before taking
// per-partition min/max (format.py:141-152; 18 s at cfg2 scale).  Here one
// streaming pass decodes each key in registers and reduces min/max per warp
// before touching the (count, order, 2) interval array with atomics.
#include <climits>

#include "alto_common.cuh"

namespace alto {

__global__ void intervals_init(long long* iv, long long n_pairs) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n_pairs; i += stride) {
    iv[2 * i] = LLONG_MAX;
    iv[2 * i + 1] = LLONG_MIN;
  }
}

__global__ void intervals_fini(long long* iv, long long n_pairs) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n_pairs; i += stride) {
    if (iv[2 * i] == LLONG_MAX) {  // empty partition (format.py:146-149)
      iv[2 * i] = 0;
      iv[2 * i + 1] = -1;
    }
  }
}

template <int W>
__global__ void partition_kernel(const __grid_constant__ DevLayout L, const uint64_t* __restrict__ tab,
                                 const uint64_t* __restrict__ keys, long long m, long long base,
                                 long long extra, long long* __restrict__ iv) {
  extern __shared__ uint64_t s_dec[];
  copy_to_smem(s_dec, tab + static_cast<long long>(L.dec_off) * W, L.dec_bytes * 256 * W);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  // Loop bound is warp-uniform so that shuffles see full warps.
  const long long m_pad = (m + 31) & ~31ll;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m_pad; i += stride) {
    const bool valid = i < m;
    Key<W> p;
#pragma unroll
    for (int w = 0; w < W; ++w) p.w[w] = 0;
    long long l = -1;
    if (valid) {
      p = decode_packed<W>(s_dec, L.dec_bytes, load_key<W>(keys, i));
      l = partition_of(i, base, extra);
    }
    const long long l0 = __shfl_sync(0xffffffffu, l, 0);
    const bool uniform = __all_sync(0xffffffffu, (!valid) || l == l0) && l0 >= 0;
    for (int n = 0; n < L.order; ++n) {
      const long long c = packed_field<W>(p, L.pack_off[n], L.bits[n]);
      if (uniform) {
        long long lo = valid ? c : LLONG_MAX, hi = valid ? c : LLONG_MIN;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
          hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) {
          atomicMin(iv + (l0 * L.order + n) * 2, lo);
          atomicMax(iv + (l0 * L.order + n) * 2 + 1, hi);
        }
      } else if (valid) {
        atomicMin(iv + (l * L.order + n) * 2, c);
        atomicMax(iv + (l * L.order + n) * 2 + 1, c);
      }
    }
  }
}

template <int W>
__global__ void spans_kernel(const uint64_t* __restrict__ keys, long long m, long long count, long long base,
                             long long extra, uint64_t* __restrict__ spans) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long l = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; l < count; l += stride) {
    const long long lo = l < extra ? l * (base + 1) : extra * (base + 1) + (l - extra) * base;
    const long long sz = l < extra ? base + 1 : base;
    if (sz == 0) continue;
    const Key<W> a = load_key<W>(keys, lo);
    const Key<W> b = load_key<W>(keys, lo + sz - 1);
#pragma unroll
    for (int w = 0; w < W; ++w) {
      spans[(l * 2 + 0) * W + w] = a.w[w];
      spans[(l * 2 + 1) * W + w] = b.w[w];
    }
  }
}

template <int W>
__global__ void flags_kernel(const __grid_constant__ DevLayout L, const uint64_t* __restrict__ tab,
                             const uint64_t* __restrict__ keys, long long m, long long base, long long extra,
                             int mode, int flag_bit, const long long* __restrict__ ov_ptr,
                             const long long* __restrict__ ov_lo, const long long* __restrict__ ov_hi,
                             const long long* __restrict__ offs, long long count, uint64_t* __restrict__ out) {
  extern __shared__ uint64_t s_dec[];
  copy_to_smem(s_dec, tab + static_cast<long long>(L.dec_off) * W, L.dec_bytes * 256 * W);
  __syncthreads();
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m; i += stride) {
    Key<W> k = load_key<W>(keys, i);
    const Key<W> p = decode_packed<W>(s_dec, L.dec_bytes, k);
    const long long c = packed_field<W>(p, L.pack_off[mode], L.bits[mode]);
    long long l;
    if (offs) {
      // arbitrary partition offsets: the last l with offs[l] <= i (skips empty partitions)
      long long a0 = 0, b0 = count;
      while (b0 - a0 > 1) {
        const long long mid = (a0 + b0) >> 1;
        if (offs[mid] <= i) a0 = mid; else b0 = mid;
      }
      l = a0;
    } else {
      l = partition_of(i, base, extra);
    }
    long long a = ov_ptr[l], b = ov_ptr[l + 1];  // ranges [a, b)
    // last range with lo <= c
    while (a < b) {
      const long long mid = (a + b) >> 1;
      if (ov_lo[mid] <= c) a = mid + 1; else b = mid;
    }
    const long long r = a - 1;
    if (r >= ov_ptr[l] && c <= ov_hi[r]) k.w[flag_bit >> 6] |= 1ull << (flag_bit & 63);
    store_key<W>(out, i, k);
  }
}

template <int W>
__global__ void read_flags_kernel(const uint64_t* __restrict__ keys, long long m, int fb, unsigned char* out) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m; i += stride)
    out[i] = static_cast<unsigned char>((keys[i * W + (fb >> 6)] >> (fb & 63)) & 1ull);
}

template <int W>
__global__ void clear_flags_kernel(const uint64_t* __restrict__ keys, long long m, int fb, uint64_t* out) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m; i += stride) {
    Key<W> k = load_key<W>(keys, i);
    k.w[fb >> 6] &= ~(1ull << (fb & 63));
    store_key<W>(out, i, k);
  }
}

// Per-tile per-mode min/max (int32), one CTA per tile.
template <int W>
__global__ void __launch_bounds__(256) tile_iv_kernel(const __grid_constant__ DevLayout L,
                                                      const uint64_t* __restrict__ tab,
                                                      const uint64_t* __restrict__ keys, long long m, int tile,
                                                      int* __restrict__ tlo, int* __restrict__ thi) {
  extern __shared__ uint64_t s_dec[];
  __shared__ int s_lo[8][ALTO_MAX_ORDER], s_hi[8][ALTO_MAX_ORDER];
  copy_to_smem(s_dec, tab + static_cast<long long>(L.dec_off) * W, L.dec_bytes * 256 * W);
  __syncthreads();
  int lo[ALTO_MAX_ORDER], hi[ALTO_MAX_ORDER];
#pragma unroll
  for (int n = 0; n < ALTO_MAX_ORDER; ++n) { lo[n] = INT_MAX; hi[n] = INT_MIN; }
  const long long t0 = static_cast<long long>(blockIdx.x) * tile;
  const long long t1 = min(t0 + tile, m);
  for (long long i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
    const Key<W> p = decode_packed<W>(s_dec, L.dec_bytes, load_key<W>(keys, i));
#pragma unroll
    for (int n = 0; n < ALTO_MAX_ORDER; ++n)
      if (n < L.order) {
        const int c = static_cast<int>(packed_field<W>(p, L.pack_off[n], L.bits[n]));
        lo[n] = min(lo[n], c);
        hi[n] = max(hi[n], c);
      }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int n = 0; n < ALTO_MAX_ORDER; ++n) {
    int a = lo[n], b = hi[n];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (lane == 0) { s_lo[warp][n] = a; s_hi[warp][n] = b; }
  }
  __syncthreads();
  if (threadIdx.x < L.order) {
    const int n = threadIdx.x;
    int a = INT_MAX, b = INT_MIN;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a = min(a, s_lo[w][n]); b = max(b, s_hi[w][n]); }
    tlo[static_cast<long long>(blockIdx.x) * L.order + n] = a;
    thi[static_cast<long long>(blockIdx.x) * L.order + n] = b;
  }
}

template <typename K>
static int set_smem(K kernel, size_t smem) {
  ALTO_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return ALTO_OK;
}

}  // namespace alto

using namespace alto;

extern "C" {

int alto_partition(const alto_layout* lay, const void* d_tables, const uint64_t* keys, int64_t m, int64_t count,
                   int64_t* intervals, uint64_t* spans, void* stream) {
  ALTO_REQUIRE(lay && lay->order >= 1 && lay->order <= ALTO_MAX_ORDER, "bad layout");
  ALTO_REQUIRE(count >= 1 && count <= (m > 1 ? m : 1), "partition count out of range");
  const DevLayout d = make_dev_layout(lay);
  cudaStream_t s = as_stream(stream);
  const long long base = m / count, extra = m % count;
  auto* iv = reinterpret_cast<long long*>(intervals);
  const long long pairs = count * d.order;
  intervals_init<<<grid_for(pairs, 256), 256, 0, s>>>(iv, pairs);
  const size_t smem = static_cast<size_t>(d.dec_bytes) * 256 * d.n_words * 8;
  const auto* tab = static_cast<const uint64_t*>(d_tables);
  if (m > 0) {
    const int grid = grid_for(m, 256, kSMs * 8);
    if (d.n_words == 1) {
      if (set_smem(partition_kernel<1>, smem)) return ALTO_ECUDA;
      partition_kernel<1><<<grid, 256, smem, s>>>(d, tab, keys, m, base, extra, iv);
      spans_kernel<1><<<grid_for(count, 256), 256, 0, s>>>(keys, m, count, base, extra, spans);
    } else {
      if (set_smem(partition_kernel<2>, smem)) return ALTO_ECUDA;
      partition_kernel<2><<<grid, 256, smem, s>>>(d, tab, keys, m, base, extra, iv);
      spans_kernel<2><<<grid_for(count, 256), 256, 0, s>>>(keys, m, count, base, extra, spans);
    }
  }
  intervals_fini<<<grid_for(pairs, 256), 256, 0, s>>>(iv, pairs);
  ALTO_LAUNCH_CHECK("alto_partition");
  return ALTO_OK;
}

int alto_apply_flags(const alto_layout* lay, const void* d_tables, const uint64_t* keys, int64_t m, int64_t count,
                     int32_t mode, int32_t flag_bit, const int64_t* ov_ptr, const int64_t* ov_lo,
                     const int64_t* ov_hi, const int64_t* d_offsets, uint64_t* out_keys, void* stream) {
  ALTO_REQUIRE(lay && lay->order >= 1 && lay->order <= ALTO_MAX_ORDER, "bad layout");
  ALTO_REQUIRE(mode >= 0 && mode < lay->order, "mode out of range");
  ALTO_REQUIRE(flag_bit >= lay->total_bits && flag_bit < 64 * lay->n_words, "flag bit must be an unused index bit");
  ALTO_REQUIRE(count >= 1 && (d_offsets || count <= (m > 1 ? m : 1)), "partition count out of range");
  if (m <= 0) return ALTO_OK;
  const DevLayout d = make_dev_layout(lay);
  cudaStream_t s = as_stream(stream);
  const long long base = m / count, extra = m % count;
  const size_t smem = static_cast<size_t>(d.dec_bytes) * 256 * d.n_words * 8;
  const auto* tab = static_cast<const uint64_t*>(d_tables);
  const int grid = grid_for(m, 256, kSMs * 8);
  auto* p = reinterpret_cast<const long long*>(ov_ptr);
  auto* lo = reinterpret_cast<const long long*>(ov_lo);
  auto* hi = reinterpret_cast<const long long*>(ov_hi);
  auto* offs = reinterpret_cast<const long long*>(d_offsets);
  if (d.n_words == 1) {
    if (set_smem(flags_kernel<1>, smem)) return ALTO_ECUDA;
    flags_kernel<1><<<grid, 256, smem, s>>>(d, tab, keys, m, base, extra, mode, flag_bit, p, lo, hi, offs, count,
                                            out_keys);
  } else {
    if (set_smem(flags_kernel<2>, smem)) return ALTO_ECUDA;
    flags_kernel<2><<<grid, 256, smem, s>>>(d, tab, keys, m, base, extra, mode, flag_bit, p, lo, hi, offs, count,
                                            out_keys);
  }
  ALTO_LAUNCH_CHECK("alto_apply_flags");
  return ALTO_OK;
}

int alto_read_flags(const uint64_t* keys, int64_t m, int32_t n_words, int32_t flag_bit, uint8_t* out, void* stream) {
  ALTO_REQUIRE(n_words == 1 || n_words == 2, "n_words must be 1 or 2");
  ALTO_REQUIRE(flag_bit >= 0 && flag_bit < 64 * n_words, "flag bit out of range");
  if (m <= 0) return ALTO_OK;
  cudaStream_t s = as_stream(stream);
  if (n_words == 1)
    read_flags_kernel<1><<<grid_for(m, 256), 256, 0, s>>>(keys, m, flag_bit, out);
  else
    read_flags_kernel<2><<<grid_for(m, 256), 256, 0, s>>>(keys, m, flag_bit, out);
  ALTO_LAUNCH_CHECK("alto_read_flags");
  return ALTO_OK;
}

int alto_clear_flags(const uint64_t* keys, int64_t m, int32_t n_words, int32_t flag_bit, uint64_t* out_keys,
                     void* stream) {
  ALTO_REQUIRE(n_words == 1 || n_words == 2, "n_words must be 1 or 2");
  ALTO_REQUIRE(flag_bit >= 0 && flag_bit < 64 * n_words, "flag bit out of range");
  if (m <= 0) return ALTO_OK;
  cudaStream_t s = as_stream(stream);
  if (n_words == 1)
    clear_flags_kernel<1><<<grid_for(m, 256), 256, 0, s>>>(keys, m, flag_bit, out_keys);
  else
    clear_flags_kernel<2><<<grid_for(m, 256), 256, 0, s>>>(keys, m, flag_bit, out_keys);
  ALTO_LAUNCH_CHECK("alto_clear_flags");
  return ALTO_OK;
}

int64_t alto_mttkrp_ntiles(int64_t m, int32_t tile) {
  if (tile <= 0 || m <= 0) return 0;
  return (m + tile - 1) / tile;
}

int alto_tile_intervals(const alto_layout* lay, const void* d_tables, const uint64_t* keys, int64_t m, int32_t tile,
                        int32_t* tile_lo, int32_t* tile_hi, void* stream) {
  ALTO_REQUIRE(lay && lay->order >= 1 && lay->order <= ALTO_MAX_ORDER, "bad layout");
  ALTO_REQUIRE(tile > 0, "tile must be positive");
  for (int n = 0; n < lay->order; ++n)
    ALTO_REQUIRE(lay->dims[n] <= INT_MAX, "streaming kernel needs mode extents below 2^31");
  const long long nt = alto_mttkrp_ntiles(m, tile);
  if (nt == 0) return ALTO_OK;
  const DevLayout d = make_dev_layout(lay);
  cudaStream_t s = as_stream(stream);
  const size_t smem = static_cast<size_t>(d.dec_bytes) * 256 * d.n_words * 8;
  const auto* tab = static_cast<const uint64_t*>(d_tables);
  if (d.n_words == 1) {
    if (set_smem(tile_iv_kernel<1>, smem)) return ALTO_ECUDA;
    tile_iv_kernel<1><<<static_cast<unsigned>(nt), 256, smem, s>>>(d, tab, keys, m, tile, tile_lo, tile_hi);
  } else {
    if (set_smem(tile_iv_kernel<2>, smem)) return ALTO_ECUDA;
    tile_iv_kernel<2><<<static_cast<unsigned>(nt), 256, smem, s>>>(d, tab, keys, m, tile, tile_lo, tile_hi);
  }
  ALTO_LAUNCH_CHECK("alto_tile_intervals");
  return ALTO_OK;
}

}  // extern "C"
