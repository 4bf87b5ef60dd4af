// alto_plan.cu — per-tensor / per-mode plans of the streaming MTTKRP:
// mode-contiguous key re-encoding and the row-sorted sub-tile order (see
// alto_fast.cuh, "planned variant").  Built once (like the reference's
// per-mode plans and flagged copies in _make_backend, cpd.py:149-181).
#include "alto_mstream.cuh"

namespace alto {

template <int W>
__global__ void pack_keys_kernel(const __grid_constant__ DevLayout L, const uint64_t* __restrict__ tab,
                                 const uint64_t* __restrict__ keys, long long m, uint64_t* __restrict__ packed) {
  extern __shared__ uint64_t s_dec[];
  copy_to_smem(s_dec, tab + static_cast<long long>(L.dec_off) * W, L.dec_bytes * 256 * W);
  __syncthreads();
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m; i += stride)
    store_key<W>(packed, i, decode_packed<W>(s_dec, L.dec_bytes, load_key<W>(keys, i)));
}

// One warp per 128-element sub-tile; deterministic (stable) slots: for each
// of the 4 element rounds, equal rows form a __match_any_sync group whose
// leader reserves the group's slots; rounds run in order.
template <int W>
__global__ void subtile_order_kernel(const __grid_constant__ DevLayout L, const uint64_t* __restrict__ packed,
                                     long long m, int mode, unsigned char* __restrict__ pos) {
  __shared__ int s_bins[kTileThreads / 32][kFastBins];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* bin = s_bins[warp];
  const long long nsub = (m + kFastTile - 1) / kFastTile;
  const long long nwarps = static_cast<long long>(gridDim.x) * (kTileThreads / 32);
  const unsigned ltm = (1u << lane) - 1u;
  for (long long sub = static_cast<long long>(blockIdx.x) * (kTileThreads / 32) + warp; sub < nsub; sub += nwarps) {
    const long long e0 = sub * kFastTile;
    const int cnt = static_cast<int>(min(static_cast<long long>(kFastTile), m - e0));
    int row[4];
    int lo = INT_MAX, hi = INT_MIN;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = lane + 32 * k;
      row[k] = -1;
      if (e < cnt) {
        row[k] = static_cast<int>(packed_field32<W>(load_key<W>(packed, e0 + e), L.pack_off[mode], L.bits[mode]));
        lo = min(lo, row[k]);
        hi = max(hi, row[k]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const int span = hi - lo + 1;
    if (span > kFastBins) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (row[k] >= 0) pos[e0 + lane + 32 * k] = static_cast<unsigned char>(lane + 32 * k);
      continue;
    }
    for (int i = lane; i < span; i += 32) bin[i] = 0;
    __syncwarp();
    unsigned peers[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool ok = row[k] >= 0;
      peers[k] = __match_any_sync(0xffffffffu, ok ? row[k] : -1 - lane);
      if (ok && (peers[k] & ltm) == 0) bin[row[k] - lo] += __popc(peers[k]);  // one writer per bin per round
      __syncwarp();
    }
    int carry = 0;
    for (int base = 0; base < span; base += 32) {
      const int i = base + lane;
      const int v = i < span ? bin[i] : 0;
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (i < span) bin[i] = carry + x - v;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool ok = row[k] >= 0;
      const int leader = __ffs(peers[k]) - 1;
      int b = 0;
      if (ok && leader == lane) {
        b = bin[row[k] - lo];
        bin[row[k] - lo] = b + __popc(peers[k]);
      }
      b = __shfl_sync(0xffffffffu, b, leader);
      if (ok) pos[e0 + lane + 32 * k] = static_cast<unsigned char>(b + __popc(peers[k] & ltm));
      __syncwarp();
    }
  }
}


// ---- per-mode stream (alto_mstream.cuh) ----------------------------------------
// ckey = (tile << b_mode) | row, idx = element: a stable sort of these pairs is
// the per-tile stable sort by output row.
template <int W>
__global__ void mstream_keys_kernel(const __grid_constant__ DevLayout L, const uint64_t* __restrict__ packed,
                                    long long m, int mode, int tile, int row_major, uint64_t* __restrict__ ckey,
                                    unsigned* __restrict__ idx) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m; i += stride) {
    const unsigned row = packed_field32<W>(load_key<W>(packed, i), L.pack_off[mode], L.bits[mode]);
    ckey[i] = row_major ? row : ((static_cast<uint64_t>(i / tile) << L.bits[mode]) | row);
    idx[i] = static_cast<unsigned>(i);
  }
}

template <int W, typename V>
__global__ void mstream_scatter_kernel(const __grid_constant__ DevLayout L, const __grid_constant__ MsFields F,
                                       const uint64_t* __restrict__ packed, const V* __restrict__ vals,
                                       const unsigned* __restrict__ idx, long long m, int mode, int tile,
                                       int round_robin, const int* __restrict__ hot_slot,
                                       uint64_t* __restrict__ skeys, V* __restrict__ svals,
                                       const uint64_t* __restrict__ srows, int* __restrict__ base_rows,
                                       int* __restrict__ overflow, int blk_u, int blk_gpw) {
  const int ch = tile / kMsSlices;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < m; q += stride) {
    const long long src = idx[q];
    const long long t = q / tile;
    const int p = static_cast<int>(q - t * tile);
    // slices: lane group s takes sorted positions [s*ch, (s+1)*ch) of the tile,
    // stored interleaved; round robin: group s takes positions s, s+8, ...
    // (consecutive elements in one instruction), stored in sorted order
    long long dst = round_robin ? q : t * tile + static_cast<long long>(p % ch) * kMsSlices + p / ch;
    if (round_robin == 2) {
      // blocked: a warp step is blk_gpw * blk_u consecutive sorted elements;
      // group s takes elements s, s + gpw, ... of the step (round robin) and
      // its blk_u elements are stored contiguously (one vector load)
      const int bsz = blk_gpw * blk_u;
      const int pb = p % bsz;
      dst = q - pb + (pb % blk_gpw) * blk_u + pb / blk_gpw;
    }
    const Key<W> k = load_key<W>(packed, src);
    const unsigned row = packed_field32<W>(k, L.pack_off[mode], L.bits[mode]);
    const bool hot = hot_slot && hot_slot[row] >= 0;
    if (base_rows) {
      // delta stream: inputs + increment from the group's previous element
      // (srows = the sorted row of every position, so its neighbour is known)
      const bool rr1 = round_robin == 1;
      int gs = rr1 ? (p % kMsSlices) : (p / ch);
      int gj = rr1 ? (p / kMsSlices) : (p % ch);
      long long prev = rr1 ? q - kMsSlices : q - 1;
      int ngroups = kMsSlices;
      if (round_robin == 2) {
        // blocked: group s takes sorted positions s, s + gpw, ... of the tile
        gs = p % blk_gpw;
        gj = p / blk_gpw;
        prev = q - blk_gpw;
        ngroups = blk_gpw;
      }
      uint64_t w = 0;
      for (int n = 0; n < L.order; ++n) {
        if (n == mode) continue;
        w |= static_cast<uint64_t>(packed_field32<W>(k, L.pack_off[n], L.bits[n])) << F.sh[n];
      }
      unsigned dlt = 0;
      if (gj == 0) {
        base_rows[t * ngroups + gs] = static_cast<int>(row);
      } else {
        dlt = row - static_cast<unsigned>(srows[prev]);
        if (dlt > F.mask[mode]) atomicExch(overflow, 1);
      }
      w |= static_cast<uint64_t>(dlt & F.mask[mode]) << F.sh[mode];
      if (hot) w |= 1ull << 63;
      skeys[dst] = w;
      svals[dst] = vals[src];
      continue;
    }
    Key<W> o{};
    for (int n = 0; n < L.order; ++n) {
      const uint64_t c = packed_field32<W>(k, L.pack_off[n], L.bits[n]);
      o.w[W == 1 ? 0 : F.word[n]] |= c << F.sh[n];
    }
    if (hot) o.w[W - 1] |= 1ull << 63;
    store_key<W>(skeys, dst, o);
    svals[dst] = vals[src];
  }
}

}  // namespace alto

using namespace alto;

extern "C" {

int alto_pack_keys(const alto_layout* lay, const void* d_tables, const uint64_t* keys, int64_t m, uint64_t* packed,
                   void* stream) {
  ALTO_REQUIRE(lay && lay->order >= 1 && lay->order <= ALTO_MAX_ORDER, "bad layout");
  if (m <= 0) return ALTO_OK;
  const DevLayout d = make_dev_layout(lay);
  cudaStream_t s = as_stream(stream);
  const size_t smem = static_cast<size_t>(d.dec_bytes) * 256 * d.n_words * 8;
  const auto* tab = static_cast<const uint64_t*>(d_tables);
  if (d.n_words == 1) {
    if (prep(pack_keys_kernel<1>, smem)) return ALTO_ECUDA;
    pack_keys_kernel<1><<<grid_for(m, 256, kSMs * 8), 256, smem, s>>>(d, tab, keys, m, packed);
  } else {
    if (prep(pack_keys_kernel<2>, smem)) return ALTO_ECUDA;
    pack_keys_kernel<2><<<grid_for(m, 256, kSMs * 8), 256, smem, s>>>(d, tab, keys, m, packed);
  }
  ALTO_LAUNCH_CHECK("alto_pack_keys");
  return ALTO_OK;
}

int alto_subtile_order(const alto_layout* lay, const uint64_t* packed, int64_t m, int32_t mode, uint8_t* pos,
                       void* stream) {
  ALTO_REQUIRE(lay && mode >= 0 && mode < lay->order, "mode out of range");
  ALTO_REQUIRE(lay->bits[mode] <= 31, "sub-tile order needs mode extents below 2^31");
  if (m <= 0) return ALTO_OK;
  const DevLayout d = make_dev_layout(lay);
  cudaStream_t s = as_stream(stream);
  const long long nsub = (m + kFastTile - 1) / kFastTile;
  const int grid = grid_for(nsub, kTileThreads / 32, kSMs * 8);
  if (d.n_words == 1)
    subtile_order_kernel<1><<<grid, kTileThreads, 0, s>>>(d, packed, m, mode, pos);
  else
    subtile_order_kernel<2><<<grid, kTileThreads, 0, s>>>(d, packed, m, mode, pos);
  ALTO_LAUNCH_CHECK("alto_subtile_order");
  return ALTO_OK;
}

size_t alto_mode_stream_workspace_bytes(int64_t m) {
  if (m < 0) m = 0;
  const size_t a = (static_cast<size_t>(m) * 8 + 255) & ~size_t(255);
  const size_t b = (static_cast<size_t>(m) * 4 + 255) & ~size_t(255);
  return a + b + alto_sort_workspace_bytes(m, 1, 4);
}

int alto_mode_stream(const alto_layout* lay, const uint64_t* packed, const void* values, int32_t value_dtype,
                     int64_t m, int32_t mode, int32_t tile, int32_t flags, const int32_t* hot_slot, uint64_t* skeys,
                     void* svals, int32_t* base_rows, int32_t* d_overflow, void* ws, size_t ws_bytes,
                     void* stream) {
  ALTO_REQUIRE(lay && lay->order >= 1 && lay->order <= ALTO_MAX_ORDER, "bad layout");
  ALTO_REQUIRE(mode >= 0 && mode < lay->order, "mode out of range");
  ALTO_REQUIRE(lay->bits[mode] <= 31, "mode stream needs mode extents below 2^31");
  ALTO_REQUIRE(value_dtype == ALTO_F32 || value_dtype == ALTO_F64, "unsupported value dtype");
  ALTO_REQUIRE(tile >= 128 && tile % 128 == 0, "tile must be a positive multiple of 128");
  ALTO_REQUIRE(m >= 0 && m < (1ll << 32) - 1, "mode stream supports fewer than 2^32 elements");
  const DevLayout d = make_dev_layout(lay);
  const bool delta = (flags & ALTO_MS_DELTA) != 0;
  ALTO_REQUIRE(!delta || ((flags & ALTO_MS_ROW_MAJOR) && base_rows && d_overflow),
               "delta stream needs row-major order, base_rows and d_overflow");
  const bool blocked = (flags & ALTO_MS_BLOCKED) != 0;
  const int blk_u = (flags >> 8) & 15, blk_gpw = (flags >> 12) & 15;
  ALTO_REQUIRE(!blocked || ((flags & ALTO_MS_ROW_MAJOR) && blk_u >= 1 && blk_u <= 8 && blk_gpw >= 1 && blk_gpw <= 8 &&
                            tile % (blk_u * blk_gpw) == 0),
               "blocked stream needs row-major order and ALTO_MS_BLOCK(u, groups) dividing the tile");
  const int gmode = blocked ? 2 : ((flags & ALTO_MS_ROUND_ROBIN) ? 1 : 0);
  const MsFields F = delta ? ms_fields_delta(d, mode) : ms_fields(d, mode);
  if (!F.ok) {
    set_error("mode stream: the mode's field layout does not fit the key width");
    return ALTO_EUNSUPPORTED;
  }
  const int sw = delta ? 1 : d.n_words;  // stream key words
  const long long ntiles = (m + tile - 1) / tile;
  const int row_major = (flags & ALTO_MS_ROW_MAJOR) ? 1 : 0;
  int tbits = 0;
  while (!row_major && (1ll << tbits) < ntiles) ++tbits;
  ALTO_REQUIRE(tbits + lay->bits[mode] <= 64, "too many tiles for the sort key");
  cudaStream_t s = as_stream(stream);
  const size_t vb = value_dtype == ALTO_F32 ? 4 : 8;
  const size_t padded = static_cast<size_t>(ntiles) * tile;
  if (delta) ALTO_CUDA_TRY(cudaMemsetAsync(d_overflow, 0, sizeof(int32_t), s));
  if (padded > static_cast<size_t>(m)) {
    ALTO_CUDA_TRY(cudaMemsetAsync(skeys + static_cast<size_t>(m) * sw, 0, (padded - m) * 8 * sw, s));
    ALTO_CUDA_TRY(cudaMemsetAsync(static_cast<char*>(svals) + m * vb, 0, (padded - m) * vb, s));
  }
  if (m <= 0) return ALTO_OK;
  ALTO_REQUIRE(ws && ws_bytes >= alto_mode_stream_workspace_bytes(m), "mode stream workspace too small");
  auto* ckey = static_cast<uint64_t*>(ws);
  const size_t a = (static_cast<size_t>(m) * 8 + 255) & ~size_t(255);
  const size_t b = (static_cast<size_t>(m) * 4 + 255) & ~size_t(255);
  auto* idx = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + a);
  void* sws = static_cast<char*>(ws) + a + b;
  const int grid = grid_for(m, 256, kSMs * 8);
  if (d.n_words == 1)
    mstream_keys_kernel<1><<<grid, 256, 0, s>>>(d, packed, m, mode, tile, row_major, ckey, idx);
  else
    mstream_keys_kernel<2><<<grid, 256, 0, s>>>(d, packed, m, mode, tile, row_major, ckey, idx);
  ALTO_LAUNCH_CHECK("alto_mode_stream/keys");
  const int st = alto_sort_pairs(ckey, idx, m, 1, 4, tbits + lay->bits[mode], sws,
                                 ws_bytes - a - b, stream);
  if (st) return st;
  const int* hs = reinterpret_cast<const int*>(hot_slot);
#define ALTO_MS_SCATTER(WW, VT)                                                                              \
  mstream_scatter_kernel<WW, VT><<<grid, 256, 0, s>>>(d, F, packed, static_cast<const VT*>(values), idx, m, mode, \
                                                      tile, gmode, hs,                                            \
                                                      skeys, static_cast<VT*>(svals), delta ? ckey : nullptr,    \
                                                      delta ? base_rows : nullptr, d_overflow, blk_u, blk_gpw)
  if (d.n_words == 1) {
    if (vb == 4) ALTO_MS_SCATTER(1, float); else ALTO_MS_SCATTER(1, double);
  } else {
    if (vb == 4) ALTO_MS_SCATTER(2, float); else ALTO_MS_SCATTER(2, double);
  }
#undef ALTO_MS_SCATTER
  ALTO_LAUNCH_CHECK("alto_mode_stream/scatter");
  return ALTO_OK;
}

}  // extern "C"

// ---- plan 2: per-mode 64-bit plan words and hot-input row selection ----------
namespace alto {

__global__ void topk_keys_kernel(const long long* __restrict__ row_ptr, long long dim, uint64_t* __restrict__ keys) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; r < dim; r += stride) {
    const unsigned long long c = static_cast<unsigned long long>(row_ptr[r + 1] - row_ptr[r]);
    keys[r] = (min(c, 0xffffffffull) << 32) | (0xffffffffull - static_cast<unsigned long long>(r));
  }
}

__global__ void topk_finish_kernel(const uint64_t* __restrict__ sorted, long long dim, int k,
                                   unsigned long long min_count, int* __restrict__ rows, int* __restrict__ slot_map,
                                   int* __restrict__ count) {
  // sorted ascending: slot s holds the s-th largest count; rows with count
  // <= min_count get no slot, so assigned slots form the prefix [0, *count)
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < k; s += gridDim.x * blockDim.x) {
    const long long idx = dim - 1 - s;
    int r = -1;
    if (idx >= 0 && (sorted[idx] >> 32) > min_count)
      r = static_cast<int>(0xffffffffull - (sorted[idx] & 0xffffffffull));
    rows[s] = r;
    if (r >= 0) {
      slot_map[r] = s;
      if (count) atomicMax(count, s + 1);
    }
  }
}

__global__ void fill_i32(int* p, long long n, int v) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride) p[i] = v;
}

}  // namespace alto

extern "C" {

size_t alto_topk_rows_workspace_bytes(int64_t dim) {
  if (dim < 1) dim = 1;
  return ((static_cast<size_t>(dim) * 8 + 255) & ~size_t(255)) + alto_sort_workspace_bytes(dim, 1, 0);
}

int alto_hot_rows(const int64_t* row_ptr, int64_t dim, int32_t k, int64_t min_count, int32_t* rows,
                  int32_t* slot_map, int32_t* d_count, void* ws, size_t ws_bytes, void* stream) {
  ALTO_REQUIRE(dim >= 1 && dim <= INT_MAX, "hot rows need 1 <= dim < 2^31");
  ALTO_REQUIRE(k >= 1 && k <= (1 << 20), "hot rows k must be in [1, 2^20]");
  ALTO_REQUIRE(ws && ws_bytes >= alto_topk_rows_workspace_bytes(dim), "hot rows workspace too small");
  cudaStream_t s = as_stream(stream);
  auto* keys = static_cast<uint64_t*>(ws);
  const size_t a = (static_cast<size_t>(dim) * 8 + 255) & ~size_t(255);
  topk_keys_kernel<<<grid_for(dim, 256), 256, 0, s>>>(reinterpret_cast<const long long*>(row_ptr), dim, keys);
  fill_i32<<<grid_for(dim, 256), 256, 0, s>>>(slot_map, dim, -1);
  ALTO_CUDA_TRY(cudaMemsetAsync(d_count, 0, sizeof(int32_t), s));
  ALTO_LAUNCH_CHECK("alto_hot_rows");
  const int st = alto_sort_pairs(keys, nullptr, dim, 1, 0, 64, static_cast<char*>(ws) + a, ws_bytes - a, stream);
  if (st) return st;
  topk_finish_kernel<<<grid_for(k, 256), 256, 0, s>>>(keys, dim, k, static_cast<unsigned long long>(min_count), rows,
                                                       slot_map, d_count);
  ALTO_LAUNCH_CHECK("alto_hot_rows/finish");
  return ALTO_OK;
}


}  // extern "C"
