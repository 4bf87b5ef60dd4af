// alto_plan.cu — per-tensor / per-mode plans of the streaming MTTKRP:
// mode-contiguous key re-encoding and the row-sorted sub-tile order (see
// alto_fast.cuh, "planned variant").  Built once (like the reference's
// per-mode plans and flagged copies in _make_backend, cpd.py:149-181).
#include "alto_fast.cuh"

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

}  // extern "C"
