// alto_mttkrp.cu — ALTO MTTKRP on B200.
//
//   out[i_n, r] = sum over elements x: x.value * prod_{m != n} F_m[x.coord_m, r]
//   (pkg/src/altotensor/mttkrp.py:1-14, contributions :80-105)
//
// 1. Streaming tile kernel (K7/K8, the fast path).  A CTA owns a tile of the
//    sorted ALTO stream (contiguous elements, so a compact coordinate box).
//    Phase A streams the tile's keys/values with coalesced loads, decodes all
//    modes in registers through the byte tables, and parks coordinates and
//    values in shared memory, reducing the output-mode interval [lo, hi].
//    Phase B, when hi-lo+1 fits the on-chip buffer (the paper's per-partition
//    interval buffer, Alg. 2 / mttkrp.py:148-156, at CTA granularity), each
//    warp owns the buffer rows r with (r-lo) % 8 == warp and applies the
//    contributions of its rows in element order (no shared-memory atomics:
//    on sm_100a those compile to CAS loops).  Factor rows are gathered as
//    coalesced 64/128-byte row segments (LPE lanes per element).  Touched
//    rows are then pushed to the float64 output with one RED per (row, rank)
//    — the pull/merge step.  Tiles whose interval is too wide use direct
//    float64 atomics per element (the Atomic scheme, mttkrp.py:178-224).
// 2. Exact-order engine (deterministic): per output row, contributions are
//    summed sequentially in element order, restarted at partition boundaries,
//    and partition partials combined in ascending order — the arithmetic
//    order of _par_buffered (mttkrp.py:148-172) and mttkrp_seq (:108-117), in
//    float64 with contraction disabled, hence bitwise equal to the reference
//    on float64 inputs.
// 3. COO kernel (mttkrp_oracle, mttkrp.py:64-77) over a coordinate list.
#include <algorithm>
#include <climits>

#include "alto_common.cuh"

namespace alto {

constexpr int kTileThreads = 256;
constexpr int kTileWarps = kTileThreads / 32;

template <typename T>
__device__ __forceinline__ double to_d(T x) { return static_cast<double>(x); }

template <typename T>
__device__ __forceinline__ T ld_nc(const T* p) { return __ldg(p); }

// fp32 configs accumulate tiles in fp32 (<= tile adds per row, then fp64
// across tiles); fp64 configs accumulate in fp64 throughout.
template <typename V, typename F>
struct AccOf { using type = double; };
template <>
struct AccOf<float, float> { using type = float; };

struct TileParams {
  const uint64_t* keys;
  const void* values;
  long long m;
  int mode;
  int rank;
  const void* factors[ALTO_MAX_ORDER];
  double* out;
  int tile;      // elements per tile
  int cap;       // rows of the on-chip buffer
  long long ntiles;
};

// LPE: lanes per element (16 -> two elements per warp step, 32 -> one).
template <int W, typename V, typename F, int LPE>
__global__ void __launch_bounds__(kTileThreads, 1)
mttkrp_tile_kernel(const __grid_constant__ DevLayout L, const uint64_t* __restrict__ tab,
                   const __grid_constant__ TileParams P) {
  using A = typename AccOf<V, F>::type;
  constexpr int EPW = 32 / LPE;  // elements per warp step
  extern __shared__ __align__(16) unsigned char smem[];
  const int N = L.order;
  const int T = P.tile;
  const int R = P.rank;
  uint64_t* s_dec = reinterpret_cast<uint64_t*>(smem);
  size_t off = static_cast<size_t>(L.dec_bytes) * 256 * W * 8;
  A* s_acc = reinterpret_cast<A*>(smem + off);
  off += static_cast<size_t>(P.cap) * R * sizeof(A);
  V* s_val = reinterpret_cast<V*>(smem + off);
  off += static_cast<size_t>(T) * sizeof(V);
  int* s_row = reinterpret_cast<int*>(smem + off);  // [N][T]
  off += static_cast<size_t>(N) * T * sizeof(int);
  unsigned char* s_touch = smem + off;               // [cap]
  __shared__ int s_lo[kTileWarps], s_hi[kTileWarps];

  copy_to_smem(s_dec, tab + static_cast<long long>(L.dec_off) * W, L.dec_bytes * 256 * W);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mode = P.mode;
  const F* __restrict__ fac[ALTO_MAX_ORDER];
#pragma unroll
  for (int n = 0; n < ALTO_MAX_ORDER; ++n) fac[n] = static_cast<const F*>(P.factors[n]);
  const V* __restrict__ vals = static_cast<const V*>(P.values);
  double* __restrict__ out = P.out;
  const int sub = lane / LPE;       // element slot within the warp step
  const int rl = lane % LPE;        // rank lane

  for (long long tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x) {
    __syncthreads();  // previous tile fully consumed; tables visible (first pass)
    const long long t0 = tile * T;
    const int cnt = static_cast<int>(min(static_cast<long long>(T), P.m - t0));
    // ---- Phase A: stream + decode -------------------------------------------
    int lo = INT_MAX, hi = INT_MIN;
    for (int e = threadIdx.x; e < cnt; e += kTileThreads) {
      const Key<W> k = load_key<W>(P.keys, t0 + e);
      const Key<W> p = decode_packed<W>(s_dec, L.dec_bytes, k);
      s_val[e] = ld_nc(vals + t0 + e);
      for (int n = 0; n < N; ++n) {
        const int c = static_cast<int>(packed_field<W>(p, L.pack_off[n], L.bits[n]));
        s_row[n * T + e] = c;
        if (n == mode) { lo = min(lo, c); hi = max(hi, c); }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) { s_lo[warp] = lo; s_hi[warp] = hi; }
    __syncthreads();
    lo = s_lo[0]; hi = s_hi[0];
#pragma unroll
    for (int w = 1; w < kTileWarps; ++w) { lo = min(lo, s_lo[w]); hi = max(hi, s_hi[w]); }
    const int span = hi - lo + 1;

    if (span <= P.cap) {
      // ---- Phase B (buffered tile) ----------------------------------------
      for (int i = threadIdx.x; i < span * R; i += kTileThreads) s_acc[i] = A(0);
      for (int i = threadIdx.x; i < span; i += kTileThreads) s_touch[i] = 0;
      __syncthreads();
      for (int base = 0; base < cnt; base += 32) {
        const int e0 = base + lane;
        const int rr = e0 < cnt ? s_row[mode * T + e0] - lo : -1;
        unsigned mine = __ballot_sync(0xffffffffu, rr >= 0 && (rr & (kTileWarps - 1)) == warp);
        while (mine) {
          int sel[EPW];
#pragma unroll
          for (int q = 0; q < EPW; ++q) {
            sel[q] = mine ? __ffs(mine) - 1 : -1;
            if (mine) mine &= mine - 1;
          }
          const int my = sel[sub];
          const int e = my >= 0 ? base + my : -1;
          const int row = e >= 0 ? s_row[mode * T + e] - lo : -1;
          int row_other = row;
          if constexpr (EPW == 2) row_other = __shfl_xor_sync(0xffffffffu, row, 16);
          for (int r0 = 0; r0 < R; r0 += LPE) {
            const int r = r0 + rl;
            A x = A(0);
            if (e >= 0 && r < R) {
              x = static_cast<A>(s_val[e]);
              for (int n = 0; n < N; ++n) {
                if (n == mode) continue;
                const long long c = s_row[n * T + e];
                x *= static_cast<A>(ld_nc(fac[n] + c * R + r));
              }
            }
            if constexpr (EPW == 2) {
              const A xo = __shfl_xor_sync(0xffffffffu, x, 16);
              if (sub == 0 && row >= 0 && row == row_other) x += xo;  // pair on one row: slot 0 applies both
            }
            const bool writer = e >= 0 && r < R && !(EPW == 2 && sub == 1 && row == row_other);
            if (writer) s_acc[row * R + r] += x;
          }
          if (e >= 0 && rl == 0) s_touch[row] = 1;
          __syncwarp();
        }
      }
      __syncthreads();
      // merge: one fp64 RED per touched (row, rank)
      for (int i = threadIdx.x; i < span * R; i += kTileThreads) {
        const int row = i / R;
        if (s_touch[row]) atomicAdd(out + static_cast<long long>(lo + row) * R + (i - row * R), to_d(s_acc[i]));
      }
    } else {
      // ---- wide tile: direct fp64 atomics per element ------------------------
      for (int e = warp * EPW + sub; e < cnt + (EPW - 1); e += kTileWarps * EPW) {
        const bool ok = e < cnt;
        const int row = ok ? s_row[mode * T + e] : 0;
        for (int r0 = 0; r0 < R; r0 += LPE) {
          const int r = r0 + rl;
          if (ok && r < R) {
            A x = static_cast<A>(s_val[e]);
            for (int n = 0; n < N; ++n) {
              if (n == mode) continue;
              const long long c = s_row[n * T + e];
              x *= static_cast<A>(ld_nc(fac[n] + c * R + r));
            }
            atomicAdd(out + static_cast<long long>(row) * R + r, to_d(x));
          }
        }
      }
    }
  }
}

// ---- exact-order engine ------------------------------------------------------

__global__ void row_ptr_kernel(const uint64_t* __restrict__ sorted_rows, long long m, long long dim,
                               long long* __restrict__ row_ptr) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i <= m; i += stride) {
    const long long prev = i > 0 ? static_cast<long long>(sorted_rows[i - 1]) : -1;
    const long long cur = i < m ? static_cast<long long>(sorted_rows[i]) : dim;
    for (long long r = prev + 1; r <= cur && r <= dim; ++r) row_ptr[r] = i;
  }
}

__global__ void iota_u32(unsigned* p, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride)
    p[i] = static_cast<unsigned>(i);
}

template <int W, typename V, typename F>
__global__ void __launch_bounds__(256)
mttkrp_exact_kernel(const __grid_constant__ DevLayout L, const uint64_t* __restrict__ tab,
                    const __grid_constant__ TileParams P, const int* __restrict__ row_perm,
                    const long long* __restrict__ row_ptr, const long long* __restrict__ part_off,
                    long long count, long long dim) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* s_dec = reinterpret_cast<uint64_t*>(smem);
  copy_to_smem(s_dec, tab + static_cast<long long>(L.dec_off) * W, L.dec_bytes * 256 * W);
  __syncthreads();
  const int N = L.order, R = P.rank, mode = P.mode;
  const int lane = threadIdx.x & 31;
  const long long gwarp = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  const V* __restrict__ vals = static_cast<const V*>(P.values);
  for (long long row = gwarp; row < dim; row += nwarps) {
    const long long j0 = row_ptr[row], j1 = row_ptr[row + 1];
    for (int r0 = 0; r0 < R; r0 += 32) {
      const int r = r0 + lane;
      double total = 0.0, part = 0.0;
      long long l = 0;
      bool have_part = false;
      for (long long j = j0; j < j1; ++j) {
        const long long e = row_perm[j];
        while (l + 1 < count && part_off[l + 1] <= e) {  // crossed into a later partition
          if (have_part) { total = __dadd_rn(total, part); part = 0.0; have_part = false; }
          ++l;
        }
        const Key<W> p = decode_packed<W>(s_dec, L.dec_bytes, load_key<W>(P.keys, e));
        double x = static_cast<double>(vals[e]);
        if (r < R) {
          for (int n = 0; n < N; ++n) {
            if (n == mode) continue;
            const long long c = packed_field<W>(p, L.pack_off[n], L.bits[n]);
            const F* f = static_cast<const F*>(P.factors[n]);
            x = __dmul_rn(x, static_cast<double>(f[c * R + r]));
          }
        }
        part = __dadd_rn(part, x);
        have_part = true;
      }
      if (have_part) total = __dadd_rn(total, part);
      if (r < R) P.out[row * R + r] = total;
    }
  }
}

// ---- COO kernel (mttkrp_oracle) ------------------------------------------------

struct CooParams {
  const long long* coords;
  const double* values;
  long long m;
  int order, mode, rank;
  const double* factors[ALTO_MAX_ORDER];
  double* out;
};

__global__ void mttkrp_coo_kernel(const __grid_constant__ CooParams P) {
  const long long total = P.m * P.rank;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total; t += stride) {
    const long long e = t / P.rank;
    const int r = static_cast<int>(t - e * P.rank);
    double x = P.values[e];
    for (int n = 0; n < P.order; ++n) {
      if (n == P.mode) continue;
      x = __dmul_rn(x, P.factors[n][P.coords[e * P.order + n] * P.rank + r]);
    }
    atomicAdd(P.out + P.coords[e * P.order + P.mode] * P.rank + r, x);
  }
}

// ---- launch helpers ----------------------------------------------------------------

template <typename K>
static int prep_smem(K kernel, size_t smem) {
  ALTO_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return ALTO_OK;
}

constexpr size_t kSmemBudget = 200 * 1024;

template <int W, typename V, typename F, int LPE>
static int launch_tile(const DevLayout& d, const uint64_t* tab, TileParams P, cudaStream_t s) {
  using A = typename AccOf<V, F>::type;
  const size_t fixed = static_cast<size_t>(d.dec_bytes) * 256 * W * 8 + static_cast<size_t>(P.tile) * sizeof(V) +
                       static_cast<size_t>(d.order) * P.tile * sizeof(int) + 64;
  if (fixed >= kSmemBudget) { set_error("tile too large for shared memory"); return ALTO_EINVAL; }
  const size_t per_row = static_cast<size_t>(P.rank) * sizeof(A) + 1;
  int cap = static_cast<int>((kSmemBudget - fixed) / per_row);
  cap = std::min(cap, 4096);
  P.cap = cap;
  const size_t smem = fixed + static_cast<size_t>(cap) * per_row + 16;
  auto kern = mttkrp_tile_kernel<W, V, F, LPE>;
  if (prep_smem(kern, smem)) return ALTO_ECUDA;
  int blocks_per_sm = 1;
  ALTO_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, kTileThreads, smem));
  int dev = 0, sms = kSMs;
  ALTO_CUDA_TRY(cudaGetDevice(&dev));
  ALTO_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const long long grid = std::min<long long>(P.ntiles, static_cast<long long>(sms) * std::max(blocks_per_sm, 1));
  kern<<<static_cast<unsigned>(grid), kTileThreads, smem, s>>>(d, tab, P);
  ALTO_LAUNCH_CHECK("alto_mttkrp");
  return ALTO_OK;
}

template <int W, typename V, typename F>
static int dispatch_lpe(const DevLayout& d, const uint64_t* tab, const TileParams& P, cudaStream_t s) {
  if (P.rank <= 16) return launch_tile<W, V, F, 16>(d, tab, P, s);
  return launch_tile<W, V, F, 32>(d, tab, P, s);
}

template <int W>
static int dispatch_types(const DevLayout& d, const uint64_t* tab, const TileParams& P, int vd, int fd,
                          cudaStream_t s) {
  if (vd == ALTO_F32 && fd == ALTO_F32) return dispatch_lpe<W, float, float>(d, tab, P, s);
  if (vd == ALTO_F64 && fd == ALTO_F64) return dispatch_lpe<W, double, double>(d, tab, P, s);
  if (vd == ALTO_F32 && fd == ALTO_F64) return dispatch_lpe<W, float, double>(d, tab, P, s);
  return dispatch_lpe<W, double, float>(d, tab, P, s);
}

static int check_args(const alto_mttkrp_args* a) {
  ALTO_REQUIRE(a && a->lay && a->d_tables, "mttkrp args incomplete");
  ALTO_REQUIRE(a->lay->order >= 1 && a->lay->order <= ALTO_MAX_ORDER, "bad layout order");
  ALTO_REQUIRE(a->mode >= 0 && a->mode < a->lay->order, "mode out of range");
  ALTO_REQUIRE(a->rank >= 1, "rank must be positive");
  ALTO_REQUIRE((a->value_dtype == ALTO_F32 || a->value_dtype == ALTO_F64) &&
                   (a->factor_dtype == ALTO_F32 || a->factor_dtype == ALTO_F64),
               "unsupported dtype");
  ALTO_REQUIRE(a->out != nullptr, "out is NULL");
  return ALTO_OK;
}

static TileParams to_params(const alto_mttkrp_args* a) {
  TileParams P{};
  P.keys = a->keys;
  P.values = a->values;
  P.m = a->m;
  P.mode = a->mode;
  P.rank = a->rank;
  for (int n = 0; n < ALTO_MAX_ORDER; ++n) P.factors[n] = n < a->lay->order ? a->factors[n] : nullptr;
  P.out = a->out;
  P.tile = a->tile > 0 ? a->tile : 1024;
  P.ntiles = a->m > 0 ? (a->m + P.tile - 1) / P.tile : 0;
  return P;
}

}  // namespace alto

using namespace alto;

extern "C" {

int alto_mttkrp(const alto_mttkrp_args* a, void* stream) {
  int st = check_args(a);
  if (st) return st;
  for (int n = 0; n < a->lay->order; ++n)
    ALTO_REQUIRE(a->lay->dims[n] <= INT_MAX, "streaming kernel needs mode extents below 2^31");
  const DevLayout d = make_dev_layout(a->lay);
  cudaStream_t s = as_stream(stream);
  const long long dim = d.dims[a->mode];
  if (a->zero_out)
    ALTO_CUDA_TRY(cudaMemsetAsync(a->out, 0, static_cast<size_t>(dim) * a->rank * sizeof(double), s));
  if (a->m <= 0) return ALTO_OK;
  const TileParams P = to_params(a);
  ALTO_REQUIRE(P.tile >= 32 && P.tile <= 8192, "tile must be in [32, 8192]");
  const auto* tab = static_cast<const uint64_t*>(a->d_tables);
  if (d.n_words == 1) return dispatch_types<1>(d, tab, P, a->value_dtype, a->factor_dtype, s);
  return dispatch_types<2>(d, tab, P, a->value_dtype, a->factor_dtype, s);
}

size_t alto_row_index_workspace_bytes(int64_t m, int64_t dim) {
  (void)dim;
  if (m < 0) m = 0;
  const size_t a = ((static_cast<size_t>(m) * 8 + 255) & ~size_t(255));
  return a + alto_sort_workspace_bytes(m, 1, 4);
}

int alto_row_index(const alto_layout* lay, const void* d_tables, const uint64_t* keys, int64_t m, int32_t mode,
                   int32_t* row_perm, int64_t* row_ptr, void* workspace, size_t workspace_bytes, void* stream) {
  ALTO_REQUIRE(lay && mode >= 0 && mode < lay->order, "mode out of range");
  ALTO_REQUIRE(workspace_bytes >= alto_row_index_workspace_bytes(m, lay->dims[mode]), "row index workspace too small");
  cudaStream_t s = as_stream(stream);
  const long long dim = lay->dims[mode];
  if (m <= 0) {
    ALTO_CUDA_TRY(cudaMemsetAsync(row_ptr, 0, static_cast<size_t>(dim + 1) * 8, s));
    return ALTO_OK;
  }
  auto* rows = static_cast<uint64_t*>(workspace);
  const size_t a = ((static_cast<size_t>(m) * 8 + 255) & ~size_t(255));
  void* sort_ws = static_cast<char*>(workspace) + a;
  int st = alto_delinearize(lay, d_tables, keys, m, mode, reinterpret_cast<int64_t*>(rows), stream);
  if (st) return st;
  iota_u32<<<grid_for(m, 256), 256, 0, s>>>(reinterpret_cast<unsigned*>(row_perm), m);
  ALTO_LAUNCH_CHECK("alto_row_index/iota");
  st = alto_sort_pairs(rows, row_perm, m, 1, 4, lay->bits[mode], sort_ws, workspace_bytes - a, stream);
  if (st) return st;
  row_ptr_kernel<<<grid_for(m + 1, 256), 256, 0, s>>>(rows, m, dim, reinterpret_cast<long long*>(row_ptr));
  ALTO_LAUNCH_CHECK("alto_row_index/row_ptr");
  return ALTO_OK;
}

int alto_mttkrp_exact(const alto_mttkrp_args* a, const int32_t* row_perm, const int64_t* row_ptr,
                      const int64_t* part_off, int64_t count, void* stream) {
  int st = check_args(a);
  if (st) return st;
  ALTO_REQUIRE(count >= 1 && part_off != nullptr, "partition offsets required");
  const DevLayout d = make_dev_layout(a->lay);
  cudaStream_t s = as_stream(stream);
  const long long dim = d.dims[a->mode];
  if (a->m <= 0 || dim <= 0) {
    ALTO_CUDA_TRY(cudaMemsetAsync(a->out, 0, static_cast<size_t>(dim) * a->rank * sizeof(double), s));
    return ALTO_OK;
  }
  TileParams P = to_params(a);
  const auto* tab = static_cast<const uint64_t*>(a->d_tables);
  const size_t smem = static_cast<size_t>(d.dec_bytes) * 256 * d.n_words * 8;
  const int grid = grid_for(dim * 32, 256, kSMs * 8);
  auto go = [&](auto kern) -> int {
    if (prep_smem(kern, smem)) return ALTO_ECUDA;
    kern<<<grid, 256, smem, s>>>(d, tab, P, reinterpret_cast<const int*>(row_perm),
                                 reinterpret_cast<const long long*>(row_ptr),
                                 reinterpret_cast<const long long*>(part_off), count, dim);
    ALTO_LAUNCH_CHECK("alto_mttkrp_exact");
    return ALTO_OK;
  };
  const bool v32 = a->value_dtype == ALTO_F32, f32 = a->factor_dtype == ALTO_F32;
  if (d.n_words == 1) {
    if (v32 && f32) return go(mttkrp_exact_kernel<1, float, float>);
    if (!v32 && !f32) return go(mttkrp_exact_kernel<1, double, double>);
    if (v32) return go(mttkrp_exact_kernel<1, float, double>);
    return go(mttkrp_exact_kernel<1, double, float>);
  }
  if (v32 && f32) return go(mttkrp_exact_kernel<2, float, float>);
  if (!v32 && !f32) return go(mttkrp_exact_kernel<2, double, double>);
  if (v32) return go(mttkrp_exact_kernel<2, float, double>);
  return go(mttkrp_exact_kernel<2, double, float>);
}

int alto_mttkrp_coo(const int64_t* coords, const double* values, int64_t m, int32_t order, int32_t mode,
                    int32_t rank, const double* const* factors_host_array, double* out, int64_t out_rows,
                    void* stream) {
  ALTO_REQUIRE(order >= 1 && order <= ALTO_MAX_ORDER, "order out of range");
  ALTO_REQUIRE(mode >= 0 && mode < order, "mode out of range");
  ALTO_REQUIRE(rank >= 1, "rank must be positive");
  cudaStream_t s = as_stream(stream);
  ALTO_CUDA_TRY(cudaMemsetAsync(out, 0, static_cast<size_t>(out_rows) * rank * sizeof(double), s));
  if (m <= 0) return ALTO_OK;
  CooParams P{};
  P.coords = reinterpret_cast<const long long*>(coords);
  P.values = values;
  P.m = m;
  P.order = order;
  P.mode = mode;
  P.rank = rank;
  for (int n = 0; n < order; ++n) P.factors[n] = factors_host_array[n];
  P.out = out;
  mttkrp_coo_kernel<<<grid_for(m * rank, 256), 256, 0, s>>>(P);
  ALTO_LAUNCH_CHECK("alto_mttkrp_coo");
  return ALTO_OK;
}

}  // extern "C"
