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
constexpr int kSortBins = 2048;   // in-tile counting sort when the output interval fits

template <typename T>
__device__ __forceinline__ double to_d(T x) { return static_cast<double>(x); }

// fp32 configs accumulate per (tile, row) segments in fp32 (<= tile adds),
// then merge into the float64 output; fp64 configs use fp64 throughout.
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
  int tile;      // elements per tile (multiple of kTileThreads, <= 4 * kTileThreads)
  int n_hot;     // hot-row slots (0: no hot plan)
  long long ntiles;
  const int* hot_slot;
  int hot_copies;
  double* hot_buf;
};

// Element record staged in shared memory: NW 32-bit words = N coordinates
// followed by the value bits.
template <int N, typename V>
struct RecWords {
  static constexpr int raw = N + static_cast<int>(sizeof(V) / 4);
  static constexpr int value = (raw + 3) & ~3;  // whole 16-byte vectors
};

// rec[mode] without dynamic register indexing.
template <int NMAX>
__device__ __forceinline__ unsigned pick(const unsigned* w, int mode) {
  unsigned r = w[0];
#pragma unroll
  for (int n = 1; n < NMAX; ++n)
    if (n == mode) r = w[n];
  return r;
}

template <typename F>
struct Vec4 {
  F v[4];
};

template <typename F, bool VEC>
__device__ __forceinline__ Vec4<F> load4(const F* __restrict__ p, int r, int R) {
  Vec4<F> o;
  if constexpr (VEC) {
    if constexpr (sizeof(F) == 4) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(p + r));
      o.v[0] = t.x; o.v[1] = t.y; o.v[2] = t.z; o.v[3] = t.w;
    } else {
      const double2 a = __ldg(reinterpret_cast<const double2*>(p + r));
      const double2 b = __ldg(reinterpret_cast<const double2*>(p + r + 2));
      o.v[0] = a.x; o.v[1] = a.y; o.v[2] = b.x; o.v[3] = b.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) o.v[q] = (r + q < R) ? __ldg(p + r + q) : F(0);
  }
  return o;
}

// Streaming ALTO MTTKRP tile kernel (see file header).  NT = compile-time
// order (0 = generic runtime order), G = lanes per element (each lane owns
// 4 consecutive ranks), VEC = rank is a multiple of 4 (vector gathers).
template <int W, typename V, typename F, int NT, int G, bool VEC>
__global__ void __launch_bounds__(kTileThreads, 2)
mttkrp_tile_kernel(const __grid_constant__ DevLayout L, const uint64_t* __restrict__ tab,
                   const __grid_constant__ TileParams P) {
  using A = typename AccOf<V, F>::type;
  constexpr int NMAX = NT > 0 ? NT : ALTO_MAX_ORDER;
  constexpr int NW = RecWords<NMAX, V>::value;
  constexpr int EPT = 4;  // max elements per thread in phase A (tile <= 1024)
  extern __shared__ __align__(16) unsigned char smem[];
  const int N = NT > 0 ? NT : L.order;
  const int T = P.tile;
  const int R = P.rank;
  const int mode = P.mode;
  uint64_t* s_dec = reinterpret_cast<uint64_t*>(smem);
  size_t off = (static_cast<size_t>(L.dec_bytes) * 256 * W * 8 + 15) & ~size_t(15);
  unsigned* s_rec = reinterpret_cast<unsigned*>(smem + off);  // [T][NW]
  off += static_cast<size_t>(T) * NW * 4;
  int* s_bin = reinterpret_cast<int*>(smem + off);            // [kSortBins + 32]
  __shared__ int s_lo[kTileWarps], s_hi[kTileWarps];

  copy_to_smem(s_dec, tab + static_cast<long long>(L.dec_off) * W, L.dec_bytes * 256 * W);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const F* __restrict__ fac[NMAX];
#pragma unroll
  for (int n = 0; n < NMAX; ++n) fac[n] = static_cast<const F*>(P.factors[n]);
  const V* __restrict__ vals = static_cast<const V*>(P.values);
  double* __restrict__ out = P.out;
  const int* __restrict__ hot_slot = P.n_hot > 0 ? P.hot_slot : nullptr;
  constexpr int NGROUPS = kTileThreads / G;
  const int grp = tid / G;
  const int gl = tid % G;  // lane within the element group

  for (long long tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x) {
    __syncthreads();  // previous tile consumed; decode tables visible
    const long long t0 = tile * T;
    const int cnt = static_cast<int>(min(static_cast<long long>(T), P.m - t0));
    // ---- phase A: coalesced stream + table decode into registers ----------
    unsigned rec[EPT][NW];
    int myrow[EPT];
    int lo = INT_MAX, hi = INT_MIN;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int e = tid + k * kTileThreads;
      myrow[k] = -1;
      if (e < cnt) {
        const Key<W> p = decode_packed<W>(s_dec, L.dec_bytes, load_key<W>(P.keys, t0 + e));
#pragma unroll
        for (int n = 0; n < NMAX; ++n)
          if (n < N) rec[k][n] = static_cast<unsigned>(packed_field<W>(p, L.pack_off[n], L.bits[n]));
        const V v = __ldg(vals + t0 + e);
        if constexpr (sizeof(V) == 4) {
          rec[k][NMAX] = __float_as_uint(static_cast<float>(v));
        } else {
          const unsigned long long u = __double_as_longlong(static_cast<double>(v));
          rec[k][NMAX] = static_cast<unsigned>(u);
          rec[k][NMAX + 1] = static_cast<unsigned>(u >> 32);
        }
        const int r = static_cast<int>(pick<NMAX>(rec[k], mode));
        myrow[k] = r;
        lo = min(lo, r);
        hi = max(hi, r);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) { s_lo[warp] = lo; s_hi[warp] = hi; }
    for (int i = tid; i < kSortBins; i += kTileThreads) s_bin[i] = 0;
    __syncthreads();
    lo = s_lo[0]; hi = s_hi[0];
#pragma unroll
    for (int w = 1; w < kTileWarps; ++w) { lo = min(lo, s_lo[w]); hi = max(hi, s_hi[w]); }
    const int span = hi - lo + 1;
    // ---- in-tile counting sort by output row (short intervals) --------------
    if (span <= kSortBins) {
#pragma unroll
      for (int k = 0; k < EPT; ++k)
        if (myrow[k] >= 0) atomicAdd(&s_bin[myrow[k] - lo], 1);
      __syncthreads();
      // exclusive scan of s_bin[0..span) (8 bins per thread)
      constexpr int BPT = kSortBins / kTileThreads;
      int loc[BPT];
      int sum = 0;
#pragma unroll
      for (int q = 0; q < BPT; ++q) {
        loc[q] = s_bin[tid * BPT + q];
        sum += loc[q];
      }
      int x = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      __syncthreads();
      if (lane == 31) s_bin[kSortBins + warp] = x;
      __syncthreads();
      int wpre = 0;
#pragma unroll
      for (int w = 0; w < kTileWarps; ++w) wpre += (w < warp) ? s_bin[kSortBins + w] : 0;
      int run = wpre + x - sum;
#pragma unroll
      for (int q = 0; q < BPT; ++q) {
        s_bin[tid * BPT + q] = run;
        run += loc[q];
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < EPT; ++k)
        if (myrow[k] >= 0) {
          const int slot = atomicAdd(&s_bin[myrow[k] - lo], 1);
#pragma unroll
          for (int q = 0; q < NW; ++q) s_rec[slot * NW + q] = rec[k][q];
        }
    } else {
#pragma unroll
      for (int k = 0; k < EPT; ++k)
        if (myrow[k] >= 0) {
          const int e = tid + k * kTileThreads;
#pragma unroll
          for (int q = 0; q < NW; ++q) s_rec[e * NW + q] = rec[k][q];
        }
    }
    __syncthreads();
    // ---- phase B: each element group walks a contiguous run of records ------
    double* __restrict__ hot_base =
        P.hot_buf ? P.hot_buf + (tile % P.hot_copies) * static_cast<long long>(P.n_hot) * R : nullptr;
    const int chunk = (cnt + NGROUPS - 1) / NGROUPS;
    const int j0 = grp * chunk;
    const int j1 = min(cnt, j0 + chunk);
    constexpr int U = 4;  // elements in flight per group (gathers issued ahead of use)
    for (int r0 = 0; r0 < R; r0 += 4 * G) {
      const int r = r0 + 4 * gl;
      const bool rank_ok = r < R;
      A acc[4] = {A(0), A(0), A(0), A(0)};
      int cur = -1, cur_hot = -1;
      for (int jb = j0; jb < j1; jb += U) {
        int rows[U];
        int hots[U];
        A vv[U];
        Vec4<F> g[U][NMAX];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = jb + u;
          rows[u] = -1;
          if (j < j1) {
            const unsigned* rc = s_rec + j * NW;
            unsigned cw[NW];
#pragma unroll
            for (int q = 0; q < NW; q += 4) {
              const uint4 t = *reinterpret_cast<const uint4*>(rc + q);
              cw[q] = t.x; cw[q + 1] = t.y; cw[q + 2] = t.z; cw[q + 3] = t.w;
            }
            rows[u] = static_cast<int>(pick<NMAX>(cw, mode));
            hots[u] = hot_slot ? __ldg(hot_slot + rows[u]) : -1;
            if constexpr (sizeof(V) == 4) {
              vv[u] = static_cast<A>(__uint_as_float(cw[NMAX]));
            } else {
              vv[u] = static_cast<A>(__longlong_as_double(static_cast<long long>(
                  (static_cast<unsigned long long>(cw[NMAX + 1]) << 32) | cw[NMAX])));
            }
#pragma unroll
            for (int n = 0; n < NMAX; ++n) {
              if (n >= N || n == mode) continue;
              if (rank_ok) g[u][n] = load4<F, VEC>(fac[n] + static_cast<long long>(cw[n]) * R, r, R);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (rows[u] < 0) continue;
          A x[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) x[q] = vv[u];
          if (rank_ok) {
#pragma unroll
            for (int n = 0; n < NMAX; ++n) {
              if (n >= N || n == mode) continue;
#pragma unroll
              for (int q = 0; q < 4; ++q) x[q] *= static_cast<A>(g[u][n].v[q]);
            }
          }
          if (rows[u] != cur) {
            if (cur >= 0 && rank_ok) {
              double* o = cur_hot >= 0 ? hot_base + static_cast<long long>(cur_hot) * R + r
                                       : out + static_cast<long long>(cur) * R + r;
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (r + q < R) atomicAdd(o + q, to_d(acc[q]));
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = x[q];
            cur = rows[u];
            cur_hot = hots[u];
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] += x[q];
          }
        }
      }
      if (cur >= 0 && rank_ok) {
        double* o = cur_hot >= 0 ? hot_base + static_cast<long long>(cur_hot) * R + r
                                 : out + static_cast<long long>(cur) * R + r;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (r + q < R) atomicAdd(o + q, to_d(acc[q]));
      }
    }
  }
}

// Sum the replicated hot-row partials in copy order into out; re-zero them.
__global__ void hot_reduce_kernel(double* __restrict__ buf, const int* __restrict__ hot_rows, int n_hot,
                                  int copies, int R, double* __restrict__ out) {
  const long long n = static_cast<long long>(n_hot) * R;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    double s = 0.0;
    for (int k = 0; k < copies; ++k) {
      double* p = buf + k * n + i;
      s += *p;
      *p = 0.0;
    }
    const long long h = i / R;
    out[static_cast<long long>(hot_rows[h]) * R + (i - h * R)] += s;
  }
}

__global__ void hot_plan_kernel(const long long* __restrict__ row_ptr, long long dim, long long tau, int hmax,
                                int* __restrict__ hot_slot, int* __restrict__ hot_rows, int* __restrict__ nhot) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; r < dim; r += stride) {
    int slot = -1;
    if (row_ptr[r + 1] - row_ptr[r] > tau) {
      const int s = atomicAdd(nhot, 1);
      if (s < hmax) {
        slot = s;
        hot_rows[s] = static_cast<int>(r);
      }
    }
    hot_slot[r] = slot;
  }
}

__global__ void clamp_count(int* n, int hmax) {
  if (*n > hmax) *n = hmax;
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

template <int W, typename V, typename F, int NT, int G, bool VEC>
static int launch_tile(const DevLayout& d, const uint64_t* tab, TileParams P, cudaStream_t s) {
  constexpr int NMAX = NT > 0 ? NT : ALTO_MAX_ORDER;
  constexpr int NW = RecWords<NMAX, V>::value;
  const size_t smem = ((static_cast<size_t>(d.dec_bytes) * 256 * W * 8 + 15) & ~size_t(15)) +
                      static_cast<size_t>(P.tile) * NW * 4 + (kSortBins + 32) * sizeof(int);
  auto kern = mttkrp_tile_kernel<W, V, F, NT, G, VEC>;
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

template <int W, typename V, typename F, int NT>
static int dispatch_rank(const DevLayout& d, const uint64_t* tab, const TileParams& P, cudaStream_t s) {
  const bool vec = (P.rank % 4) == 0;
  const int groups = (P.rank + 3) / 4;
  if (vec) {
    if (groups <= 1) return launch_tile<W, V, F, NT, 1, true>(d, tab, P, s);
    if (groups <= 2) return launch_tile<W, V, F, NT, 2, true>(d, tab, P, s);
    if (groups <= 4) return launch_tile<W, V, F, NT, 4, true>(d, tab, P, s);
    return launch_tile<W, V, F, NT, 8, true>(d, tab, P, s);
  }
  if (groups <= 1) return launch_tile<W, V, F, NT, 1, false>(d, tab, P, s);
  if (groups <= 4) return launch_tile<W, V, F, NT, 4, false>(d, tab, P, s);
  return launch_tile<W, V, F, NT, 8, false>(d, tab, P, s);
}

template <int W, typename V, typename F>
static int dispatch_order(const DevLayout& d, const uint64_t* tab, const TileParams& P, cudaStream_t s) {
  switch (d.order) {
    case 3: return dispatch_rank<W, V, F, 3>(d, tab, P, s);
    case 4: return dispatch_rank<W, V, F, 4>(d, tab, P, s);
    case 5: return dispatch_rank<W, V, F, 5>(d, tab, P, s);
    default: return dispatch_rank<W, V, F, 0>(d, tab, P, s);
  }
}

template <int W>
static int dispatch_types(const DevLayout& d, const uint64_t* tab, const TileParams& P, int vd, int fd,
                          cudaStream_t s) {
  if (vd == ALTO_F32 && fd == ALTO_F32) return dispatch_order<W, float, float>(d, tab, P, s);
  if (vd == ALTO_F64 && fd == ALTO_F64) return dispatch_order<W, double, double>(d, tab, P, s);
  if (vd == ALTO_F32 && fd == ALTO_F64) return dispatch_order<W, float, double>(d, tab, P, s);
  return dispatch_order<W, double, float>(d, tab, P, s);
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
  P.n_hot = (a->hot_slot && a->hot_buf && a->n_hot > 0 && a->hot_copies > 0) ? a->n_hot : 0;
  P.hot_slot = a->hot_slot;
  P.hot_copies = a->hot_copies > 0 ? a->hot_copies : 1;
  P.hot_buf = P.n_hot ? a->hot_buf : nullptr;
  return P;
}

}  // namespace alto

using namespace alto;

extern "C" {

int alto_mttkrp(const alto_mttkrp_args* a, void* stream) {
  int st = check_args(a);
  ALTO_REQUIRE(a->n_hot <= 0 || a->hot_rows != nullptr, "hot plan needs hot_rows");
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
  ALTO_REQUIRE(P.tile >= kTileThreads && P.tile <= 4 * kTileThreads && P.tile % kTileThreads == 0,
               "tile must be a multiple of 256 in [256, 1024]");
  const auto* tab = static_cast<const uint64_t*>(a->d_tables);
  st = d.n_words == 1 ? dispatch_types<1>(d, tab, P, a->value_dtype, a->factor_dtype, s)
                      : dispatch_types<2>(d, tab, P, a->value_dtype, a->factor_dtype, s);
  if (st) return st;
  if (P.n_hot > 0) {
    hot_reduce_kernel<<<grid_for(static_cast<long long>(P.n_hot) * a->rank, 256), 256, 0, s>>>(
        P.hot_buf, a->hot_rows, P.n_hot, P.hot_copies, a->rank, a->out);
    ALTO_LAUNCH_CHECK("alto_mttkrp/hot_reduce");
  }
  return ALTO_OK;
}

int alto_hot_plan(const int64_t* row_ptr, int64_t dim, int64_t tau, int32_t hmax, int32_t* hot_slot,
                  int32_t* hot_rows, int32_t* d_nhot, void* stream) {
  ALTO_REQUIRE(dim >= 0 && dim <= INT_MAX, "hot plan needs mode extents below 2^31");
  ALTO_REQUIRE(hmax >= 0, "hmax must be nonnegative");
  cudaStream_t s = as_stream(stream);
  ALTO_CUDA_TRY(cudaMemsetAsync(d_nhot, 0, sizeof(int32_t), s));
  if (dim > 0)
    hot_plan_kernel<<<grid_for(dim, 256), 256, 0, s>>>(reinterpret_cast<const long long*>(row_ptr), dim, tau, hmax,
                                                        hot_slot, hot_rows, d_nhot);
  clamp_count<<<1, 1, 0, s>>>(d_nhot, hmax);
  ALTO_LAUNCH_CHECK("alto_hot_plan");
  return ALTO_OK;
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
